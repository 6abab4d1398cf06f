"""B200-native single-path polynomial homotopy tracker (D / DD / QD).

Hot path (BASELINE.json north_star): track_path on an sm_100a device, through
the C-ABI in include/pathtrack_b200.h.  See DESIGN.md.
"""
from .tracker import (  # noqa: F401
    FAILURE_KINDS,
    Homotopy,
    PolynomialSystem,
    PrecisionMode,
    StepControlParams,
    TrackOutcome,
    arith,
    augment_with_linear,
    chandrasekhar,
    complex_from_limbs,
    cyclic_system,
    device_count,
    gamma_from_seed,
    least_squares_solve,
    limbs_from_complex,
    make_homotopy,
    random_dense,
    total_degree_start,
    unit_complex,
)
from . import monodromy, workloads  # noqa: F401

__version__ = "0.1.0"
