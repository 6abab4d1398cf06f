"""B200-native single-path polynomial homotopy tracker (D / DD / QD).

Hot path (BASELINE.json north_star): track_path on an sm_100a device, through
the C-ABI in include/pathtrack_b200.h.  See DESIGN.md.

Importing the package loads only the host-only inputs library
(libpt_inputs.so: systems, generators, file formats); the CUDA tracker
library is loaded on first use of a tracker name (make_homotopy,
least_squares_solve, ...), so input construction never maps the product.
"""
from .systems import (  # noqa: F401
    CyclicDegreeFact,
    PolynomialSystem,
    PrecisionMode,
    Solution,
    StepControlParams,
    augment_with_linear,
    canonical,
    chandrasekhar,
    complex_from_limbs,
    cyclic_degree,
    cyclic_system,
    gamma_from_seed,
    hex_decode_limb,
    hex_encode_limb,
    hex_limbs,
    limbs_from_complex,
    parse_hex_limbs,
    parse_system,
    random_dense,
    read_solutions,
    serialize_system,
    stack_systems,
    total_degree_start,
    unit_complex,
    write_solutions,
)

__version__ = "0.2.0"

_TRACKER_NAMES = {"FAILURE_KINDS", "Homotopy", "TrackOutcome", "arith", "device_count", "eval_bench", "least_squares_solve",
                  "make_homotopy"}
_SUBMODULES = {"monodromy", "workloads", "pieri", "multi", "cli", "tracker"}


def __getattr__(name):  # PEP 562: load the CUDA tracker library lazily
    if name in _TRACKER_NAMES:
        from . import tracker
        return getattr(tracker, name)
    if name in _SUBMODULES:
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
