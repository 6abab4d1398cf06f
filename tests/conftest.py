import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.orc import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def ref_oracle():
    from oracle.orc import REFERENCE, Oracle
    if not os.path.exists(REFERENCE):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def ref_oracle_or_restated():
    """The reference-header oracle where it was built (oracle/_ref travels
    with gpurun), else the restatement (pinned to it by the CPU suite)."""
    from oracle.orc import REFERENCE, Oracle
    return Oracle("reference" if os.path.exists(REFERENCE) else "restatement")


@pytest.fixture(scope="session")
def gpu():
    from paper_1501_06625_b200 import device_count
    if device_count() == 0:
        pytest.fail("GPU test scheduled but no CUDA device is visible")
    return 0


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bits_equal(a, b, what=""):
    a, b = bits(a), bits(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.flatnonzero(a.reshape(-1) != b.reshape(-1))
    assert bad.size == 0, f"{what}: {bad.size} of {a.size} limbs differ (first at {bad[:5]})"


def assert_bits_equal_nan(a, b, what=""):
    """Bitwise equality where any two NaNs count as equal: the GPU's FP64
    units return the canonical NaN, x86 propagates the operand's payload
    (DESIGN.md section 3); every non-NaN limb must match bit for bit."""
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    both_nan = np.isnan(a) & np.isnan(b)
    bad = np.flatnonzero((a.view(np.uint64) != b.view(np.uint64)) & ~both_nan)
    assert bad.size == 0, f"{what}: {bad.size} of {a.size} limbs differ (first at {bad[:5]}: {a[bad[:3]]} vs {b[bad[:3]]})"
