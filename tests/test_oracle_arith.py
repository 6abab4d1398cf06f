"""CPU: the oracle's arithmetic and the host build of the device arithmetic
(csrc/mp.cuh), pinned against the reference headers and SPEC known answers.

Pins, in order of strength:
  1. bitwise vs the UNMODIFIED reference headers (oracle/_ref, built here);
  2. bitwise vs tests/golden/arith_*.npz (outputs of the reference build,
     committed, so the pin also holds where /root/reference is absent);
  3. SPEC.md example values;
  4. mpmath error bounds (acceptance criterion 5).
"""
import os

import numpy as np
import pytest

from arith_inputs import OPS, random_operands
from conftest import assert_bits_equal

import paper_1501_06625_b200 as pt

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALL_OPS = ["add", "sub", "mul", "mul_d", "div", "sqrt", "renorm", "cmul", "cadd", "conj_mul", "norm_sqr",
           "modulus_double", "powi", "cscale", "cpowi"]


def _operands(prec, op, count, oracle):
    a = random_operands(prec, count, 11, positive=(op == "sqrt"), oracle=oracle)
    b = random_operands(prec, count, 12, small_int=op in ("powi", "cpowi"), oracle=oracle)
    return a, b


@pytest.mark.parametrize("prec", [0, 1, 2], ids=["d", "dd", "qd"])
@pytest.mark.parametrize("op", ALL_OPS)
def test_restatement_matches_reference_headers(ref_oracle, oracle, prec, op):
    a, b = _operands(prec, op, 2000 if prec == 2 else 10000, ref_oracle)
    want = ref_oracle.arith(prec, OPS[op], a, b)
    assert_bits_equal(oracle.arith(prec, OPS[op], a, b), want, "oracle restatement")
    assert_bits_equal(pt.arith(pt.PrecisionMode(prec), OPS[op], a, b, device=None), want, "mp.cuh host build")


@pytest.mark.parametrize("prec", [0, 1, 2], ids=["d", "dd", "qd"])
def test_golden_arith_vectors(oracle, prec):
    path = os.path.join(GOLDEN, f"arith_{('d', 'dd', 'qd')[prec]}.npz")
    data = np.load(path)
    for op in ALL_OPS:
        a, b, want = data[f"{op}_a"], data[f"{op}_b"], data[f"{op}_out"]
        assert_bits_equal(oracle.arith(prec, OPS[op], a, b), want, f"oracle {op}")
        assert_bits_equal(pt.arith(pt.PrecisionMode(prec), OPS[op], a, b, device=None), want, f"host {op}")


def _one(prec, op, a_limbs, b_limbs, impl):
    L = (1, 2, 4)[prec]
    a = np.zeros((1, 2, L))
    b = np.zeros((1, 2, L))
    a.reshape(-1)[: len(a_limbs)] = a_limbs
    b.reshape(-1)[: len(b_limbs)] = b_limbs
    return impl(prec, OPS[op], a, b).reshape(-1)


IMPLS = {
    "oracle": None,  # filled per test
    "host": lambda prec, op, a, b: pt.arith(pt.PrecisionMode(prec), op, a, b, device=None),
}


@pytest.fixture(params=["oracle", "host"])
def impl(request, oracle):
    return oracle.arith if request.param == "oracle" else IMPLS["host"]


def test_spec_two_sum_two_prod_examples(impl):
    # two_sum through DD addition of binary64 values
    assert list(_one(1, "add", [1.0, 0], [2.0, 0], impl)[:2]) == [3.0, 0.0]
    assert list(_one(1, "add", [1.0, 0], [2.0 ** -100, 0], impl)[:2]) == [1.0, 2.0 ** -100]
    assert list(_one(1, "add", [2.0 ** 53, 0], [1.0, 0], impl)[:2]) == [2.0 ** 53, 1.0]
    # two_prod through DD multiplication
    assert list(_one(1, "mul", [3.0, 0], [4.0, 0], impl)[:2]) == [12.0, 0.0]
    v = 2.0 ** 27 + 1
    assert list(_one(1, "mul", [v, 0], [v, 0], impl)[:2]) == [2.0 ** 54 + 2.0 ** 28, 1.0]
    assert list(_one(1, "mul", [2.0 ** -30, 0], [2.0 ** -30, 0], impl)[:2]) == [2.0 ** -60, 0.0]


def test_spec_dd_qd_examples(impl):
    assert list(_one(1, "add", [1.0, 0], [2.0 ** -80, 0], impl)[:2]) == [1.0, 2.0 ** -80]
    assert list(_one(1, "sub", [1.0, 2.0 ** -80], [1.0, 0], impl)[:2]) == [2.0 ** -80, 0.0]
    q = _one(2, "add", [1.0, 0, 0, 0], [2.0 ** -180, 0, 0, 0], impl)[:4]
    assert sorted(q.tolist(), key=abs, reverse=True)[:2] == [1.0, 2.0 ** -180] and q.sum() == 1.0
    x = [np.pi, 1.2246467991473532e-16, -2.994769809718339e-33, 1.1124542208633657e-49]
    assert not np.any(_one(2, "sub", x, x, impl)[:4])
    assert list(_one(1, "sqrt", [4.0, 0], [0, 0], impl)[:2]) == [2.0, 0.0]
    assert list(_one(2, "sqrt", [0.0] * 4, [0] * 4, impl)[:4]) == [0.0] * 4


def test_spec_complex_examples(impl):
    z = _one(0, "cmul", [1.0, 2.0], [3.0, 4.0], impl)
    assert list(z[:2]) == [-5.0, 10.0]
    z = _one(0, "conj_mul", [1.25, -3.5], [1.25, -3.5], impl)
    assert z[1] == 0.0 and z[0] == 1.25 ** 2 + 3.5 ** 2
    assert _one(0, "modulus_double", [3.0, 4.0], [0, 0], impl)[0] == 5.0


mp = pytest.importorskip("mpmath")


def _to_mp(limbs):
    return sum((mp.mpf(float(v)) for v in limbs), mp.mpf(0))


@pytest.mark.parametrize("prec,bound", [(1, 2.0 ** -104), (2, 2.0 ** -209)], ids=["dd", "qd"])
@pytest.mark.parametrize("op", ["add", "mul", "div", "sqrt"])
def test_error_bounds_vs_bigfloat(oracle, prec, bound, op):
    mp.mp.prec = 320
    L = (1, 2, 4)[prec]
    a, b = _operands(prec, op, 400, oracle)
    b[:, 0, 0] = np.where(b[:, 0, 0] == 0.0, 1.0, b[:, 0, 0])
    out = oracle.arith(prec, OPS[op], a, b)
    lim = bound * (4 if op in ("div", "sqrt") else 1)  # 2^-102 / 2^-206 for div, sqrt
    worst = 0.0
    for i in range(a.shape[0]):
        x, y = _to_mp(a[i, 0]), _to_mp(b[i, 0])
        exact = {"add": lambda: x + y, "mul": lambda: x * y, "div": lambda: x / y,
                 "sqrt": lambda: mp.sqrt(x)}[op]()
        if exact == 0:
            continue
        got = _to_mp(out[i, 0])
        worst = max(worst, float(abs((got - exact) / exact)))
    assert worst <= lim, (op, worst, lim)
    assert L > 1


def test_glibc_hypot_replay_matches_the_host_libm():
    """modulus_double (complex.hpp:113-116) calls std::hypot, which glibc does
    not round correctly; the device replays glibc's kernel (mp.cuh
    glibc_hypot).  Its host build (the same source) against this host's libm
    (numpy.hypot) on 4e6 pairs: random mantissas with exponents over the
    whole range (the 2^511 / 2^-459 scaling branches, subnormals), signs
    mixed, plus ties and exact cases -- bit for bit."""
    import paper_1501_06625_b200 as pt
    rng = np.random.default_rng(2024)
    n = 4_000_000
    e1 = rng.integers(-1070, 1020, n)
    e2 = np.clip(e1 + rng.integers(-60, 61, n), -1074, 1023)
    x = np.ldexp(rng.uniform(0.5, 1.0, n), e1) * rng.choice([-1.0, 1.0], n)
    y = np.ldexp(rng.uniform(0.5, 1.0, n), e2) * rng.choice([-1.0, 1.0], n)
    x[:1000], y[:1000] = 3.0 * np.arange(1000), 4.0 * np.arange(1000)  # exact 3-4-5 cases
    a = np.zeros((n, 2))
    a[:, 0], a[:, 1] = x, y
    out = pt.arith(pt.PrecisionMode.D, 11, a, np.zeros_like(a), device=None)
    got = out.reshape(n, 2)[:, 0]
    want = np.hypot(x, y)
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (bad.size, x[bad[:3]], y[bad[:3]], got[bad[:3]], want[bad[:3]])
