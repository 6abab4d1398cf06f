"""Pieri homotopies (acceptance
criterion 3).  CPU: minor expansion, special matrix and the whole bootstrap
tracked by the CPU oracle (test infrastructure).  GPU: the same sequence
through the product tracker is bit-identical stage by stage."""
import time

import numpy as np
import pytest

from conftest import assert_bits_equal
from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import pieri as PI


def oracle_tracker(orc):
    def run(g, f, gamma, start, params):
        end, st, _ = orc.track_path(int(g.prec), g, f, gamma, 1, start, params)
        return end, st.status == 0, st.steps, st.newton_iters
    return run


def _eval(sysm, x):
    """Evaluate equation 0 of a D-precision system at complex128 x."""
    v = 0j
    for sup, c in sysm.terms(0):
        t = c
        for var, e in sup:
            t *= x[var] ** e
        v += t
    return v


def test_event_order_is_the_papers_n4_sequence():
    # PAPER.md 4.1: x_{3,2}, x_{4,2}, x_{2,1}, x_{3,1} (1-based row, column)
    assert PI.pieri_events(2, 2) == [(2, 1), (3, 1), (1, 0), (2, 0)]
    ev = PI.pieri_events(3, 2)
    assert len(ev) == 6 and ev[:3] == [(2, 1), (3, 1), (4, 1)]


def test_minor_n2_example():
    # n=2, m=1, A=(a1;a2), X=(1;x) -> det = a1 x - a2
    A = np.zeros((2, 1, 2))
    A[0, 0] = [0.75, -1.5]
    A[1, 0] = [0.25, 2.0]
    s = PI.minor_expand(1, 1, 1, A, PM.D)
    assert s.terms(0) == [([], -(-1.5 + 2.0j)), ([(0, 1)], 0.75 + 0.25j)]


@pytest.mark.parametrize("m,p,k", [(2, 2, 4), (2, 2, 2), (3, 2, 6), (2, 3, 5), (4, 4, 16), (4, 4, 9)])
def test_minor_matches_numeric_determinant(m, p, k):
    """SPEC.md invariant: the expansion evaluates equal to det([A|X]) (1e-12 rel, D)."""
    A = PI.pieri_planes(m, p, 1, 100 + k, PM.D)[0]
    s = PI.minor_expand(m, p, k, A, PM.D)
    rng = np.random.default_rng(k)
    for _ in range(4):
        x = rng.uniform(-1, 1, k) + 1j * rng.uniform(-1, 1, k)
        xl = np.stack([x.real, x.imag])[:, None, :]
        d = PI.pieri_det(m, p, k, A, xl, PM.D)
        assert abs(_eval(s, x) - d) <= 1e-12 * max(1.0, abs(d))


def test_constant_pattern_is_the_numeric_determinant():
    A = PI.pieri_planes(2, 2, 1, 3, PM.D)[0]
    s = PI.minor_expand(2, 2, 0, A, PM.D)
    d = PI.pieri_det(2, 2, 0, A, np.zeros((2, 1, 0)), PM.D)
    assert len(s.terms(0)) == 1 and s.terms(0)[0][0] == [] and abs(s.terms(0)[0][1] - d) < 1e-15


def test_special_matrix_spec_example():
    # n=4 stage 1 (new variable x_{3,2}): S_X = (e2, e4) qualifies -- and is the first
    S = PI.choose_special_matrix(2, 2, 1, np.zeros((2, 1, 1)), PM.D)
    cols = [np.flatnonzero(S[0, 0, c * 4:(c + 1) * 4]).tolist() for c in range(2)]
    assert cols == [[1], [3]]


@pytest.mark.parametrize("m,p", [(2, 2), (3, 2), (2, 3)])
def test_special_matrix_postconditions(m, p):
    """det([S_X|X_k(x0)]) = 0 and d/d(new variable) != 0 at the start point."""
    rng = np.random.default_rng(m * 10 + p)
    for k in range(2, m * p + 1):
        x0 = np.zeros((2, 1, k))
        x0[:, 0, : k - 1] = rng.uniform(-1, 1, (2, k - 1))
        S = PI.choose_special_matrix(m, p, k, x0, PM.D)
        assert abs(PI.pieri_det(m, p, k, S, x0, PM.D)) <= 1e-12
        x1 = x0.copy()
        x1[0, 0, k - 1] = 1.0  # det is linear in the new variable
        assert abs(PI.pieri_det(m, p, k, S, x1, PM.D)) > 1e-6


def test_pieri_4_2_2_double(oracle):
    """Acceptance criterion 3, first half: pieri_sequence(4,2,2) in D, residual <= 1e-10."""
    r = PI.pieri_sequence(2, 2, 7, PM.D, tracker=oracle_tracker(oracle))
    assert r.residual <= 1e-10, r.residual
    assert [s.stage for s in r.stages] == [1, 2, 3, 4] and all(s.success for s in r.stages)
    assert r.stages[0].steps == 0  # the first stage is linear (PAPER.md 4.1)


def test_pieri_8_4_4_double_double(oracle):
    """Acceptance criterion 3, second half: pieri_sequence(8,4,4) in DD, residual <= 1e-8, < 60 s."""
    t0 = time.perf_counter()
    r = PI.pieri_sequence(4, 4, 7, PM.DD, tracker=oracle_tracker(oracle))
    assert time.perf_counter() - t0 < 60
    assert r.residual <= 1e-8, r.residual
    assert len(r.stages) == 16 and all(10 <= s.steps <= 500 for s in r.stages[1:])


def test_pieri_deterministic(oracle):
    a = PI.pieri_sequence(2, 2, 11, PM.DD, tracker=oracle_tracker(oracle))
    b = PI.pieri_sequence(2, 2, 11, PM.DD, tracker=oracle_tracker(oracle))
    assert_bits_equal(a.point, b.point, "same seed, same bits")


def test_pieri_rejects_bad_shape():
    with pytest.raises(ValueError):
        PI.pieri_sequence(0, 2, 1, PM.D, tracker=lambda *a: None)


@pytest.mark.gpu
@pytest.mark.parametrize("m,p,prec", [(2, 2, PM.D), (4, 4, PM.DD), (2, 3, PM.QD)])
def test_pieri_on_device_bitwise(gpu, oracle, m, p, prec):
    """Every stage tracked by the CUDA path ends on the oracle's bits."""
    got = PI.pieri_sequence(m, p, 7, prec, tracker=PI.gpu_path_tracker(gpu))
    want = PI.pieri_sequence(m, p, 7, prec, tracker=oracle_tracker(oracle))
    assert [(s.steps, s.newton_iters) for s in got.stages] == [(s.steps, s.newton_iters) for s in want.stages]
    assert_bits_equal(got.point, want.point, "final Pieri point")
    assert got.residual <= (1e-10 if prec == PM.D else 1e-8)
