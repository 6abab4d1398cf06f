"""Monodromy driver.

CPU: the driver logic over the CPU oracle tracker -- cyclic-4 family 1
stabilises at 2 points (Fig. 4), stabilizationLoops = 0
returns the start set, the endpoints satisfy (f, L).
GPU: the same loops through the batch kernel are bit-identical to the
oracle's, deterministic, and the cyclic-16 Backelin component has degree 4
(Table 5).
"""
import numpy as np
import pytest

from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import monodromy as MD
from paper_1501_06625_b200 import workloads as W
from paper_1501_06625_b200.tracker import augment_with_linear, limbs_from_complex, complex_from_limbs


def oracle_tracker(orc):
    def run(g, f, gamma, starts, params):
        ends = np.zeros_like(starts)
        ok = np.zeros(starts.shape[0], dtype=bool)
        for p in range(starts.shape[0]):
            ends[p], st, _ = orc.track_path(int(g.prec), g, f, gamma, 1, starts[p], params)
            ok[p] = st.status == 0
        return ends, ok
    return run


def oracle_evaluator(orc):
    def run(sysm, points):
        one = np.zeros(2 * sysm.prec.limbs)
        one[0] = 1.0
        return np.array([orc.eval_homotopy(int(sysm.prec), sysm, sysm, one, 1, p, 1.0)[2] for p in points])
    return run


def witness(m, prec):
    n, dim = m * m, m - 1
    fL = augment_with_linear(n, dim, 1, prec)
    return fL, limbs_from_complex(W.backelin_witness(fL, m, dim), prec)


def residual(sys_, x):
    z = complex_from_limbs(x)
    worst = 0.0
    for i in range(sys_.n_eqs):
        v = 0j
        for sup, coef in sys_.terms(i):
            term = coef
            for var, e in sup:
                term *= z[var] ** e
            v += term
        worst = max(worst, abs(v))
    return worst


@pytest.mark.parametrize("prec", [PM.D, PM.DD], ids=lambda p: p.name)
def test_cyclic4_family1_has_degree_2(oracle, prec):
    """Acceptance criterion 2: one internally constructed family-1 witness
    point (cyclic4_witness) stabilises at exactly 2 points,
    every stored point's (f, L) residual below the corrector tolerance."""
    fL = augment_with_linear(4, 1, 1, prec)
    pts = W.cyclic4_witness(W.slice_rows(fL, 1)[0], family=1)
    assert all(residual(fL, limbs_from_complex(p, prec)) < 1e-12 for p in pts)
    w0 = limbs_from_complex(pts[0], prec)
    # polish to working precision with the tracker's t = 0 Newton pass
    ends, ok = oracle_tracker(oracle)(fL, fL, np.r_[1.0, np.zeros(2 * prec.limbs - 1)], w0[None],
                                      MD.StepControlParams.defaults(prec))
    ws = MD.monodromy_degree(4, 1, [ends[0]], seed=11, stabilization_loops=3, prec=prec,
                             tracker=oracle_tracker(oracle), evaluator=oracle_evaluator(oracle))
    assert ws.degree == 2
    tol = MD.StepControlParams.defaults(prec).newton_tol
    assert all(r < tol for r in ws.residuals[1:]) and len(ws.residuals) == 2


def test_cyclic4_witness_spec_examples():
    # family 1 at a = i is (i, -i, -i, i), a cyclic-4 root
    row = np.array([-1j, 1, 0, 0, 0], dtype=complex)  # the slice x_0 - i = 0
    pts = W.cyclic4_witness(row, 1)
    assert any(np.allclose(p, [1j, -1j, -1j, 1j]) for p in pts)
    with pytest.raises(ValueError):  # c1 = c3, c2 = c4 in our indexing (constant first): vanishing quadratic
        W.cyclic4_witness(np.array([1, 0.5, 0.25, 0.5, 0.25], dtype=complex), 1)


def test_zero_stabilization_loops_returns_start(oracle):
    _, w0 = witness(2, PM.DD)
    ws = MD.monodromy_degree(4, 1, [w0], seed=11, stabilization_loops=0, prec=PM.DD,
                             tracker=oracle_tracker(oracle), evaluator=oracle_evaluator(oracle))
    assert ws.degree == 1 and ws.loops == 0
    assert np.array_equal(ws.points[0].view(np.uint64), w0.view(np.uint64))


def test_empty_start_set_is_rejected():
    with pytest.raises(ValueError):
        MD.monodromy_degree(4, 1, [], seed=1, stabilization_loops=1)


@pytest.mark.gpu
def test_gpu_loop_bitwise_equals_oracle(gpu, oracle):
    fL, w0 = witness(4, PM.DD)
    fK = augment_with_linear(16, 3, 5, PM.DD)
    alpha, beta = W.gamma_from_seed(21, PM.DD), W.gamma_from_seed(22, PM.DD)
    got = MD.monodromy_loop(fL, fK, w0[None], alpha, beta, tracker=MD.gpu_batch_tracker(gpu))
    want = MD.monodromy_loop(fL, fK, w0[None], alpha, beta, tracker=oracle_tracker(oracle))
    assert np.array_equal(got.success, want.success)
    assert np.array_equal(got.mid.view(np.uint64), want.mid.view(np.uint64))
    assert np.array_equal(got.points.view(np.uint64), want.points.view(np.uint64))
    again = MD.monodromy_loop(fL, fK, w0[None], alpha, beta, tracker=MD.gpu_batch_tracker(gpu))
    assert np.array_equal(again.points.view(np.uint64), got.points.view(np.uint64))  # determinism


@pytest.mark.gpu
def test_gpu_cyclic16_monodromy_degree_is_4(gpu):
    """SPEC.md:581 / PAPER.md Table 5: the cyclic-16 Backelin component has
    degree 4.  The family x_{4a+b} = i^a r_b with prod x = 1 is the union of 4
    components {prod r = zeta, zeta^4 = 1}; the loops' endpoints that jump to a
    sibling component (prod r changes) are path-crossing failures and are
    rejected by the component key, so the witness set stabilises at the
    start component's 4 points, all on (f, L) below the corrector tolerance."""
    fL, w0 = witness(4, PM.DD)
    key = W.backelin_component_key(4)
    ws = MD.monodromy_degree(16, 3, [w0], seed=3, stabilization_loops=4, prec=PM.DD,
                             tracker=MD.gpu_batch_tracker(gpu), evaluator=MD.gpu_evaluator(gpu),
                             component_key=key, residual_tol=1e-12)
    assert ws.degree == 4, ws.log
    k0 = key(ws.points[0])
    for p in ws.points:
        assert residual(fL, p) < 1e-10
        assert abs(key(p) - k0) < 1e-9
        z = complex_from_limbs(p)
        for b in range(4):
            for a in range(4):
                assert abs(z[4 * a + b] - (1j ** a) * z[b]) < 1e-12 * max(1.0, abs(z[b]))
