"""GPU parity on the BASELINE.json configurations themselves (VERDICT r1
"Next round" 1): the CUDA path against the CPU oracle, bit for bit (NaN
payloads aside), at the sizes the bench runs.

  C3 rand96 degree 4, M = 65,536   evaluation (DD, QD) + a DD prefix track
  C4 cyclic-256 QD                 evaluation, the 271 x 256 least squares
                                   (D / DD / QD: the grid group MGS with
                                   N > 256), a 1-trial prefix track
  C5 batch of dim-32 paths (DD)    256 real paths of the 8192-path batch,
                                   failing paths included, stats and ends
Shapes: SPEC.md:529-555 (cyclic + slices), :497 (concurrent trackers).
The oracle runs on all host cores (OpenMP inside a path, a thread pool
over paths for the batch)."""
import os

import numpy as np
import pytest

from conftest import assert_bits_equal_nan

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import workloads as W

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def orc(oracle):
    oracle.set_threads(THREADS)
    return oracle


def _perturbed(w, scale=1e-3, seed=0):
    rng = np.random.default_rng(seed)
    x = np.array(w.start, copy=True)
    x[:, 0, :] += scale * rng.uniform(-1, 1, size=x[:, 0, :].shape)
    return x


def _eval_parity(orc, w, t, seed):
    x = _perturbed(w, seed=seed)
    h_ref, J_ref, r_ref = orc.eval_homotopy(int(w.prec), w.g, w.f, w.gamma, w.k, x, t)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=0)
    h, J, r = hom.evaluate(x, t)
    assert_bits_equal_nan(h, h_ref, "h")
    assert_bits_equal_nan(J, J_ref, "J")
    assert_bits_equal_nan(np.array([r]), np.array([r_ref]), "max|h|")


def _compare_track(out, end_ref, st_ref, tr_ref):
    assert (out.success, out.steps, out.accepted, out.newton_iters, out.start_iters, out.solves) == (
        st_ref.status == 0, st_ref.steps, st_ref.accepted, st_ref.newton_iters, st_ref.start_iters, st_ref.solves)
    assert_bits_equal_nan(np.array([out.final_residual, out.final_update, out.t_end]),
                          np.array([st_ref.final_residual, st_ref.final_update, st_ref.t_end]), "stats")
    assert len(out.trace) == len(tr_ref)
    for a, b in zip(out.trace, tr_ref):
        assert (a.ok, a.iters) == (b.ok, b.iters)
        assert_bits_equal_nan(np.array([a.t, a.residual, a.update]), np.array([b.t, b.residual, b.update]), "trace")
    assert_bits_equal_nan(out.end, end_ref, "end point")


# ---- C3 ---------------------------------------------------------------------
@pytest.fixture(scope="module")
def rand96():
    return {p: W.random_system(96, 4, 65536, p) for p in (PM.DD, PM.QD)}


@pytest.mark.parametrize("prec,t,seed", [(PM.DD, 0.31, 1), (PM.DD, 0.87, 2), (PM.QD, 0.31, 3), (PM.QD, 0.87, 4)])
def test_rand96_evaluation(gpu, orc, rand96, prec, t, seed):
    _eval_parity(orc, rand96[prec], t, seed)


def test_rand96_dd_prefix_track(gpu, orc, rand96):
    """Start validation + the first two trials of the C3 DD path, every trial traced."""
    w = rand96[PM.DD]
    w.params.max_steps = 1
    cap = w.params.max_steps + 2
    ref = orc.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.start, w.params, cap)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    assert hom.engine == "grid"
    _compare_track(hom.track_path(w.start, w.params, trace=True), *ref)


# ---- C4 ---------------------------------------------------------------------
@pytest.fixture(scope="module")
def cyclic256():
    return W.cyclic_leg(16, PM.QD)


def test_cyclic256_qd_evaluation(gpu, orc, cyclic256):
    _eval_parity(orc, cyclic256, 0.43, 5)


@pytest.mark.parametrize("prec", [PM.D, PM.DD, PM.QD], ids=lambda p: p.name)
def test_lstsq_271x256(gpu, orc, prec):
    """The C4 solve shape: N = 271 > 256 exercises the group MGS with
    more elements than canonical partials (device.cuh mgs_reduce)."""
    N, n, L = 271, 256, prec.limbs
    rng = np.random.default_rng(271 + int(prec))
    A = np.zeros((2, L, N * n))
    b = np.zeros((2, L, N))
    A[:, 0] = rng.uniform(-1, 1, (2, N * n))
    b[:, 0] = rng.uniform(-1, 1, (2, N))
    want = orc.lstsq(int(prec), A, b)
    got = pt.least_squares_solve(A, b, prec, device=gpu)
    assert_bits_equal_nan(got, want, "x")


def test_cyclic256_qd_prefix_track(gpu, orc, cyclic256):
    """Start validation on the Backelin witness + the first trial of the C4 leg."""
    w = cyclic256
    w.params.max_steps = 0
    cap = 4
    ref = orc.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.start, w.params, cap)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    _compare_track(hom.track_path(w.start, w.params, trace=True), *ref)


# ---- C5 ---------------------------------------------------------------------
def test_batch32_real_paths(gpu, orc):
    """256 paths of the 8192-path C5 batch (every 32nd path, so the shard
    spans the whole index range), failing paths included: statuses, failure
    kinds, counters, residuals and end points bitwise."""
    w = W.batch(prec=PM.DD)
    idx = np.arange(0, 8192, 32)
    starts = np.ascontiguousarray(w.starts[idx])
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(starts, w.params)
    ends_ref, st_ref = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, starts, w.params, THREADS)
    fails = 0
    for p in range(idx.size):
        o, s = outs[p], st_ref[p]
        assert (o.success, o.failure_kind, o.steps, o.accepted, o.newton_iters, o.start_iters, o.solves) == (
            s.status == 0, pt.FAILURE_KINDS[s.failure_kind], s.steps, s.accepted, s.newton_iters, s.start_iters,
            s.solves), f"path {idx[p]}"
        assert_bits_equal_nan(np.array([o.final_residual, o.final_update, o.t_end]),
                              np.array([s.final_residual, s.final_update, s.t_end]), f"stats of path {idx[p]}")
        fails += not o.success
    assert_bits_equal_nan(ends, ends_ref, "end points")
    assert fails > 0, "the shard should contain failing paths"


# ---- plans sharing a kernel function ------------------------------
def test_large_plan_survives_a_smaller_plan(gpu, orc):
    """cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the kernel
    function: creating a small plan after a large one must not break the
    large plan's launches (the attribute is set per launch)."""
    big = W.chandra(64, PM.DD)
    hb = pt.make_homotopy(big.g, big.f, big.gamma, big.k, device=gpu)
    small = W.random_system(n=6, degree=2, n_monomials=8, prec=PM.DD, seed=3)
    hs = pt.make_homotopy(small.g, small.f, small.gamma, small.k, device=gpu)
    hs.track_path(small.start, small.params)
    for engine in ("cluster", "grid"):
        hb.set_engine(engine)
        out = hb.track_path(big.start, big.params)
        end_ref, st_ref, _ = orc.track_path(int(big.prec), big.g, big.f, big.gamma, big.k, big.start, big.params)
        assert out.success and out.steps == st_ref.steps
        assert_bits_equal_nan(out.end, end_ref, "end point after a smaller plan")
    _, outs = hb.track_batch(np.repeat(big.starts, 2, axis=0), big.params)
    assert all(o.success for o in outs)


# ---- non-finite values: the exact DD re-track (pathtrack_b200.h PT_STAT_NONFINITE) ----
def _overflow_homotopy(prec):
    """f = 1e308 x^2 + 1e308 x - 3 overflows at x = 1 (not at x = 0.001);
    g = (x - 1)(x - 0.001) has both as start roots."""
    f = pt.PolynomialSystem.from_terms(1, [[([], -3.0), ([(0, 1)], 1e308), ([(0, 2)], 1e308)]], prec)
    g = pt.PolynomialSystem.from_terms(1, [[([], 0.001), ([(0, 1)], -1.001), ([(0, 2)], 1.0)]], prec)
    starts = np.stack([pt.limbs_from_complex([v], prec) for v in (1.0, 0.001, 1.0, 0.001, 1.0)])
    return g, f, pt.gamma_from_seed(5, prec), starts


@pytest.mark.parametrize("engine", ["grid", "cluster"])
def test_nonfinite_path_is_retracked_exactly(gpu, orc, engine):
    """A DD path that meets inf / NaN is flagged by the fast kernels and
    re-tracked by the exact ones: its results follow the reference's
    non-finite rules (multiprec.hpp:102-107) bit for bit (NaN payloads aside)."""
    prec = PM.DD
    g, f, gamma, starts = _overflow_homotopy(prec)
    params = pt.StepControlParams.defaults(prec)
    hom = pt.make_homotopy(g, f, gamma, 2, device=gpu)
    hom.set_engine(engine)
    for p in (0, 1):
        out = hom.track_path(starts[p], params, trace=True)
        ref = orc.track_path(int(prec), g, f, gamma, 2, starts[p], params, params.max_steps + 2)
        _compare_track(out, *ref)
        # start 0 overflows for sure; start 1 may meet an inf on a rejected
        # trial (the flag is conservative -- its results are exact either way)
        if p == 0:
            assert out.flags & 1, out.flags


def test_nonfinite_paths_in_a_batch(gpu, orc):
    prec = PM.DD
    g, f, gamma, starts = _overflow_homotopy(prec)
    params = pt.StepControlParams.defaults(prec)
    hom = pt.make_homotopy(g, f, gamma, 2, device=gpu)
    ends, outs = hom.track_batch(starts, params)
    ends_ref, st_ref = orc.track_batch(int(prec), g, f, gamma, 2, starts, params, 2)
    for p, (o, s) in enumerate(zip(outs, st_ref)):
        assert (o.success, o.steps, o.newton_iters, o.solves) == (s.status == 0, s.steps, s.newton_iters, s.solves)
        assert_bits_equal_nan(np.array([o.final_residual, o.final_update, o.t_end]),
                              np.array([s.final_residual, s.final_update, s.t_end]), f"stats {p}")
        if p % 2 == 0:
            assert o.flags & 1, (p, o.flags)
    assert_bits_equal_nan(ends, ends_ref, "ends")


def test_finite_paths_are_not_flagged(gpu):
    w = W.chandra(64, PM.DD)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    assert hom.track_path(w.start, w.params).flags == 0


# ---- batch kernel shapes ---------------------------------------------------------
# The batch kernel's own paths: lane tasks in warp bundles over coalesced
# contribution streams (plan.hpp Bundle) and the column-item MGS (mgs_batch,
# N <= 64: one and two elements per leaf, partial and full items), each
# against the unbundled / warp-MGS variants and the oracle.  Short prefixes
# keep the CPU oracle fast; every counter, residual and end point bitwise.
@pytest.mark.parametrize("variant", ["new", "old", "allimbs"])
@pytest.mark.parametrize("n,prec", [(5, PM.D), (12, PM.DD), (32, PM.QD), (40, PM.DD), (64, PM.D), (48, PM.QD),
                                    (64, PM.DD)])
def test_batch_kernel_shapes_bitwise(gpu, orc, monkeypatch, n, prec, variant):
    """new: bundles + column-item MGS; old: unbundled lane / group sums + warp
    MGS; allimbs: bundles whose streams keep every coefficient limb (the
    random coefficients are binary64, so by default only the leading limbs
    are streamed)."""
    flag = "0" if variant == "old" else "1"
    monkeypatch.setenv("PT_BUNDLES", flag)
    monkeypatch.setenv("PT_MGS_BATCH", flag)
    monkeypatch.setenv("PT_STREAM_HI", "0" if variant == "allimbs" else "1")
    w = W.random_system(n=n, degree=2, n_monomials=3 * n, prec=prec, seed=100 + n, n_paths=12)
    w.params.max_steps = 4
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(w.starts, w.params)
    ends_ref, st_ref = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts, w.params, THREADS)
    for p, (o, s) in enumerate(zip(outs, st_ref)):
        assert (o.success, o.failure_kind, o.steps, o.accepted, o.newton_iters, o.solves) == (
            s.status == 0, pt.FAILURE_KINDS[s.failure_kind], s.steps, s.accepted, s.newton_iters, s.solves), p
        assert_bits_equal_nan(np.array([o.final_residual, o.final_update, o.t_end]),
                              np.array([s.final_residual, s.final_update, s.t_end]), f"stats of path {p}")
    assert_bits_equal_nan(ends, ends_ref, "end points")


def test_batch_nonsquare_cyclic_leg_bitwise(gpu, orc):
    """19 x 16 (cyclic-16 monodromy leg, N > n): the column-item MGS with
    partial items and the bundles of a system without a shared support."""
    w = W.cyclic_leg(4, PM.DD)
    starts = np.repeat(w.starts, 4, axis=0)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(starts, w.params)
    ends_ref, st_ref = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, starts, w.params, THREADS)
    for p, (o, s) in enumerate(zip(outs, st_ref)):
        assert (o.success, o.steps, o.newton_iters, o.solves) == (s.status == 0, s.steps, s.newton_iters, s.solves)
    assert_bits_equal_nan(ends, ends_ref, "end points")


@pytest.mark.parametrize("n", [1, 2, 3])
def test_batch_kernel_tiny_systems_bitwise(gpu, orc, n):
    """n = 1 (the right-hand side is column 1, taken by the critical warp),
    n = 2, 3 (the items own only the right-hand side)."""
    w = W.random_system(n=n, degree=3, n_monomials=1 if n == 1 else 2 + n, prec=PM.DD, seed=200 + n, n_paths=8)
    w.params.max_steps = 6
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(w.starts, w.params)
    ends_ref, st_ref = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts, w.params, THREADS)
    for p, (o, s) in enumerate(zip(outs, st_ref)):
        assert (o.success, o.steps, o.newton_iters, o.solves) == (s.status == 0, s.steps, s.newton_iters, s.solves), p
    assert_bits_equal_nan(ends, ends_ref, "end points")


@pytest.mark.parametrize("prec", [PM.DD, PM.D])
def test_batch_split_bundles_bitwise(gpu, orc, prec):
    """Long slot sums split over D lanes (the value slot: K = 1501, width 128,
    D = 8; the Jacobian slots: K ~ 375, width 32, D = 4) and merged after the
    bundle pass -- bitwise against the oracle and the unbundled kernel."""
    w = W.random_system(n=16, degree=4, n_monomials=1500, prec=prec, seed=31, n_paths=8)
    w.params.max_steps = 3
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(w.starts, w.params)
    ends_ref, st_ref = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts, w.params, THREADS)
    for p, (o, s) in enumerate(zip(outs, st_ref)):
        assert (o.success, o.steps, o.newton_iters, o.solves) == (s.status == 0, s.steps, s.newton_iters, s.solves), p
        assert_bits_equal_nan(np.array([o.final_residual, o.final_update]),
                              np.array([s.final_residual, s.final_update]), f"stats of path {p}")
    assert_bits_equal_nan(ends, ends_ref, "end points")
