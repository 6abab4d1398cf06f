"""GPU parity: the CUDA path against the CPU oracle, bit for bit.

Every comparison is exact (uint64 views of the binary64 limbs): the device
replicates the reference operation sequences and the oracle's pinned
summation trees, so any difference is a bug.
"""
import numpy as np
import pytest

from conftest import assert_bits_equal, assert_bits_equal_nan
from arith_inputs import OPS, edge_operands, random_operands

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import workloads as W

pytestmark = pytest.mark.gpu

PRECS = [PM.D, PM.DD, PM.QD]


@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
@pytest.mark.parametrize("op", ["add", "sub", "mul", "mul_d", "div", "sqrt", "renorm", "cmul", "cadd",
                                "conj_mul", "norm_sqr", "modulus_double", "powi", "cscale", "cpowi"])
def test_arith_device_bitwise(gpu, oracle, prec, op):
    count = 4096 if prec == PM.QD else 20000
    a = random_operands(int(prec), count, 1, positive=(op == "sqrt"), oracle=oracle)
    b = random_operands(int(prec), count, 2, small_int=op in ("powi", "cpowi"), oracle=oracle)
    want = oracle.arith(int(prec), OPS[op], a, b)
    got = pt.arith(prec, OPS[op], a, b, device=gpu)
    if op == "modulus_double":
        want, got = want[:, 0, 0], got[:, 0, 0]
    elif op in ("add", "sub", "mul", "mul_d", "div", "sqrt", "renorm", "norm_sqr", "powi"):
        want, got = want[:, 0], got[:, 0]
    assert_bits_equal(got, want, f"{prec.name} {op}")


@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
@pytest.mark.parametrize("op", ["add", "sub", "mul", "mul_d", "div", "sqrt", "renorm", "cmul", "cadd",
                                "conj_mul", "norm_sqr", "modulus_double", "cscale"])
def test_arith_device_edge_operands(gpu, ref_oracle_or_restated, prec, op):
    """The whole binary64 range: exponents -1074..1023, subnormals, +-0,
    +-inf, NaN, the glibc hypot scaling thresholds.  Bitwise against the
    reference-header oracle (NaN payloads aside), non-finite DD values
    included (dd_norm's {h, 0} rule, multiprec.hpp:102-107)."""
    orc = ref_oracle_or_restated
    count = 4096 if prec == PM.QD else 20000
    a = edge_operands(int(prec), count, 11, positive=(op == "sqrt"), oracle=orc)
    b = edge_operands(int(prec), count, 12, oracle=orc)
    want = orc.arith(int(prec), OPS[op], a, b)
    got = pt.arith(prec, OPS[op], a, b, device=gpu)
    assert_bits_equal_nan(got, want, f"{prec.name} {op} (edge operands)")


def _perturbed(w, scale=1e-3, seed=0):
    rng = np.random.default_rng(seed)
    x = np.array(w.start, copy=True)
    x[:, 0, :] += scale * rng.uniform(-1, 1, size=x[:, 0, :].shape)
    return x


@pytest.mark.parametrize("name,prec,t", [("cyclic16", PM.DD, 0.37), ("cyclic16", PM.QD, 0.81),
                                         ("chandra64", PM.D, 0.5), ("chandra64", PM.DD, 0.5),
                                         ("chandra64", PM.QD, 0.25)])
def test_eval_homotopy_bitwise(gpu, oracle, name, prec, t):
    w = W.by_name(name, prec)
    x = _perturbed(w)
    h_ref, J_ref, r_ref = oracle.eval_homotopy(int(prec), w.g, w.f, w.gamma, w.k, x, t)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    h, J, r = hom.evaluate(x, t)
    assert_bits_equal(h, h_ref, "h")
    assert_bits_equal(J, J_ref, "J")
    assert_bits_equal(np.array([r]), np.array([r_ref]), "max|h|")


@pytest.mark.parametrize("prec", PRECS, ids=lambda p: p.name)
@pytest.mark.parametrize("N,n", [(4, 4), (19, 16), (64, 64), (97, 96), (40, 33)])
def test_lstsq_bitwise(gpu, oracle, prec, N, n):
    rng = np.random.default_rng(N * 1000 + n)
    L = prec.limbs
    A = np.zeros((2, L, N * n))
    b = np.zeros((2, L, N))
    A[:, 0] = rng.uniform(-1, 1, (2, N * n))
    b[:, 0] = rng.uniform(-1, 1, (2, N))
    want = oracle.lstsq(int(prec), A, b)
    got = pt.least_squares_solve(A, b, prec, device=gpu)
    assert_bits_equal(got, want, "x")


def _compare_track(w, out, end_ref, st_ref, tr_ref):
    assert out.success == (st_ref.status == 0)
    assert (out.steps, out.accepted, out.newton_iters, out.start_iters) == (
        st_ref.steps, st_ref.accepted, st_ref.newton_iters, st_ref.start_iters)
    assert_bits_equal(np.array([out.final_residual, out.final_update, out.t_end]),
                      np.array([st_ref.final_residual, st_ref.final_update, st_ref.t_end]), "stats")
    assert len(out.trace) == len(tr_ref)
    for a, b in zip(out.trace, tr_ref):
        assert (a.ok, a.iters) == (b.ok, b.iters)
        assert_bits_equal(np.array([a.t, a.residual, a.update]), np.array([b.t, b.residual, b.update]), "trace")
    assert_bits_equal(out.end, end_ref, "end point")


_REF_TRACKS = {}


def _ref_track(oracle, name, prec):
    key = (name, prec)
    if key not in _REF_TRACKS:
        w = W.by_name(name, prec)
        cap = w.params.max_steps + 2
        _REF_TRACKS[key] = (w, oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, cap))
    return _REF_TRACKS[key]


@pytest.mark.parametrize("engine", ["grid", "cluster"])
@pytest.mark.parametrize("name,prec", [("cyclic16", PM.DD), ("cyclic16", PM.D), ("chandra64", PM.D),
                                       ("chandra64", PM.DD), ("chandra64", PM.QD)])
def test_track_path_bitwise(gpu, oracle, name, prec, engine):
    w, (end_ref, st_ref, tr_ref) = _ref_track(oracle, name, prec)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    hom.set_engine(engine)
    out = hom.track_path(w.start, w.params, trace=True)
    _compare_track(w, out, end_ref, st_ref, tr_ref)
    if name == "chandra64":
        assert out.success


def test_track_batch_bitwise(gpu, oracle):
    w = W.random_system(n=8, degree=3, n_monomials=40, prec=PM.DD, n_paths=48)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    ends, outs = hom.track_batch(w.starts, w.params)
    for p in range(w.starts.shape[0]):
        end_ref, st_ref, _ = oracle.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts[p], w.params)
        assert (outs[p].steps, outs[p].newton_iters, outs[p].success) == (st_ref.steps, st_ref.newton_iters,
                                                                         st_ref.status == 0)
        assert_bits_equal(ends[p], end_ref, f"path {p}")


# Mid-size systems: the warp MGS with E = 3..4 rows per lane (width_mgs = 64,
# lane-local off = 32 level), both hand-off variants (TMA multicast when the
# Q buffer fits in shared memory, DSMEM + flags otherwise), and the canonical
# trees with partial (N < 32 E) and full (N = 32 E) warps.  Short prefixes
# keep the CPU oracle fast; every trial, the stats and the end point must be
# bit-identical, whatever the path does.
@pytest.mark.parametrize("engine", ["grid", "cluster"])
@pytest.mark.parametrize("n,prec", [(80, PM.D), (80, PM.DD), (128, PM.DD), (72, PM.QD)])
def test_track_midsize_bitwise(gpu, oracle, n, prec, engine):
    w = W.random_system(n=n, degree=2, n_monomials=24, prec=prec, seed=n)
    w.params.max_steps = 3
    cap = w.params.max_steps + 2
    end_ref, st_ref, tr_ref = oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, cap)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    hom.set_engine(engine)
    out = hom.track_path(w.start, w.params, trace=True)
    _compare_track(w, out, end_ref, st_ref, tr_ref)
