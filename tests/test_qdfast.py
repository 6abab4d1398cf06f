"""The tolerance-parity QD arithmetic (mp_qdfast.cuh, pt_plan_set_arith).

CPU: its host build against mpmath at 320 bits -- every operation within a
few units of 2^-209 of the exact result (relative to the operands for
add / sub, whose sloppy form bounds the error by |a| + |b|).
GPU: the device kernels equal the host build bit for bit, and fast QD tracks
agree with the reference tracker (oracle) within the north-star tolerance --
end points to 1e-55 relative -- with identical step and Newton counts."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

mpmath = pytest.importorskip("mpmath")
mp = mpmath.mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EPS = 2.0 ** -209


@pytest.fixture(scope="module")
def qdf(tmp_path_factory):
    so = tmp_path_factory.mktemp("qdf") / "libqdf.so"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-DPT_QD_FAST",
                    "-DPT_QD_FAST_HOST", os.path.join(ROOT, "tests", "qdfast_host.cpp"), "-o", str(so)],
                   check=True, capture_output=True)
    lib = C.CDLL(str(so))
    dp = C.POINTER(C.c_double)
    lib.qdf_arith.argtypes = [C.c_int, C.c_long, dp, dp, dp]
    return lib


def to_mp(limbs):
    return sum((mp.mpf(float(v)) for v in limbs), mp.mpf(0))


def from_mp(x):
    out = []
    r = x
    for _ in range(4):
        v = float(r)
        out.append(v)
        r = r - mp.mpf(v)
    return out


def random_qd(rng, count, lo=-30, hi=30, positive=False):
    mp.prec = 320
    vals = []
    for _ in range(count):
        # 265 random bits: every limb of the quad-double is populated
        m = mp.mpf(0.5) + sum(mp.mpf(int(rng.integers(0, 2**53))) * mp.mpf(2) ** (-53 * (k + 1)) for k in range(5))
        x = m * mp.mpf(2) ** int(rng.integers(lo, hi))
        if not positive and rng.random() < 0.5:
            x = -x
        vals.append(from_mp(x))
    return np.array(vals)


def run(lib, op, a, b):
    out = np.zeros_like(a)
    dp = C.POINTER(C.c_double)
    assert lib.qdf_arith(op, a.shape[0], a.ctypes.data_as(dp), b.ctypes.data_as(dp), out.ctypes.data_as(dp)) == 0
    return out


@pytest.mark.parametrize("op,bound", [(0, 4), (1, 4), (2, 8), (3, 4), (4, 16), (5, 16), (6, 16)])
def test_host_fast_qd_accuracy(qdf, op, bound):
    rng = np.random.default_rng(op)
    n = 400
    a = random_qd(rng, n, positive=op in (5, 6))
    b = random_qd(rng, n)
    if op == 3:
        b[:, 1:] = 0.0
    got = run(qdf, op, a, b)
    mp.prec = 320
    worst = 0.0
    for i in range(n):
        x, y = to_mp(a[i]), to_mp(b[i])
        exact = {0: x + y, 1: x - y, 2: x * y, 3: x * y, 4: x / y, 5: mp.sqrt(x), 6: 1 / mp.sqrt(x)}[op]
        scale = abs(x) + abs(y) if op in (0, 1) else abs(exact)
        err = abs(to_mp(got[i]) - exact) / scale
        worst = max(worst, float(err / EPS))
        # a valid quad-double: limbs non-overlapping (|c_{l+1}| <= ulp(c_l))
        for l in range(3):
            assert abs(got[i][l + 1]) <= abs(got[i][l]) * 2.0 ** -52 or got[i][l + 1] == 0.0, (op, got[i])
    print(f"op {op}: worst {worst:.3f}")
    assert worst <= bound, f"op {op}: worst error {worst:.2f} units of 2^-209"


def test_host_fast_qd_cancellation(qdf):
    """a - b with |a - b| << |a|: the sloppy add stays within its |a| + |b| bound."""
    rng = np.random.default_rng(9)
    a = random_qd(rng, 200)
    b = a.copy()
    b[:, 3] *= 1.5  # differ in the last limb only
    got = run(qdf, 1, a, b)
    mp.prec = 320
    for i in range(a.shape[0]):
        x, y = to_mp(a[i]), to_mp(b[i])
        assert abs(to_mp(got[i]) - (x - y)) <= 4 * EPS * (abs(x) + abs(y))


@pytest.mark.gpu
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5])
def test_device_fast_qd_equals_host_build(qdf, gpu, op):
    import paper_1501_06625_b200 as pt
    rng = np.random.default_rng(100 + op)
    n = 2000
    a = random_qd(rng, n, positive=op == 5)
    b = random_qd(rng, n)
    if op == 3:
        b[:, 1:] = 0.0
    want = run(qdf, op, a, b)
    # device element layout: (re limbs, im limbs) per element; the real ops read re
    A = np.zeros((n, 2, 4))
    B = np.zeros((n, 2, 4))
    A[:, 0] = a
    B[:, 0] = b
    out = pt.arith(pt.PrecisionMode.QD, op, A, B, device=gpu, fast=True)
    got = out.reshape(n, 2, 4)[:, 0]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def _rel_err(a, b):
    """max over the coordinates of |a - b| / max(|b|, 1e-300), QD limbs (2, 4, n) summed in float."""
    mp.prec = 320
    worst = 0.0
    n = a.shape[-1]
    for i in range(n):
        za = mp.mpc(to_mp(a[0, :, i]), to_mp(a[1, :, i]))
        zb = mp.mpc(to_mp(b[0, :, i]), to_mp(b[1, :, i]))
        den = max(abs(zb), mp.mpf(1e-300))
        worst = max(worst, float(abs(za - zb) / den))
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("name,engine", [("chandra64", "cluster"), ("chandra64", "grid"), ("cyclic16", "cluster")])
def test_fast_qd_track_within_tolerance(gpu, oracle, name, engine):
    """North-star tolerance parity: a fast-QD track ends within 1e-55 (relative)
    of the reference tracker's end point, with the same step, accepted-step
    and Newton counts."""
    import paper_1501_06625_b200 as pt
    from paper_1501_06625_b200 import workloads as W
    w = W.by_name(name, pt.PrecisionMode.QD)
    end_ref, st_ref, _ = oracle.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.start, w.params)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    hom.set_engine(engine)
    hom.set_arith("fast")
    out = hom.track_path(w.start, w.params)
    assert (out.success, out.steps, out.accepted, out.newton_iters) == (
        st_ref.status == 0, st_ref.steps, st_ref.accepted, st_ref.newton_iters)
    err = _rel_err(out.end.reshape(2, 4, -1), end_ref.reshape(2, 4, -1))
    assert err <= 1e-55, err


@pytest.mark.gpu
def test_fast_qd_batch_within_tolerance(gpu, oracle):
    import paper_1501_06625_b200 as pt
    from paper_1501_06625_b200 import workloads as W
    w = W.random_system(n=12, degree=2, n_monomials=36, prec=pt.PrecisionMode.QD, seed=5, n_paths=16)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=gpu)
    hom.set_arith("fast")
    ends, outs = hom.track_batch(w.starts, w.params)
    for p in range(w.starts.shape[0]):
        end_ref, st_ref, _ = oracle.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts[p], w.params)
        assert (outs[p].success, outs[p].steps, outs[p].newton_iters) == (st_ref.status == 0, st_ref.steps,
                                                                          st_ref.newton_iters), p
        if outs[p].success:
            assert _rel_err(ends[p].reshape(2, 4, -1), end_ref.reshape(2, 4, -1)) <= 1e-55, p


def test_fast_arith_symbols_exported():
    """pt_plan_set_arith / pt_arith_device_mode are part of the C-ABI."""
    from paper_1501_06625_b200 import _native as nat
    assert nat.lib.pt_plan_set_arith(None, 1) != 0  # null plan: PT_E_INVAL, no device needed
    assert hasattr(nat.lib, "pt_arith_device_mode")
