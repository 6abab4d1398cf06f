"""CPU: SPEC.md's acceptance criteria 4, 6 (DD), 7, 8 and 9
on the oracle -- the SPEC tracker the CUDA path equals bit for bit
(tests/test_gpu_*.py), pinned to the unmodified reference headers
(tests/test_oracle_tracker.py).  Criteria 1-3 and 5 live in test_inputs.py,
test_monodromy.py, test_pieri.py and test_oracle_arith.py."""
import numpy as np
import pytest

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PolynomialSystem, PrecisionMode as PM
from paper_1501_06625_b200 import workloads as W

mpmath = pytest.importorskip("mpmath")
mp = mpmath.mp

EPS = {PM.D: 2.0 ** -52, PM.DD: 2.0 ** -104, PM.QD: 2.0 ** -209}


def to_mp(limbs):
    return sum((mp.mpf(float(v)) for v in limbs), mp.mpf(0))


def from_mp(x, L):
    out, r = [], x
    for _ in range(L):
        v = float(r)
        out.append(v)
        r = r - mp.mpf(v)
    return out


def mpc_vec(limbs):
    """(2, L, S) limb array -> list of mpc."""
    return [mp.mpc(to_mp(limbs[0, :, i]), to_mp(limbs[1, :, i])) for i in range(limbs.shape[-1])]


def limbs_vec(zs, prec):
    L = prec.limbs
    out = np.zeros((2, L, len(zs)))
    for i, z in enumerate(zs):
        out[0, :, i] = from_mp(mp.mpf(z.real), L)
        out[1, :, i] = from_mp(mp.mpf(z.imag), L)
    return out


# ---- criterion 4: precision escalation -----------------------------------------
@pytest.mark.parametrize("tol,fails,succeeds", [(1e-25, PM.D, PM.DD), (1e-50, PM.DD, PM.QD)])
def test_precision_escalation_on_cyclic4_leg(oracle, tol, fails, succeeds):
    """with corrector tolerance 1e-25 D fails and DD succeeds;
    with 1e-50 DD fails and QD succeeds (the cyclic-4 monodromy leg)."""
    for prec, ok in ((fails, False), (succeeds, True)):
        w = W.cyclic_leg(2, prec)
        w.params.newton_tol = tol
        _, st, _ = oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params)
        assert (st.status == 0) == ok, (prec, tol, st.status, st.failure_kind)


# ---- criterion 6 in DD ------------------------------------------------------------
def test_ad_vs_bruteforce_random_systems_dd(oracle):
    """SPEC.md:709 in DD: relative error <= 1e-28 against a 256-bit evaluation
    of the same polynomials; structural zeros exactly zero."""
    mp.prec = 256
    rng = np.random.default_rng(11)
    prec = PM.DD
    for trial in range(100):
        n = int(rng.integers(1, 9))
        eqs = []
        for i in range(n):
            terms = []
            for _ in range(int(rng.integers(1, 21))):
                vs = sorted(rng.choice(n, size=int(rng.integers(0, min(n, 6) + 1)), replace=False).tolist())
                terms.append(([(v, int(rng.integers(1, 4))) for v in vs], complex(*rng.uniform(-1, 1, 2))))
            eqs.append(terms)
        f = PolynomialSystem.from_terms(n, eqs, prec)
        x = [complex(*rng.uniform(-1, 1, 2)) for _ in range(n)]
        xl = pt.limbs_from_complex(np.array(x), prec)
        gam = pt.limbs_from_complex([1.0], prec).reshape(-1)
        h, J, _ = oracle.eval_homotopy(int(prec), f, f, gam, 1, xl, 1.0)
        hv, Jv = mpc_vec(h), mpc_vec(J)  # J column-major: entry (i, j) at j * n + i
        xm = [mp.mpc(z) for z in x]
        for i, terms in enumerate(eqs):
            val = mp.fsum(mp.mpc(c) * mp.fprod(xm[v] ** e for v, e in sup) for sup, c in terms)
            assert abs(hv[i] - val) <= 1e-28 * max(1, abs(val)), (trial, i)
            for j in range(n):
                d = mp.fsum(mp.mpc(c) * mp.fprod((e * xm[v] ** (e - 1)) if v == j else xm[v] ** e for v, e in sup)
                            for sup, c in terms if j in [v for v, _ in sup])
                assert abs(Jv[j * n + i] - d) <= 1e-28 * max(1, abs(d)), (trial, i, j)
                if all(j not in [v for v, _ in sup] for sup, _ in terms):
                    assert J[:, :, j * n + i].tolist() == [[0.0, 0.0], [0.0, 0.0]]


# ---- criterion 7: least squares ----------------------------------------------------
@pytest.mark.parametrize("prec", [PM.D, PM.DD, PM.QD], ids=lambda p: p.name)
@pytest.mark.parametrize("n", [4, 17, 64])
def test_lstsq_residual_orthogonal_to_columns(oracle, prec, n):
    """the least-squares residual r = b - A x is orthogonal to
    the column space, |A^H r|_max <= 16 n eps |A|_max (|A|_max |x|_max + |b|_max),
    for random complex N x n matrices (N = n + 3) in every mode."""
    mp.prec = 320
    rng = np.random.default_rng(n)
    N = n + 3
    A = rng.uniform(-1, 1, (N, n)) + 1j * rng.uniform(-1, 1, (N, n))
    b = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
    Al = pt.limbs_from_complex(A.T.reshape(-1), prec)
    bl = pt.limbs_from_complex(b, prec)
    x = mpc_vec(oracle.lstsq(int(prec), Al, bl))
    Am = [[mp.mpc(A[i, j]) for j in range(n)] for i in range(N)]
    r = [mp.mpc(b[i]) - mp.fsum(Am[i][j] * x[j] for j in range(n)) for i in range(N)]
    ahr = max(abs(mp.fsum(mp.conj(Am[i][j]) * r[i] for i in range(N))) for j in range(n))
    amax = max(abs(z) for z in A.reshape(-1))
    bound = 16 * n * EPS[prec] * amax * (amax * max(abs(z) for z in x) + max(abs(z) for z in b))
    assert ahr <= bound, (float(ahr), bound)


# ---- criterion 8: Newton convergence ------------------------------------------------
@pytest.mark.parametrize("prec", [PM.D, PM.DD, PM.QD], ids=lambda p: p.name)
def test_newton_quadratic_convergence_on_cyclic4(oracle, prec):
    """from a point of cyclic-4's family-1 curve (a, 1/a, -a, -1/a)
    perturbed by 1e-3 (the curve made isolated by a slice c . x = c . x*
    through the point), the corrector steps x += lstsq(J, -h) contract
    quadratically, e_{k+1} <= 10 e_k^2, until the mode's precision.  (At SPEC's
    own point a = i, i.e. (i, -i, -i, i), the sliced system has a double root
    -- the iterates halve their error each step -- so a generic a is used.)"""
    mp.prec = 400
    a = 0.7 + 0.4j
    xs = [a, 1 / a, -a, -1 / a]
    cyc = pt.cyclic_system(4, prec)
    coef = [1.0, 2.0, 3.0, 5.0]
    const = -sum(c * z for c, z in zip(coef, xs))
    rows = [cyc.terms(i) for i in range(4)] + [[([], const)] + [([(j, 1)], coef[j]) for j in range(4)]]
    f = PolynomialSystem.from_terms(4, rows, prec)
    gam = pt.limbs_from_complex([1.0], prec).reshape(-1)
    rng = np.random.default_rng(8)
    x = [mp.mpc(z) + mp.mpc(*(1e-3 * rng.uniform(-1, 1, 2))) for z in xs]
    iterates = [x]
    for _ in range(8):
        xl = limbs_vec(x, prec)
        h, J, _ = oracle.eval_homotopy(int(prec), f, f, gam, 1, xl, 1.0)
        dx = oracle.lstsq(int(prec), J, -h)
        assert dx is not None
        x = [a + d for a, d in zip(x, mpc_vec(dx))]
        x = mpc_vec(limbs_vec(x, prec))  # the iterate in working precision
        iterates.append(x)
    lim = iterates[-1]
    err = [max(abs(a - b) for a, b in zip(it, lim)) for it in iterates[:-1]]
    floor = 1e4 * EPS[prec]
    checked = 0
    for k in range(len(err) - 1):
        if err[k + 1] <= floor or err[k] <= floor:
            break
        assert err[k + 1] <= 10 * err[k] ** 2, (k, [float(e) for e in err])
        checked += 1
    # quadratic contractions observed before the floor (D reaches it after one)
    assert checked >= (1 if prec == PM.D else 2), [float(e) for e in err]
    assert err[-1] <= floor


def test_residual_increase_fires_on_overshoot(oracle):
    """SPEC.md:711 (second half): a start whose Newton step overshoots makes
    the residual grow; Fig. 2 stops with residual-increase, which the tracker
    reports as a failed start (t = 0, no steps)."""
    prec = PM.D
    # x^3 - 2x + 2 = 0 from x = 0: the Newton iterates cycle 0 -> 1 -> 0 with
    # residual 2 -> 1 -> 2, so the residual increases at the third iterate
    g = PolynomialSystem.from_terms(1, [[([], 2.0), ([(0, 1)], -2.0), ([(0, 3)], 1.0)]], prec)
    params = pt.StepControlParams.defaults(prec)
    start = pt.limbs_from_complex([0.0], prec)
    _, st, _ = oracle.track_path(int(prec), g, g, pt.gamma_from_seed(1, prec), 1, start, params)
    assert st.status != 0 and pt.FAILURE_KINDS[st.failure_kind] == "start" and st.steps == 0
    assert st.start_iters == 3 and st.solves == 2


# ---- criterion 9: tracker invariants over 500 randomized homotopies -----------------
def test_tracker_invariants_500_random_homotopies(oracle):
    """monotone t, step bound, budget and trace completeness on
    500 randomized small homotopies; bit-determinism of repeated runs."""
    rng = np.random.default_rng(500)
    prec = PM.D
    for trial in range(500):
        n = int(rng.integers(1, 4))
        deg = int(rng.integers(1, 4))
        params = pt.StepControlParams.defaults(prec)
        params.max_steps = int(rng.integers(5, 60))
        params.max_step = float(rng.choice([0.05, 0.1, 0.25]))
        g = pt.total_degree_start(n, deg, prec)
        from math import comb
        f = pt.random_dense(n, deg, min(3 * n, comb(n + deg - 1, deg)), int(rng.integers(1, 1 << 30)), prec)
        gamma = pt.gamma_from_seed(int(rng.integers(1, 1 << 30)), prec)
        start = W.total_degree_starts(n, deg, 1, prec)[0]
        cap = params.max_steps + 2
        end, st, tr = oracle.track_path(int(prec), g, f, gamma, 2, start, params, cap)
        end2, st2, tr2 = oracle.track_path(int(prec), g, f, gamma, 2, start, params, cap)
        assert np.array_equal(end.view(np.uint64), end2.view(np.uint64)) and st.steps == st2.steps  # determinism
        assert len(tr) == st.steps, trial                           # trace completeness
        assert st.steps <= params.max_steps + 1, trial              # budget
        assert st.accepted == sum(1 for e in tr if e.ok)
        t_acc = 0.0
        for e in tr:
            assert e.t > t_acc and e.t <= 1.0, trial                  # monotone t (every trial moves ahead)
            assert e.t - t_acc <= params.max_step * (1 + 1e-12), trial  # step bound
            if e.ok:
                t_acc = e.t
        assert st.t_end == t_acc
        if st.status == 0:
            assert t_acc == 1.0
