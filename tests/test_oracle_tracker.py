"""CPU: the oracle tracker, pinned against the reference-header build, the
committed golden runs, and the SPEC.md examples of every hot-path module."""
import os

import numpy as np
import pytest

from conftest import assert_bits_equal
import structured

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PolynomialSystem, PrecisionMode as PM, StepControlParams
from paper_1501_06625_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _one(z, prec=PM.D):
    return pt.limbs_from_complex(np.atleast_1d(z), prec)


def _gamma(z, prec):
    return pt.limbs_from_complex([z], prec).reshape(-1)


@pytest.mark.parametrize("name,prec", [("cyclic16", PM.DD), ("cyclic16", PM.D), ("chandra64", PM.D),
                                       ("chandra64", PM.DD), ("cyclic16", PM.QD), ("chandra64", PM.QD)])
def test_restatement_tracker_matches_reference_build(oracle, ref_oracle, name, prec):
    w = W.by_name(name, prec)
    e1, s1, t1 = oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, 600)
    e2, s2, t2 = ref_oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, 600)
    assert (s1.steps, s1.newton_iters, s1.status) == (s2.steps, s2.newton_iters, s2.status)
    assert_bits_equal(e1, e2, "end point")
    assert len(t1) == len(t2)


@pytest.mark.parametrize("name,prec", [("cyclic16", PM.DD), ("cyclic16", PM.D), ("chandra64", PM.D),
                                       ("chandra64", PM.DD), ("cyclic16", PM.QD), ("chandra64", PM.QD)])
def test_golden_tracks(oracle, name, prec):
    g = np.load(os.path.join(GOLDEN, f"track_{name}_{prec.name.lower()}.npz"))
    w = W.by_name(name, prec)
    end, st, tr = oracle.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, 600)
    assert [st.status, st.failure_kind, st.steps, st.accepted, st.newton_iters, st.start_iters] == g["stats"].tolist()
    assert_bits_equal(np.array([st.final_residual, st.final_update, st.t_end]), g["fstats"], "stats")
    assert_bits_equal(np.array([[e.t, e.ok, e.iters, e.residual, e.update] for e in tr]), g["trace"], "trace")
    assert_bits_equal(end, g["end"], "end")


# ---- evaldiff ---------------------------------------------
def _eval_target(oracle, f, x, prec=PM.D):
    """f(x) and J_f(x) via evaluate_homotopy at t = 1 (h = f)."""
    g = f
    h, J, r = oracle.eval_homotopy(int(prec), g, f, _gamma(1.0, prec), 1, x, 1.0)
    N, n = f.n_eqs, f.n_vars
    hc = pt.complex_from_limbs(h)
    Jc = pt.complex_from_limbs(J).reshape(n, N).T
    return hc, Jc, r


def test_speelpenning_example(oracle):
    f = PolynomialSystem.from_terms(6, [[([(2, 1), (3, 1), (4, 1), (5, 1)], 1.0)]], PM.D)
    x = _one([9.0, 9.0, 2.0, 3.0, 5.0, 7.0])
    h, J, _ = _eval_target(oracle, f, x)
    assert h[0] == 210.0
    assert J[0].tolist() == [0, 0, 105.0, 70.0, 42.0, 30.0]


def test_power_rule_example(oracle):
    f = PolynomialSystem.from_terms(2, [[([(0, 2), (1, 1)], 1.0)], [([(0, 1)], 1.0)]], PM.D)
    h, J, _ = _eval_target(oracle, f, _one([2.0, 3.0]))
    assert h[0] == 12.0 and J[0].tolist() == [12.0, 4.0]
    assert h[1] == 2.0 and J[1].tolist() == [1.0, 0.0]


def test_cyclic4_vanishes(oracle):
    f = pt.cyclic_system(4, PM.D)
    h, J, r = _eval_target(oracle, f, _one([1j, -1j, -1j, 1j]))
    assert np.all(h == 0) and r == 0.0


def test_ad_vs_bruteforce_random_systems(oracle):
    """Acceptance criterion 6, D mode."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(1, 8))
        eqs = []
        for i in range(n):
            terms = []
            for _ in range(int(rng.integers(1, 12))):
                vs = sorted(rng.choice(n, size=int(rng.integers(0, min(n, 6) + 1)), replace=False).tolist())
                terms.append(([(v, int(rng.integers(1, 4))) for v in vs], complex(*rng.uniform(-1, 1, 2))))
            eqs.append(terms)
        f = PolynomialSystem.from_terms(n, eqs, PM.D)
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        h, J, _ = _eval_target(oracle, f, _one(x))
        for i, terms in enumerate(eqs):
            val = sum(c * np.prod([x[v] ** e for v, e in sup]) for sup, c in terms)
            assert abs(h[i] - val) <= 1e-13 * max(1, abs(val))
            for j in range(n):
                d = 0
                for sup, c in terms:
                    if j in [v for v, _ in sup]:
                        d += c * np.prod([(e * x[v] ** (e - 1)) if v == j else x[v] ** e for v, e in sup])
                assert abs(J[i, j] - d) <= 1e-12 * max(1, abs(d))
                if all(j not in [v for v, _ in sup] for sup, _ in terms):
                    assert J[i, j] == 0  # structural zero


def test_homotopy_weights_examples(oracle):
    """SPEC.md:171-182 through h(x,t) of g = x - 1, f = x - 2."""
    g = PolynomialSystem.from_terms(1, [[([], -1.0), ([(0, 1)], 1.0)]], PM.D)
    f = PolynomialSystem.from_terms(1, [[([], -2.0), ([(0, 1)], 1.0)]], PM.D)
    x = _one([5.0])
    h, _, _ = oracle.eval_homotopy(0, g, f, _gamma(1j, PM.D), 2, x, 0.0)
    assert pt.complex_from_limbs(h)[0] == 4j                      # gamma * g at t = 0
    h, _, _ = oracle.eval_homotopy(0, g, f, _gamma(1.0, PM.D), 2, x, 0.5)
    assert pt.complex_from_limbs(h)[0] == 0.25 * 4 + 0.25 * 3     # k=2, t=1/2
    h, _, _ = oracle.eval_homotopy(0, g, f, _gamma(1.0, PM.D), 1, x, 1.0)
    assert pt.complex_from_limbs(h)[0] == 3.0                     # f at t = 1


# ---- linalg -----------------------------------------------
def _lstsq(oracle, A, b, prec=PM.D):
    A = np.asarray(A, dtype=np.complex128)
    N, n = A.shape
    Al = pt.limbs_from_complex(A.T.reshape(-1), prec)
    bl = pt.limbs_from_complex(b, prec)
    x = oracle.lstsq(int(prec), Al, bl)
    return None if x is None else pt.complex_from_limbs(x)


def test_lstsq_examples(oracle):
    assert _lstsq(oracle, np.eye(3), [1, 2j, 3]).tolist() == [1, 2j, 3]
    assert abs(_lstsq(oracle, [[1.0], [1.0]], [1.0, 3.0])[0] - 2.0) < 1e-15
    x = _lstsq(oracle, [[2.0, 1.0], [0.0, 4.0]], [4.0, 8.0])
    assert np.allclose(x, [1.0, 2.0], rtol=0, atol=1e-15)
    x = _lstsq(oracle, [[3.0, 0.0], [4.0, 0.0], [0.0, 1.0]], [3.0, 4.0, 2.0])
    assert np.allclose(x, [1.0, 2.0], rtol=0, atol=1e-15)
    assert _lstsq(oracle, [[1.0, 2.0], [2.0, 4.0]], [1.0, 1.0]) is None             # rank deficiency


@pytest.mark.parametrize("prec,tol", [(PM.D, 1e-12), (PM.DD, 1e-28)], ids=["d", "dd"])
def test_lstsq_residual_property(oracle, prec, tol):
    rng = np.random.default_rng(7)
    n = 32
    A = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    x = _lstsq(oracle, A, b, prec)
    assert np.max(np.abs(A @ x - b)) <= 1e-12 * np.max(np.abs(b)) * 1e3  # binary64 check of a DD solve


# ---- newton / tracker ---------------------
def test_tracker_one_variable_example(oracle):
    g = PolynomialSystem.from_terms(1, [[([], -1.0), ([(0, 1)], 1.0)]], PM.DD)
    f = PolynomialSystem.from_terms(1, [[([], -2.0), ([(0, 1)], 1.0)]], PM.DD)
    sp = StepControlParams.defaults(PM.DD)
    end, st, tr = oracle.track_path(1, g, f, W.gamma_from_seed(4, PM.DD), 2, _one([1.0], PM.DD), sp, 600)
    assert st.status == 0 and st.t_end == 1.0
    assert abs(pt.complex_from_limbs(end)[0] - 2.0) < 1e-25
    # monotone t, bounded steps, one event per trial
    ts = [e.t for e in tr if e.ok]
    assert all(b > a for a, b in zip(ts, ts[1:])) and ts[-1] == 1.0
    assert st.steps == len(tr) <= sp.max_steps + 1


def test_tracker_max_steps_one_fails(oracle):
    w = W.cyclic_leg(4, PM.DD)
    sp = StepControlParams.defaults(PM.DD)
    sp.max_steps = 1
    _, st, _ = oracle.track_path(1, w.g, w.f, w.gamma, w.k, w.start, sp)
    assert st.status == 1 and st.failure_kind == 2 and st.steps == 2  # SPEC.md:474, budget steps <= max+1


def test_newton_quadratic_start_validation(oracle):
    """x^2 - 1 from x0 = 2 as the t = 0 corrector pass."""
    g = PolynomialSystem.from_terms(1, [[([], -1.0), ([(0, 2)], 1.0)]], PM.D)
    sp = StepControlParams(newton_tol=1e-12, newton_max_iter=10, max_steps=0)
    _, st, _ = oracle.track_path(0, g, g, _gamma(1.0, PM.D), 2, _one([2.0]), sp)
    assert st.start_iters <= 7


def test_step_doubling_rule(oracle):
    """Trace of a smooth path: after 3 consecutive successes the step doubles
    up to max_step; failures halve it."""
    w = W.cyclic_leg(4, PM.DD)
    sp = StepControlParams.defaults(PM.DD)
    _, st, tr = oracle.track_path(1, w.g, w.f, w.gamma, w.k, w.start, sp, 600)
    dt, succ, tacc = sp.max_step, 0, 0.0
    for e in tr:
        assert e.t == min(1.0, tacc + dt)
        if e.ok:
            tacc = e.t
            succ += 1
            if succ > 2:
                dt = min(2 * dt, sp.max_step)
        else:
            succ = 0
            dt = dt / 2


@pytest.mark.parametrize("n,prec,seed", structured.CASES,
                         ids=lambda v: str(v) if not isinstance(v, PM) else v.name)
def test_restatement_matches_reference_build_on_structured_systems(oracle, ref_oracle, n, prec, seed):
    """The oracle the device is checked against (tests/test_gpu_random.py)
    equals the reference-header build on the randomly structured systems too:
    every path's stats, trace and end point, whatever the path's outcome."""
    f, g, gamma, params, starts = structured.case(n, prec, seed, structured.max_steps(prec))
    cap = params.max_steps + 2
    for p in range(starts.shape[0]):
        e1, s1, t1 = oracle.track_path(int(prec), g, f, gamma, 2, starts[p], params, cap)
        e2, s2, t2 = ref_oracle.track_path(int(prec), g, f, gamma, 2, starts[p], params, cap)
        assert (s1.status, s1.failure_kind, s1.steps, s1.accepted, s1.newton_iters) == (
            s2.status, s2.failure_kind, s2.steps, s2.accepted, s2.newton_iters)
        assert_bits_equal(np.array([s1.final_residual, s1.final_update, s1.t_end]),
                          np.array([s2.final_residual, s2.final_update, s2.t_end]), "stats")
        assert_bits_equal(np.array([(e.t, e.residual, e.update) for e in t1]).reshape(-1),
                          np.array([(e.t, e.residual, e.update) for e in t2]).reshape(-1), "trace")
        assert_bits_equal(e1, e2, f"end point of path {p}")
