"""CPU: the drop-in boundary.  The C-ABI library loads, exports exactly what
include/pathtrack_b200.h declares, validates its inputs, refuses to compute
without an sm_100 device (no CPU fallback), and the host-side generators
build the documented systems."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import PrecisionMode as PM
from paper_1501_06625_b200 import _native as nat
from paper_1501_06625_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(pt_\w+)\s*\(", text))


def test_every_declared_symbol_is_exported():
    """Each header's functions are exported by its library, and the ctypes
    prototype tables cover exactly the declarations."""
    from paper_1501_06625_b200 import _inputs as inp
    for header, mod, at_least in (("pathtrack_b200.h", nat, 24), ("pathtrack_inputs.h", inp, 25)):
        names = declared_functions(header)
        assert len(names) >= at_least
        lib = C.CDLL(mod.LIB_PATH)
        missing = [n for n in sorted(names) if not hasattr(lib, n)]
        assert not missing, (header, missing)
        assert set(mod.PROTOTYPES) == names, (header, set(mod.PROTOTYPES) ^ names)


def test_inputs_never_load_the_tracker_library():
    """Workload construction (what the reference arm of bench.py and the
    oracle tests use) maps libpt_inputs.so only, never libpathtrack_b200.so."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1501_06625_b200 import workloads as W, PrecisionMode as PM\n"
            "w = W.chandra(8, PM.DD); W.batch(n_paths=4); W.cyclic_leg(4, PM.DD)\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('inputs' if 'libpt_inputs.so' in maps else 'no-inputs',"
            " 'TRACKER' if 'libpathtrack_b200.so' in maps else 'clean')\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["inputs", "clean"], out


def test_default_params_match_the_library():
    for prec in PM:
        sp = nat.StepParams()
        nat.check(nat.lib.pt_default_params(int(prec), C.byref(sp)))
        py = pt.StepControlParams.defaults(prec)
        assert (sp.max_step, sp.min_step, sp.max_steps, sp.pred_degree, sp.newton_max_iter, sp.newton_tol) == (
            py.max_step, py.min_step, py.max_steps, py.pred_degree, py.newton_max_iter, py.newton_tol)


def test_struct_layouts_match_header():
    assert C.sizeof(nat.StepParams) == 40
    assert C.sizeof(nat.PathStats) == 56
    assert C.sizeof(nat.TraceEvent) == 32
    from oracle import orc
    assert C.sizeof(orc.PathStats) == C.sizeof(nat.PathStats)
    assert C.sizeof(orc.StepParams) == C.sizeof(nat.StepParams)


def test_default_params_follow_spec():
    d = pt.StepControlParams.defaults(PM.D)
    dd = pt.StepControlParams.defaults(PM.DD)
    qd = pt.StepControlParams.defaults(PM.QD)
    assert (d.newton_tol, dd.newton_tol, qd.newton_tol) == (1e-8, 1e-20, 1e-44)
    assert (d.max_steps, dd.max_steps, qd.max_steps) == (500, 500, 1500)
    assert dd.max_step == 0.1 and dd.min_step == 1e-6 and dd.pred_degree == 4 and dd.newton_max_iter == 6


@pytest.mark.skipif(pt.device_count() > 0, reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    w = W.chandra(8, PM.DD)
    with pytest.raises(nat.NativeError) as e:
        pt.make_homotopy(w.g, w.f, w.gamma, w.k)
    assert e.value.code == nat.PT_E_NODEVICE
    a = np.zeros((4, 2, 2))
    with pytest.raises(nat.NativeError):
        pt.arith(PM.DD, 0, a, a, device=0)
    with pytest.raises(nat.NativeError):
        pt.least_squares_solve(np.zeros((2, 2, 4)), np.zeros((2, 2, 2)), PM.DD)


def test_plan_rejects_malformed_systems():
    f = pt.PolynomialSystem.from_terms(2, [[([(1, 1), (0, 1)], 1.0)], [([(0, 1)], 1.0)]], PM.D)  # vars not increasing
    g = pt.PolynomialSystem.from_terms(2, [[([(0, 1)], 1.0)], [([(1, 1)], 1.0)]], PM.D)
    with pytest.raises(nat.NativeError) as e:
        pt.make_homotopy(g, f, pt.limbs_from_complex([1.0], PM.D).reshape(-1), 1)
    assert e.value.code in (nat.PT_E_INVAL, nat.PT_E_NODEVICE)


def test_cyclic_generator_term_counts():
    for n in (3, 4, 8):
        s = pt.cyclic_system(n, PM.D)
        counts = np.diff(s.eq_ptr).tolist()
        assert counts == [n] * (n - 1) + [2]
    s = pt.cyclic_system(4, PM.D)
    assert sorted(sup for sup, _ in s.terms(1)) == [[(0, 1), (1, 1)], [(0, 1), (3, 1)], [(1, 1), (2, 1)],
                                                   [(2, 1), (3, 1)]]


def test_augment_is_deterministic_and_sized():
    a = pt.augment_with_linear(16, 3, 5, PM.DD)
    b = pt.augment_with_linear(16, 3, 5, PM.DD)
    assert a.n_eqs == 19 and a.n_vars == 16
    assert np.array_equal(a.coef, b.coef)
    c = pt.augment_with_linear(16, 0, 5, PM.DD)
    assert c.n_eqs == 16


def test_gamma_is_unit_in_working_precision():
    from oracle.orc import Oracle
    o = Oracle("restatement")
    for prec, tol in ((PM.DD, 1e-30), (PM.QD, 1e-62)):
        g = pt.gamma_from_seed(123, prec).reshape(1, 2, prec.limbs)
        ns = o.arith(int(prec), 10, g, g)[0, 0]  # norm_sqr
        assert abs(ns.sum() - 1.0) < tol


def test_backelin_witness_on_cyclic16():
    w = W.cyclic_leg(4, PM.D)
    x = pt.complex_from_limbs(w.start)
    n = 16
    for i in range(1, n):
        val = sum(np.prod([x[(t + k) % n] for k in range(i)]) for t in range(n))
        assert abs(val) < 1e-10
    assert abs(np.prod(x) - 1) < 1e-10


def test_workloads_shapes():
    w = W.random_system(8, 3, 20, PM.DD, n_paths=10)
    assert w.starts.shape == (10, 2, 2, 8)
    assert w.f.n_eqs == 8 and np.diff(w.f.eq_ptr).tolist() == [21] * 8
