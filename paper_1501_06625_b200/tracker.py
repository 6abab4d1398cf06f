"""Host-side mirror of the reference tracker interface (SPEC.md signatures).

The reference ships only the scalar layer (proj/include/pathtrack); the path
API is specified in SPEC.md and re-stated here with the same names and
argument meaning, over the CUDA library's C-ABI:

  PrecisionMode                multiprec.hpp:27
  PolynomialSystem             SPEC.md:133-136 (canonical form :150)
  HomotopyParameters/make_homotopy/homotopy_weights
  NewtonParams/StepControlParams
  TrackOutcome, track_path
  evaluate_homotopy
  least_squares_solve
  cyclic_system / augment_with_linear

Numbers cross the boundary as binary64 limb arrays: a complex vector of
length n in precision with L limbs is a float64 array of shape (2, L, n)
(re limbs, im limbs), exactly RealTraits<R>::components per entry.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as nat


class PrecisionMode(enum.IntEnum):  # multiprec.hpp:27
    D = 0
    DD = 1
    QD = 2

    @property
    def limbs(self) -> int:
        return (1, 2, 4)[int(self)]

    @staticmethod
    def parse(text: str) -> "PrecisionMode":  # precision.cpp:22-27
        m = {"d": PrecisionMode.D, "dd": PrecisionMode.DD, "qd": PrecisionMode.QD}
        if text not in m:
            raise ValueError(f"unknown precision mode '{text}' (expected d, dd, or qd)")
        return m[text]


def limbs_from_complex(z, prec: PrecisionMode) -> np.ndarray:
    """complex128 vector -> (2, L, n) limbs with the value in limb 0."""
    z = np.asarray(z, dtype=np.complex128).reshape(-1)
    out = np.zeros((2, prec.limbs, z.size))
    out[0, 0] = z.real
    out[1, 0] = z.imag
    return out


def complex_from_limbs(a: np.ndarray) -> np.ndarray:
    """(2, L, n) limbs -> complex128 (sum of limbs rounded to binary64)."""
    a = np.asarray(a)
    return a[0].sum(axis=0) + 1j * a[1].sum(axis=0)


@dataclass
class PolynomialSystem:
    """Canonical distributed form, pt_system_desc layout."""

    n_vars: int
    eq_ptr: np.ndarray
    term_ptr: np.ndarray
    var: np.ndarray
    exp: np.ndarray
    coef: np.ndarray  # (2, L, n_terms)
    prec: PrecisionMode

    @property
    def n_eqs(self) -> int:
        return int(self.eq_ptr.size - 1)

    @property
    def n_terms(self) -> int:
        return int(self.term_ptr.size - 1)

    def desc(self) -> nat.SystemDesc:
        for name in ("eq_ptr", "term_ptr", "var", "exp"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int32))
        self.coef = np.ascontiguousarray(self.coef, dtype=np.float64)
        d = nat.SystemDesc()
        d.n_vars, d.n_eqs, d.n_terms = self.n_vars, self.n_eqs, self.n_terms
        d.eq_ptr = nat.iptr(self.eq_ptr)
        d.term_ptr = nat.iptr(self.term_ptr)
        d.var = nat.iptr(self.var if self.var.size else np.zeros(1, np.int32))
        d.exp = nat.iptr(self.exp if self.exp.size else np.ones(1, np.int32))
        d.coef = nat.dptr(self.coef)
        return d

    def terms(self, i: int):
        """(support [(var, exp)], complex128 coefficient) of equation i."""
        out = []
        for t in range(self.eq_ptr[i], self.eq_ptr[i + 1]):
            sup = [(int(self.var[q]), int(self.exp[q])) for q in range(self.term_ptr[t], self.term_ptr[t + 1])]
            c = self.coef[0, :, t].sum() + 1j * self.coef[1, :, t].sum()
            out.append((sup, c))
        return out

    @staticmethod
    def _from_sysbuf(buf, prec: PrecisionMode) -> "PolynomialSystem":
        d = nat.SystemDesc()
        nat.check(nat.lib.pt_sysbuf_desc(buf, C.byref(d)))
        T = d.n_terms
        V = d.term_ptr[T] if T > 0 else 0
        arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n > 0 else np.zeros(0, np.int32)
        sysm = PolynomialSystem(
            n_vars=d.n_vars,
            eq_ptr=arr(d.eq_ptr, d.n_eqs + 1),
            term_ptr=arr(d.term_ptr, T + 1),
            var=arr(d.var, V),
            exp=arr(d.exp, V),
            coef=np.ctypeslib.as_array(d.coef, shape=(2 * prec.limbs * max(T, 1),)).copy()[: 2 * prec.limbs * T]
            .reshape(2, prec.limbs, T),
            prec=prec,
        )
        nat.lib.pt_sysbuf_free(buf)
        return sysm

    @staticmethod
    def from_terms(n_vars: int, equations, prec: PrecisionMode) -> "PolynomialSystem":
        """Build from [[(support, coef), ...], ...] with support [(var, exp), ...]
        (var ascending, exp >= 1) and coef a complex number or a (2, L) limb
        array.  Term order is kept as given."""
        L = prec.limbs
        eq_ptr, term_ptr, var, exp, coefs = [0], [0], [], [], []
        for eq in equations:
            for sup, c in eq:
                for v, e in sup:
                    var.append(v)
                    exp.append(e)
                term_ptr.append(len(var))
                cl = np.zeros((2, L))
                if np.ndim(c) == 0:
                    cl[0, 0], cl[1, 0] = complex(c).real, complex(c).imag
                else:
                    cl[:] = np.asarray(c, dtype=np.float64).reshape(2, L)
                coefs.append(cl)
            eq_ptr.append(len(term_ptr) - 1)
        coef = np.stack(coefs, axis=-1) if coefs else np.zeros((2, L, 0))
        return PolynomialSystem(n_vars, np.array(eq_ptr, np.int32), np.array(term_ptr, np.int32),
                                np.array(var, np.int32), np.array(exp, np.int32), coef, prec)


def _gen(fn, *args, prec: PrecisionMode) -> PolynomialSystem:
    buf = C.c_void_p()
    nat.check(fn(*args, int(prec), C.byref(buf)))
    return PolynomialSystem._from_sysbuf(buf, prec)


def cyclic_system(n: int, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """Cyclic n-roots, Eq. (5)."""
    return _gen(nat.lib.pt_gen_cyclic, n, prec=prec)


def augment_with_linear(n_cyclic: int, dim: int, seed: int,
                        prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """cyclic-n plus `dim` random affine slices, Eq. (6)."""
    fb = C.c_void_p()
    nat.check(nat.lib.pt_gen_cyclic(n_cyclic, int(prec), C.byref(fb)))
    out = C.c_void_p()
    rc = nat.lib.pt_gen_augment(fb, dim, C.c_uint64(seed), int(prec), C.byref(out))
    nat.lib.pt_sysbuf_free(fb)
    nat.check(rc)
    return PolynomialSystem._from_sysbuf(out, prec)


def chandrasekhar(n: int, c: float = 0.51234, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """Discretised Chandrasekhar H-equation (BASELINE config 2)."""
    return _gen(nat.lib.pt_gen_chandra, n, C.c_double(c), prec=prec)


def random_dense(n: int, degree: int, n_monomials: int, seed: int,
                 prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """n equations on one shared random support (BASELINE configs 3 and 5)."""
    return _gen(nat.lib.pt_gen_random_dense, n, degree, n_monomials, C.c_uint64(seed), prec=prec)


def total_degree_start(n: int, degree: int, prec: PrecisionMode = PrecisionMode.DD) -> PolynomialSystem:
    """g_i = x_i^degree - 1."""
    return _gen(nat.lib.pt_gen_total_degree, n, degree, prec=prec)


def gamma_from_seed(seed: int, prec: PrecisionMode) -> np.ndarray:
    """Rng(seed).unit<R>() (rng.hpp:38-41) as 2L limbs."""
    out = np.zeros(2 * prec.limbs)
    nat.check(nat.lib.pt_gen_gamma(C.c_uint64(seed), int(prec), nat.dptr(out)))
    return out


def unit_complex(theta: float, prec: PrecisionMode) -> np.ndarray:
    """unit_complex<R>(theta) (complex.hpp:141-148) as 2L limbs."""
    out = np.zeros(2 * prec.limbs)
    nat.check(nat.lib.pt_gen_unit_complex(C.c_double(theta), int(prec), nat.dptr(out)))
    return out


@dataclass
class StepControlParams:  # SPEC.md:448-451 + NewtonParams SPEC.md:357-359
    max_step: float = 0.1
    min_step: float = 1e-6
    max_steps: int = 500
    pred_degree: int = 4
    newton_max_iter: int = 6
    newton_tol: float = 1e-20

    @staticmethod
    def defaults(prec: PrecisionMode) -> "StepControlParams":
        sp = nat.StepParams()
        nat.check(nat.lib.pt_default_params(int(prec), C.byref(sp)))
        return StepControlParams(sp.max_step, sp.min_step, sp.max_steps, sp.pred_degree, sp.newton_max_iter,
                                 sp.newton_tol)

    def native(self) -> nat.StepParams:
        return nat.StepParams(self.max_step, self.min_step, self.max_steps, self.pred_degree,
                              self.newton_max_iter, 0, self.newton_tol)


FAILURE_KINDS = {0: "none", 1: "start", 2: "max-steps", 3: "min-step"}


@dataclass
class TrackOutcome:
    success: bool
    end: np.ndarray  # (2, L, n) limbs
    steps: int
    accepted: int
    newton_iters: int
    start_iters: int
    final_residual: float
    final_update: float
    t_end: float
    failure_kind: str
    trace: List[nat.TraceEvent] = field(default_factory=list)
    solves: int = 0  # completed least-squares solves

    @staticmethod
    def from_native(end: np.ndarray, st: nat.PathStats, trace=None) -> "TrackOutcome":
        return TrackOutcome(st.status == 0, end, st.steps, st.accepted, st.newton_iters, st.start_iters,
                            st.final_residual, st.final_update, st.t_end,
                            FAILURE_KINDS.get(st.failure_kind, str(st.failure_kind)), trace or [], st.solves)


class Homotopy:
    """h(x,t) = gamma (1-t)^k g(x) + t^k f(x), compiled for one device
    (make_homotopy + compile_plan)."""

    def __init__(self, g: PolynomialSystem, f: PolynomialSystem, gamma: np.ndarray, k: int = 2,
                 device: int = 0):
        if g.prec != f.prec:
            raise ValueError("start and target systems must share the precision")
        self.prec = g.prec
        self.n = g.n_vars
        self.N = g.n_eqs
        self.g, self.f = g, f
        self.gamma = np.ascontiguousarray(gamma, dtype=np.float64).reshape(-1)
        if self.gamma.size != 2 * self.prec.limbs:
            raise ValueError("gamma must have 2L limbs")
        self.k = int(k)
        self._plan = C.c_void_p()
        gd, fd = g.desc(), f.desc()
        nat.check(nat.lib.pt_plan_create(device, int(self.prec), C.byref(gd), C.byref(fd), nat.dptr(self.gamma),
                                         self.k, C.byref(self._plan)))

    def close(self):
        if self._plan:
            nat.lib.pt_plan_destroy(self._plan)
            self._plan = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def plan(self):
        return self._plan

    def info(self, what: int) -> int:
        return int(nat.lib.pt_plan_info(self._plan, what))

    @property
    def engine(self) -> str:
        return ("grid", "cluster")[self.info(8)]

    def set_engine(self, engine: str) -> None:
        """Force the single-path engine ("grid" or "cluster"); results are bit-identical."""
        nat.check(nat.lib.pt_plan_set_engine(self._plan, {"grid": 0, "cluster": 1}[engine]))

    def track_path(self, start: np.ndarray, params: Optional[StepControlParams] = None,
                   trace: bool = False) -> TrackOutcome:
        """track_path."""
        params = params or StepControlParams.defaults(self.prec)
        start = np.ascontiguousarray(start, dtype=np.float64).reshape(2, self.prec.limbs, self.n)
        end = np.zeros_like(start)
        st = nat.PathStats()
        sp = params.native()
        cap = params.max_steps + 2 if trace else 0
        nat.check(nat.lib.pt_plan_set_trace(self._plan, cap))
        nat.check(nat.lib.pt_track_path(self._plan, nat.dptr(start), C.byref(sp), nat.dptr(end), C.byref(st)))
        events = []
        if trace:
            buf = (nat.TraceEvent * cap)()
            cnt = C.c_int32()
            nat.check(nat.lib.pt_plan_get_trace(self._plan, buf, cap, C.byref(cnt)))
            events = list(buf[: min(cnt.value, cap)])
        return TrackOutcome.from_native(end, st, events)

    def track_batch(self, starts: np.ndarray, params: Optional[StepControlParams] = None):
        """Independent paths, one CTA each."""
        params = params or StepControlParams.defaults(self.prec)
        starts = np.ascontiguousarray(starts, dtype=np.float64).reshape(-1, 2, self.prec.limbs, self.n)
        P = starts.shape[0]
        ends = np.zeros_like(starts)
        stats = (nat.PathStats * max(P, 1))()
        sp = params.native()
        nat.check(nat.lib.pt_track_batch(self._plan, P, nat.dptr(starts), C.byref(sp), nat.dptr(ends), stats))
        return ends, [TrackOutcome.from_native(ends[p], stats[p]) for p in range(P)]

    def evaluate(self, x: np.ndarray, t: float):
        """evaluate_homotopy: (h (2,L,N), J (2,L,N*n) column-major, max|h|)."""
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(2, self.prec.limbs, self.n)
        h = np.zeros((2, self.prec.limbs, self.N))
        J = np.zeros((2, self.prec.limbs, self.N * self.n))
        r = np.zeros(1)
        nat.check(nat.lib.pt_eval_homotopy(self._plan, nat.dptr(x), C.c_double(t), nat.dptr(h), nat.dptr(J),
                                           nat.dptr(r)))
        return h, J, float(r[0])


def make_homotopy(g: PolynomialSystem, f: PolynomialSystem, gamma: np.ndarray, k: int = 2,
                  device: int = 0) -> Homotopy:
    return Homotopy(g, f, gamma, k, device)


def least_squares_solve(A: np.ndarray, b: np.ndarray, prec: PrecisionMode, device: int = 0) -> np.ndarray:
    """MGS least squares on the device.
    A: (2, L, N*n) column-major limbs, b: (2, L, N)."""
    L = prec.limbs
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    N = b.shape[-1]
    n = A.shape[-1] // N
    x = np.zeros((2, L, n))
    nat.check(nat.lib.pt_lstsq(device, int(prec), N, n, nat.dptr(A), nat.dptr(b), nat.dptr(x)))
    return x


def device_count() -> int:
    return int(nat.lib.pt_device_count())


def arith(prec: PrecisionMode, op: int, a: np.ndarray, b: np.ndarray, device: Optional[int] = 0) -> np.ndarray:
    """Bulk scalar op (parity tests). device=None runs the host build of the
    device arithmetic."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros_like(a)
    cnt = a.size // (2 * prec.limbs)
    if device is None:
        nat.check(nat.lib.pt_arith_host(int(prec), op, cnt, nat.dptr(a), nat.dptr(b), nat.dptr(out)))
    else:
        nat.check(nat.lib.pt_arith_device(device, int(prec), op, cnt, nat.dptr(a), nat.dptr(b), nat.dptr(out)))
    return out
