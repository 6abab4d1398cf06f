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


from .systems import (  # noqa: F401  (re-exported: the SPEC names live here too)
    PolynomialSystem,
    PrecisionMode,
    StepControlParams,
    augment_with_linear,
    chandrasekhar,
    complex_from_limbs,
    cyclic_system,
    gamma_from_seed,
    limbs_from_complex,
    random_dense,
    total_degree_start,
    unit_complex,
)


FAILURE_KINDS = {0: "none", 1: "start", 2: "max-steps", 3: "min-step", 4: "abort"}


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
    flags: int = 0   # PT_STAT_NONFINITE (1): met inf / NaN, re-tracked by the exact DD kernels

    @staticmethod
    def from_native(end: np.ndarray, st: nat.PathStats, trace=None) -> "TrackOutcome":
        return TrackOutcome(st.status == 0, end, st.steps, st.accepted, st.newton_iters, st.start_iters,
                            st.final_residual, st.final_update, st.t_end,
                            FAILURE_KINDS.get(st.failure_kind, str(st.failure_kind)), trace or [], st.solves,
                            st.flags)


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

    def set_arith(self, arith: str) -> None:
        """"reference" (default: the reference's operation sequences, bit
        parity) or "fast" (QD plans: tolerance-parity quad-double arithmetic,
        pt_plan_set_arith)."""
        nat.check(nat.lib.pt_plan_set_arith(self._plan, {"reference": 0, "fast": 1}[arith]))

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


def eval_bench(hom: Homotopy, x: np.ndarray, t: float, reps: int) -> float:
    """Device milliseconds per evaluation + differentiation pass (pt_eval_bench)."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(2, hom.prec.limbs, hom.n)
    ms = np.zeros(1)
    nat.check(nat.lib.pt_eval_bench(hom.plan, nat.dptr(x), C.c_double(t), int(reps), nat.dptr(ms)))
    return float(ms[0])


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


def arith(prec: PrecisionMode, op: int, a: np.ndarray, b: np.ndarray, device: Optional[int] = 0,
          fast: bool = False) -> np.ndarray:
    """Bulk scalar op (parity tests). device=None runs the host build of the
    device arithmetic; fast=True the tolerance-parity QD set on the device."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros_like(a)
    cnt = a.size // (2 * prec.limbs)
    if device is None:
        nat.check(nat.lib.pt_arith_host(int(prec), op, cnt, nat.dptr(a), nat.dptr(b), nat.dptr(out)))
    elif fast:
        nat.check(nat.lib.pt_arith_device_mode(device, int(prec), 1, op, cnt, nat.dptr(a), nat.dptr(b),
                                               nat.dptr(out)))
    else:
        nat.check(nat.lib.pt_arith_device(device, int(prec), op, cnt, nat.dptr(a), nat.dptr(b), nat.dptr(out)))
    return out
