"""Pieri homotopies over the B200 tracker -- SURVEY.md 8(f) row 3: a second
benchmark family whose evaluation cost grows with the minor expansions
(PAPER.md 4.1, Eqs. 7-8).

  pieri_events            PieriPattern variable-introduction order
  minor_expand            det([A | X_k]) fully expanded   (libpt_inputs.so)
  choose_special_matrix   S_X of Eq. (7)                  (libpt_inputs.so)
  pieri_sequence          the bootstrap: stage 1 solved as a linear system,
                          stage k = 2 .. m p tracked from the previous
                          solution extended by a zero for the new variable

Stage k tracks h = gamma (1-t) g + t f (relaxation k = 1, the Eq.-(1)
machinery) with g = {det(A^(i)|X_k) = 0, i < k} + {det(S_X|X_k) = 0} and
f = {det(A^(i)|X_k) = 0, i < k} + {det(A^(k)|X_k) = 0}: the shared
equations are summed once by the plan, and their weight gamma (1-t) + t never
vanishes for a random unit gamma, so their zero set is unchanged -- the
gamma-trick form of Eq. (8), t det(A^(k)|X) + (1-t) det(S_X|X).
Randomness: the planes A^(1..mp) come from pathtrack::Rng(seed) (box<R>
entries), gamma of stage k from Rng(seed + 1000 + k).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import _inputs as inp
from ._abi import dptr
from .systems import PolynomialSystem, PrecisionMode, StepControlParams, gamma_from_seed, stack_systems

# (g, f, gamma, start (2,L,n), params) -> (end (2,L,n), success, steps, newton_iters)
PathTracker = Callable[[PolynomialSystem, PolynomialSystem, np.ndarray, np.ndarray, StepControlParams], tuple]


def gpu_path_tracker(device: int = 0) -> PathTracker:
    """The product path: one plan per stage, one tracked path on the device."""

    def run(g, f, gamma, start, params):
        from .tracker import make_homotopy
        hom = make_homotopy(g, f, gamma, 1, device=device)
        out = hom.track_path(start, params)
        hom.close()
        return out.end, out.success, out.steps, out.newton_iters

    return run


def pieri_events(m: int, p: int) -> List[Tuple[int, int]]:
    """(row, column), 0-based, of the m p variables in introduction order."""
    rows = np.zeros(m * p, np.int32)
    cols = np.zeros(m * p, np.int32)
    inp.check(inp.lib.pt_pieri_events(m, p, rows.ctypes.data_as(C.POINTER(C.c_int32)),
                                      cols.ctypes.data_as(C.POINTER(C.c_int32))))
    return list(zip(rows.tolist(), cols.tolist()))


def pieri_planes(m: int, p: int, count: int, seed: int, prec: PrecisionMode) -> np.ndarray:
    """A^(1..count): (count, 2, L, n m) column-major complex limbs."""
    n, L = m + p, prec.limbs
    out = np.zeros((count, 2, L, n * m))
    inp.check(inp.lib.pt_pieri_planes(m, p, count, C.c_uint64(seed), int(prec), dptr(out)))
    return out


def minor_expand(m: int, p: int, k: int, A: np.ndarray, prec: PrecisionMode) -> PolynomialSystem:
    """det([A | X_k]) as a one-equation system in the k stage variables."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    buf = C.c_void_p()
    inp.check(inp.lib.pt_pieri_minor(m, p, k, dptr(A), int(prec), C.byref(buf)))
    return PolynomialSystem._from_sysbuf(buf, prec)


def pieri_det(m: int, p: int, k: int, A: np.ndarray, x: np.ndarray, prec: PrecisionMode) -> complex:
    """det([A | X_k(x)]) evaluated numerically in `prec` (leading limbs returned)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1) if k else np.zeros(1)
    out = np.zeros(2 * prec.limbs)
    inp.check(inp.lib.pt_pieri_det(m, p, k, dptr(A), dptr(x), int(prec), dptr(out)))
    L = prec.limbs
    return complex(out[:L].sum(), out[L:].sum())


def choose_special_matrix(m: int, p: int, k: int, x0: np.ndarray, prec: PrecisionMode) -> np.ndarray:
    """S_X of stage k at the start point x0 (new variable = 0), like A."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1)
    S = np.zeros((2, prec.limbs, (m + p) * m))
    inp.check(inp.lib.pt_pieri_special(m, p, k, dptr(x0), int(prec), dptr(S)))
    return S


@dataclass
class StageLog:
    stage: int
    steps: int
    newton_iters: int
    success: bool


@dataclass
class PieriResult:
    point: np.ndarray             # (2, L, m p) final solution
    residual: float               # max_i |det(A^(i) | X(point))|, i = 1 .. m p
    stages: List[StageLog] = field(default_factory=list)


class PieriStageError(RuntimeError):
    def __init__(self, stage: int, msg: str):
        super().__init__(f"Pieri stage {stage}: {msg}")
        self.stage = stage


def stage_homotopy(m: int, p: int, k: int, planes: np.ndarray, x0: np.ndarray, prec: PrecisionMode):
    """(g, f) of stage k >= 2 (start point x0 with the new variable at 0)."""
    S = choose_special_matrix(m, p, k, x0, prec)
    shared = None
    for i in range(k - 1):
        e = minor_expand(m, p, k, planes[i], prec)
        shared = e if shared is None else stack_systems(shared, e)
    g = stack_systems(shared, minor_expand(m, p, k, S, prec))
    f = stack_systems(shared, minor_expand(m, p, k, planes[k - 1], prec))
    return g, f


def pieri_sequence(m: int, p: int, seed: int, prec: PrecisionMode = PrecisionMode.DD,
                   params: Optional[StepControlParams] = None,
                   tracker: Optional[PathTracker] = None) -> PieriResult:
    """pieri_sequence(n, m, p, seed, trackerParams)."""
    if m < 1 or p < 1:
        raise ValueError("need m, p >= 1 (m + p = n)")
    params = params or StepControlParams.defaults(prec)
    tracker = tracker or gpu_path_tracker()
    L, K = prec.limbs, m * p
    planes = pieri_planes(m, p, K, seed, prec)
    x = np.zeros(2 * L)
    inp.check(inp.lib.pt_pieri_linear_start(m, p, dptr(np.ascontiguousarray(planes[0])), int(prec), dptr(x)))
    x = x.reshape(2, L, 1)
    stages = [StageLog(1, 0, 0, True)]
    for k in range(2, K + 1):
        x0 = np.zeros((2, L, k))
        x0[:, :, : k - 1] = x
        g, f = stage_homotopy(m, p, k, planes, x0, prec)
        gamma = gamma_from_seed(seed + 1000 + k, prec)
        end, ok, steps, iters = tracker(g, f, gamma, x0, params)
        stages.append(StageLog(k, int(steps), int(iters), bool(ok)))
        if not ok:
            raise PieriStageError(k, f"path failed after {steps} steps")
        x = np.asarray(end).reshape(2, L, k)
    res = max(abs(pieri_det(m, p, K, planes[i], x, prec)) for i in range(K))
    return PieriResult(x, float(res), stages)
