"""Monodromy driver over the B200 tracker -- the first SURVEY.md 8(f) "next"
row: the immediate caller of track_path for cyclic witness sets.

  monodromy_loop    SPEC.md:570-576  (Eqs. (9)-(10))
  monodromy_degree  SPEC.md:577-582  (PAPER.md 4.2)

A loop tracks h_alpha = {f = 0, alpha (1-t) L + t K = 0} from t = 0 to 1 and
then h_beta = {f = 0, beta (1-t) K + t L = 0} back, with the Eq.-(1) machinery
at k = 1 and gamma in {alpha, beta}; start and target share the f equations
(the plan sums them once).  Every known witness point goes around the loop
in ONE batch launch per leg (pt_track_batch: one CTA per path), so a degree
computation costs two kernel launches per loop.

Seeds: the slice K and the unit complex alpha, beta of loop i come from
pathtrack::Rng (rng.hpp) seeded with (seed, i), so the same seeds give the same
endpoint bits.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from .systems import (PolynomialSystem, PrecisionMode, StepControlParams, augment_with_linear,
                      gamma_from_seed)

# (g, f, gamma, starts[P,2,L,n], params) -> (ends[P,2,L,n], success[P])
BatchTracker = Callable[[PolynomialSystem, PolynomialSystem, np.ndarray, np.ndarray, StepControlParams],
                        tuple]
# (system, points[P,2,L,n]) -> max_i |f_i(point)| per point (binary64), evaluated in the system's precision
Evaluator = Callable[[PolynomialSystem, np.ndarray], np.ndarray]

# point-matching tolerance per precision (SPEC.md "DESIGN DECISIONS": 1e-6 D, 1e-12 DD)
MATCH_TOL = {PrecisionMode.D: 1e-6, PrecisionMode.DD: 1e-12, PrecisionMode.QD: 1e-12}


def gpu_batch_tracker(device: int = 0) -> BatchTracker:
    """The product path: one plan per leg, all points in one batch launch."""

    def run(g, f, gamma, starts, params):
        from .tracker import make_homotopy
        hom = make_homotopy(g, f, gamma, 1, device=device)
        ends, outs = hom.track_batch(starts, params)
        return ends, np.array([o.success for o in outs], dtype=bool)

    return run


def gpu_evaluator(device: int = 0) -> Evaluator:
    """max_modulus(f(x)) on the device: evaluate_homotopy of (f, f) at t = 1."""

    def run(sysm, points):
        from .tracker import make_homotopy
        one = np.zeros(2 * sysm.prec.limbs)
        one[0] = 1.0
        hom = make_homotopy(sysm, sysm, one, 1, device=device)
        out = np.array([hom.evaluate(p, 1.0)[2] for p in points])
        hom.close()
        return out

    return run


@dataclass
class LoopResult:
    points: np.ndarray        # [P, 2, L, n] endpoints back on (f, L)
    success: np.ndarray       # [P] both legs succeeded
    mid: np.ndarray           # [P, 2, L, n] endpoints of the first leg (on (f, K))


def loop_seeds(seed: int, i: int):
    """(K slice seed, alpha seed, beta seed) of loop i."""
    base = (seed * 1_000_003 + 7919 * (i + 1)) & 0xFFFFFFFF
    return base + 1, base + 2, base + 3


def monodromy_loop(fL: PolynomialSystem, fK: PolynomialSystem, points: np.ndarray, alpha: np.ndarray,
                   beta: np.ndarray, params: Optional[StepControlParams] = None,
                   tracker: Optional[BatchTracker] = None) -> LoopResult:
    """monodromy_loop for a batch of witness points of (f, L)."""
    params = params or StepControlParams.defaults(fL.prec)
    tracker = tracker or gpu_batch_tracker()
    points = np.ascontiguousarray(points, dtype=np.float64)
    mid, ok1 = tracker(fL, fK, alpha, points, params)        # h_alpha: (f,L) -> (f,K)
    back, ok2 = tracker(fK, fL, beta, mid, params)           # h_beta:  (f,K) -> (f,L)
    return LoopResult(back, ok1 & ok2, mid)


def _distinct(a: np.ndarray, b: np.ndarray, tol: float) -> bool:
    """Leading-limb distance of two points (re/im hi limbs) above tol (relative)."""
    za = a[0, 0] + 1j * a[1, 0]
    zb = b[0, 0] + 1j * b[1, 0]
    scale = max(1.0, float(np.max(np.abs(za))))
    return float(np.max(np.abs(za - zb))) > tol * scale


@dataclass
class WitnessSet:
    points: List[np.ndarray] = field(default_factory=list)   # each [2, L, n]
    loops: int = 0
    failed_paths: int = 0
    residuals: List[float] = field(default_factory=list)     # (f, L) residual of each stored point
    rejected_residual: int = 0   # endpoints whose (f, L) residual failed the insertion check
    jumped: int = 0              # endpoints that left the start component (path jumping)
    log: List[str] = field(default_factory=list)             # loop-by-loop discoveries

    @property
    def degree(self) -> int:
        return len(self.points)


def monodromy_degree(n_cyclic: int, dim: int, start_witness: Sequence[np.ndarray], seed: int,
                     stabilization_loops: int, prec: PrecisionMode = PrecisionMode.DD,
                     loop_budget: int = 64, slice_seed: int = 1, match_tol: Optional[float] = None,
                     params: Optional[StepControlParams] = None,
                     tracker: Optional[BatchTracker] = None,
                     evaluator: Optional[Evaluator] = None, residual_tol: Optional[float] = None,
                     component_key: Optional[Callable[[np.ndarray], complex]] = None) -> WitnessSet:
    """monodromy_degree on the cyclic-n component cut by
    `dim` affine slices L (augment_with_linear(n, dim, slice_seed)): every loop
    sends all known points around a fresh (alpha, beta, K) loop and adds the
    endpoints at distance > match_tol (default MATCH_TOL[prec]) from every
    known point; stops after `stabilization_loops` consecutive loops without a
    new point, or after `loop_budget` loops.  Raises RuntimeError when every
    path of every loop fails.

    Insertion checks (SPEC.md bench invariants): the (f, L) residual of a new
    point is re-evaluated (`evaluator`, default the device) and must be below
    `residual_tol` (default the corrector tolerance); with `component_key`
    (an invariant of the start component, e.g. workloads.backelin_component_key)
    an endpoint whose key differs from the start witness's has jumped to
    another component -- a path-crossing failure of that loop -- and is
    rejected, not counted."""
    if not start_witness:
        raise ValueError("start witness set is empty")
    params = params or StepControlParams.defaults(prec)
    tracker = tracker or gpu_batch_tracker()
    evaluator = evaluator or gpu_evaluator()
    match_tol = MATCH_TOL[prec] if match_tol is None else match_tol
    residual_tol = params.newton_tol if residual_tol is None else residual_tol
    fL = augment_with_linear(n_cyclic, dim, slice_seed, prec)
    ws = WitnessSet([np.array(p, dtype=np.float64) for p in start_witness])
    ws.residuals = [float(r) for r in evaluator(fL, np.stack(ws.points))]
    key0 = component_key(ws.points[0]) if component_key else None
    quiet, any_ok = 0, False
    while quiet < stabilization_loops and ws.loops < loop_budget:
        k_seed, a_seed, b_seed = loop_seeds(seed, ws.loops)
        fK = augment_with_linear(n_cyclic, dim, k_seed, prec)
        res = monodromy_loop(fL, fK, np.stack(ws.points), gamma_from_seed(a_seed, prec),
                             gamma_from_seed(b_seed, prec), params, tracker)
        ws.loops += 1
        ws.failed_paths += int(np.count_nonzero(~res.success))
        any_ok |= bool(res.success.any())
        cand = [np.array(p) for p, ok in zip(res.points, res.success)
                if ok and all(_distinct(p, q, match_tol) for q in ws.points)]
        if key0 is not None:
            kept = [p for p in cand if abs(component_key(p) - key0) <= 1e-6 * max(1.0, abs(key0))]
            ws.jumped += len(cand) - len(kept)
            cand = kept
        new = 0
        if cand:
            resid = evaluator(fL, np.stack(cand))
            for p, r in zip(cand, resid):
                if not (r < residual_tol):
                    ws.rejected_residual += 1
                elif all(_distinct(p, q, match_tol) for q in ws.points):
                    ws.points.append(p)
                    ws.residuals.append(float(r))
                    new += 1
        ws.log.append(f"loop {ws.loops}: {new} new, degree {ws.degree}")
        quiet = 0 if new else quiet + 1
    if ws.loops and not any_ok:
        raise RuntimeError(f"monodromy: all {ws.failed_paths} paths of {ws.loops} loops failed")
    return ws
