"""Command-line front end:

  python -m paper_1501_06625_b200.cli --mode track     --system f.sys [--start-system g.sys] [--start s.sol]
  python -m paper_1501_06625_b200.cli --mode track     --cyclic 16           (built-in monodromy leg)
  python -m paper_1501_06625_b200.cli --mode monodromy --cyclic 4 | --cyclic 16 [--witness w.sol]
  python -m paper_1501_06625_b200.cli --mode pieri     --pieri 4,2,2
  python -m paper_1501_06625_b200.cli --mode evalbench --cyclic 16 | --system f.sys  [--reps 100]

Reports use Table 9's columns (Table 9: n, s, m, time):
s = 1 for a path that reached t = 1, m = predictor-corrector trials.
Exit codes (SPEC.md "Invariants"): 0 the mathematical task succeeded,
1 it did not (a path failed, a stage failed, no witness found),
2 usage / configuration / input errors.  All randomness flows from --seed.

Tracking runs on the device through the product C-ABI (pt_track_path /
pt_track_batch / pt_eval_bench); without a CUDA device the tracker modes
fail with the library's PT_E_NODEVICE error (there is no CPU fallback).
"""
from __future__ import annotations

import argparse
import sys
import time
from typing import List, Optional

import numpy as np

from . import systems as S
from .systems import PrecisionMode, StepControlParams

EXIT_OK, EXIT_FAIL, EXIT_USAGE = 0, 1, 2


class UsageError(Exception):
    pass


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1501_06625_b200.cli",
                                 description="B200 polynomial homotopy path tracker (D / DD / QD)")
    ap.add_argument("--mode", required=True, choices=["track", "monodromy", "pieri", "evalbench"])
    ap.add_argument("--precision", default=None,
                    help="d, dd or qd (default dd; evalbench: a comma list, default d,dd,qd)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tol", type=float, default=None, help="corrector tolerance (default per precision)")
    ap.add_argument("--max-step", type=float, default=None)
    ap.add_argument("--min-step", type=float, default=None)
    ap.add_argument("--max-steps", type=int, default=None)
    ap.add_argument("--degree", type=int, default=None, help="predictor extrapolation degree")
    ap.add_argument("--system", help="target system file (polysys grammar, SPEC.md:197)")
    ap.add_argument("--start-system", help="start system file (default: total degree x_i^d_i - 1)")
    ap.add_argument("--start", help="start solutions file (default: all-ones total-degree root)")
    ap.add_argument("--witness", help="witness set file (solutions format) for --mode monodromy")
    ap.add_argument("--trace", help="write the per-trial trace here")
    ap.add_argument("--out", help="write end solutions / the witness set here (solutions format)")
    ap.add_argument("--cyclic", type=int, help="cyclic n-roots benchmark (n = m^2 for built-in witnesses)")
    ap.add_argument("--pieri", help="N,M,P with M + P = N")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--loops", type=int, default=4, help="monodromy stabilisation loops")
    ap.add_argument("--device", type=int, default=0)
    return ap


def _prec(text: Optional[str]) -> PrecisionMode:
    try:
        return PrecisionMode.parse(text or "dd")
    except ValueError as e:
        raise UsageError(str(e))


def _params(args, prec: PrecisionMode) -> StepControlParams:
    p = StepControlParams.defaults(prec)
    for name, attr in (("tol", "newton_tol"), ("max_step", "max_step"), ("min_step", "min_step"),
                       ("max_steps", "max_steps"), ("degree", "pred_degree")):
        v = getattr(args, name)
        if v is not None:
            setattr(p, attr, v)
    if not (0 < p.min_step <= p.max_step <= 1) or p.max_steps < 0 or not 0 <= p.pred_degree <= 8:
        raise UsageError("step control out of range: need 0 < min-step <= max-step <= 1, max-steps >= 0, "
                         "0 <= degree <= 8")
    return p


def _read(path: str, what: str) -> str:
    try:
        with open(path) as fh:
            return fh.read()
    except OSError as e:
        raise UsageError(f"cannot read {what} '{path}': {e.strerror}")


def _parse_system_file(path: str, prec: PrecisionMode) -> S.PolynomialSystem:
    try:
        return S.parse_system(_read(path, "system file"), prec)
    except ValueError as e:
        raise UsageError(f"{path}: {e}")


def _total_degree_start(f: S.PolynomialSystem) -> S.PolynomialSystem:
    """g_i = x_i^{d_i} - 1 with d_i = deg f_i (square systems)."""
    if f.n_eqs != f.n_vars:
        raise UsageError("the default total-degree start system needs a square target; pass --start-system")
    eqs = []
    for i in range(f.n_eqs):
        d = max([sum(e for _, e in sup) for sup, _ in f.terms(i)] or [1])
        eqs.append([([], -1.0), ([(i, max(d, 1))], 1.0)])
    return S.canonical(S.PolynomialSystem.from_terms(f.n_vars, eqs, f.prec))


def _report(rows: List[dict], out=sys.stdout) -> None:
    """Table 9 layout: n, s, m, time (seconds), plus the Newton count."""
    print(f"{'n':>5} {'prec':>4} {'s':>2} {'m':>5} {'newton':>7} {'time':>11}", file=out)
    for r in rows:
        print(f"{r['n']:>5} {r['prec']:>4} {r['s']:>2} {r['m']:>5} {r['newton']:>7} {r['time']:>11.6f}", file=out)


def run_track(args) -> int:
    """run_track."""
    prec = _prec(args.precision)
    params = _params(args, prec)
    if args.cyclic:
        from . import workloads as W
        m = int(round(args.cyclic ** 0.5))
        if m * m != args.cyclic:
            raise UsageError(f"--cyclic {args.cyclic}: the built-in Backelin witness needs n = m^2 "
                             f"(pass --system/--start for other n)")
        w = W.cyclic_leg(m, prec, seed_l=args.seed, seed_k=args.seed + 1, seed_gamma=args.seed + 2)
        g, f, gamma, k, starts = w.g, w.f, w.gamma, w.k, w.starts
    else:
        if not args.system:
            raise UsageError("--mode track needs --system FILE (or --cyclic N)")
        f = _parse_system_file(args.system, prec)
        g = _parse_system_file(args.start_system, prec) if args.start_system else _total_degree_start(f)
        if g.n_vars != f.n_vars or g.n_eqs != f.n_eqs:
            raise UsageError("start and target systems differ in shape")
        gamma, k = S.gamma_from_seed(args.seed, prec), 2
        if args.start:
            try:
                sols = S.read_solutions(_read(args.start, "start file"), prec)
            except ValueError as e:
                raise UsageError(f"{args.start}: {e}")
            if not sols or sols[0].point.shape[-1] != f.n_vars:
                raise UsageError(f"{args.start}: expected points of dimension {f.n_vars}")
            starts = np.stack([s.point for s in sols])
        else:
            starts = S.limbs_from_complex(np.ones(f.n_vars), prec)[None]
    from .tracker import make_homotopy
    hom = make_homotopy(g, f, gamma, k, device=args.device)
    rows, sols, ok_all = [], [], True
    trace_lines = []
    for p in range(starts.shape[0]):
        t0 = time.perf_counter()
        out = hom.track_path(starts[p], params, trace=bool(args.trace))
        dt = time.perf_counter() - t0
        ok_all &= out.success
        rows.append({"n": f.n_vars, "prec": prec.name.lower(), "s": int(out.success), "m": out.steps,
                     "newton": out.newton_iters, "time": dt})
        sols.append(S.Solution(out.end, out.t_end, out.final_residual, out.final_update))
        for ev in out.trace:
            trace_lines.append(f"{p} {ev.t!r} {ev.ok} {ev.iters} {ev.residual!r} {ev.update!r}")
    _report(rows)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(S.write_solutions(sols, prec))
    if args.trace:
        with open(args.trace, "w") as fh:
            fh.write("# path t ok newton_iters residual update\n" + "\n".join(trace_lines) + "\n")
    return EXIT_OK if ok_all else EXIT_FAIL


def run_monodromy(args) -> int:
    """run_monodromy: loop-by-loop discoveries and the degree."""
    from . import monodromy as MD
    from . import workloads as W
    prec = _prec(args.precision)
    params = _params(args, prec)
    n = args.cyclic
    if not n:
        raise UsageError("--mode monodromy needs --cyclic N")
    fact = S.cyclic_degree(n) if n >= 4 else None
    m = int(round(n ** 0.5))
    dim = (m - 1) if m * m == n else (fact.dim if fact else 0)
    if dim < 1:
        raise UsageError(f"cyclic-{n} has no positive-dimensional Backelin component (Table 5)")
    fL = S.augment_with_linear(n, dim, args.seed, prec)
    key = None
    if args.witness:
        try:
            start = [s.point for s in S.read_solutions(_read(args.witness, "witness file"), prec)]
        except ValueError as e:
            raise UsageError(f"{args.witness}: {e}")
        if not start:
            raise UsageError(f"{args.witness}: empty witness set")
    elif n == 4:
        pts = W.cyclic4_witness(W.slice_rows(fL, 1)[0], family=1)
        start = [S.limbs_from_complex(pts[0], prec)]
    elif m * m == n:
        start = [S.limbs_from_complex(W.backelin_witness(fL, m, dim), prec)]
        key = W.backelin_component_key(m)
    else:
        raise UsageError(f"cyclic-{n}: no built-in witness for n != m^2; pass --witness FILE "
                         f"(a solutions file of points on cyclic-{n} augmented with {dim} slices, seed {args.seed})")
    from .tracker import make_homotopy
    one = np.zeros(2 * prec.limbs)
    one[0] = 1.0
    # polish the start points with the t = 0 Newton pass of the tracker
    hom = make_homotopy(fL, fL, one, 1, device=args.device)
    ends, outs = hom.track_batch(np.stack(start), params)
    start = [e for e, o in zip(ends, outs) if o.success]
    if not start:
        print("monodromy: the start witness does not satisfy (f, L)", file=sys.stderr)
        return EXIT_FAIL
    t0 = time.perf_counter()
    ws = MD.monodromy_degree(n, dim, start, seed=args.seed, stabilization_loops=args.loops, prec=prec,
                             slice_seed=args.seed, params=params, tracker=MD.gpu_batch_tracker(args.device),
                             evaluator=MD.gpu_evaluator(args.device), component_key=key)
    for line in ws.log:
        print(line)
    print(f"cyclic-{n} degree estimate {ws.degree} ({ws.loops} loops, {ws.failed_paths} failed paths, "
          f"{ws.jumped} jumped, {time.perf_counter() - t0:.3f} s)"
          + (f"; Table 5 degree {fact.degree}" if fact else ""))
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(S.write_solutions([S.Solution(p, 1.0, r, 0.0) for p, r in zip(ws.points, ws.residuals)], prec))
    return EXIT_OK if ws.degree >= 1 and ws.loops > 0 else EXIT_FAIL


def run_pieri(args) -> int:
    """run_pieri: per-stage rows and the final residual."""
    from . import pieri as PI
    prec = _prec(args.precision)
    params = _params(args, prec)
    try:
        n, m, p = [int(v) for v in (args.pieri or "").split(",")]
    except ValueError:
        raise UsageError("--pieri takes N,M,P")
    if m + p != n or m < 1 or p < 1:
        raise UsageError(f"--pieri {n},{m},{p}: need M + P = N with M, P >= 1")
    t0 = time.perf_counter()
    try:
        r = PI.pieri_sequence(m, p, args.seed, prec, params, PI.gpu_path_tracker(args.device))
    except PI.PieriStageError as e:
        print(f"pieri: {e}", file=sys.stderr)
        return EXIT_FAIL
    print(f"{'stage':>5} {'m':>5} {'newton':>7}")
    for s in r.stages:
        print(f"{s.stage:>5} {s.steps:>5} {s.newton_iters:>7}")
    print(f"pieri {n},{m},{p} {prec.name.lower()}: final residual {r.residual:.3e}, "
          f"{time.perf_counter() - t0:.3f} s")
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(S.write_solutions([S.Solution(r.point, 1.0, r.residual, 0.0)], prec))
    return EXIT_OK


def run_evalbench(args) -> int:
    """run_evalbench: device time per evaluation +
    differentiation pass per precision, like the CPU rows of Tables 2-4."""
    precs = [_prec(x.strip()) for x in (args.precision or "d,dd,qd").split(",")]
    if args.reps < 0:
        raise UsageError("--reps must be >= 0")
    print(f"{'prec':>4} {'n':>5} {'N':>5} {'reps':>6} {'ms/eval':>12}")
    if args.reps == 0:
        return EXIT_OK
    from .tracker import eval_bench, make_homotopy
    for prec in precs:
        if args.cyclic:
            f = S.cyclic_system(args.cyclic, prec)
        elif args.system:
            f = _parse_system_file(args.system, prec)
        else:
            raise UsageError("--mode evalbench needs --system FILE or --cyclic N")
        one = np.zeros(2 * prec.limbs)
        one[0] = 1.0
        hom = make_homotopy(f, f, one, 1, device=args.device)
        rng = np.random.default_rng(args.seed)
        x = S.limbs_from_complex(np.exp(2j * np.pi * rng.uniform(size=f.n_vars)), prec)
        ms = eval_bench(hom, x, 0.5, args.reps)
        print(f"{prec.name.lower():>4} {f.n_vars:>5} {f.n_eqs:>5} {args.reps:>6} {ms:>12.6f}")
    return EXIT_OK


def main(argv: Optional[List[str]] = None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # argparse: --help (0) or a usage error (2)
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return {"track": run_track, "monodromy": run_monodromy, "pieri": run_pieri,
                "evalbench": run_evalbench}[args.mode](args)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
