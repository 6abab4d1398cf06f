#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200: tracked paths per second
(= 1 / seconds per tracked path) for the Chandrasekhar H dim-64 single path
in double-double (configs[1]); other configs via --workload / --prec.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload chandra64|cyclic16|rand96|cyclic256|batch32] [--prec d|dd|qd]

A step is one tracked path (single-path workloads) or one pass over the whole
batch (batch32).  Single paths do not shard: at N > 1 every rank tracks its
own replica ("replicas only") and value counts all ranks'
paths; batch32 shards the 8192 paths contiguously over the ranks.
value:  device time (CUDA events on the launching stream, inputs resident,
        L2 flushed between steps, max over ranks).
e2e:    the same metric through the C-ABI pt_track_path / pt_track_batch with
        pinned host buffers (H2D of the start, D2H of end point and stats
        inside the timed region), wall clock, max over ranks.
roofline: algorithmic FP64 instructions of the reference DD/QD algorithms per
        launch (pt_plan_work x the path's evaluation / solve / step counts)
        over the measured FP64 DFMA peak (profiles/fp64_peak.json).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tracked paths/s (1 / sec per tracked path); chandra64 dd single path"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="chandra64")
    ap.add_argument("--prec", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-reference", action="store_true",
                    help="skip the precision-matched CPU tracker timing (keep the CPU-D comparison)")
    ap.add_argument("--max-steps", type=int, default=None,
                    help="track only a prefix of the path (per-step timing of huge configs)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload(args):
    from paper_1501_06625_b200 import PrecisionMode, workloads as W
    prec = PrecisionMode.parse(args.prec) if args.prec else None
    if args.workload == "cyclic16":
        return W.cyclic_leg(4, (prec if prec is not None else PrecisionMode.DD))
    if args.workload == "cyclic256":
        return W.cyclic_leg(16, (prec if prec is not None else PrecisionMode.QD))
    if args.workload == "chandra64":
        return W.chandra(64, (prec if prec is not None else PrecisionMode.DD))
    if args.workload == "rand96":
        return W.random_system(96, 4, 65536, (prec if prec is not None else PrecisionMode.DD))
    if args.workload == "batch32":
        return W.batch(prec=(prec if prec is not None else PrecisionMode.DD))
    raise SystemExit(f"unknown workload {args.workload}")


def apply_overrides(args, w):
    if args.max_steps is not None:
        w.params.max_steps = args.max_steps
        w.name += f"-prefix{args.max_steps}"
    return w


def config(args, w, world):
    cfg = {"workload": w.name, "n_vars": w.n, "n_eqs": w.N, "precision": w.prec.name.lower(),
           "paths_per_step": int(w.starts.shape[0]) if args.workload == "batch32" else world,
           "parallelism": ("shard" if args.workload == "batch32" else "replicas") + f"x{world}",
           "l2": "flushed between steps (256 MiB write)"}
    return cfg


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak():
    """Measured FP64 DFMA peak (profiles/fp64_peak.json written by
    tools/measure_fp64_peak.py on the B200 pool); live fallback."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d["instr_per_s"], "measured (profiles/fp64_peak.json, DFMA microbenchmark on B200)"
    from paper_1501_06625_b200 import _native as nat
    v, ms = C.c_double(), C.c_double()
    nat.check(nat.lib.pt_fp64_peak(0, C.byref(v), C.byref(ms)))
    return v.value, "measured live (pt_fp64_peak DFMA microbenchmark)"


def path_work(hom, stats_list, degree):
    """Algorithmic FP64 instructions of the tracked path(s) (csrc/work.hpp)."""
    from paper_1501_06625_b200 import _native as nat
    buf = np.zeros(6)

    def w(kind, d=0):
        nat.check(nat.lib.pt_plan_work(hom.plan, kind, d, nat.dptr(buf)))
        return float(buf[5])

    we, ws = w(0), w(1)
    wp = [w(2, d) for d in range(degree + 1)]
    total = 0.0
    for st in stats_list:
        total += st.newton_iters * we + st.solves * ws
        for s in range(st.steps):  # predictor degree grows with the accepted count (upper bound s)
            total += wp[min(degree, s)]
    return total, we, ws


def critical_path(hom, st, prof, steps):
    """Latency view of a single path (the FP64-pipe fraction is tiny by
    construction): the MGS sweep is a chain of n dependent column steps
    (project column k+1 with q_k, normalise it, hand q_{k+1} on).  From the
    device timeline of the last sweep: median ns per column step, and the
    share of the measured MGS time that n x solves x that step explains."""
    from paper_1501_06625_b200 import _native as nat
    n = hom.n
    buf = np.zeros(6 * (n + 1))
    if nat.lib.pt_plan_mgs_timeline(hom.plan, nat.dptr(buf), buf.size) != 0:
        return None
    t = buf.reshape(n + 1, 6)
    cols = [j for j in range(2, n) if t[j, 5] > 0 and t[j - 1, 5] > 0]
    if not cols:
        return None
    col_ns = float(np.median([t[j, 5] - t[j - 1, 5] for j in cols]))
    mgs_ns = prof[2] / steps
    chain_ns = col_ns * n * st.solves
    return {"columns_per_solve": n, "solves": int(st.solves), "ns_per_column_step": col_ns,
            "chain_share_of_mgs": chain_ns / mgs_ns if mgs_ns > 0 else None,
            "mgs_share_of_phases": float(prof[2] / sum(prof[:5])) if sum(prof[:5]) > 0 else None}


def cpu_reference(args, w, seconds):
    """The reference CPU tracker on this host's cores: oracle/_ref (SPEC
    tracker on the unmodified reference headers), else the oracle port."""
    from oracle.orc import Oracle
    orc = Oracle("auto")
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    starts = w.starts if args.workload == "batch32" else w.starts[:1]
    done, t0 = 0, time.perf_counter()
    stats = None
    while True:
        for p in range(starts.shape[0]):
            _, stats, _ = orc.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, starts[p], w.params)
            done += 1
            if time.perf_counter() - t0 > seconds:
                break
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    kind = "reference" if orc.variant == "reference" else "port"
    sample = (f"{done} tracked path(s) of {w.name} in {dt:.2f}s with {threads} OpenMP threads "
              f"({'SPEC tracker on the unmodified reference arithmetic headers, oracle/_ref' if kind == 'reference' else 'oracle restatement'})")
    return {"value": done / dt, "unit": "paths/s", "cores": threads, "kind": kind, "sample": sample,
            "last_steps": stats.steps if stats else None}


def cpu_d_all_cores(args, seconds=2.0):
    """North-star comparison: the reference CPU tracker in complex DOUBLE on
    all host cores, same system and prefix (--max-steps): seconds per tracked
    path and per Newton iteration (the per-iteration figure is the fair one
    for prefixes, whose step counts differ between precisions)."""
    from paper_1501_06625_b200 import PrecisionMode
    from oracle.orc import Oracle
    a = argparse.Namespace(**vars(args))
    a.prec = "d"
    wd = apply_overrides(a, workload(a))
    if args.workload == "batch32":
        return None
    orc = Oracle("auto")
    orc.set_threads(os.cpu_count() or 1)
    n, iters, t0 = 0, 0, time.perf_counter()
    while True:
        _, st, _ = orc.track_path(int(PrecisionMode.D), wd.g, wd.f, wd.gamma, wd.k, wd.start, wd.params)
        n += 1
        iters += st.newton_iters
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"sec_per_path": dt / n, "sec_per_newton_iter": dt / max(1, iters), "cores": os.cpu_count() or 1,
            "paths": n, "newton_iters_per_path": iters / n, "workload": wd.name}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = apply_overrides(args, workload(args))
    per_step = max(args.cpu_seconds / max(args.steps, 1), 0.5)
    vals = []
    for _ in range(args.warmup):
        cpu_reference(args, w, 0.1)
    for _ in range(args.steps):
        vals.append(cpu_reference(args, w, per_step))
    value = sum(v["value"] for v in vals) / len(vals)
    base = vals[-1]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": {"D": "f64", "DD": "dd (2xf64)", "QD": "qd (4xf64)"}[w.prec.name],
            "data": "synthetic (pinned generators, SURVEY.md 8(d))", "config": config(args, w, 1),
            "cpu_baseline": {**{k: base[k] for k in ("unit", "cores", "kind", "sample")}, "value": value},
            "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if torch.cuda.is_available() else 0
    torch.cuda.set_device(device)
    import paper_1501_06625_b200 as pt
    from paper_1501_06625_b200 import _native as nat

    w = apply_overrides(args, workload(args))
    L, n = w.prec.limbs, w.n
    batch = args.workload == "batch32"
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=device)
    sp = w.params.native()
    stream = torch.cuda.Stream(device)  # kernel and its CUDA events on the same stream
    sh = C.c_void_p(stream.cuda_stream)
    if batch:
        P = w.starts.shape[0]
        lo, hi = rank * P // world, (rank + 1) * P // world
        starts_h = w.starts[lo:hi]
    else:
        starts_h = w.starts[:1]
    npaths = starts_h.shape[0]
    d_start = torch.from_numpy(np.ascontiguousarray(starts_h)).to(f"cuda:{device}")
    d_end = torch.zeros_like(d_start)
    d_stats = torch.zeros((npaths, C.sizeof(nat.PathStats)), dtype=torch.uint8, device=f"cuda:{device}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")

    def launch():
        if batch:
            nat.check(nat.lib.pt_track_batch_device(hom.plan, npaths, C.c_void_p(d_start.data_ptr()), C.byref(sp),
                                                    C.c_void_p(d_end.data_ptr()), C.c_void_p(d_stats.data_ptr()), sh))
        else:
            nat.check(nat.lib.pt_track_path_device(hom.plan, C.c_void_p(d_start.data_ptr()), C.byref(sp),
                                                   C.c_void_p(d_end.data_ptr()), C.c_void_p(d_stats.data_ptr()), sh))

    def barrier():
        torch.cuda.synchronize(device)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            launch()
    barrier()
    clocks = Clocks(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    prof = np.zeros(8)
    nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
    for e0, e1 in ev:
        with torch.cuda.stream(stream):
            flush.zero_()
            e0.record(stream)
            launch()
            e1.record(stream)
    barrier()
    nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    t_dev = sum(step_ms) / 1e3
    stats_raw = d_stats.cpu().numpy()
    stats_list = [nat.PathStats.from_buffer_copy(stats_raw[p].tobytes()) for p in range(npaths)]

    # e2e through the public C-ABI with pinned host buffers
    h_start = torch.from_numpy(np.ascontiguousarray(starts_h)).pin_memory()
    h_end = torch.zeros_like(h_start).pin_memory()
    h_stats = (nat.PathStats * npaths)()
    dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), nat._dp)

    def e2e_call():
        if batch:
            nat.check(nat.lib.pt_track_batch(hom.plan, npaths, dp(h_start), C.byref(sp), dp(h_end), h_stats))
        else:
            nat.check(nat.lib.pt_track_path(hom.plan, dp(h_start), C.byref(sp), dp(h_end), h_stats))

    e2e_call()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_call()
    t_e2e = time.perf_counter() - t0
    barrier()

    tt = torch.tensor([t_dev, t_e2e], dtype=torch.float64, device=f"cuda:{device}")
    if world > 1:
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    t_dev_max, t_e2e_max = float(tt[0]), float(tt[1])
    total_paths = (w.starts.shape[0] if batch else world) * args.steps
    value = total_paths / t_dev_max
    e2e_value = total_paths / t_e2e_max

    if rank == 0:
        work, we, ws = path_work(hom, stats_list, w.params.pred_degree)
        t_launch = t_dev / args.steps
        peak, peak_src = fp64_peak()
        achieved = work / t_launch
        traffic = None
        tr_path = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr_path):
            with open(tr_path) as fh:
                traffic = json.load(fh).get(w.name)
        ok = all(s.status == 0 for s in stats_list)
        line = {
            "metric": METRIC if args.workload == "chandra64" and w.prec.name == "DD" else
            f"tracked paths/s; {w.name}",
            "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if batch else "weak", "vs_baseline": None,
            "dtype": {"D": "f64", "DD": "dd (2xf64)", "QD": "qd (4xf64)"}[w.prec.name],
            "data": "synthetic (pinned generators, SURVEY.md 8(d)); no checkpoints",
            "config": config(args, w, world),
            "sec_per_path": t_dev_max / args.steps / (npaths if batch else 1),
            "path": {"success": ok, "steps": stats_list[0].steps, "newton_iters": stats_list[0].newton_iters,
                     "solves": stats_list[0].solves, "grid_ctas": hom.info(4), "engine": hom.engine,
                     "cluster_ctas": hom.info(9), "paths_ok": int(sum(s.status == 0 for s in stats_list)),
                     "paths": len(stats_list)},
            "e2e": {"value": e2e_value, "unit": "paths/s",
                    "h2d_bytes_per_step": int(h_start.numel() * 8),
                    "d2h_bytes_per_step": int(h_end.numel() * 8 + C.sizeof(nat.PathStats) * npaths),
                    "timing": "wall clock around the C-ABI call, max over ranks"},
            "roofline": {"bound": "fp64-pipe",
                         "kernel": "k_track_batch" if batch else ("k_track_cluster" if hom.engine == "cluster" else "k_track_grid"),
                         "achieved": achieved * 1e-12, "peak": peak * 1e-12,
                         "unit": "T FP64-instr/s (DADD/DMUL/DFMA of the reference DD/QD algorithms; FMA = 1)",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "work_per_launch_fp64_instr": work, "work_per_eval": we, "work_per_solve": ws},
            "gpu_launches": args.steps,
            "phase_ms_per_path": None if batch else {
                k: prof[i] * 1e-6 / args.steps for i, k in enumerate(
                    ["monomials", "slot_sums", "mgs", "backsub_update", "predict"])},
            "newton_iters_timed": None if batch else prof[5] / args.steps,
            "critical_path": None if batch else critical_path(hom, stats_list[0], prof, args.steps),
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            if not args.no_cpu_reference:
                line["cpu_baseline"] = cpu_reference(args, w, args.cpu_seconds)
            dall = cpu_d_all_cores(args)
            if dall is not None:
                line["cpu_d_all_cores"] = dall
                line["sec_per_newton_iter"] = t_dev_max / args.steps / max(1, stats_list[0].newton_iters)
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
