#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200.

Default line (no flags): "paths/sec/box" on configs[4], the batch of 8192
independent paths of the dim-32 random degree-4 system (M = 512) in
double-double -- the workload that shards across GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload batch32|chandra64|cyclic16|rand96|cyclic256] [--prec d|dd|qd]

A step (batch) is one k_track_batch launch over a fixed slice of
--paths-per-step (4096, half the batch) paths per rank: at step s rank r tracks paths
[((s N + r) P) mod 8192, +P) (multi.step_slice) -- weak scaling, N ranks
cover N slices per step, no collective on the data path.  A step
(single-path workloads) is one tracked path; at N > 1 each rank tracks a
replica ("replicas only").

value:  paths per second over all ranks, device time (CUDA events on the
        launching stream, inputs resident in HBM, L2 flushed between steps
        by a 256 MiB write, max over ranks).
e2e:    the same metric through the public C-ABI pt_track_batch /
        pt_track_path with pinned host buffers: H2D of the starts and D2H of
        the end points and stats inside the timed region (wall clock, max
        over ranks).
roofline: FP64-pipe bound -- algorithmic FP64 instructions of the reference
        DD/QD algorithms per launch (pt_plan_work x each path's evaluation /
        solve / step counts) over the launch time, against the measured DFMA
        peak (profiles/fp64_peak.json).
cpu_baseline: the SPEC tracker on the unmodified reference headers
        (oracle/_ref) on this host's cores -- a thread pool over paths for the
        batch, plus the 1-thread single-path figure (i).
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

BATCH_METRIC = "paths/sec/box; batch of 8192 dim-32 random degree-4 paths (M=512), dd"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="batch32")
    ap.add_argument("--prec", default=None)
    # 4096: the launch tail (the last long paths of a launch, ~1.5 s) costs 4 % of a
    # 13 s step; 2048 / 4096 / 8192 measured 295 / 308 / 316 paths/s (profiles/r02)
    ap.add_argument("--paths-per-step", type=int, default=4096, help="batch: paths per rank per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-paths", type=int, default=96, help="batch: CPU sample paths per reference step")
    ap.add_argument("--no-cpu-reference", action="store_true",
                    help="skip the precision-matched CPU tracker timing (keep the CPU-D comparison)")
    ap.add_argument("--arith", default="reference", choices=["reference", "fast"],
                    help="QD only: fast = tolerance-parity quad-double arithmetic (pt_plan_set_arith)")
    ap.add_argument("--max-steps", type=int, default=None,
                    help="track only a prefix of the path (per-step timing of huge configs)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def is_batch(args):
    return args.workload == "batch32"


def workload(args):
    """Inputs only (libpt_inputs.so): never loads the tracker library."""
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
    if args.arith == "fast":
        w.name += "-fastqd"
    return w


def metric_of(args, w):
    if is_batch(args) and w.prec.name == "DD":
        return BATCH_METRIC
    return f"tracked paths/s (1 / sec per tracked path); {w.name}"


def config(args, w, world):
    cfg = {"workload": w.name, "n_vars": w.n, "n_eqs": w.N, "precision": w.prec.name.lower(),
           "arith": "reference (bit parity)" if args.arith == "reference" else "fast (tolerance parity)",
           "l2": "flushed between steps (256 MiB write)"}
    if is_batch(args):
        cfg.update({"batch_paths": int(w.starts.shape[0]), "paths_per_step_per_gpu": args.paths_per_step,
                    "paths_per_step": args.paths_per_step * world,
                    "parallelism": f"batch shards x{world} (multi.step_slice, no collective)"})
    else:
        cfg.update({"paths_per_step": world, "parallelism": f"replicas x{world}"})
    return cfg


def dtype_of(w):
    return {"D": "f64", "DD": "dd (2xf64)", "QD": "qd (4xf64)"}[w.prec.name]


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
    """Latency view of a single path: the MGS sweep is a chain of n dependent
    column steps; from the device timeline of the last sweep: median ns per
    column step and the share of the measured MGS time it explains."""
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


# ---------------------------------------------------------------------------
# CPU baselines (oracle/_ref: the SPEC tracker on the unmodified reference
# arithmetic headers; the oracle restatement where _ref was not built)
# ---------------------------------------------------------------------------
def _oracle():
    from oracle.orc import Oracle
    return Oracle("auto")


def cpu_batch_pool(w, n_paths, offset=0):
    """(iii): a thread pool over paths on all host cores, one single-threaded
    tracker per path."""
    orc = _oracle()
    threads = os.cpu_count() or 1
    idx = (offset + np.arange(n_paths)) % w.starts.shape[0]
    starts = np.ascontiguousarray(w.starts[idx])
    t0 = time.perf_counter()
    _, stats = orc.track_batch(int(w.prec), w.g, w.f, w.gamma, w.k, starts, w.params, threads)
    dt = time.perf_counter() - t0
    kind = "reference" if orc.variant == "reference" else "port"
    return {"value": n_paths / dt, "unit": "paths/s", "cores": threads, "kind": kind,
            "sample": f"{n_paths} paths [{int(idx[0])}..) of {w.name} in {dt:.2f}s on a pool of {threads} host "
                      f"threads, one single-threaded tracker per path "
                      f"({'oracle/_ref: SPEC tracker on the unmodified reference headers' if kind == 'reference' else 'oracle restatement'})",
            "paths_ok": int(sum(s.status == 0 for s in stats))}


def cpu_single(w, seconds, threads):
    """(i) one path on 1 thread, or (ii) one path with OpenMP inside it."""
    orc = _oracle()
    orc.set_threads(threads)
    done, t0 = 0, time.perf_counter()
    p = 0
    while True:
        orc.track_path(int(w.prec), w.g, w.f, w.gamma, w.k, w.starts[p % w.starts.shape[0]], w.params)
        done += 1
        p += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    kind = "reference" if orc.variant == "reference" else "port"
    return {"value": done / dt, "unit": "paths/s", "cores": threads, "kind": kind,
            "sample": f"{done} tracked path(s) of {w.name} in {dt:.2f}s, {threads} OpenMP thread(s) inside the path"}


def cpu_d_all_cores(args, seconds=2.0):
    """North-star comparison for single paths: the reference CPU tracker in
    complex DOUBLE on the host cores, same system and prefix (--max-steps).
    The per-path OpenMP of the tracker does not always pay in D (a 64 x 64
    column sweep is a few microseconds of work per fork), so both 1 thread
    and all cores are timed and the FASTER one is the baseline."""
    from paper_1501_06625_b200 import PrecisionMode
    a = argparse.Namespace(**vars(args))
    a.prec = "d"
    wd = apply_overrides(a, workload(a))
    orc = _oracle()
    best = None
    for threads in sorted({1, os.cpu_count() or 1}, reverse=True):
        orc.set_threads(threads)
        n, iters, t0 = 0, 0, time.perf_counter()
        while True:
            _, st, _ = orc.track_path(int(PrecisionMode.D), wd.g, wd.f, wd.gamma, wd.k, wd.start, wd.params)
            n += 1
            iters += st.newton_iters
            if time.perf_counter() - t0 > seconds / 2:
                break
        dt = time.perf_counter() - t0
        r = {"sec_per_path": dt / n, "sec_per_newton_iter": dt / max(1, iters), "cores": threads,
             "paths": n, "newton_iters_per_path": iters / n, "workload": wd.name}
        if best is None or r["sec_per_path"] < best["sec_per_path"]:
            best = r
    best["cores_available"] = os.cpu_count() or 1
    return best


def run_reference(args):
    """--impl reference: the reference CPU tracker (oracle/_ref) on the box's
    host cores, same metric/config/unit; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = apply_overrides(args, workload(args))
    vals = []
    if is_batch(args):
        for s in range(args.warmup):
            cpu_batch_pool(w, min(16, args.cpu_paths), offset=s * 16)
        for s in range(args.steps):
            vals.append(cpu_batch_pool(w, args.cpu_paths, offset=s * args.cpu_paths))
    else:
        per_step = max(args.cpu_seconds / max(args.steps, 1), 0.5)
        threads = os.cpu_count() or 1
        for _ in range(args.warmup):
            cpu_single(w, 0.1, threads)
        for _ in range(args.steps):
            vals.append(cpu_single(w, per_step, threads))
    value = sum(v["value"] for v in vals) / len(vals)
    base = vals[-1]
    line = {"impl": "reference", "metric": metric_of(args, w), "value": value, "unit": "paths/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(w),
            "data": "synthetic (pinned generators, SURVEY.md 8(d))", "config": config(args, w, 1),
            "cpu_baseline": {**{k: base[k] for k in ("unit", "cores", "kind", "sample")}, "value": value},
            "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line["ms_per_step"] = 1e3 * (args.cpu_paths if is_batch(args) else 1) / value
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
    from paper_1501_06625_b200.multi import step_slice

    w = apply_overrides(args, workload(args))
    batch = is_batch(args)
    hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k, device=device)
    if args.arith == "fast":
        hom.set_arith("fast")  # tolerance parity (tests/test_qdfast.py), QD plans only
    sp = w.params.native()
    stream = torch.cuda.Stream(device)  # kernel and its CUDA events on the same stream
    sh = C.c_void_p(stream.cuda_stream)
    PS = 2 * w.prec.limbs * w.n  # doubles per start point
    total_batch = w.starts.shape[0]
    P = args.paths_per_step if batch else 1
    # every start resident in HBM; each step points into its slice
    d_all = torch.from_numpy(np.ascontiguousarray(w.starts if batch else w.starts[:1])).to(f"cuda:{device}")
    d_end = torch.zeros((P,) + tuple(w.starts.shape[1:]), dtype=torch.float64, device=f"cuda:{device}")
    d_stats = torch.zeros((P, C.sizeof(nat.PathStats)), dtype=torch.uint8, device=f"cuda:{device}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")

    def slice_of(step):
        return step_slice(total_batch, P, step, rank, world) if batch else (0, 1)

    def launch(step):
        lo, _ = slice_of(step)
        src = C.c_void_p(d_all.data_ptr() + lo * PS * 8)
        if batch:
            nat.check(nat.lib.pt_track_batch_device(hom.plan, P, src, C.byref(sp), C.c_void_p(d_end.data_ptr()),
                                                    C.c_void_p(d_stats.data_ptr()), sh))
        else:
            nat.check(nat.lib.pt_track_path_device(hom.plan, src, C.byref(sp), C.c_void_p(d_end.data_ptr()),
                                                   C.c_void_p(d_stats.data_ptr()), sh))

    def barrier():
        torch.cuda.synchronize(device)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(device)

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            launch(s)
    barrier()
    clocks = Clocks(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    prof = np.zeros(8)
    nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
    stats_all = []
    for s, (e0, e1) in enumerate(ev):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0.record(stream)
            launch(s)
            e1.record(stream)
            if batch:  # per-step statistics feed the work count (stream-ordered copy, outside the events)
                stats_all.append((s, d_stats.clone()))
    barrier()
    nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    t_dev = sum(step_ms) / 1e3
    if batch:
        stats_list = []
        for _, t in stats_all:
            raw = t.cpu().numpy()
            stats_list.extend(nat.PathStats.from_buffer_copy(raw[p].tobytes()) for p in range(P))
    else:  # every step tracks the same path: identical statistics per launch
        raw = d_stats.cpu().numpy()
        stats_list = [nat.PathStats.from_buffer_copy(raw[0].tobytes())] * args.steps

    # e2e through the public C-ABI with pinned host buffers (H2D starts, D2H ends + stats per step)
    h_starts = torch.from_numpy(np.ascontiguousarray(w.starts if batch else w.starts[:1])).pin_memory()
    h_end = torch.zeros((P,) + tuple(w.starts.shape[1:]), dtype=torch.float64).pin_memory()
    h_stats = (nat.PathStats * P)()
    dp = lambda t, off=0: C.cast(C.c_void_p(t.data_ptr() + off), nat._dp)
    e2e_steps = max(2, args.steps // 5) if batch else args.steps

    def e2e_call(step):
        lo, _ = slice_of(step)
        if batch:
            nat.check(nat.lib.pt_track_batch(hom.plan, P, dp(h_starts, lo * PS * 8), C.byref(sp), dp(h_end), h_stats))
        else:
            nat.check(nat.lib.pt_track_path(hom.plan, dp(h_starts), C.byref(sp), dp(h_end), h_stats))

    e2e_call(0)
    barrier()
    t0 = time.perf_counter()
    for s in range(e2e_steps):
        e2e_call(s)
    t_e2e = time.perf_counter() - t0
    barrier()

    tt = torch.tensor([t_dev, t_e2e], dtype=torch.float64, device=f"cuda:{device}")
    if world > 1:
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    t_dev_max, t_e2e_max = float(tt[0]), float(tt[1])
    paths_per_step = P * world
    value = paths_per_step * args.steps / t_dev_max
    e2e_value = paths_per_step * e2e_steps / t_e2e_max

    if rank == 0:
        work, we, ws = path_work(hom, stats_list, w.params.pred_degree)
        t_launch = t_dev / args.steps
        peak, peak_src = fp64_peak()
        achieved = work / args.steps / t_launch
        traffic = None
        tr_path = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr_path):
            with open(tr_path) as fh:
                tr = json.load(fh)
            # single paths: bytes per launch; the batch: bytes per path x paths per launch
            traffic = tr.get(w.name)
            if traffic is None and batch and f"{w.name}/path" in tr:
                traffic = tr[f"{w.name}/path"] * P
        ok = [s.status == 0 for s in stats_list]
        line = {
            "metric": metric_of(args, w),
            "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(w),
            "data": "synthetic (pinned generators, SURVEY.md 8(d)); no checkpoints",
            "config": config(args, w, world),
            "sec_per_path": t_dev_max / args.steps / P,
            "paths": {"tracked": len(stats_list), "ok": int(sum(ok)),
                      "mean_steps": float(np.mean([s.steps for s in stats_list])),
                      "mean_newton_iters": float(np.mean([s.newton_iters for s in stats_list])),
                      "engine": "batch" if batch else hom.engine, "ctas": hom.info(6 if batch else 4)},
            "e2e": {"value": e2e_value, "unit": "paths/s",
                    "h2d_bytes_per_step": int(P * PS * 8),
                    "d2h_bytes_per_step": int(P * PS * 8 + C.sizeof(nat.PathStats) * P),
                    "steps": e2e_steps, "timing": "wall clock around the C-ABI call, max over ranks"},
            "roofline": {"bound": "fp64-pipe",
                         "kernel": "k_track_batch" if batch else ("k_track_cluster" if hom.engine == "cluster"
                                                                  else "k_track_grid"),
                         "achieved": achieved * 1e-12, "peak": peak * 1e-12,
                         "unit": "T FP64-instr/s (DADD/DMUL/DFMA of the reference DD/QD algorithms; FMA = 1)",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "work_per_launch_fp64_instr": work / args.steps, "work_per_eval": we, "work_per_solve": ws},
            "gpu_launches": args.steps,
            "clocks": clk,
        }
        if not batch:
            line["path"] = {"success": bool(ok[0]), "steps": stats_list[0].steps,
                            "newton_iters": stats_list[0].newton_iters, "solves": stats_list[0].solves}
            line["phase_ms_per_path"] = {k: prof[i] * 1e-6 / args.steps for i, k in enumerate(
                ["monomials", "slot_sums", "mgs", "backsub_update", "predict"])}
            line["critical_path"] = critical_path(hom, stats_list[0], prof, args.steps)
        if world == 1 and not args.no_cpu_baseline:
            if batch:
                line["cpu_baseline"] = cpu_batch_pool(w, args.cpu_paths)
                one = cpu_single(w, min(args.cpu_seconds, 5.0), 1)
                line["cpu_single_thread"] = one
            else:
                if not args.no_cpu_reference:
                    line["cpu_baseline"] = cpu_single(w, args.cpu_seconds, os.cpu_count() or 1)
                    line["cpu_single_thread"] = cpu_single(w, min(args.cpu_seconds, 5.0), 1)
                dall = cpu_d_all_cores(args)
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
