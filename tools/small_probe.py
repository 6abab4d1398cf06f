"""Phase timers of ONE path of a small system on the batch engine (one CTA,
k_track_batch) next to the single-path engine's wall time:
    python tools/small_probe.py [workload] [prec] [reps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import _native as nat, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cyclic16"
prec = pt.PrecisionMode.parse(sys.argv[2] if len(sys.argv) > 2 else "dd")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = W.by_name(name, prec)
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
start = np.ascontiguousarray(w.start)
names = ["monomials", "slot_sums", "mgs", "backsub", "predict"]
out = {"workload": name, "prec": prec.name.lower()}
for n in (1, 8):
    starts = np.ascontiguousarray(np.stack([start] * n))
    hom.track_batch(starts, w.params)  # workspace + first launch
    prof = np.zeros(8)
    best = 1e9
    for _ in range(reps):
        nat.check(nat.lib.pt_plan_batch_profile(hom.plan, 0, nat.dptr(prof), 1))
        t0 = time.perf_counter()
        _, outs = hom.track_batch(starts, w.params)
        best = min(best, time.perf_counter() - t0)
    nat.check(nat.lib.pt_plan_batch_profile(hom.plan, 0, nat.dptr(prof), 1))
    it = max(1.0, prof[5])
    out[f"batch_{n}"] = {"ms_per_launch": round(best * 1e3, 3), "cta0_newton_iters": prof[5],
                         "cta0_us_per_iter": {k: round(prof[i] * 1e-3 / it, 2) for i, k in enumerate(names)},
                         "ok": int(sum(o.success for o in outs))}
hom.track_path(start, w.params)
best = 1e9
for _ in range(reps):
    t0 = time.perf_counter()
    o = hom.track_path(start, w.params)
    best = min(best, time.perf_counter() - t0)
out["single_path_ms"] = round(best * 1e3, 3)
out["single_path_iters"] = o.newton_iters
print(json.dumps(out))
