"""Phase timers of batch CTA 0 (k_track_batch): python tools/prof_batch.py [prec] [paths] [max_steps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import _native as nat, workloads as W  # noqa: E402

prec = pt.PrecisionMode.parse(sys.argv[1] if len(sys.argv) > 1 else "dd")
npaths = int(sys.argv[2]) if len(sys.argv) > 2 else 296
w = W.batch(prec=prec)
if len(sys.argv) > 3:
    w.params.max_steps = int(sys.argv[3])
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
starts = np.ascontiguousarray(w.starts[:npaths])
hom.track_batch(starts[:8], w.params)  # allocate the batch workspace
prof = np.zeros(8)
nat.check(nat.lib.pt_plan_batch_profile(hom.plan, 0, nat.dptr(prof), 1))
t0 = time.perf_counter()
_, outs = hom.track_batch(starts, w.params)
dt = time.perf_counter() - t0
nat.check(nat.lib.pt_plan_batch_profile(hom.plan, 0, nat.dptr(prof), 1))
names = ["monomials", "slot_sums", "mgs", "backsub", "predict"]
it = max(1.0, prof[5])
print(json.dumps({"paths": npaths, "batch_ctas": int(hom.info(6)), "wall_s": round(dt, 3),
                  "cta0_newton_iters": prof[5],
                  "cta0_us_per_iter": {k: round(prof[i] * 1e-3 / it, 2) for i, k in enumerate(names)},
                  "ok": int(sum(o.success for o in outs))}))
