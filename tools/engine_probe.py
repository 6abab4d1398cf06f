"""Single path on the cluster / grid engines vs one CTA (the batch kernel with
one path): device ms per tracked path.  python tools/engine_probe.py <workload> <prec> [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import workloads as W  # noqa: E402

w = W.by_name(sys.argv[1], pt.PrecisionMode.parse(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
res = {}
for eng in ("cluster", "grid"):
    try:
        hom.set_engine(eng)
    except Exception:
        continue
    hom.track_path(w.start, w.params)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = hom.track_path(w.start, w.params)
    res[eng] = (time.perf_counter() - t0) / reps * 1e3
ends, outs = hom.track_batch(w.starts[:1], w.params)
t0 = time.perf_counter()
for _ in range(reps):
    ends, outs = hom.track_batch(w.starts[:1], w.params)
res["one_cta"] = (time.perf_counter() - t0) / reps * 1e3
same = np.array_equal(ends[0].view(np.uint64), out.end.view(np.uint64))
print(w.name, {k: round(v, 2) for k, v in res.items()}, "steps", out.steps, "newton", out.newton_iters, "bitwise_same", same)
