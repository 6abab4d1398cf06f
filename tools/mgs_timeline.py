"""Per-column MGS timeline of the last tracked path (pt_plan_mgs_timeline)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import _native as nat, workloads as W  # noqa: E402

name, prec, engine = sys.argv[1], sys.argv[2], sys.argv[3]
w = W.by_name(name, pt.PrecisionMode.parse(prec))
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
hom.set_engine(engine)
for _ in range(2):
    hom.track_path(w.start, w.params)
n = w.n
buf = np.zeros(6 * (n + 1))
nat.check(nat.lib.pt_plan_mgs_timeline(hom.plan, nat.dptr(buf), buf.size))
t = buf.reshape(n + 1, 6)
cols = range(2, n)
med = lambda v: float(np.median(v))
out = {"workload": w.name, "engine": engine, "per_column_median": {
    "wait_ns (gtimer: publish j-1 -> seen)": med([t[j, 0] - t[j - 1, 5] for j in cols]),
    "q_load_cycles": med([t[j, 2] - t[j, 1] for j in cols]),
    "project_cycles": med([t[j, 3] - t[j, 2] for j in cols]),
    "normalize_publish_cycles": med([t[j, 4] - t[j, 3] for j in cols])},
    "total_ns": float(t[n - 1, 5] - t[1, 0])}
print(json.dumps(out))
