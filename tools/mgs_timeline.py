"""Per-column MGS timeline of the last tracked path (pt_plan_mgs_timeline):
python tools/mgs_timeline.py <workload> <prec> [engine] [arith]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import _native as nat, workloads as W  # noqa: E402

name, prec = sys.argv[1], sys.argv[2]
w = W.by_name(name, pt.PrecisionMode.parse(prec))
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
if len(sys.argv) > 3:
    hom.set_engine(sys.argv[3])
if len(sys.argv) > 4:
    hom.set_arith(sys.argv[4])
for _ in range(2):
    hom.track_path(w.start, w.params)
n = w.n
buf = np.zeros(6 * (n + 1))
nat.check(nat.lib.pt_plan_mgs_timeline(hom.plan, nat.dptr(buf), buf.size))
t = buf.reshape(n + 1, 6)
cols = range(2, n)
med = lambda v: float(np.median(v))
out = {"workload": w.name, "engine": hom.engine, "per_column_median": {
    "handoff_ns (q_{j-1} pushed -> q loaded by owner j, globaltimer)": med([t[j, 0] - t[j - 1, 5] for j in cols]),
    "wait_and_load_cycles": med([t[j, 2] - t[j, 1] for j in cols]),
    "project_cycles": med([t[j, 3] - t[j, 2] for j in cols]),
    "normalize_cycles": med([t[j, 4] - t[j, 3] for j in cols]),
    "column_ns (q_{j-1} pushed -> q_j pushed)": med([t[j, 5] - t[j - 1, 5] for j in cols])},
    "total_ns": float(t[n - 1, 5] - t[1, 0])}
print(json.dumps(out))
if os.environ.get("MGS_FINE"):  # library built with -DPT_MGS_FINE
    f = np.zeros(14 * (n + 2))
    # pt_plan_mgs_timeline returns prof[kProfSlots:...]; fine markers follow the 6 (n+2) timeline words
    big = np.zeros(6 * (n + 2) + 8 * (n + 2))
    nat.check(nat.lib.pt_plan_mgs_timeline(hom.plan, nat.dptr(big), big.size))
    fm = big[6 * (n + 2):].reshape(n + 2, 8)
    names = ["load_col", "conj_mul", "tree", "bcast", "axpy"]
    print(json.dumps({"fine_cycles_median": {names[q]: float(np.median([fm[j, q + 1] - fm[j, q] for j in cols])) for q in range(5)}}))
if os.environ.get("MGS_DUMP"):
    print(" ".join(f"{j}:{int(t[j, 3] - t[j, 2])}/{int(t[j, 4] - t[j, 3])}" for j in cols))
