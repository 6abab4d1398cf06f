"""Device phase timers of one tracked path: python tools/prof_path.py <workload> <prec>"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import _native as nat, workloads as W  # noqa: E402

w = W.by_name(sys.argv[1], pt.PrecisionMode.parse(sys.argv[2]))
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
hom.track_path(w.start, w.params)
prof = np.zeros(8)
nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
out = hom.track_path(w.start, w.params)
nat.check(nat.lib.pt_plan_profile(hom.plan, nat.dptr(prof), 1))
names = ["monomials_ns", "slot_sums_ns", "mgs_ns", "backsub_ns", "predict_ns", "newton_iters", "bs_chain_cycles", "bs_chain_steps"]
d = dict(zip(names, prof.tolist()))
d["bs_cycles_per_step"] = d["bs_chain_cycles"] / max(1, d["bs_chain_steps"])
d["backsub_ns_per_solve"] = d["backsub_ns"] / max(1, out.solves)
print(json.dumps({"workload": w.name, **{k: round(v, 1) for k, v in d.items()}}))
