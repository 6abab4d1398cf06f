"""One evaluation + differentiation pass (k_eval) of a BASELINE system, for
profilers: python tools/eval_once.py <workload> <prec> [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import workloads as W  # noqa: E402

w = W.by_name(sys.argv[1], pt.PrecisionMode.parse(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
ms = pt.eval_bench(hom, w.start, 0.37, reps)
print(w.name, "ms per evaluation", round(ms, 4), "grid CTAs", hom.info(4))
