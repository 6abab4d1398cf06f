"""Track a prefix of one path (for profilers):
python tools/one_prefix.py <workload> <prec> <max_steps> [engine]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import workloads as W  # noqa: E402

w = W.by_name(sys.argv[1], pt.PrecisionMode.parse(sys.argv[2]))
w.params.max_steps = int(sys.argv[3])
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
if len(sys.argv) > 4:
    hom.set_engine(sys.argv[4])
out = hom.track_path(w.start, w.params)
print(w.name, hom.engine, out.success, out.steps, out.newton_iters)
