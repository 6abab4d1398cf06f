import sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import structured as S
import paper_1501_06625_b200 as pt
from oracle.orc import Oracle
ci, engine = int(sys.argv[1]), sys.argv[2]
n, prec, seed = S.CASES[ci]
f, g, gamma, params, starts = S.case(n, prec, seed, S.max_steps(prec))
hom = pt.make_homotopy(g, f, gamma, 2, device=0)
o = Oracle("restatement")
try:
    if engine == "batch":
        ends, outs = hom.track_batch(starts, params)
        bad = 0
        for p in range(starts.shape[0]):
            e, st, _ = o.track_path(int(prec), g, f, gamma, 2, starts[p], params)
            bad += int(not np.array_equal(ends[p].view(np.uint64), e.view(np.uint64)) or outs[p].steps != st.steps)
        print(ci, n, prec.name, engine, "mismatches", bad)
    else:
        hom.set_engine(engine)
        for p in range(2):
            e, st, tr = o.track_path(int(prec), g, f, gamma, 2, starts[p], params, params.max_steps + 2)
            out = hom.track_path(starts[p], params, trace=True)
            same = np.array_equal(out.end.view(np.uint64), e.view(np.uint64)) and out.steps == st.steps
            print(ci, n, prec.name, engine, p, "same" if same else "DIFF", out.steps, st.steps)
except Exception as ex:
    print(ci, n, prec.name, engine, "ERROR", str(ex)[:200])
