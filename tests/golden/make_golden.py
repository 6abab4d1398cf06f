"""Generate the golden fixtures from the UNMODIFIED reference headers.

Run here (where /root/reference exists) after `make ref`:
    python tests/golden/make_golden.py
Outputs (committed, small):
  arith_{d,dd,qd}.npz   inputs and reference outputs per scalar op
  track_*.npz           oracle/_ref tracker runs (end point, stats, trace)
The generating oracle is oracle/_ref/liborc_ref.so, i.e. the SPEC tracker
compiled on /root/reference/proj/include/pathtrack/{multiprec,complex}.hpp.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from arith_inputs import OPS, random_operands  # noqa: E402
from oracle.orc import Oracle  # noqa: E402

import paper_1501_06625_b200 as pt  # noqa: E402
from paper_1501_06625_b200 import workloads as W  # noqa: E402

ALL_OPS = ["add", "sub", "mul", "mul_d", "div", "sqrt", "renorm", "cmul", "cadd", "conj_mul", "norm_sqr",
           "modulus_double", "powi", "cscale", "cpowi"]

TRACKS = [("cyclic16", pt.PrecisionMode.DD), ("cyclic16", pt.PrecisionMode.D), ("chandra64", pt.PrecisionMode.D),
          ("chandra64", pt.PrecisionMode.DD), ("cyclic16", pt.PrecisionMode.QD), ("chandra64", pt.PrecisionMode.QD)]


def main(tracks_only=False):
    """tracks_only (argv "--tracks"): regenerate the track fixtures only."""
    ref = Oracle("reference")
    assert ref.variant == "reference"
    for prec, tag in enumerate(("d", "dd", "qd")):
        if tracks_only:
            break
        blob = {}
        for op in ALL_OPS:
            a = random_operands(prec, 256, 101, positive=(op == "sqrt"), oracle=ref)
            b = random_operands(prec, 256, 102, small_int=op in ("powi", "cpowi"), oracle=ref)
            blob[f"{op}_a"] = a
            blob[f"{op}_b"] = b
            blob[f"{op}_out"] = ref.arith(prec, OPS[op], a, b)
        np.savez_compressed(os.path.join(HERE, f"arith_{tag}.npz"), **blob)
    for name, prec in TRACKS:
        w = W.by_name(name, prec)
        cap = w.params.max_steps + 2
        end, st, tr = ref.track_path(int(prec), w.g, w.f, w.gamma, w.k, w.start, w.params, cap)
        stats = np.array([st.status, st.failure_kind, st.steps, st.accepted, st.newton_iters, st.start_iters])
        fstats = np.array([st.final_residual, st.final_update, st.t_end])
        trace = np.array([[e.t, e.ok, e.iters, e.residual, e.update] for e in tr])
        np.savez_compressed(os.path.join(HERE, f"track_{name}_{prec.name.lower()}.npz"), end=end, stats=stats,
                            fstats=fstats, trace=trace)
        print(name, prec.name, "steps", st.steps, "status", st.status)


if __name__ == "__main__":
    main(tracks_only="--tracks" in sys.argv)
