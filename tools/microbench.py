"""Latency microbenchmarks on the B200 (pt_microbench): FP64 / DD / QD op
latency, grid barrier and cross-SM flag latency.  Output: JSON line."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_06625_b200 import _native as nat  # noqa: E402

out = {}
b = np.zeros(16)
nat.check(nat.lib.pt_microbench(0, 0, nat.dptr(b)))
out["cycles_per_op"] = dict(zip(["dadd", "dd_add", "dd_mul", "qd_add", "qd_mul", "cplx_dd_mul", "hypot"],
                                b[:7].round(1).tolist()))
nat.check(nat.lib.pt_microbench(0, 1, nat.dptr(b)))
out["grid_barrier_ns"] = float(b[0])
nat.check(nat.lib.pt_microbench(0, 2, nat.dptr(b)))
out["flag_one_way_ns"] = float(b[0])
nat.check(nat.lib.pt_microbench(0, 3, nat.dptr(b)))
out["mgs_pieces_cycles"] = dict(zip(["tree_cplx_dd", "project_dd_N64", "conj_mul_dd", "sqrt_dd", "div_dd"],
                                    b[:5].tolist()))
print(json.dumps(out))
