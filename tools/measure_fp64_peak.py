"""Measure the B200 FP64-pipe peak (thread-level DFMA/s) and write
profiles/fp64_peak.json -- the roofline denominator bench.py uses
(MEASURED_PEAKS.json has no FP64 figure)."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1501_06625_b200 import _native as nat  # noqa: E402

best = 0.0
for _ in range(5):
    v, ms = C.c_double(), C.c_double()
    nat.check(nat.lib.pt_fp64_peak(0, C.byref(v), C.byref(ms)))
    best = max(best, v.value)
clk = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
out = {"instr_per_s": best, "tflops_equiv_fma2": 2 * best * 1e-12,
       "how": "k_fp64_peak: 148*4 CTAs x 256 threads x 4096 iters x 8 independent __fma_rn chains; best of 5x5 "
              "CUDA-event timings; thread-level DFMA instructions per second (FMA counted once)",
       "nvidia_smi_after": clk}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
dst = os.path.join(ROOT, "gpurun_out", "fp64_peak.json") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else \
    os.path.join(ROOT, "profiles", "fp64_peak.json")
with open(dst, "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
