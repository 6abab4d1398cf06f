import sys, numpy as np
sys.path.insert(0, '.')
from paper_1501_06625_b200 import PrecisionMode as PM, monodromy as MD, workloads as W
from paper_1501_06625_b200.tracker import augment_with_linear, limbs_from_complex, complex_from_limbs
fL = augment_with_linear(16, 3, 1, PM.DD)
w0 = limbs_from_complex(W.backelin_witness(fL, 4, 3), PM.DD)
ws = MD.monodromy_degree(16, 3, [w0], seed=3, stabilization_loops=4, prec=PM.DD)
print("degree", ws.degree, "loops", ws.loops, "failed", ws.failed_paths)
Z = [complex_from_limbs(p) for p in ws.points]
for i, z in enumerate(Z):
    # Backelin structure: x_{a m + b} / x_b should be omega^a
    m = 4
    ratios = [z[a*m+1]/z[1] for a in range(m)]
    prod = np.prod(z)
    print(i, np.round(z[:4], 5), "ratios", np.round(ratios, 4), "prod", np.round(prod, 6))
