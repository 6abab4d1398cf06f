"""Write chandra64 DD's [J | -h] at the start point (t = 0.5) as SoA planes for tools/mgs_bench.cu."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06625_b200 as pt
from paper_1501_06625_b200 import workloads as W
w = W.chandra(64, pt.PrecisionMode.DD)
hom = pt.make_homotopy(w.g, w.f, w.gamma, w.k)
x = np.array(w.start, copy=True)
h, J, r = hom.evaluate(x, 0.5)
N, n, L = w.N, w.n, 2
SA = N * (n + 1)
A = np.zeros((2 * L, SA))
J = J.reshape(2 * L, N * n)
h = h.reshape(2 * L, N)
A[:, :N * n] = J
A[:, N * n:] = -h
A.astype(np.float64).tofile(sys.argv[1])
print("wrote", sys.argv[1], A.shape, "max|h|", r)
