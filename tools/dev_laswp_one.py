import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
n, npiv, cols = 16384, 256, 16384
A = mla.alloc_matrix(n, n); mla.fill_random(A, 1, 2.0, -1.0)
rng = np.random.default_rng(0)
ipiv = np.array([rng.integers(t, n) for t in range(npiv)], dtype=np.int64)
for _ in range(3):
    mla.laswp(A[:, :cols], ipiv)
torch.cuda.synchronize()
print("ok")
