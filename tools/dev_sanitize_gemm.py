"""Smallest racecheck target: the update's tile engine alone (k_gemm; chained tiles + bulk-reduction epilogue,
the code in which round 2 found the shared-memory race), a fused update step (k_apply_panel) and the 128-row
triangular solve.
   compute-sanitizer --tool racecheck python tools/dev_sanitize_gemm.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.kernels import apply_panel
c = mla.alloc_matrix(640, 512); x = mla.alloc_matrix(640, 256); y = mla.alloc_matrix(256, 512)
for t in (c, x, y): mla.fill_random(t, 1)
mla.gemm_malleable(c, x, y, 1.0, -1.0); torch.cuda.synchronize(); print("gemm ok", flush=True)
l = mla.alloc_matrix(256, 256); b = mla.alloc_matrix(256, 300)
mla.fill_random(l, 2); mla.fill_random(b, 3)
mla.trsm_llu(l, b); torch.cuda.synchronize(); print("trsm ok", flush=True)
rows, w, cols = 700, 256, 300
p = mla.alloc_matrix(rows, w); t = mla.alloc_matrix(rows, cols)
mla.fill_random(p, 4, 2.0, -1.0); mla.fill_random(t, 5)
piv = np.arange(w, dtype=np.int64) + 3
apply_panel(p, w, t, piv); torch.cuda.synchronize(); print("apply_panel ok", flush=True)
