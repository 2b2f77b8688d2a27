"""Deterministic factorizations whose packed factors + pivots are written to a file; run once with the normal
library and once with the -DMLA_RACE_STRESS build (MLA_B200_LIB), then compared bit for bit (tools/race_stress.sh).
    python tools/dev_race_stress.py out.npz"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.kernels import apply_panel
out = {}
for n, b_o, b_i, t_pf in [(3072, 256, 32, 12), (2048, 512, 64, 32), (1500, 128, 16, 5)]:
    a = mla.alloc_matrix(n, n); mla.fill_random(a, 21, 2.0, -1.0)
    r = mla.lu_la(a, mla.Policy("lu_mb", mla.BlockConfig(b_o, b_i), t_pf=t_pf))
    out[f"lu_{n}"] = mla.to_numpy(a); out[f"piv_{n}"] = r.ipiv.ipiv
c = mla.alloc_matrix(1280, 1024); x = mla.alloc_matrix(1280, 512); y = mla.alloc_matrix(512, 1024)
for t in (c, x, y): mla.fill_random(t, 1)
mla.gemm_malleable(c, x, y, 1.0, -1.0); out["gemm"] = mla.to_numpy(c)
p = mla.alloc_matrix(1800, 256); t = mla.alloc_matrix(1800, 700)
mla.fill_random(p, 4, 2.0, -1.0); mla.fill_random(t, 5)
apply_panel(p, 256, t, np.arange(256, dtype=np.int64) + 5); out["apply"] = mla.to_numpy(t)
q = mla.alloc_matrix(4000, 128); mla.fill_random(q, 9, 2.0, -1.0)
r = mla.lu_blk_ll(q, 32, team_sms=6); out["panel"] = mla.to_numpy(q); out["panel_piv"] = r.ipiv.ipiv
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1], {k: v.shape for k, v in out.items()})
