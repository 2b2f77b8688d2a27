"""Small factorizations meant for compute-sanitizer (memcheck / racecheck / synccheck):
   compute-sanitizer --tool racecheck python tools/dev_sanitize.py
(the tool is closed on the round-1 GPU pool, so tests/test_gpu_lu.py::test_repeated_runs_are_bitwise_identical
stands in for racecheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
pool = mla.default_pool()
for n, bo, bi, v, tpf in [(768, 128, 32, "lu_et", 8), (1200, 256, 64, "lu_mb", 4), (640, 64, 16, "lu", None)]:
    a = mla.alloc_matrix(n, n); mla.fill_random(a, 7, 2.0, -1.0)
    a0 = a.clone()
    r = mla.lu_la(a, mla.Policy(v, mla.BlockConfig(bo, bi), t_pf=tpf), pool)
    res = mla.residual_packed(a0, a, r.ipiv) if hasattr(mla, "residual_packed") else float("nan")
    print(n, v, "panels", len(r.widths), "residual", float(res))
p = mla.alloc_matrix(3000, 96); mla.fill_random(p, 3, 2.0, -1.0)
print("panel", mla.lu_blk_ll(p, 32, team_sms=3).cols_factored)
c = mla.alloc_matrix(512, 384); x = mla.alloc_matrix(512, 256); y = mla.alloc_matrix(256, 384)
for t in (c, x, y): mla.fill_random(t, 1)
mla.gemm_malleable(c, x, y, 1.0, -1.0); torch.cuda.synchronize(); print("gemm ok")
