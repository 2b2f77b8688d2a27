"""Headline factorization time for small fixed panel teams that may grow when the panel becomes the critical
path (SmPool.t_pf_max): does a smaller team in the update-bound iterations return SM-time to the update?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b_o, b_i = 512, 64
pool = mla.default_pool()
a0 = mla.alloc_matrix(n, n)
mla.fill_random(a0, 3, 2.0, -1.0)
for t_pf, t_max in [(32, 0), (16, 32), (24, 32), (16, 48), (20, 40), (12, 48), (32, 64)]:
    pool.t_pf_max = t_max
    ts = []
    for i in range(3):
        a = a0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = mla.lu_la(a, mla.Policy("lu_et", mla.BlockConfig(b_o, b_i), t_pf=t_pf), pool)
        e1.record(); torch.cuda.synchronize()
        if i: ts.append(e0.elapsed_time(e1))
        del a
    ms = float(np.mean(ts))
    print(f"n={n} t_pf={t_pf} t_pf_max={t_max}: {ms:.1f} ms {2*n**3/3/ms*1e-9:.2f} TFLOP/s panels {len(r.widths)} et {r.et_events} peak team {r.t_pf_peak}", flush=True)
pool.t_pf_max = 0
