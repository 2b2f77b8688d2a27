"""Timing of the block-cyclic driver's per-GPU step in the degenerate P=1 layout (one GPU available): per
iteration update || look-ahead panel on two streams, worker sharing by a joining launch, ET through the
step flag -- next to lu_la (the persistent kernel) on the same matrix.
    python tools/dev_dist_time.py n b [variant] [panel_sms]
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.distributed import DistLU
from paper_1611_06365_b200.workloads import LuConfig
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
b = int(sys.argv[2]) if len(sys.argv) > 2 else 512
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["lu", "lu_la", "lu_mb", "lu_et"]
psms = int(sys.argv[4]) if len(sys.argv) > 4 else 32
cfg = LuConfig("t", n, "uniform", 4, b, b // 8)
a0 = mla.alloc_matrix(n, n, device="cuda")
mla.fill_random(a0, cfg.seed, 2.0, -1.0)
a = mla.alloc_matrix(n, n, device="cuda")
def timed(fn):
    ms = []
    for rep in range(3):
        a.copy_(a0); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms[1:]), r
ms, r = timed(lambda: mla.lu_la(a, mla.Policy("lu_et", mla.BlockConfig(b, b // 8), t_pf=psms)))
ref_piv = r.ipiv.ipiv.copy()
print(f"lu_la lu_et (persistent kernel) n={n} b={b}: {ms:.1f} ms  {mla.flops_lu(n, n) / ms / 1e9:.2f} TFLOP/s", flush=True)
for v in variants:
    dlu = DistLU(n, b, b // 8, cfg, "cuda", variant=v, rank=0, world=1, panel_sms=psms, storage=a)
    ms, piv = timed(dlu.factor)
    print(f"DistLU P=1 {v:6s} n={n} b={b}: {ms:.1f} ms  {mla.flops_lu(n, n) / ms / 1e9:.2f} TFLOP/s  panels {len(dlu.widths)} "
          f"et_events {dlu.et_events} host_waits {dlu.host_waits} launches {dlu.launches_per_factor} "
          f"pivots==lu_la {bool(np.array_equal(piv, ref_piv))}", flush=True)
