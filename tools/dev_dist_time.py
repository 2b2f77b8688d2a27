"""Timing of the block-cyclic driver's per-GPU work in the degenerate P=1 layout (one GPU available):
panel (lu_blk_ll kernel) + fused apply-panel launch per iteration, no broadcast."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.distributed import DistLU
from paper_1611_06365_b200.workloads import LuConfig
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
b = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = LuConfig("t", n, "uniform", 4, b, b // 8)
dlu = DistLU(n, b, b // 8, cfg, "cuda", rank=0, world=1, panel_sms=int(sys.argv[3]) if len(sys.argv) > 3 else 32,
             overlap_panel=len(sys.argv) > 4 and sys.argv[4] == "overlap")   # overlap: experimental, races
dlu.generate()
for rep in range(2):
    dlu.restore(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dlu.factor(); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"DistLU P=1 n={n} b={b}: {ms:.1f} ms  {mla.flops_lu(n, n) / ms / 1e9:.2f} TFLOP/s  launches {dlu.launches_per_factor}")
