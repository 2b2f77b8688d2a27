"""Regression check for the round-1 corruption of the two-stream driver (panel kernel co-resident with the
update kernel; root cause: a shared-memory race in the tile epilogue, fixed in round 2): P=1 DistLU in every
variant on a device-generated uniform matrix; pivots compared with lu_la's, backward error from the device
residual.
    python tools/dev_overlap_repro.py n b [reps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.distributed import DistLU
from paper_1611_06365_b200.workloads import LuConfig
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = LuConfig("t", n, "uniform", 4, b, b // 8)
eps = np.finfo(np.float64).eps
# reference pivots from the persistent kernel (parity-tested against the oracle)
a0 = mla.alloc_matrix(n, n, device="cuda")
mla.fill_random(a0, cfg.seed, 2.0, -1.0)
ref_piv = None
if n <= 40000:
    a = mla.alloc_matrix(n, n, device="cuda"); a.copy_(a0)
    r = mla.lu_la(a, mla.Policy("lu_mb", mla.BlockConfig(b, b // 8)))
    ref_piv = r.ipiv.ipiv.copy()
    del a
bad = 0
for overlap in ("lu", "lu_la", "lu_mb", "lu_et"):
    dlu = DistLU(n, b, b // 8, cfg, "cuda", rank=0, world=1, variant=overlap)
    for rep in range(reps):
        dlu.a.copy_(a0); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); piv = dlu.factor(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        chk = mla.alloc_matrix(n, n, device="cuda"); chk.copy_(a0)
        berr = mla.residual_packed(chk, dlu.a, mla.PivotVector(piv)) / (n * eps)
        del chk
        same = None if ref_piv is None else bool(np.array_equal(piv, ref_piv))
        ok = berr <= 10 and same is not False
        bad += (not ok)
        print(f"variant={overlap} et_events={dlu.et_events} n={n} b={b} rep={rep}: {ms:.1f} ms  backward err {berr:.4g} n eps  pivots==lu_la {same}  {'OK' if ok else 'CORRUPT'}", flush=True)
    del dlu
sys.exit(1 if bad else 0)
