"""Library reference (measurement only, never on the product path): cuSOLVER's FP64 getrf through
torch.linalg.lu_factor on the same matrices as the configs, next to lu_la.
    python tools/cusolver_getrf_ref.py [n ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
ns = [int(x) for x in sys.argv[1:]] or [2048, 8192, 16384, 32768]
for n in ns:
    a0 = mla.alloc_matrix(n, n); mla.fill_random(a0, 3, 2.0, -1.0)
    best = 1e9
    for rep in range(3):
        x = a0.clone()           # column-major (stride (1, n)): what cuSOLVER wants
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); lu, piv = torch.linalg.lu_factor(x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
        del lu, x
    b_o = 512 if n >= 16384 else 256
    ours = 1e9
    for rep in range(3):
        x = a0.clone(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = mla.lu_la(x, mla.Policy("lu_et", mla.BlockConfig(b_o, b_o // 8))); e1.record(); torch.cuda.synchronize()
        ours = min(ours, e0.elapsed_time(e1))
    same = bool(np.array_equal(piv.cpu().numpy().astype(np.int64) - 1, r.ipiv.ipiv))
    f = mla.flops_lu(n, n)
    print(f"n={n}: cuSOLVER getrf (torch.linalg.lu_factor) {best:.1f} ms = {f / best / 1e9:.2f} TFLOP/s;  lu_la lu_et b={b_o} "
          f"{ours:.1f} ms = {f / ours / 1e9:.2f} TFLOP/s;  pivots identical: {same}", flush=True)
