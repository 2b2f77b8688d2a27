"""Does a power-of-two leading dimension cost anything?  lu_la and laswp on the same matrix stored with
ld = n, n + 16, n + 64, n + 528 (column stride no longer a multiple of 256 KiB).  usage: dev_ld_pad.py [n]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b_o, b_i = 512, 64
pool = mla.default_pool()
L = _capi.lib()
for pad in (0, 16, 64, 528, 2064):
    a0 = mla.alloc_matrix(n, n, ld=n + pad)
    mla.fill_random(a0, 3, 2.0, -1.0)
    work = mla.alloc_matrix(n, n, ld=n + pad)
    ts = []
    for i in range(3):
        work.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = mla.lu_la(work, mla.Policy("lu_et", mla.BlockConfig(b_o, b_i)), pool)
        e1.record(); torch.cuda.synchronize()
        if i: ts.append(e0.elapsed_time(e1))
    ms = float(np.mean(ts))
    # laswp: 512 pivots over all columns
    piv = torch.randint(0, n, (512,), dtype=torch.int32, device="cuda")
    piv = torch.maximum(piv, torch.arange(512, dtype=torch.int32, device="cuda"))
    s = torch.cuda.current_stream().cuda_stream
    def lw():
        rc = L.mla_laswp_async(pool.handle, work.data_ptr(), n, n, work.stride(1), piv.data_ptr(), 512, 0, s)
        assert rc == 0
    lw(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): lw()
    e1.record(); torch.cuda.synchronize()
    lms = e0.elapsed_time(e1) / 5
    print(f"n={n} ld=n+{pad}: lu_et {ms:.1f} ms {2*n**3/3/ms*1e-9:.2f} TFLOP/s (panels {len(r.widths)}); laswp 512 pivots x {n} cols {lms*1e3:.0f} us", flush=True)
    del a0, work
