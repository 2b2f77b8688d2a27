import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
pool = mla.default_pool()
L = _capi.lib()
def timed(m, w, b, team, reps=3):
    a0 = mla.from_numpy(mla.make_matrix("uniform", w, 5, m))
    piv = torch.empty(w, dtype=torch.int32, device="cuda")
    info = _capi.LuInfo()
    best = 1e9
    for _ in range(reps):
        a = a0.clone().t().contiguous().t() if False else mla.alloc_matrix(m, w); a.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.mla_panel_ll(pool.handle, a.data_ptr(), m, w, a.stride(1), piv.data_ptr(), b, 0, 0, team, ctypes.byref(info), torch.cuda.current_stream().cuda_stream)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    prof = (ctypes.c_uint64 * 16)()
    L.mla_panel_profile(pool.handle, prof, 1)
    pr = [x / 1e3 / reps for x in prof[:6]]
    print(f"panel m={m} w={w} b={b} team={team}: {best*1e3:.0f} us  ({best*1e3/w:.2f} us/col)  trsm {pr[0]:.0f} gemm {pr[1]:.0f} steps {pr[2]:.0f} (xchg {pr[5]:.0f}) wb+swap {pr[3]:.0f} bar {pr[4]:.0f}", flush=True)
for m, w, b, team in [(2048, 32, 32, 1), (2048, 32, 32, 4), (2048, 32, 32, 16), (2048, 32, 32, 64), (8192, 32, 32, 16), (8192, 32, 32, 64),
                      (2048, 256, 32, 16), (2048, 256, 32, 64), (8192, 256, 32, 16), (8192, 256, 32, 32), (8192, 256, 32, 64), (32768, 256, 32, 64), (32768, 256, 32, 148), (16384, 512, 64, 64)]:
    timed(m, w, b, team)
