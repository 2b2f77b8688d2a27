import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
L = _capi.lib(); pool = mla.default_pool(); h = pool.handle
def cm(m, n): return torch.randn(n, m, dtype=torch.float64, device="cuda").t()
dbg = (ctypes.c_uint64 * 8)()
for m, k in [(2048, 512), (16384, 512), (32768, 512), (16384, 256)]:
    A = cm(m, k); B = cm(k, m); C = cm(m, m); s = torch.cuda.current_stream().cuda_stream
    L.mla_gemm(h, C.data_ptr(), m, m, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, 1.0, -1.0, None, 0, s)
    torch.cuda.synchronize(); L.mla_getrf_debug(h, dbg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): L.mla_gemm(h, C.data_ptr(), m, m, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, 1.0, -1.0, None, 0, s)
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 3
    L.mla_getrf_debug(h, dbg)
    t = max(1, dbg[0])
    ideal = 128 * 128 * k * 2 / 512 * 16 / 4 / 2   # clk: DMMAs per SMSP * 16
    print(f"m={m} k={k}: {2.0*m*m*k/ms*1e-9:.2f} TF; CTA0: {t} tiles, {dbg[1]/t:.0f} clk/tile, wait+sync {dbg[2]/t:.0f}, epilogue {dbg[3]/t:.0f} (stage half0 {dbg[4]/t:.0f}, issue+wait_read {dbg[5]/t:.0f}; start wait + issue of half 1 {dbg[6]/t:.0f}, fence of half 1 {dbg[7]/t:.0f})")
