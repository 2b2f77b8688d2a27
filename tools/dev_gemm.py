import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_06365_b200 import _capi
L = _capi.lib()
h = ctypes.c_void_p()
assert L.mla_create(0, ctypes.byref(h)) == 0
def cm(m, n, ld=None):
    ld = ld or m
    return torch.randn(n, ld, dtype=torch.float64, device="cuda").t()[:m]
def run(m, n, k, alpha=1.0, beta=-1.0, lda=None, check=True, reps=0):
    A = cm(m, k, lda); B = cm(k, n); C = cm(m, n)
    ref = alpha * C + beta * (A @ B) if check else None
    s = torch.cuda.current_stream().cuda_stream
    rc = L.mla_gemm(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, alpha, beta, None, 0, s)
    torch.cuda.synchronize()
    assert rc == 0, rc
    if check:
        err = (C - ref).abs().max().item()
        print(f"gemm {m}x{n}x{k} a={alpha} b={beta} maxerr {err:.3e}")
        assert err < 1e-10 * max(1, k)
    if reps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            L.mla_gemm(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, alpha, beta, None, 0, s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"   {ms:.3f} ms  {2.0*m*n*k/ms*1e-9:.2f} TFLOP/s")
run(128, 128, 16)
run(256, 384, 64)
run(517, 333, 129, 0.5, 2.0)
run(130, 70, 300, lda=131)
run(1000, 1000, 256)
for m, k in [(4096, 256), (8192, 256), (16384, 256), (16384, 512), (32768, 256), (32768, 512), (32768, 128)]:
    run(m, m, k, check=False, reps=3)
