"""Stand-alone mla_gemm at the shapes of the phased entry point's catch-up updates: C (m x n) -= A (m x k) B (k x n)
for k from one panel (512) to a whole phase (12288).  TFLOP/s per k."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_06365_b200 import _capi
L = _capi.lib()
h = ctypes.c_void_p()
assert L.mla_create(0, ctypes.byref(h)) == 0
def cm(m, n):
    return (torch.rand(n, m, dtype=torch.float64, device="cuda") - 0.5).t()
def run(m, n, k, reps=3, check=False):
    A = cm(m, k); B = cm(k, n); C = cm(m, n)
    s = torch.cuda.current_stream().cuda_stream
    def go():
        rc = L.mla_gemm(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, 1.0, -1.0, None, 0, s)
        assert rc == 0, rc
    if check:
        ref = C - A @ B
        go(); torch.cuda.synchronize()
        err = (C - ref).abs().max().item()
        print(f"gemm {m}x{n}x{k} maxerr {err:.3e}")
        assert err < 1e-10 * k
        return
    go(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): go()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"gemm {m}x{n}x{k}: {ms:.3f} ms  {2.0*m*n*k/ms*1e-9:.2f} TFLOP/s", flush=True)
run(1024, 1152, 2048, check=True)
run(2048, 640, 5000, check=True)
for m in (20480, 12288):
    for k in (512, 1024, 2048, 4096, 8192, 12288):
        run(m, m, k)
