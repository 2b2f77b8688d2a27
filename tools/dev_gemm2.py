import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_06365_b200 import _capi
L = _capi.lib()
h = ctypes.c_void_p()
assert L.mla_create(0, ctypes.byref(h)) == 0
def cm(m, n):
    return torch.randn(n, m, dtype=torch.float64, device="cuda").t()
def run(m, n, k, reps=3):
    A = cm(m, k); B = cm(k, n); C = cm(m, n)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: L.mla_gemm(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, 1.0, -1.0, None, 0, s)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"gemm {m}x{n}x{k}: {ms:.3f} ms  {2.0*m*n*k/ms*1e-9:.2f} TFLOP/s", flush=True)
sizes = [(8192, 8192, 256), (8192, 8192, 4096)] if len(sys.argv) < 2 else [tuple(int(x) for x in sys.argv[1:4])]
for m, n, k in sizes:
    run(m, n, k, reps=int(sys.argv[4]) if len(sys.argv) > 4 else 3)
