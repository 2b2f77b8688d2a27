import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_06365_b200 import _capi
L = ctypes.CDLL(_capi.LIB_PATH)
h = ctypes.c_void_p(); assert _capi.lib().mla_create(0, ctypes.byref(h)) == 0
i64, vp = ctypes.c_int64, ctypes.c_void_p
L.mla_gemm_half_experiment.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, i64, i64, ctypes.c_int, vp]
MODE = int(sys.argv[1]) if len(sys.argv) > 1 else 0
def cm(m, n): return torch.randn(n, m, dtype=torch.float64, device="cuda").t()
def run(m, n, k, check=False, reps=3):
    A, B, C = cm(m, k), cm(k, n), cm(m, n)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: L.mla_gemm_half_experiment(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, MODE, s)
    if check:
        ref = C - A @ B; f(); torch.cuda.synchronize()
        print("maxerr", (C - ref).abs().max().item())
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"mode {MODE} half-tile gemm {m}x{n}x{k}: {ms:.3f} ms  {2.0*m*n*k/ms*1e-9:.2f} TFLOP/s", flush=True)
run(1024, 1024, 256, check=True)
for m, k in [(8192, 256), (16384, 256), (16384, 512), (32768, 256)]:
    run(m, m, k)
