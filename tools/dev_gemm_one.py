"""One mla_gemm shape, launched a few times (for an ncu capture): dev_gemm_one.py m n k [reps]"""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1611_06365_b200 import _capi
L = _capi.lib(); h = ctypes.c_void_p(); assert L.mla_create(0, ctypes.byref(h)) == 0
m, n, k = (int(x) for x in sys.argv[1:4]); reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cm = lambda r, c: (torch.rand(c, r, dtype=torch.float64, device="cuda") - 0.5).t()
A, B, C = cm(m, k), cm(k, n), cm(m, n)
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    if i == 1: e0.record()
    assert L.mla_gemm(h, C.data_ptr(), m, n, C.stride(1), A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), k, 1.0, -1.0, None, 0, s) == 0
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / max(1, reps - 1)
print(f"gemm {m}x{n}x{k}: {ms:.3f} ms {2.0*m*n*k/ms*1e-9:.2f} TFLOP/s")
