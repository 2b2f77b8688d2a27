"""cuBLAS DGEMM sustained rate on this B200 (measurement reference only, never the product path)."""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n, k in [(8192, 8192), (16384, 256), (16384, 512), (32768, 256)]:
    a = torch.randn(n, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cublas dgemm m=n={n} k={k}: {ms:.3f} ms  {2.0*n*n*k/ms*1e-9:.2f} TFLOP/s")
    del a, b, c
