import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
pool = mla.default_pool(); L = _capi.lib(); s = torch.cuda.current_stream().cuda_stream
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
n = 16384
A = mla.alloc_matrix(n, n); mla.fill_random(A, 1, 2.0, -1.0)
for w in (128, 256, 512):
    for c in (128 * 148, 128 * 148 * 2):
        c = min(c, n - w)
        us = t(lambda: L.mla_trsm_llu(pool.handle, A.data_ptr(), w, n, A[:, w:].data_ptr(), c, n, s))
        strips = (c + 127) // 128
        print(f"trsm w={w} c={c}: {us:.0f} us  ({us / ((strips + 147) // 148):.0f} us per strip round, {w*w*c/us*1e-6:.2f} TFLOP/s)")
for npiv in (64, 256, 512):
    rng = np.random.default_rng(0)
    ipiv = torch.from_numpy(np.array([rng.integers(t_, n) for t_ in range(npiv)], dtype=np.int32)).cuda()
    for cols in (4096, 16384):
        us = t(lambda: L.mla_laswp_async(pool.handle, A.data_ptr(), n, cols, n, ipiv.data_ptr(), npiv, 0, s))
        print(f"laswp npiv={npiv} cols={cols}: {us:.0f} us  algorithmic {32.0*npiv*cols/us*1e-3:.0f} GB/s")
