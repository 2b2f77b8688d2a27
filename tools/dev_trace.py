import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
n = int(sys.argv[1]); variant = sys.argv[2] if len(sys.argv) > 2 else "lu_et"
bo = int(sys.argv[3]) if len(sys.argv) > 3 else 256; bi = bo // 8
tpf = int(sys.argv[4]) if len(sys.argv) > 4 else None
pool = mla.default_pool()
if len(sys.argv) > 5: pool.t_pf_max = int(sys.argv[5])
if len(sys.argv) > 6: bi = int(sys.argv[6])
a0 = mla.alloc_matrix(n, n); mla.fill_random(a0, 3, 2.0, -1.0)
a = mla.alloc_matrix(n, n)
for rep in range(2):
    a.copy_(a0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); res = mla.lu_la(a, mla.Policy(variant, mla.BlockConfig(bo, bi), t_pf=tpf), pool); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"n={n} {variant} b={bo}/{bi}: {ms:.2f} ms  {mla.flops_lu(n,n)/ms/1e9:.2f} TFLOP/s  panels {len(res.widths)} et {res.et_events} ws {res.ws_joins} t_pf_max {pool.t_pf_max} peak {res.t_pf_peak}")
rows = len(res.widths) - 1
buf = (ctypes.c_uint64 * (5 * 1024))()
got = _capi.lib().mla_getrf_trace(pool.handle, buf, 1024)
t = np.array(buf[:5 * min(rows, got)], dtype=np.uint64).reshape(-1, 5).astype(np.int64)
prof = (ctypes.c_uint64 * 16)(); _capi.lib().mla_panel_profile(pool.handle, prof, 1)
dbg = (ctypes.c_uint64 * 8)(); _capi.lib().mla_getrf_debug(pool.handle, dbg)
print("  RU CTA: gemm %.1f ms in %d tiles (%.2f us/tile), prep %.2f ms in %d (%.1f us each), left %.2f ms, barriers %.2f ms, kernel %.1f ms, chained-tile gaps %.2f ms" % (
    dbg[0] / 1e6, dbg[1], dbg[0] / 1e3 / max(1, dbg[1]), dbg[2] / 1e6, dbg[3], dbg[2] / 1e3 / max(1, dbg[3]), dbg[4] / 1e6, dbg[5] / 1e6, dbg[6] / 1e6, dbg[7] / 1e6))
print("  it   w  knew   pq_us panel_us   rq_us  iter_us   (pq: start->panel may start; panel: PF panel; rq: start->remainder done)")
tot = {"pq": 0, "panel": 0, "rq": 0, "iter": 0}
for i in range(len(t)):
    s0, pq, pe, rq, wk = t[i]
    nxt = t[i + 1][0] if i + 1 < len(t) else max(pe, rq)
    w, k = int(wk) >> 32, int(wk) & 0xffffffff
    row = ((pq - s0) / 1e3, (pe - pq) / 1e3, (rq - s0) / 1e3 if rq else 0.0, (nxt - s0) / 1e3)
    tot["pq"] += row[0]; tot["panel"] += row[1]; tot["rq"] += row[2]; tot["iter"] += row[3]
    if i < 6 or i % max(1, len(t) // 24) == 0 or i > len(t) - 4 or os.environ.get('TRACE_ALL'):
        print(f"{i+1:4d} {w:4d} {k:5d} {row[0]:7.0f} {row[1]:8.0f} {row[2]:7.0f} {row[3]:8.0f}")
ub = [(int(t[i][3]) - int(t[i][0])) >= (int(t[i][2]) - int(t[i][0])) for i in range(len(t))]
it_us = [((t[i + 1][0] if i + 1 < len(t) else max(t[i][2], t[i][3])) - t[i][0]) / 1e3 for i in range(len(t))]
print("  update-bound iterations: %d, %.1f ms;  panel-bound iterations: %d, %.1f ms (of which panel+pq %.1f ms)" % (
    sum(ub), sum(x for x, u in zip(it_us, ub) if u) / 1e3, len(ub) - sum(ub), sum(x for x, u in zip(it_us, ub) if not u) / 1e3,
    sum((int(t[i][2]) - int(t[i][0])) / 1e3 for i in range(len(t)) if not ub[i]) / 1e3))
cum_c, marks, nxtm = 0, [], 4096
for i in range(len(t)):
    cum_c += res.widths[i]
    while cum_c >= nxtm:
        marks.append((nxtm, (int(t[i][0]) - int(t[0][0])) / 1e6)); nxtm += 4096
print("  time (ms) at which the iteration that factors past column q starts: " + "  ".join(f"{q}:{ms_:.1f}" for q, ms_ in marks))
print("  totals (ms):", {k: round(v / 1e3, 2) for k, v in tot.items()})
print("  panel phases of all panels (ms): trsm %.2f gemm %.2f steps %.2f (xchg %.2f) wb+swap %.2f bar %.2f" % tuple(x / 1e6 / 2 for x in prof[:3] + prof[5:6] + prof[3:5]))
