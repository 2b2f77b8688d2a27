import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_06365_b200 as mla
import oracle
from paper_1611_06365_b200.workloads import make_matrix

def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))

stage = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)

if stage in ("all", "laswp"):
    for rows, cols, npiv in [(30, 9, 10), (500, 300, 64), (4096, 1000, 256), (2000, 77, 1)]:
        a = np.asfortranarray(rng.standard_normal((rows, cols)))
        ipiv = np.array([rng.integers(t, rows) for t in range(npiv)], dtype=np.int64)
        for rev in (False, True):
            d = mla.from_numpy(a); mla.laswp(d, ipiv, reverse=rev)
            r = a.copy(order="F"); oracle.laswp(r, ipiv, reverse=rev)
            assert np.array_equal(mla.to_numpy(d), r), ("laswp", rows, cols, npiv, rev)
    try:
        mla.laswp(mla.from_numpy(a), [1, 99999]); raise SystemExit("no IndexError")
    except IndexError: pass
    print("laswp ok", flush=True)

if stage in ("all", "trsm"):
    for w, c in [(2, 1), (24, 17), (32, 128), (100, 300), (256, 1000), (512, 260)]:
        L = np.asfortranarray(rng.uniform(-1, 1, (w, w))); B = np.asfortranarray(rng.standard_normal((w, c)))
        d = mla.from_numpy(B); mla.trsm_llu(mla.from_numpy(L), d)
        r = B.copy(order="F"); oracle.trsm_llu(L, r)
        e = rel(mla.to_numpy(d), r); print("trsm", w, c, e, flush=True)
        assert e < 1e-9
    print("trsm ok", flush=True)

if stage in ("all", "panel"):
    for m, w, b, team in [(64, 48, 8, 1), (64, 48, 8, 4), (200, 96, 32, 3), (2048, 256, 32, 16), (5000, 256, 32, 8), (40000, 128, 32, 16), (1000, 192, 64, 148)]:
        a = make_matrix("uniform", w, 5, m)
        d = mla.from_numpy(a); t0 = time.perf_counter(); res = mla.lu_blk_ll(d, b, team_sms=team); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        r = a.copy(order="F"); ro = oracle.lu_blk_ll(r, b)
        same = np.array_equal(res.ipiv.ipiv, ro.ipiv)
        e = rel(mla.to_numpy(d), r)
        print("panel", m, w, b, team, "pivots_equal", same, "relerr", e, "cols", res.cols_factored, f"{dt*1e3:.2f} ms", flush=True)
        assert same and e < 1e-9
    # ET semantics
    a = make_matrix("uniform", 128, 3, 128)
    d = mla.from_numpy(a); res = mla.lu_blk_ll(d, 32, stop=mla.CountingStop(1), team_sms=4)
    r = a.copy(order="F"); ro = oracle.lu_blk_ll(r, 32, stop_trip=1)
    assert res.cols_factored == 32 == ro.cols_factored and rel(mla.to_numpy(d), r) < 1e-10
    d = mla.from_numpy(a); res = mla.lu_blk_ll(d, 32, stop=mla.CountingStop(3), team_sms=4)
    assert res.cols_factored == 96
    print("panel ok", flush=True)

if stage in ("all", "lu"):
    for n, bo, bi, variant in [(100, 16, 4, "lu"), (300, 64, 16, "lu"), (300, 64, 16, "lu_la"), (1000, 128, 32, "lu_mb"), (1000, 128, 32, "lu_et"), (2048, 256, 32, "lu"), (2048, 256, 32, "lu_la"), (2048, 256, 32, "lu_et"), (2048, 256, 32, "lu_ws_static")]:
        a = make_matrix("uniform", n, 0)
        d = mla.from_numpy(a)
        t0 = time.perf_counter(); res = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(bo, bi))); dt = time.perf_counter() - t0
        r = a.copy(order="F")
        sched = mla.et_schedule_from(res.widths, n, bo, bi)
        ro = oracle.lu_la(r, bo, bi, et_sched=sched)
        same = np.array_equal(res.ipiv.ipiv, ro.ipiv)
        e = rel(mla.to_numpy(d), r)
        print("lu_la", n, bo, bi, variant, "pivots_equal", same, "relerr", e, "et", res.et_events, res.et_widths[:6], "ws", res.ws_joins, "widths_ok", tuple(res.widths) == tuple(ro.widths), f"{dt*1e3:.1f} ms", flush=True)
        assert same and e < 1e-9
    print("lu ok", flush=True)
