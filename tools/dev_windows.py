"""The windowed (two-level) factorization: correctness against the oracle (clamped replay) at small sizes with a
small window, bitwise repeatability, host entry point == device path, and timing at full size.
usage: python tools/dev_windows.py [check] [time n [W ...]] [e2e n]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi

L = _capi.lib()
pool = mla.default_pool()
EPS = np.finfo(np.float64).eps

def host_call(host_t, m, n, b_o, b_i, variant):
    ipiv = torch.empty(n, dtype=torch.int32).pin_memory()
    info = _capi.LuInfo()
    t0 = time.perf_counter()
    rc = L.mla_getrf_la_host(pool.handle, host_t.data_ptr(), m, n, m, ipiv.data_ptr(), b_o, b_i,
                             _capi.VARIANT_CODES[variant], pool.t_pf, 4, ctypes.byref(info))
    dt = time.perf_counter() - t0
    _capi.check(rc, pool.handle, "mla_getrf_la_host")
    return ipiv.numpy().astype(np.int64), info, dt

def check():
    cases = [(2048, 2048, 128, 32, 512, 256), (3000, 2500, 256, 32, 512, 256), (3333, 3333, 128, 16, 1024, 384),
             (4096, 4096, 256, 64, 1024, 0), (2304, 2304, 128, 32, 768, 128)]
    for (m, n, b_o, b_i, W, fc) in cases:
        pool.set_windows(W, 1024, fc)
        rng = np.random.default_rng(7)
        a = np.asfortranarray(rng.uniform(-1, 1, size=(m, n)))
        first = {}
        for variant in ("lu", "lu_la", "lu_mb", "lu_et"):
            d = mla.from_numpy(a)
            r = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(b_o, b_i)), pool)
            got = mla.to_numpy(d)
            assert r.window == W // b_o * b_o, (r.window, W)
            ref = a.copy(order="F")
            ro = oracle.lu_la(ref, b_o, b_i, et_sched=mla.et_schedule_from(r.widths, n, b_o, b_i, r.window), clamp=r.window)
            assert tuple(ro.widths) == tuple(r.widths), (ro.widths, r.widths)
            same_piv = np.array_equal(r.ipiv.ipiv, ro.ipiv)
            scale = np.maximum(np.abs(ref), np.abs(ref).max(axis=0, keepdims=True))
            err = float((np.abs(got - ref) / scale).max())
            berr = oracle.residual_lu(a, got, r.ipiv.ipiv) / (n * EPS)
            print(f"{m}x{n} b={b_o}/{b_i} W={W} {variant}: pivots {'same' if same_piv else 'DIFFER'}, err {err:.2e}, "
                  f"backward {berr:.4f} n eps, panels {len(r.widths)}, et {r.et_events}", flush=True)
            assert same_piv and err < 1e-10 and berr < 10
            if variant != "lu_et":
                if not first: first["f"] = got
                else: assert np.array_equal(first["f"], got), "variants differ bitwise"
            # host entry point: same factors (bitwise without ET)
            pristine = torch.from_numpy(np.array(a.T, order="C", copy=True))
            host = pristine.clone().pin_memory()
            ipiv, info, _ = host_call(host, m, n, b_o, b_i, variant)
            hgot = host.numpy().T
            herr = float((np.abs(hgot - ref) / scale).max())
            assert np.array_equal(ipiv, ro.ipiv) and herr < 1e-10, herr
            if variant != "lu_et":
                assert np.array_equal(hgot, got), "host entry differs from the device path"
                assert info.n_panels == len(r.widths)
            print(f"      host entry: err {herr:.2e}, bitwise {np.array_equal(hgot, got)}, panels {info.n_panels}", flush=True)
    pool.set_windows(4096, 16384, 1024)
    print("check OK")

def timing(n, widths):
    b_o, b_i = 512, 64
    a0 = mla.alloc_matrix(n, n)
    mla.fill_random(a0, 3, 2.0, -1.0)
    for W in widths:
        pool.set_windows(W, 8192 if W else 16384, 1024)
        for variant in os.environ.get("VARIANTS", "lu_et,lu_mb").split(","):
            ts = []
            for i in range(3):
                a = a0.clone()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r = mla.lu_la(a, mla.Policy(variant, mla.BlockConfig(b_o, b_i)), pool)
                e1.record(); torch.cuda.synchronize()
                if i: ts.append(e0.elapsed_time(e1))
            resid = mla.residual_packed(a0.clone(), a, r.ipiv) / (n * EPS)
            ms = float(np.mean(ts))
            print(f"n={n} W={W} {variant}: {ms:.1f} ms  {2*n**3/3/ms*1e-9:.2f} TFLOP/s  panels {len(r.widths)} et {r.et_events} "
                  f"backward {resid:.4f} n eps", flush=True)
            del a
    pool.set_windows(4096, 16384, 1024)

def e2e(n, widths):
    b_o, b_i = 512, 64
    a = mla.alloc_matrix(n, n)
    mla.fill_random(a, 3, 2.0, -1.0)
    host_t = a.t().contiguous().cpu().pin_memory()
    del a
    work = torch.empty_like(host_t).pin_memory()
    for W in widths:
        for fc in (1024,):
            pool.set_windows(W, 8192 if W else 16384, fc)
            for variant in os.environ.get("VARIANTS", "lu_et").split(","):
                ts = []
                for i in range(3):
                    work.copy_(host_t)
                    ipiv, info, dt = host_call(work, n, n, b_o, b_i, variant)
                    if i: ts.append(dt)
                print(f"e2e n={n} W={W} first_chunk={fc} {variant}: {np.mean(ts)*1e3:.1f} ms (min {min(ts)*1e3:.1f}) panels {info.n_panels} et {info.et_events}", flush=True)
    pool.set_windows(4096, 16384, 1024)

if __name__ == "__main__":
    args = sys.argv[1:] or ["check"]
    if "check" in args: check()
    if "time" in args:
        i = args.index("time")
        rest = [int(x) for x in args[i + 1:] if x.isdigit()]
        timing(rest[0] if rest else 32768, rest[1:] or [0, 4096])
    if "e2e" in args:
        i = args.index("e2e")
        rest = [int(x) for x in args[i + 1:] if x.isdigit()]
        e2e(rest[0] if rest else 32768, rest[1:] or [0, 4096])
