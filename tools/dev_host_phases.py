"""The phased host entry point (mla_getrf_la_host + mla_set_host_phases): correctness against the device path
(bitwise for lu_mb, windows cut anywhere) and end-to-end time at n = 32768 for several window layouts.
usage: python tools/dev_host_phases.py [check] [time [n]]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi

L = _capi.lib()
pool = mla.default_pool()

def set_phases(bounds, deep=0):
    if bounds is None:
        rc = L.mla_set_host_phases(pool.handle, None, -1, deep)
    else:
        arr = (ctypes.c_int64 * max(1, len(bounds)))(*bounds)
        rc = L.mla_set_host_phases(pool.handle, arr, len(bounds), deep)
    assert rc == 0, rc

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
    for (m, n, b_o, b_i, bounds) in [(3000, 3000, 256, 32, [256, 768, 1536]), (5000, 3500, 256, 32, [1024, 2048]),
                                     (6144, 6144, 512, 64, [512, 1024, 3072, 5632]), (4096, 4096, 128, 32, [128, 256, 384, 512, 4000]),
                                     (2500, 2500, 256, 32, [700, 1900])]:
        rng = np.random.default_rng(5)
        a = np.asfortranarray(rng.uniform(-1, 1, size=(m, n)))
        for variant in ("lu_mb", "lu", "lu_la", "lu_et"):
            d = mla.from_numpy(a)
            r = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(b_o, b_i)), pool)
            want = mla.to_numpy(d)
            pristine = torch.from_numpy(np.array(a.T, order="C", copy=True))
            for deep in (0, 512, 100000):
                set_phases(bounds, deep)
                host = pristine.clone().pin_memory()
                ipiv, info, _ = host_call(host, m, n, b_o, b_i, variant)
                got = host.numpy().T
                same_piv = np.array_equal(ipiv, r.ipiv.ipiv)
                bitwise = np.array_equal(got, want)
                scale = np.maximum(np.abs(want), np.abs(want).max(axis=0, keepdims=True))
                err = float((np.abs(got - want) / scale).max())
                print(f"{m}x{n} b={b_o}/{b_i} {variant} deep={deep} bounds={bounds}: pivots {'same' if same_piv else 'DIFFER'}, "
                      f"bitwise {bitwise}, max col-scaled diff {err:.2e}, panels {info.n_panels} (device {len(r.widths)}), et {info.et_events}",
                      flush=True)
                assert same_piv and err < 1e-10
                if variant != "lu_et" and deep == 0:
                    assert bitwise
                    assert info.n_panels == len(r.widths)
    set_phases(None)
    print("check OK")

def timing(n):
    b_o, b_i = 512, 64
    pool.t_pf_max = int(os.environ.get("T_PF_MAX", "0"))       # malleable panel team inside the windows
    a = mla.alloc_matrix(n, n)
    mla.fill_random(a, 3, 2.0, -1.0)
    host_t = a.t().contiguous().cpu().pin_memory()          # (n, n): rows are the matrix's columns
    del a
    work = torch.empty_like(host_t).pin_memory()
    f = n // 32
    layouts = [("one phase", [], 0), ("default", None, 4096)]
    for spec in os.environ.get("LAYOUTS", "1,4,12,22;1,4,12,20;1,4,12,18,25;1,4,10,20;1,4,12,17,22,27").split(";"):
        layouts.append((f"{spec} /32", [int(float(x) * f) for x in spec.split(",")], 4096))
    for variant in VARIANTS:
        for name, bounds, deep in layouts:
            set_phases(bounds, deep)
            ts = []
            for i in range(3):
                work.copy_(host_t)
                ipiv, info, dt = host_call(work, n, n, b_o, b_i, variant)
                if i: ts.append(dt)
            print(f"n={n} {variant} {name}: {np.mean(ts)*1e3:.1f} ms (min {min(ts)*1e3:.1f}), panels {info.n_panels}, et {info.et_events}", flush=True)
    set_phases(None)

VARIANTS = tuple(os.environ.get("VARIANTS", "lu_et,lu_mb").split(","))

if __name__ == "__main__":
    args = sys.argv[1:] or ["check"]
    if "check" in args: check()
    if "time" in args:
        i = args.index("time")
        timing(int(args[i + 1]) if len(args) > i + 1 else 32768)
