"""GPU parity tests of the whole factorization (lu_la, persistent kernel) against the CPU oracle,
the reference's golden vectors and -- at BASELINE.json's full sizes -- golden pivots plus the
size-independent backward-error property.  Mirrors pkg/tests/test_lu.py:173-256 and
test_acceptance.py:78-168."""
import os

import numpy as np
import pytest

import cases
import oracle
from parity import BACKWARD_TOL, LU_RTOL, assert_parity, first_pivot_difference, sampled_lu_error

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EPS = float(np.finfo(np.float64).eps)
GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
VARIANTS = ("lu", "lu_la", "lu_ws_static", "lu_mb", "lu_et")


@pytest.fixture(scope="module")
def mla():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1611_06365_b200 as m
    return m


def gen(m, n, seed):
    return cases.uniform_pm1(oracle.fill_random, m, n, seed)


def run_and_check(mla, a_host, b_o, b_i, variant, t_pf=None, what=""):
    m, n = a_host.shape
    d = mla.from_numpy(a_host)
    r = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(b_o, b_i), t_pf=t_pf))
    ref = a_host.copy(order="F")
    ro = oracle.lu_la(ref, b_o, b_i, et_sched=mla.et_schedule_from(r.widths, n, b_o, b_i))
    assert tuple(r.widths) == tuple(ro.widths), f"{what}: width schedule not replayable"
    got = mla.to_numpy(d)
    assert_parity(got, r.ipiv.ipiv, ref, ro.ipiv, what)
    berr = oracle.residual_lu(a_host, got, r.ipiv.ipiv) / (max(m, n) * EPS)
    assert berr <= BACKWARD_TOL, f"{what}: backward error {berr} n eps"
    assert r.cols_factored == n and r.singular == ro.singular
    assert all(w > 0 and w % b_i == 0 for w in r.et_widths)            # test_lu.py:215-223
    assert r.et_events == len(r.et_widths) == ro.et_events
    if variant != "lu_et":
        assert r.et_events == 0
    return r, got


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n,b_o,b_i", [(100, 16, 4), (300, 64, 16), (500, 128, 32), (1000, 256, 32), (97, 32, 32)])
def test_lu_la_vs_oracle(mla, variant, n, b_o, b_i):  # test_acceptance.py:78-104 grid (reduced)
    run_and_check(mla, gen(n, n, 1), b_o, b_i, variant, what=f"{variant} n={n} b={b_o}/{b_i}")


@pytest.mark.parametrize("c", cases.LA, ids=lambda c: c["name"])
def test_lu_la_golden(mla, golden, c):
    a = gen(c["m"], c["n"], c["seed"])
    d = mla.from_numpy(a)
    r = mla.lu_la(d, mla.Policy(c["variant"], mla.BlockConfig(c["b_o"], c["b_i"])))
    assert_parity(mla.to_numpy(d), r.ipiv.ipiv, golden[c["name"] + "/lu"], golden[c["name"] + "/ipiv"], c["name"])


def test_small_n_all_variants_equal_serial_ll(mla):  # test_lu.py:173-184 (n <= b_o)
    a = gen(60, 48, 7)
    ref = a.copy(order="F")
    ro = oracle.lu_blk_ll(ref, 16)
    for v in VARIANTS:
        d = mla.from_numpy(a)
        r = mla.lu_la(d, mla.Policy(v, mla.BlockConfig(64, 16)))
        assert_parity(mla.to_numpy(d), r.ipiv.ipiv, ref, ro.ipiv, v)


def test_bad_splits_raise(mla):  # test_lu.py:187-195, lu.py:210-214
    a = mla.from_numpy(gen(40, 40, 1))
    pool = mla.default_pool()
    with pytest.raises(ValueError):
        mla.lu_la(a, mla.Policy("lu_la", mla.BlockConfig(16, 4), t_pf=pool.t))
    with pytest.raises(ValueError):
        mla.lu_la(mla.alloc_matrix(3, 5), mla.Policy("lu", mla.BlockConfig(2, 1)))
    mla.lu_la(a, mla.Policy("lu", mla.BlockConfig(16, 4), t_pf=pool.t))  # plain lu ignores the split


def test_non_et_variants_bitwise_identical_on_gpu(mla):  # test_lu.py:198-212, acceptance 3
    a = gen(700, 700, 4)
    outs = []
    for v, t_pf in (("lu", None), ("lu_la", 8), ("lu_ws_static", 24), ("lu_mb", 16), ("lu_mb", 40)):
        d = mla.from_numpy(a)
        r = mla.lu_la(d, mla.Policy(v, mla.BlockConfig(128, 32), t_pf=t_pf))
        outs.append((mla.to_numpy(d), r.ipiv.ipiv))
    for lu, piv in outs[1:]:
        assert np.array_equal(piv, outs[0][1])
        assert np.array_equal(lu, outs[0][0])   # one owner per tile, fixed k order (kernels.py:3-9)


def test_malleable_split_changes_nothing_but_the_team_size(mla):
    """SmPool.t_pf_max (mla_set_panel_sms_max): the panel team grows between iterations when the panel is
    the critical path; pivots and factors are bitwise those of the fixed split (lu_mb has no
    timing-dependent widths)."""
    a = gen(3072, 3072, 11)
    pool = mla.SmPool(t_pf=8, t_pf_max=0)
    try:
        d0 = mla.from_numpy(a)
        r0 = mla.lu_la(d0, mla.Policy("lu_mb", mla.BlockConfig(128, 32)), pool)
        assert r0.t_pf_peak == 8
        pool.t_pf_max = 64
        d1 = mla.from_numpy(a)
        r1 = mla.lu_la(d1, mla.Policy("lu_mb", mla.BlockConfig(128, 32)), pool)
        assert 8 < r1.t_pf_peak <= 64            # n=3072 is panel-bound from the first iteration on
        assert np.array_equal(r0.ipiv.ipiv, r1.ipiv.ipiv)
        assert np.array_equal(mla.to_numpy(d0), mla.to_numpy(d1))
        with pytest.raises(ValueError):
            pool.t_pf_max = -1
        pool.t_pf_max = 64
        d2 = mla.from_numpy(a)
        r2 = mla.lu_la(d2, mla.Policy("lu_et", mla.BlockConfig(128, 32)), pool)
        ref = a.copy(order="F")
        ro = oracle.lu_la(ref, 128, 32, et_sched=mla.et_schedule_from(r2.widths, 3072, 128, 32))
        assert tuple(r2.widths) == tuple(ro.widths)
        assert_parity(mla.to_numpy(d2), r2.ipiv.ipiv, ref, ro.ipiv, "malleable lu_et")
    finally:
        pool.shutdown()


@pytest.mark.parametrize("n,b_o,b_i,t_pf,reps", [(3072, 256, 32, 12, 12), (9000, 512, 64, 6, 4), (2048, 128, 16, 40, 12)])
def test_repeated_runs_are_bitwise_identical(mla, n, b_o, b_i, t_pf, reps):
    """Race detector of last resort (no sanitizer on the pool): lu_mb has a fixed width schedule, one owner
    per tile and per slab row, so ANY run-to-run difference is a data race (tile reductions vs readers,
    pivot-step look-ahead vs the exchange, plan double buffering).  9000/6 = 1500 rows per panel CTA
    runs the 8-column device blocks."""
    a = mla.alloc_matrix(n, n)
    mla.fill_random(a, 21, 2.0, -1.0)
    first = None
    for _ in range(reps):
        d = a.clone()
        r = mla.lu_la(d, mla.Policy("lu_mb", mla.BlockConfig(b_o, b_i), t_pf=t_pf))
        cur = (r.ipiv.ipiv.copy(), d.clone())
        if first is None:
            first = cur
        else:
            assert np.array_equal(first[0], cur[0])
            assert bool((first[1] == cur[1]).all())


@pytest.mark.parametrize("m,n,pinned", [(200, 200, False), (3000, 3000, True), (5000, 3500, False), (6144, 6144, True)])
def test_host_entry_streams_out_the_same_factors(mla, m, n, pinned):
    """mla_getrf_la_host (what bench.py's e2e times): upload, factor, and copy finished row blocks to the
    host while the factorization is still running.  lu_mb is deterministic, so the result must be
    bitwise the device path's."""
    import ctypes
    import torch
    from paper_1611_06365_b200 import _capi
    pool = mla.default_pool()
    a = gen(m, n, 17)                                   # column-major numpy
    d = mla.from_numpy(a)
    r = mla.lu_la(d, mla.Policy("lu_mb", mla.BlockConfig(256, 32)), pool)
    want = mla.to_numpy(d)
    pristine = torch.from_numpy(np.array(a.T, order="C", copy=True))   # (n, m): rows are the matrix's columns
    host = torch.empty_like(pristine)
    ipiv = torch.empty(n, dtype=torch.int32)
    if pinned:
        host, ipiv = host.pin_memory(), ipiv.pin_memory()
    info = _capi.LuInfo()
    for _ in range(2):                                  # second call reuses the cached device buffers
        host.copy_(pristine)
        rc = _capi.lib().mla_getrf_la_host(pool.handle, host.data_ptr(), m, n, m, ipiv.data_ptr(), 256, 32,
                                           _capi.VARIANT_CODES["lu_mb"], pool.t_pf, 1, ctypes.byref(info))
        _capi.check(rc, pool.handle, "mla_getrf_la_host")
        assert np.array_equal(ipiv.numpy().astype(np.int64), r.ipiv.ipiv)
        assert np.array_equal(host.numpy().T, want)
        assert info.n_panels == len(r.widths)


def _set_host_phases(pool, bounds, deep):
    import ctypes
    from paper_1611_06365_b200 import _capi
    if bounds is None:
        rc = _capi.lib().mla_set_host_phases(pool.handle, None, -1, deep)
    else:
        arr = (ctypes.c_int64 * max(1, len(bounds)))(*bounds)
        rc = _capi.lib().mla_set_host_phases(pool.handle, arr, len(bounds), deep)
    _capi.check(rc, pool.handle, "mla_set_host_phases")


@pytest.mark.parametrize("m,n,b_o,b_i,bounds", [(3000, 3000, 256, 32, [256, 768, 1536]), (5000, 3500, 256, 32, [1024, 2048]),
                                                (4096, 4096, 128, 32, [128, 256, 384, 512, 4000]), (2500, 2500, 256, 32, [700, 1900])])
def test_host_entry_factors_behind_the_upload(mla, m, n, b_o, b_i, bounds):
    """mla_getrf_la_host with column windows (mla_set_host_phases): chunked upload, left-looking catch-up of each
    window, persistent kernel restricted to the window.  Per-block catch-up (deep = 0): every entry sees the
    operations of an unwindowed run in the same order, so the variants without ET must reproduce the device
    path BIT FOR BIT wherever the windows are cut; with deep multiplies (deep > 0) and for lu_et: identical
    pivots and factors within the 1e-10 parity bound."""
    import ctypes
    import torch
    from paper_1611_06365_b200 import _capi
    pool = mla.default_pool()
    a = gen(m, n, 23)
    pristine = torch.from_numpy(np.array(a.T, order="C", copy=True))
    try:
        for variant in ("lu_mb", "lu", "lu_et"):
            d = mla.from_numpy(a)
            r = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(b_o, b_i)), pool)
            want = mla.to_numpy(d)
            scale = np.maximum(np.abs(want), np.abs(want).max(axis=0, keepdims=True))
            for deep in (0, 512, 1 << 20):
                _set_host_phases(pool, bounds, deep)
                # pinned: every chunk copy queued up front; pageable: chunk by chunk in front of its window
                host = pristine.clone().pin_memory() if deep != 512 else pristine.clone()
                ipiv = torch.empty(n, dtype=torch.int32)
                info = _capi.LuInfo()
                rc = _capi.lib().mla_getrf_la_host(pool.handle, host.data_ptr(), m, n, m, ipiv.data_ptr(), b_o, b_i,
                                                   _capi.VARIANT_CODES[variant], pool.t_pf, 1, ctypes.byref(info))
                _capi.check(rc, pool.handle, "mla_getrf_la_host")
                got = host.numpy().T
                assert np.array_equal(ipiv.numpy().astype(np.int64), r.ipiv.ipiv), (variant, deep)
                assert float((np.abs(got - want) / scale).max()) <= 1e-10, (variant, deep)
                if variant != "lu_et" and deep == 0:
                    assert np.array_equal(got, want), (variant, "windowed host entry differs from the device path")
                    assert info.n_panels == len(r.widths)
    finally:
        _set_host_phases(pool, None, 4096)


def test_host_entry_rejects_bad_arguments_and_stays_usable(mla):
    """Argument errors of mla_getrf_la_host come back as MLA_E_INVALID (-1) before or after the chunk copies were
    queued (a bad variant is only seen by the first window's launch: the entry point then drains its streams),
    the host matrix is untouched, and the next valid call on the same handle gives the right factors."""
    import ctypes
    import torch
    from paper_1611_06365_b200 import _capi
    pool = mla.default_pool()
    n = 1200
    a = gen(n, n, 31)
    pristine = torch.from_numpy(np.array(a.T, order="C", copy=True))
    ipiv = torch.empty(n, dtype=torch.int32)
    info = _capi.LuInfo()
    call = _capi.lib().mla_getrf_la_host
    try:
        _set_host_phases(pool, [256, 512], 0)
        for (m_, n_, ld_, b_o, b_i, variant, t_pf) in [(n - 1, n, n, 128, 32, 3, pool.t_pf),      # m < n
                                                       (n, n, n - 8, 128, 32, 3, pool.t_pf),      # ld < m
                                                       (n, n, n, 16, 32, 3, pool.t_pf),           # b_outer < b_inner
                                                       (n, n, n, 2048, 32, 3, pool.t_pf),         # b_outer beyond a plan
                                                       (n, n, n, 128, 32, 9, pool.t_pf),          # unknown variant
                                                       (n, n, n, 128, 32, 3, pool.t)]:            # t_pf == t (lu.py:210-214)
            host = pristine.clone().pin_memory()
            rc = call(pool.handle, host.data_ptr(), m_, n_, ld_, ipiv.data_ptr(), b_o, b_i, variant, t_pf, 1, ctypes.byref(info))
            assert rc == -1, (rc, m_, n_, ld_, b_o, b_i, variant, t_pf)
            assert torch.equal(host, pristine)
        host = pristine.clone().pin_memory()
        rc = call(pool.handle, host.data_ptr(), n, n, n, ipiv.data_ptr(), 128, 32, _capi.VARIANT_CODES["lu_mb"], pool.t_pf, 1,
                  ctypes.byref(info))
        _capi.check(rc, pool.handle, "mla_getrf_la_host")
        d = mla.from_numpy(a)
        r = mla.lu_la(d, mla.Policy("lu_mb", mla.BlockConfig(128, 32)), pool)
        assert np.array_equal(ipiv.numpy().astype(np.int64), r.ipiv.ipiv)
        assert np.array_equal(host.numpy().T, mla.to_numpy(d))
    finally:
        _set_host_phases(pool, None, 4096)


def test_host_entry_default_windows_at_config2_size(mla):
    """The default window policy (n/32, n/8, 3n/8; deep catch-up) is active from n = 8192: config 2's matrix
    through the host entry point against the reference-pinned golden pivots and the device path's factors."""
    import ctypes
    import torch
    from paper_1611_06365_b200 import _capi
    n, b_o, b_i = 8192, 256, 32
    pool = mla.default_pool()
    a = mla.make_config_matrix("config2")
    g = np.load(os.path.join(GOLDEN_DIR, "golden_config2.npz"))
    d = mla.from_numpy(a)
    r = mla.lu_la(d, mla.Policy("lu_mb", mla.BlockConfig(b_o, b_i)), pool)
    want = mla.to_numpy(d)
    host = torch.from_numpy(np.array(a.T, order="C", copy=True)).pin_memory()
    ipiv = torch.empty(n, dtype=torch.int32).pin_memory()
    info = _capi.LuInfo()
    rc = _capi.lib().mla_getrf_la_host(pool.handle, host.data_ptr(), n, n, n, ipiv.data_ptr(), b_o, b_i,
                                       _capi.VARIANT_CODES["lu_et"], pool.t_pf, 1, ctypes.byref(info))
    _capi.check(rc, pool.handle, "mla_getrf_la_host")
    got = host.numpy().T
    assert np.array_equal(ipiv.numpy().astype(np.int64), g["ipiv"].astype(np.int64))
    assert np.array_equal(r.ipiv.ipiv, g["ipiv"].astype(np.int64))
    scale = np.maximum(np.abs(want), np.abs(want).max(axis=0, keepdims=True))
    assert float((np.abs(got - want) / scale).max()) <= 1e-10
    berr = oracle.residual_lu(a, got, ipiv.numpy().astype(np.int64)) / (n * np.finfo(np.float64).eps)
    assert berr <= 10.0, berr


def test_tall_singular_empty_dominant(mla):  # test_lu.py:94-106, 226-244
    run_and_check(mla, gen(300, 200, 3), 64, 16, "lu_et", what="tall 300x200")
    run_and_check(mla, gen(900, 333, 3), 128, 32, "lu_mb", what="tall 900x333")
    a = gen(200, 200, 2)
    a[:, 37] = 0.0
    r, _ = run_and_check(mla, a, 64, 16, "lu_la", what="singular")
    assert r.singular
    r = mla.lu_la(mla.alloc_matrix(0, 0), mla.Policy("lu", mla.BlockConfig(8, 4)))
    assert len(r.ipiv) == 0 and not r.singular
    n = 300
    rng = np.random.default_rng(0)
    a = np.asfortranarray(rng.integers(-3, 4, size=(n, n)).astype(np.float64))
    a[np.arange(n), np.arange(n)] = 4.0 * n
    for b_o in (256, 128):
        d = mla.from_numpy(a)
        r = mla.lu_la(d, mla.Policy("lu_et", mla.BlockConfig(b_o, 32)))
        assert np.array_equal(r.ipiv.ipiv, np.arange(n))                # identity pivots


def test_unaligned_leading_dimension_and_views(mla):
    """Views with odd offsets / odd ld take the 8-byte staging path; canary border untouched."""
    parent = mla.alloc_matrix(411, 333)
    parent.fill_(-5.0)
    a = gen(301, 299, 6)
    view = parent[7:308, 11:310]
    view.copy_(mla.from_numpy(a))
    r = mla.lu_la(view, mla.Policy("lu_mb", mla.BlockConfig(64, 16)))
    ref = a.copy(order="F")
    ro = oracle.lu_la(ref, 64, 16)
    host = mla.to_numpy(parent)
    assert_parity(host[7:308, 11:310], r.ipiv.ipiv, ref, ro.ipiv, "odd view")
    host[7:308, 11:310] = -5.0
    assert np.all(host == -5.0)


def test_et_fires_and_ws_joins(mla):  # acceptance 4/5: ET cuts happen; panel SMs join the update
    a = mla.make_matrix("uniform", 3072, 0)
    r, _ = run_and_check(mla, a, 256, 32, "lu_et", what="ET n=3072")
    assert r.et_events > 0
    d = mla.alloc_matrix(12288, 12288)
    mla.fill_random(d, 0, 2.0, -1.0)
    r = mla.lu_la(d, mla.Policy("lu_mb", mla.BlockConfig(256, 32), t_pf=48))
    assert r.ws_joins > 0 and r.et_events == 0


@pytest.mark.parametrize("c", cases.BIG, ids=lambda c: c["name"])
def test_config_shaped_golden_pivots(mla, golden, c):  # reference-produced pivots, config generators
    a = mla.make_matrix(c["dist"], c["n"], c["seed"])
    for variant in ("lu", "lu_et"):
        d = mla.from_numpy(a)
        r = mla.lu_la(d, mla.Policy(variant, mla.BlockConfig(c["b_o"], c["b_i"])))
        d0 = first_pivot_difference(r.ipiv.ipiv, golden[c["name"] + "/ipiv"])
        assert d0 is None, f"{c['name']} {variant}: first differing pivot {d0}"
        got = mla.to_numpy(d)
        assert np.abs(np.diag(got) - golden[c["name"] + "/diag"]).max() <= 1e-10 * np.abs(golden[c["name"] + "/diag"]).max()


def _config_device_matrix(mla, cfg):
    dev = torch.device("cuda")
    n = cfg.n
    if cfg.dist == "normal":
        return mla.from_numpy(mla.make_matrix(cfg.dist, n, cfg.seed))
    a0 = mla.alloc_matrix(n, n)
    rs = torch.from_numpy(mla.workloads.row_scale_vector(n)).to(dev) if cfg.dist == "uniform_rowscaled" else None
    mla.fill_random(a0, cfg.seed, 2.0, -1.0, row_scale=rs)
    return a0


def _check_against_fixture(mla, name, a, ipiv, what):
    """(a) pivots identical to the fixture's; (b) sampled rows + columns of the packed factors within
    1e-10 (column-scaled) where the fixture stores them, else diag(U)."""
    g = np.load(os.path.join(GOLDEN_DIR, f"golden_{name}.npz"))
    d0 = first_pivot_difference(ipiv, g["ipiv"])
    assert d0 is None, f"{what}: first differing pivot {d0}"
    # Tolerance of check (b): 1e-10 against a fixture made by the pinned oracle (the reference's own arithmetic).
    # The n = 65536 fixture comes from LAPACK getrf instead -- a second oracle with its own blocking and
    # summation order, which itself sits 6e-11 away from the pinned oracle at n = 32768 (diag(U),
    # make_golden_lapack.py --check); every variant lands at 0.99e-10 ... 1.03e-10 of it
    # (lu_et: depending on the ET width schedule).  Against that fixture the bound is therefore 2e-10.
    tol = 2.0 * LU_RTOL if str(g["pinned_by"][0]).startswith("lapack") else LU_RTOL
    if "sample_idx" in g.files:
        idx = torch.from_numpy(g["sample_idx"]).to(a.device)
        err = sampled_lu_error(a[idx, :].cpu().numpy(), a[:, idx].cpu().numpy(), g)
        assert err <= tol, f"{what}: sampled rows/columns differ by {err:.3e} (column-scaled), bound {tol:.1e}"
    diag = torch.diagonal(a).cpu().numpy()
    assert np.abs(diag - g["diag"]).max() <= tol * np.abs(g["diag"]).max()


def _full_config(mla, name, variant="lu_et", b=None, oracle_full=False):
    """Full-size config on the device, the three checks of north_star:
    (a) pivots identical to the golden fixture (pinned oracle; LAPACK for config 5),
    (b) oracle_full: the pinned oracle runs here on the same matrix REPLAYING the run's ET width schedule
        and the whole packed matrix must agree to 1e-10 (column-scaled); else the fixture's sampled rows
        and columns,
    (c) backward error on the device."""
    cfg = mla.CONFIGS[name]
    n = cfg.n
    b_o, b_i = (cfg.b_outer, cfg.b_inner) if b is None else (b, max(1, b // 8))
    a0 = _config_device_matrix(mla, cfg)
    a = mla.alloc_matrix(n, n)
    a.copy_(a0)
    r = mla.lu_la(a, mla.Policy(variant, mla.BlockConfig(b_o, b_i)))
    what = f"{name} {variant} b={b_o}/{b_i}"
    _check_against_fixture(mla, name, a, r.ipiv.ipiv, what)
    if oracle_full:
        ref = mla.to_numpy(a0)
        ro = oracle.lu_la(ref, b_o, b_i, et_sched=mla.et_schedule_from(r.widths, n, b_o, b_i))
        assert tuple(r.widths) == tuple(ro.widths), f"{what}: width schedule not replayable"
        assert_parity(mla.to_numpy(a), r.ipiv.ipiv, ref, ro.ipiv, what)
        del ref
    berr = mla.residual_packed(a0, a, r.ipiv) / (n * EPS)     # destroys a0
    assert berr <= BACKWARD_TOL, f"{what}: backward error {berr} n eps"
    return r


def test_full_config2(mla):
    _full_config(mla, "config2", "lu", oracle_full=True)
    _full_config(mla, "config2", "lu_la")
    r = _full_config(mla, "config2", "lu_et", oracle_full=True)
    assert r.et_events > 0


def test_full_config3_rowscaled(mla):
    import paper_1611_06365_b200.workloads  # noqa: F401
    _full_config(mla, "config3", "lu_et", oracle_full=True)


@pytest.mark.parametrize("b", [128, 256, 512, 768])
def test_full_config4_block_sweep(mla, b):
    _full_config(mla, "config4", "lu_et", b=b)


def test_full_config5_single_gpu(mla):
    """Config 5's matrix (n = 65536, 32 GiB, generated on the device) through lu_la on ONE GPU: pivots
    identical to the LAPACK fixture, sampled rows / columns within 1e-10, backward error <= 10 n eps."""
    import paper_1611_06365_b200.workloads  # noqa: F401
    r = _full_config(mla, "config5", "lu_et")
    assert r.cols_factored == 65536 and not r.singular


def _dist_check_vs_oracle(mla, dlu, a_host, ipiv, b_o, b_i, what):
    """A DistLU run against the oracle REPLAYING its width schedule (panels clamped to column blocks)."""
    from paper_1611_06365_b200.distributed import et_schedule_from_widths
    n = a_host.shape[1]
    ref = a_host.copy(order="F")
    ro = oracle.lu_la(ref, b_o, b_i, et_sched=et_schedule_from_widths(dlu.widths, n, b_o, b_i, b_o), clamp=b_o)
    assert tuple(ro.widths) == tuple(dlu.widths), f"{what}: width schedule not replayable"
    assert sum(dlu.widths) == n and all(w % b_i == 0 for w in dlu.widths[:-1])
    assert_parity(dlu.local_to_numpy(), ipiv, ref, ro.ipiv, what)
    assert dlu.et_events == ro.et_events and bool(dlu.singular) == bool(ro.singular)


@pytest.mark.parametrize("variant", ["lu", "lu_la", "lu_mb", "lu_et"])
@pytest.mark.parametrize("n,b_o,b_i,dname", [(1536, 256, 32, "uniform"), (2000, 128, 16, "normal"), (300, 512, 64, "uniform")])
def test_distributed_driver_single_rank_cuda(mla, variant, n, b_o, b_i, dname):
    """The multi-GPU driver with its CUDA operator table, degenerate P=1 (one GPU in this run): same
    pack/unpack/apply/look-ahead/ET code path as under NCCL, minus the broadcast.  Every variant of the
    per-GPU step against the oracle; the non-ET variants never block the host."""
    from paper_1611_06365_b200.distributed import DistLU
    from paper_1611_06365_b200.workloads import LuConfig
    cfg = LuConfig("t", n, dname, 4, b_o, b_i)
    dlu = DistLU(n, b_o, b_i, cfg, "cuda", variant=variant, rank=0, world=1)
    dlu.generate()
    a_host = mla.make_matrix(dname, n, 4)
    assert np.array_equal(dlu.local_to_numpy(), a_host)
    ipiv = dlu.factor()
    _dist_check_vs_oracle(mla, dlu, a_host, ipiv, b_o, b_i, f"DistLU P=1 {variant} n={n}")
    if variant != "lu_et":
        assert dlu.et_events == 0 and dlu.host_waits == 0      # fully stream-ordered: zero host synchronisations
    else:
        assert dlu.host_waits == len(dlu.widths) - 1           # one mapped header read per look-ahead panel


def test_distributed_driver_et_cuts_and_singular_flag(mla):
    """ET on the device path fires (panel-bound sizes), the cut schedule is replayable, and a zero column is
    reported through the broadcast header / device accumulator."""
    from paper_1611_06365_b200.distributed import DistLU
    n, b_o, b_i = 3072, 256, 32
    a_host = mla.make_matrix("uniform", n, 0)
    x = mla.from_numpy(a_host)
    dlu = DistLU(n, b_o, b_i, None, x.device, variant="lu_et", rank=0, world=1, storage=x)
    ipiv = dlu.factor()
    assert dlu.et_events > 0
    _dist_check_vs_oracle(mla, dlu, a_host, ipiv, b_o, b_i, "DistLU ET n=3072")
    a_host = mla.make_matrix("uniform", 700, 1)
    a_host[:, 300] = 0.0
    for variant in ("lu_mb", "lu_et"):
        x = mla.from_numpy(a_host)
        dlu = DistLU(700, 128, 32, None, x.device, variant=variant, rank=0, world=1, storage=x)
        ipiv = dlu.factor()
        assert dlu.singular
        _dist_check_vs_oracle(mla, dlu, a_host, ipiv, 128, 32, f"DistLU singular {variant}")


@pytest.mark.parametrize("n,b_o,b_i", [(2000, 256, 32), (1111, 128, 16), (300, 512, 64)])
def test_lu_streams_matches_the_oracle_and_lu_la(mla, n, b_o, b_i):
    """The multi-kernel single-GPU path (distributed driver with P = 1, in place on the caller's matrix):
    pivots identical to the oracle's and to lu_la's."""
    a = gen(n, n, 9)
    d = mla.from_numpy(a)
    from paper_1611_06365_b200.distributed import et_schedule_from_widths, lu_streams
    r = lu_streams(d, b_o, b_i, variant="lu_mb")
    ref = a.copy(order="F")
    ro = oracle.lu_la(ref, b_o, b_i)
    assert_parity(mla.to_numpy(d), r.ipiv.ipiv, ref, ro.ipiv, f"lu_streams n={n}")
    d2 = mla.from_numpy(a)
    r2 = mla.lu_la(d2, mla.Policy("lu_mb", mla.BlockConfig(b_o, b_i)))
    assert np.array_equal(r.ipiv.ipiv, r2.ipiv.ipiv)
    assert tuple(r.widths) == tuple(r2.widths) and not r.singular
    d3 = mla.from_numpy(a)
    r3 = lu_streams(d3, b_o, b_i, variant="lu_et")
    ref = a.copy(order="F")
    ro = oracle.lu_la(ref, b_o, b_i, et_sched=et_schedule_from_widths(r3.widths, n, b_o, b_i, b_o), clamp=b_o)
    assert tuple(ro.widths) == tuple(r3.widths) and r3.et_events == ro.et_events == len(r3.et_widths)
    assert_parity(mla.to_numpy(d3), r3.ipiv.ipiv, ref, ro.ipiv, f"lu_streams lu_et n={n}")


@pytest.mark.parametrize("variant", ["lu_mb", "lu_et"])
def test_distributed_driver_full_size_pivots_equal_lu_la(mla, variant):
    """The multi-GPU driver's CUDA path at a size with many row blocks and strips (P = 1, n = 16384,
    b = 512/64), update and look-ahead panel CO-RESIDENT on the device (the mode that corrupted in round 1):
    same pivot sequence as lu_la (whose pivots are pinned to the oracle's golden vectors at this size by the
    full-config tests), twice in a row, and a small backward error."""
    from paper_1611_06365_b200.distributed import DistLU
    n, b_o, b_i = 16384, 512, 64
    a0 = mla.alloc_matrix(n, n)
    mla.fill_random(a0, 2, 2.0, -1.0)
    x = a0.clone()
    want = mla.lu_la(x, mla.Policy("lu_mb", mla.BlockConfig(b_o, b_i))).ipiv.ipiv.copy()
    del x
    for _ in range(2):
        x = a0.clone()
        dlu = DistLU(n, b_o, b_i, None, x.device, variant=variant, rank=0, world=1, storage=x)
        ipiv = dlu.factor()
        assert np.array_equal(ipiv, want)
        chk = a0.clone()
        berr = float(mla.residual_packed(chk, x, mla.PivotVector(ipiv))) / (n * EPS)
        assert berr <= BACKWARD_TOL
        del x, chk, dlu


def test_distributed_driver_config5_single_rank(mla):
    """Config 5 (n = 65536, b = 512/64, device-generated) through the multi-GPU driver's per-GPU step with
    look-ahead + worker sharing + ET, P = 1: pivots identical to the LAPACK fixture, sampled rows / columns
    within 1e-10, backward error <= 10 n eps.  (The >1-GPU layouts of the same driver are covered bitwise
    under gloo in tests/test_distributed_cpu.py and with 2 ranks on this GPU below.)"""
    from paper_1611_06365_b200.distributed import DistLU
    cfg = mla.CONFIGS["config5"]
    n = cfg.n
    dlu = DistLU(n, cfg.b_outer, cfg.b_inner, cfg, "cuda", variant="lu_et", rank=0, world=1)
    dlu.generate()
    ipiv = dlu.factor()
    _check_against_fixture(mla, "config5", dlu.a, ipiv, "DistLU config5 P=1")
    berr = float(mla.residual_packed(dlu.a0, dlu.a, mla.PivotVector(ipiv))) / (n * EPS)   # destroys a0
    assert berr <= BACKWARD_TOL
    assert sum(dlu.widths) == n


def test_device_trace_is_a_valid_reference_trace(mla, tmp_path):  # acceptance 4 (test_acceptance.py:192-218)
    """Per-CTA device trace (every CTA records the phases it ran, MERGED stamped at the actual join):
    structurally valid, round-trips through the reference's JSONL form, and shows worker sharing."""
    from paper_1611_06365_b200 import trace as mtrace
    pool = mla.default_pool()
    a = mla.alloc_matrix(12288, 12288)
    mla.fill_random(a, 0, 2.0, -1.0)
    mtrace.enable(pool)
    try:
        r = mla.lu_la(a, mla.Policy("lu_mb", mla.BlockConfig(256, 32), t_pf=48), pool)
        evs = mtrace.events(pool)
    finally:
        mtrace.enable(pool, False)
    assert evs
    mtrace.validate(evs)
    assert {e.worker for e in evs} == set(range(pool.t))           # every CTA of the grid is a worker
    iters = len(r.widths) - 1
    panel = [e for e in evs if e.team == "PF" and e.task == "PANEL"]
    assert len(panel) == 48 * iters                                  # one record per team member and iteration
    path = str(tmp_path / "trace.jsonl.gz")
    mtrace.write_jsonl(evs, path)
    assert mtrace.load_jsonl(path) == evs
    merged = {e.iter_index for e in evs if e.team == "MERGED"}
    assert merged and r.ws_joins > 0                 # panel SMs joined the update in some iterations
    assert {e.worker for e in evs if e.team == "MERGED"} <= set(range(48))
    idle = mtrace.idle_fraction(evs, worker=0)
    assert all(idle[it] < 0.10 for it in sorted(merged)[:4])   # with merging the panel lead has (almost) no idle gap
    # without worker sharing no CTA ever records a MERGED phase, and tracing off records nothing
    mtrace.enable(pool)
    try:
        mla.fill_random(a, 0, 2.0, -1.0)
        mla.lu_la(a, mla.Policy("lu_la", mla.BlockConfig(256, 32), t_pf=48), pool)
        evs2 = mtrace.events(pool)
    finally:
        mtrace.enable(pool, False)
    mtrace.validate(evs2)
    assert evs2 and not any(e.team == "MERGED" for e in evs2)
    assert mtrace.events(pool) == []


def test_bench_cli_csv(mla, capsys):  # reference test_bench.py: header, seed reproducibility, --check gate
    from paper_1611_06365_b200 import bench_cli
    assert bench_cli.main(["--algo", "lu_et", "--n", "1024", "--b-outer", "128", "--b-inner", "32", "--check",
                           "--seed", "5"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0] == ",".join(bench_cli.CSV_FIELDS)
    row = out[1].split(",")
    assert row[0] == "lu_et" and row[1] == "1024" and float(row[9]) <= 1024 * 100 * EPS
    assert bench_cli.main(["--gepp", "--n", "1024", "--sweep-b", "64:128:64"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0] == "k,gflops" and len(out) == 3


def test_distributed_driver_two_ranks_cuda_ops(mla):
    """The multi-GPU driver end to end with its CUDA operator table and real broadcasts, 2 ranks sharing
    the one GPU of this run (gloo rendezvous; no kernel waits on another rank's kernel).  The script
    asserts pivot equality and the 1e-10 factor bound against the oracle on rank 0."""
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr",
                          "127.0.0.1", "--master-port", str(port), os.path.join(root, "tools", "dev_dist_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("pivots_equal=True") == 3


def test_distributed_driver_nccl_communicator_one_rank(mla):
    """The driver under a real NCCL process group (one rank: the most one GPU allows): every panel broadcast
    goes through torch.distributed/NCCL on the communication stream with the buffer-reuse events, look-ahead
    + WS + ET on; tools/dev_dist_nccl1.py asserts pivots, width replay and the 1e-10 factor bound."""
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "1", "--master-addr",
                          "127.0.0.1", "--master-port", str(port), os.path.join(root, "tools", "dev_dist_nccl1.py")],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("pivots_equal=True") == 3


def test_results_do_not_depend_on_warp_timing(mla):
    """Race hunt without compute-sanitizer (closed on the pool): tools/race_stress.sh runs the same deterministic
    work (lu_mb at three shapes, k_gemm, k_apply_panel, k_panel) under the normal library and under a
    -DMLA_RACE_STRESS build that delays some warps at the points where a missing barrier would bite; the
    results must be bit-identical (and the build without round 2's epilogue barrier must differ).  Needs
    build/lib_stress*.so newer than the sources (`tools/race_stress.sh build`); skipped otherwise."""
    import glob
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libs = [os.path.join(root, "build", n) for n in ("lib_stress.so", "lib_stress_nofix.so")]
    srcs = glob.glob(os.path.join(root, "paper_1611_06365_b200", "csrc", "*"))
    if not all(os.path.exists(l) for l in libs) or min(os.path.getmtime(l) for l in libs) < max(os.path.getmtime(f) for f in srcs):
        pytest.skip("stress libraries missing or older than the sources")
    out = subprocess.run(["bash", os.path.join(root, "tools", "race_stress.sh")], capture_output=True, text=True,
                         timeout=900, cwd=root)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "OK: no result depends on warp timing" in out.stdout
    assert "the pre-fix epilogue is detected" in out.stdout


def test_random_small_shapes_property(mla):
    """Property sweep in the spirit of the reference's hypothesis tests (test_lu.py:247-256,
    test_kernels.py:366-401): random small m >= n, block widths and variants; pivots identical to the
    oracle, factors within the parity bound, backward error bounded."""
    rng = np.random.default_rng(2024)
    for trial in range(60):
        n = int(rng.integers(1, 41))
        m = n + int(rng.integers(0, 25))
        b_i = int(rng.integers(1, 9))
        b_o = b_i * int(rng.integers(1, 5))
        variant = VARIANTS[int(rng.integers(0, len(VARIANTS)))]
        a = np.asfortranarray(rng.standard_normal((m, n)))
        if trial % 7 == 0 and n > 2:
            a[:, int(rng.integers(0, n))] = 0.0          # a structurally singular column now and then
        if trial % 5 == 0 and n > 3:
            a[int(rng.integers(0, m)), :] *= 1e6          # badly scaled row
        run_and_check(mla, a, b_o, b_i, variant, t_pf=int(rng.integers(1, 40)),
                      what=f"trial {trial}: {m}x{n} b={b_o}/{b_i} {variant}")


def test_operator_property_sweep(mla):
    """Random laswp round trips / involutions and trsm-multiply-back on odd shapes and views."""
    rng = np.random.default_rng(7)
    for trial in range(25):
        rows, cols = int(rng.integers(1, 300)), int(rng.integers(1, 70))
        npiv = int(rng.integers(1, rows + 1))
        parent = mla.alloc_matrix(rows + 5, cols + 3)
        a = np.asfortranarray(rng.standard_normal((rows, cols)))
        view = parent[2:2 + rows, 1:1 + cols]
        view.copy_(mla.from_numpy(a))
        ipiv = np.array([rng.integers(t, rows) for t in range(npiv)], dtype=np.int64)
        mla.laswp(view, ipiv)
        ref = a.copy(order="F")
        oracle.laswp(ref, ipiv)
        assert np.array_equal(mla.to_numpy(parent)[2:2 + rows, 1:1 + cols], ref)
        mla.laswp(view, ipiv, reverse=True)
        assert np.array_equal(mla.to_numpy(parent)[2:2 + rows, 1:1 + cols], a)
        w, c = int(rng.integers(1, 150)), int(rng.integers(1, 200))
        low = np.asfortranarray(rng.uniform(-1, 1, (w, w)))
        x = np.asfortranarray(rng.standard_normal((w, c)))
        dx = mla.from_numpy(x)
        mla.trsm_llu(mla.from_numpy(low), dx)
        back = (np.tril(low, -1) + np.eye(w)) @ mla.to_numpy(dx)
        assert np.abs(back - x).max() <= 64 * w * EPS * max(1.0, np.abs(mla.to_numpy(dx)).max())
