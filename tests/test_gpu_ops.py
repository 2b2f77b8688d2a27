"""GPU parity tests of the operators (gemm / trsm / laswp / panel) through the C ABI, against the
CPU oracle and the reference's golden vectors.  Mirrors pkg/tests/test_kernels.py and the panel
part of pkg/tests/test_lu.py (line numbers cited per test)."""
import numpy as np
import pytest

import cases
import oracle
from parity import assert_parity, lu_error

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EPS = float(np.finfo(np.float64).eps)


@pytest.fixture(scope="module")
def mla():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1611_06365_b200 as m
    return m


def gen(m, n, seed):
    return cases.uniform_pm1(oracle.fill_random, m, n, seed)


# ---- fill_random -------------------------------------------------------------------------------

def test_fill_random_bitwise(mla, golden):  # matrix.py:44-63, test_matrix.py:81-113
    a = mla.alloc_matrix(7, 5, ld=9)
    mla.fill_random(a, 3)
    assert np.array_equal(mla.to_numpy(a), golden["fill_7x5_seed3"])
    b = mla.alloc_matrix(100, 37, ld=104)
    mla.fill_random(b, 12345, 2.0, -1.0)
    assert np.array_equal(mla.to_numpy(b), gen(100, 37, 12345))
    # column block of a larger matrix (multi-GPU layout)
    c = mla.alloc_matrix(100, 8)
    mla.fill_random(c, 12345, 2.0, -1.0, col0=16, total_rows=100)
    assert np.array_equal(mla.to_numpy(c), gen(100, 37, 12345)[:, 16:24])


# ---- gemm ---------------------------------------------------------------------------------------

GEMM_SHAPES = [(1, 1, 1), (7, 5, 3), (37, 29, 21), (128, 128, 32), (130, 70, 300), (517, 333, 129),
               (256, 384, 64), (1000, 999, 257), (700, 600, 24), (900, 800, 40), (2048, 2048, 64),
               (3000, 2900, 33)]


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
def test_gemm_vs_oracle(mla, m, n, k):  # test_kernels.py:184-226, tol 4 k eps max|A| max|B|
    a, b, c = gen(m, k, 1), gen(k, n, 2), gen(m, n, 3)
    ref = c.copy(order="F")
    oracle.gemm(ref, a, b, 1.0, -1.0)
    dc = mla.from_numpy(c)
    mla.gemm_malleable(dc, mla.from_numpy(a), mla.from_numpy(b), 1.0, -1.0)
    tol = 4 * k * EPS * np.abs(a).max() * np.abs(b).max()
    assert np.abs(mla.to_numpy(dc) - ref).max() <= tol


@pytest.mark.parametrize("c", cases.GEMM, ids=lambda c: c["name"])
def test_gemm_golden_alpha_beta(mla, golden, c):  # test_kernels.py:205-215
    a, b, cc = gen(c["m"], c["k"], c["seed"]), gen(c["k"], c["n"], c["seed"] + 100), gen(c["m"], c["n"], c["seed"] + 200)
    dc = mla.from_numpy(cc)
    mla.gemm_malleable(dc, mla.from_numpy(a), mla.from_numpy(b), c["alpha"], c["beta"])
    tol = 4 * c["k"] * EPS * max(abs(c["beta"]), 1.0) + 4 * EPS
    assert np.abs(mla.to_numpy(dc) - golden[c["name"] + "/c"]).max() <= tol


def test_gemm_views_and_canary(mla):  # test_kernels.py:229-247: no out-of-view writes, odd offsets
    big = mla.alloc_matrix(300, 260)
    big.fill_(7.0)
    a, b = gen(101, 33, 4), gen(33, 57, 5)
    cv = big[13:114, 9:66]
    cv.copy_(torch.zeros_like(cv))
    mla.gemm_malleable(cv, mla.from_numpy(a), mla.from_numpy(b), 1.0, 1.0)
    ref = np.zeros((101, 57), order="F")
    oracle.gemm(ref, a, b, 1.0, 1.0)
    host = mla.to_numpy(big)
    assert np.abs(host[13:114, 9:66] - ref).max() <= 4 * 33 * EPS
    host[13:114, 9:66] = 7.0
    assert np.all(host == 7.0)


def test_gemm_edge_cases(mla):  # kernels.py:217-232
    c = mla.from_numpy(gen(5, 4, 1))
    with pytest.raises(ValueError):
        mla.gemm_malleable(c, mla.alloc_matrix(5, 3), mla.alloc_matrix(2, 4))
    mla.gemm_malleable(mla.alloc_matrix(0, 4), mla.alloc_matrix(0, 3), mla.alloc_matrix(3, 4))  # empty: no-op
    before = mla.to_numpy(c)
    mla.gemm_malleable(c, mla.alloc_matrix(5, 0), mla.alloc_matrix(0, 4), 0.5, 1.0)  # k == 0 scales
    assert np.array_equal(mla.to_numpy(c), 0.5 * before)


def test_gemm_worker_sharing_flag(mla):  # checkpoint_merge semantics, pool.py:377-414
    m, n, k = 1500, 1400, 128
    a, b, c = gen(m, k, 1), gen(k, n, 2), gen(m, n, 3)
    ref = mla.from_numpy(c)
    mla.gemm_malleable(ref, mla.from_numpy(a), mla.from_numpy(b), 1.0, -1.0)
    for preset in (True, False):   # donors join at once / never join: same bits either way
        flag = mla.CompletionFlag("PF")
        if preset:
            mla.signal_complete(flag)
        dc = mla.from_numpy(c)
        mla.gemm_malleable(dc, mla.from_numpy(a), mla.from_numpy(b), 1.0, -1.0, flag=flag, donor_sms=40)
        assert torch.equal(dc, ref)


# ---- trsm ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("w,c", [(1, 3), (2, 1), (24, 17), (32, 128), (100, 300), (256, 1000), (512, 130), (768, 40)])
def test_trsm_vs_oracle(mla, w, c):  # test_kernels.py:270-319: multiply-back bound 8*64*eps scaled
    low, x = gen(w, w, 41), gen(w, c, 141)
    ref = x.copy(order="F")
    oracle.trsm_llu(low, ref)
    dx = mla.from_numpy(x)
    mla.trsm_llu(mla.from_numpy(low), dx)
    err, _ = lu_error(mla.to_numpy(dx), ref)
    assert err <= 1e-10


def test_trsm_kat_and_errors(mla, golden):  # test_kernels.py:279-283, test_oracle.py:29-36
    low = mla.from_numpy(np.array([[9.0, 0.0], [2.0, 9.0]]))
    x = mla.from_numpy(np.array([[1.0], [5.0]]))
    mla.trsm_llu(low, x)
    assert np.array_equal(mla.to_numpy(x), [[1.0], [3.0]])
    c = cases.TRSM[0]
    dx = mla.from_numpy(gen(c["w"], c["c"], c["seed"] + 100))
    mla.trsm_llu(mla.from_numpy(gen(c["w"], c["w"], c["seed"])), dx)
    assert np.abs(mla.to_numpy(dx) - golden[c["name"] + "/x"]).max() <= 1e-12
    with pytest.raises(ValueError):
        mla.trsm_llu(mla.alloc_matrix(3, 2), mla.alloc_matrix(3, 1))
    with pytest.raises(ValueError):
        mla.trsm_llu(mla.alloc_matrix(3, 3), mla.alloc_matrix(2, 1))


# ---- laswp --------------------------------------------------------------------------------------

@pytest.mark.parametrize("rows,cols,npiv", [(30, 9, 10), (500, 300, 64), (4096, 1000, 256), (2000, 77, 1),
                                            (3000, 50, 768), (5000, 33, 1500)])
def test_laswp_bitwise_and_roundtrip(mla, rows, cols, npiv):  # test_kernels.py:322-344
    rng = np.random.default_rng(rows + npiv)
    a = np.asfortranarray(rng.standard_normal((rows, cols)))
    ipiv = np.array([rng.integers(t, rows) for t in range(npiv)], dtype=np.int64)
    d = mla.from_numpy(a)
    mla.laswp(d, ipiv)
    ref = a.copy(order="F")
    oracle.laswp(ref, ipiv)
    assert np.array_equal(mla.to_numpy(d), ref)
    mla.laswp(d, mla.PivotVector(ipiv), reverse=True)
    assert np.array_equal(mla.to_numpy(d), a)


def test_laswp_golden_and_validation(mla, golden):  # test_kernels.py:329-332, 346-352
    c = cases.LASWP[0]
    d = mla.from_numpy(gen(c["rows"], c["cols"], c["seed"]))
    mla.laswp(d, c["ipiv"])
    assert np.array_equal(mla.to_numpy(d), golden[c["name"] + "/fwd"])
    mla.laswp(d, c["ipiv"], reverse=True)
    assert np.array_equal(mla.to_numpy(d), golden[c["name"] + "/back"])
    a = mla.from_numpy(np.arange(12.0).reshape(4, 3))
    mla.laswp(a, [2])
    h = mla.to_numpy(a)
    assert np.array_equal(h[0], [6.0, 7.0, 8.0]) and np.array_equal(h[2], [0.0, 1.0, 2.0])
    with pytest.raises(IndexError):
        mla.laswp(a, [1, 4])          # validated before anything is touched
    assert np.array_equal(mla.to_numpy(a), h)
    mla.laswp(a, [])                  # empty pivot list: no-op
    mla.laswp(mla.alloc_matrix(5, 0), [1, 2])  # no columns: no-op


def test_laswp_long_pivot_vectors_any_in_range_index(mla):
    """More pivots than one device plan holds (1024): applied chunk by chunk inside the library.  The
    reference's laswp accepts ANY index in [0, rows), also ipiv[t] < t (kernels.py:316-327) -- the chunks
    must too -- and a bad index anywhere, including the last chunk, leaves the matrix untouched."""
    rng = np.random.default_rng(99)
    for rows, cols, npiv in [(3000, 40, 2500), (2100, 17, 2100), (1500, 9, 1025)]:
        a = np.asfortranarray(rng.standard_normal((rows, cols)))
        ipiv = rng.integers(0, rows, size=npiv).astype(np.int64)      # unconstrained: above and below t
        d = mla.from_numpy(a)
        mla.laswp(d, ipiv)
        ref = a.copy(order="F")
        oracle.laswp(ref, ipiv)
        assert np.array_equal(mla.to_numpy(d), ref)
        mla.laswp(d, ipiv, reverse=True)
        assert np.array_equal(mla.to_numpy(d), a)
        bad = ipiv.copy()
        bad[-1] = rows                                                 # out of range in the LAST chunk
        with pytest.raises(IndexError):
            mla.laswp(d, bad)
        assert np.array_equal(mla.to_numpy(d), a)                      # nothing was touched
    # small vectors with indices above their position as well
    a = np.asfortranarray(rng.standard_normal((50, 7)))
    ipiv = np.array([49, 0, 1, 0, 48, 2], dtype=np.int64)
    d = mla.from_numpy(a)
    mla.laswp(d, ipiv)
    ref = a.copy(order="F")
    oracle.laswp(ref, ipiv)
    assert np.array_equal(mla.to_numpy(d), ref)


def test_caller_supplied_ipiv_is_written_in_place(mla):
    """lu_unb / lu_blk_ll / lu_blk_rl honour a caller's pivot array like the reference (lu.py:82-90,
    97-103, 123-137): 1-d int64 of length >= n, else ValueError; filled in place."""
    a = gen(90, 60, 5)
    for fn, kw in ((mla.lu_unb, {}), (lambda x, **k: mla.lu_blk_ll(x, 16, **k), {}),
                   (lambda x, **k: mla.lu_blk_rl(x, 16, **k), {})):
        mine = np.full(64, -7, dtype=np.int64)
        r = fn(mla.from_numpy(a), ipiv=mine)
        assert np.array_equal(mine[:60], r.ipiv.ipiv) and np.all(mine[60:] == -7)
        dev = torch.full((60,), -7, dtype=torch.int64, device="cuda")
        r2 = fn(mla.from_numpy(a), ipiv=dev)
        assert np.array_equal(dev.cpu().numpy(), r2.ipiv.ipiv) and np.array_equal(r2.ipiv.ipiv, r.ipiv.ipiv)
        for wrong in (np.zeros(59, dtype=np.int64), np.zeros(60, dtype=np.int32), np.zeros((60, 1), dtype=np.int64),
                      torch.zeros(60, dtype=torch.int32)):
            with pytest.raises(ValueError):
                fn(mla.from_numpy(a), ipiv=wrong)


# ---- panel (lu_unb / lu_blk_ll) -------------------------------------------------------------------

def test_panel_kats(mla):  # test_lu.py:29-57
    a = mla.from_numpy(np.array([[3.0]]))
    r = mla.lu_unb(a)
    assert list(r.ipiv.ipiv) == [0] and mla.to_numpy(a)[0, 0] == 3.0
    a = mla.from_numpy(np.array([[0.0, 1.0], [1.0, 0.0]]))
    r = mla.lu_unb(a)
    assert list(r.ipiv.ipiv) == [1, 1] and not r.singular
    assert np.array_equal(mla.to_numpy(a), [[1.0, 0.0], [0.0, 1.0]])
    a = mla.from_numpy(np.array([[0.0, 2.0], [0.0, 3.0]]))
    r = mla.lu_unb(a)
    assert r.singular and list(r.ipiv.ipiv) == [0, 1]
    assert np.array_equal(mla.to_numpy(a)[:, 0], [0.0, 0.0])
    with pytest.raises(ValueError):
        mla.lu_unb(mla.alloc_matrix(2, 3))
    r = mla.lu_blk_ll(mla.alloc_matrix(0, 0), 4)
    assert len(r.ipiv) == 0 and r.cols_factored == 0


@pytest.mark.parametrize("c", cases.UNB + [x for x in cases.LL if x["stop_trip"] == 0], ids=lambda c: c["name"])
def test_panel_golden(mla, golden, c):
    a = gen(c["m"], c["n"], c["seed"])
    d = mla.from_numpy(a)
    r = mla.lu_blk_ll(d, c.get("b", c["n"]), team_sms=3)
    assert_parity(mla.to_numpy(d), r.ipiv.ipiv, golden[c["name"] + "/lu"], golden[c["name"] + "/ipiv"], c["name"])


@pytest.mark.parametrize("m,w,b,team", [(64, 48, 8, 1), (200, 96, 32, 3), (2048, 256, 32, 16), (5000, 256, 32, 8),
                                        (40000, 128, 32, 16), (1000, 192, 64, 148), (3000, 96, 96, 7), (777, 130, 16, 5),
                                        # slab fitting: 2000 rows per CTA -> 8-column device blocks; 1000 -> 16
                                        (4000, 64, 32, 2), (16000, 128, 64, 16)])
def test_panel_vs_oracle(mla, m, w, b, team):  # test_lu.py:121-129 (same pivots), any team size
    a = gen(m, w, 5)
    d = mla.from_numpy(a)
    r = mla.lu_blk_ll(d, b, team_sms=team)
    ref = a.copy(order="F")
    ro = oracle.lu_blk_ll(ref, b)
    assert r.cols_factored == w
    assert_parity(mla.to_numpy(d), r.ipiv.ipiv, ref, ro.ipiv, f"panel {m}x{w} b={b} team={team}")


def test_panel_et_cut_semantics(mla, golden):  # test_lu.py:132-170
    a = gen(128, 128, 3)
    d = mla.from_numpy(a)
    r = mla.lu_blk_ll(d, 32, stop=mla.CountingStop(1), team_sms=4)   # pre-set flag
    assert r.cols_factored == 32 and len(r.ipiv) == 32
    ref = a.copy(order="F")
    oracle.laswp(ref[:, 32:], r.ipiv.ipiv)
    assert np.array_equal(mla.to_numpy(d)[:, 32:], ref[:, 32:])       # right columns carry exactly the swaps
    d = mla.from_numpy(a)
    assert mla.lu_blk_ll(d, 32, stop=mla.CountingStop(3), team_sms=4).cols_factored == 96  # polled once per block
    d = mla.from_numpy(gen(64, 32, 3))
    assert mla.lu_blk_ll(d, 32, stop=mla.CountingStop(1)).cols_factored == 32             # single block never cut
    flag = mla.CompletionFlag("RU")
    mla.signal_complete(flag)
    d = mla.from_numpy(a)
    assert mla.lu_blk_ll(d, 32, stop=flag, team_sms=4).cols_factored == 32                # device flag
    for c in (x for x in cases.LL if x["stop_trip"] > 0):
        d = mla.from_numpy(gen(c["m"], c["n"], c["seed"]))
        r = mla.lu_blk_ll(d, c["b"], stop=mla.CountingStop(c["stop_trip"]), team_sms=2)
        assert r.cols_factored == int(golden[c["name"] + "/cols"][0])
        assert_parity(mla.to_numpy(d), r.ipiv.ipiv, golden[c["name"] + "/lu"], golden[c["name"] + "/ipiv"], c["name"])


def test_panel_team_size_independent_pivots(mla):  # test_kernels.py:250-267 analogue
    a = gen(1500, 128, 9)
    out = []
    for team in (1, 2, 5, 16):
        d = mla.from_numpy(a)
        out.append(mla.lu_blk_ll(d, 32, team_sms=team).ipiv.ipiv)
    assert all(np.array_equal(out[0], o) for o in out[1:])


def test_blk_rl_matches_ll_pivots(mla, golden):  # test_lu.py:85-91, 121-129
    for c in cases.RL:
        a = gen(c["m"], c["n"], c["seed"])
        d = mla.from_numpy(a)
        r = mla.lu_blk_rl(d, c["b"], inner_b=c["inner_b"])
        assert_parity(mla.to_numpy(d), r.ipiv.ipiv, golden[c["name"] + "/lu"], golden[c["name"] + "/ipiv"], c["name"])


@pytest.mark.parametrize("rows,w,cols", [(700, 128, 300), (2048, 256, 1000), (333, 32, 77), (1500, 64, 129)])
def test_apply_panel_equals_operator_chain(mla, rows, w, cols):
    """The fused multi-GPU update step (one persistent launch) is bit-identical to the reference's
    operator chain laswp -> trsm_llu -> gemm_malleable (lu.py:251-253, 280-281) run through the
    stand-alone operators, and agrees with the oracle."""
    from paper_1611_06365_b200.kernels import apply_panel
    rng = np.random.default_rng(rows + w)
    panel = np.asfortranarray(rng.uniform(-1, 1, (rows, w)))
    tgt = np.asfortranarray(rng.standard_normal((rows, cols)))
    ipiv = np.array([rng.integers(t, rows) for t in range(w)], dtype=np.int64)
    dp = mla.from_numpy(panel)
    a = mla.from_numpy(tgt)
    apply_panel(dp, w, a, ipiv)
    b = mla.from_numpy(tgt)
    mla.laswp(b, ipiv)
    mla.trsm_llu(dp[:w, :w], b[:w, :])
    mla.gemm_malleable(b[w:, :], dp[w:, :w], b[:w, :], 1.0, -1.0)
    assert torch.equal(a, b)
    ref = tgt.copy(order="F")
    oracle.laswp(ref, ipiv)
    oracle.trsm_llu(panel[:w, :w], ref[:w, :])
    oracle.gemm(ref[w:, :], panel[w:, :w], ref[:w, :], 1.0, -1.0)
    err, _ = lu_error(mla.to_numpy(a), ref)
    assert err <= 1e-10


def test_apply_panel_second_launch_joins_the_queue(mla):
    """Worker sharing across kernels (distributed driver): one update step prepared once, drained by a
    launch on 100 SMs and a second launch on 40 SMs of another stream that joins the same queue; the
    result is bitwise that of the single launch (one owner per tile either way)."""
    from paper_1611_06365_b200.kernels import apply_panel, apply_panel_launch, apply_panel_prepare
    rows, w, cols = 6000, 256, 5000
    rng = np.random.default_rng(7)
    panel = np.asfortranarray(rng.uniform(-1, 1, (rows, w)))
    tgt = np.asfortranarray(rng.standard_normal((rows, cols)))
    ipiv = np.array([rng.integers(t, rows) for t in range(w)], dtype=np.int64)
    dp = mla.from_numpy(panel)
    want = mla.from_numpy(tgt)
    apply_panel(dp, w, want, ipiv)
    got = mla.from_numpy(tgt)
    piv_dev = torch.as_tensor(ipiv, dtype=torch.int32, device=got.device)
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    apply_panel_prepare(dp, piv_dev, w)
    ready = torch.cuda.Event()
    ready.record(main)
    apply_panel_launch(dp, w, got, 100)
    with torch.cuda.stream(side):
        side.wait_event(ready)
        apply_panel_launch(dp, w, got, 40)
    main.wait_stream(side)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
