"""Blocked LU factorizations with partial pivoting and the look-ahead driver -- the reference's
lu.py:33-334 entry points over CUDA tensors.

Factors overwrite the input: unit-lower L strictly below the diagonal, U on and above; pivots are
view-local with ipiv[k] >= k, ties go to the lowest row, an exactly-zero pivot column is recorded
and skipped (singular flag).  All arithmetic happens in libmla_b200.so (include/mla_b200.h).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .config import Policy
from .kernels import gemm_malleable, laswp, trsm_llu
from .matrix import PivotVector, _stream, check_colmajor
from .pool import CompletionFlag, SmPool, default_pool


@dataclass
class LuResult:
    """Outcome of a factorization; the factors live in the input matrix (reference lu.py:33-41).
    `widths` (extension) lists every panel's factored width in order, which makes an ET run
    replayable on the CPU oracle; `ws_joins` counts iterations in which panel SMs joined the update;
    `t_pf_peak` is the largest panel team an adaptive split (pool.t_pf_max) used."""

    ipiv: PivotVector
    cols_factored: int
    singular: bool = False
    et_events: int = 0
    et_widths: tuple = ()
    widths: tuple = ()
    ws_joins: int = 0
    t_pf_peak: int = 0


def _check_tall(a: torch.Tensor) -> tuple[int, int, int]:
    m, n, ld = check_colmajor(a, "a")
    if m < n:
        raise ValueError(f"need m >= n, got {m} x {n}")
    return m, n, ld


def _caller_ipiv(ipiv, n: int):
    """Validate a caller-supplied pivot array like the reference's _shared_ipiv (lu.py:82-90): it must be
    a 1-d int64 array of length >= n (numpy, or a torch tensor on the host or the device); the pivots are
    written into its first n entries in place.  Returns a writer callback (or None)."""
    if ipiv is None:
        return None
    if isinstance(ipiv, torch.Tensor):
        if ipiv.dtype != torch.int64 or ipiv.dim() != 1 or ipiv.shape[0] < n:
            raise ValueError("ipiv must be a 1-d int64 array of length >= n")
        return lambda host, dev=None: ipiv[:host.shape[0]].copy_(
            dev.to(torch.int64) if (dev is not None and ipiv.is_cuda) else torch.from_numpy(host))
    arr = ipiv if isinstance(ipiv, np.ndarray) else np.asarray(ipiv)
    if arr.dtype != np.int64 or arr.ndim != 1 or arr.shape[0] < n:
        raise ValueError("ipiv must be a 1-d int64 array of length >= n")
    # (anything that is not already an ndarray was converted to a private copy, exactly as
    # np.asarray does in the reference: it validates, but the caller does not see the result)

    def write(host, dev=None):
        arr[:host.shape[0]] = host
    return write


class CountingStop:
    """Deterministic ET injection: behaves like a flag that is set from poll number `trip` on --
    the reference tests' CountingFlag fake (test_lu.py:149-156); trip=1 is a pre-set flag."""

    def __init__(self, trip: int) -> None:
        self.trip = int(trip)


def lu_blk_ll(a: torch.Tensor, b: int, ipiv=None, stop=None, team=None, cfg=None,
              pool: SmPool | None = None, team_sms: int | None = None) -> LuResult:
    """Left-looking blocked panel LU, optionally stoppable between block steps (lu.py:140-180).

    `stop` may be a CompletionFlag (device word polled once per finished inner block) or a
    CountingStop.  Pivots are panel-local.
    """
    m, n, ld = _check_tall(a)
    if b < 1:
        raise ValueError("block size must be >= 1")
    put = _caller_ipiv(ipiv, n)
    pool = pool or default_pool(a.device.index)
    if n == 0:
        return LuResult(PivotVector(np.empty(0, dtype=np.int64)), 0, False)
    dev_piv = torch.empty(n, dtype=torch.int32, device=a.device)
    info = _capi.LuInfo()
    flag_ptr, trip = 0, 0
    if isinstance(stop, CompletionFlag):
        flag_ptr = stop.ptr
    elif isinstance(stop, CountingStop):
        trip = stop.trip
    elif stop is not None:
        raise ValueError("stop must be a CompletionFlag or CountingStop")
    _capi.check(_capi.lib().mla_panel_ll(pool.handle, a.data_ptr(), m, n, ld, dev_piv.data_ptr(), int(b),
                                         flag_ptr, trip, int(team_sms or 0), ctypes.byref(info),
                                         _stream(a)), pool.handle, "lu_blk_ll")
    cols = int(info.cols_factored)
    host_piv = dev_piv[:cols].cpu().numpy().astype(np.int64)
    if put is not None:
        put(host_piv, dev_piv[:cols])        # in place, like the reference (lu.py:160, 175)
    return LuResult(PivotVector(host_piv, device=dev_piv[:cols]), cols,
                    bool(info.singular), int(info.et_events),
                    (cols,) if cols < n else ())


def lu_unb(a: torch.Tensor, ipiv=None, pool: SmPool | None = None) -> LuResult:
    """Unblocked pivoted LU (lu.py:97-103): the panel kernel with one block spanning the width
    (the device factors it in steps of at most 128 columns, which changes no pivot rule)."""
    m, n, _ = _check_tall(a)
    return lu_blk_ll(a, max(n, 1), ipiv=ipiv, pool=pool)


def lu_blk_ll_async(a: torch.Tensor, b: int, pool: SmPool, team_sms: int = 0,
                    singular_accum: torch.Tensor | None = None, stop: tuple[int, int] | None = None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """Stream-ordered lu_blk_ll for drivers that never look at the result on the host: returns the
    panel-local pivots as a device int32 tensor (`out` if given); `singular_accum` (device int32[1]) is
    OR-ed with the singular flag; `stop` = (device address of a flag word, tag) is the ET flag of
    lu.py:177-179 -- the panel is cut after a finished inner block once the word equals the tag.  The
    factored width stays on the device (pool handle's info record; kernels.pack_panel reads it)."""
    m, n, ld = _check_tall(a)
    if b < 1:
        raise ValueError("block size must be >= 1")
    dev_piv = out if out is not None else torch.empty(n, dtype=torch.int32, device=a.device)
    if n == 0:
        return dev_piv
    acc = 0 if singular_accum is None else singular_accum.data_ptr()
    flag_ptr, tag = (0, 0) if stop is None else (int(stop[0]), int(stop[1]))
    _capi.check(_capi.lib().mla_panel_ll_async(pool.handle, a.data_ptr(), m, n, ld, dev_piv.data_ptr(), int(b),
                                               int(team_sms), acc, flag_ptr, tag, _stream(a)), pool.handle,
                "lu_blk_ll_async")
    return dev_piv


def lu_blk_rl(a: torch.Tensor, b: int, ipiv=None, team=None, cfg=None, inner_b: int | None = None,
              pool: SmPool | None = None) -> LuResult:
    """Right-looking blocked LU (lu.py:106-137): panel, pivots left and right, trsm, gemm --
    composed from the device operators, one panel at a time."""
    m, n, _ = _check_tall(a)
    if b < 1:
        raise ValueError("block size must be >= 1")
    put = _caller_ipiv(ipiv, n)
    pool = pool or default_pool(a.device.index)
    ipiv_all = np.empty(n, dtype=np.int64)
    singular = False
    for j in range(0, n, b):
        w = min(b, n - j)
        panel = a[j:m, j:j + w]
        sub = lu_blk_ll(panel, inner_b if (inner_b is not None and inner_b < w) else w, pool=pool)
        singular = singular or sub.singular
        laswp(a[j:m, :j], sub.ipiv, pool=pool)
        laswp(a[j:m, j + w:n], sub.ipiv, pool=pool)
        ipiv_all[j:j + w] = sub.ipiv.ipiv + j
        trsm_llu(a[j:j + w, j:j + w], a[j:j + w, j + w:n], pool=pool)
        gemm_malleable(a[j + w:m, j + w:n], a[j + w:m, j:j + w], a[j:j + w, j + w:n], 1.0, -1.0, pool=pool)
    if put is not None:
        put(ipiv_all)                          # global pivots, in place (lu.py:123-137)
    return LuResult(PivotVector(ipiv_all), n, singular)


def lu_la(a: torch.Tensor, policy: Policy, pool: SmPool | None = None, cfg=None) -> LuResult:
    """Factor A in place under the given policy (lu.py:197-334): one persistent kernel launch.

    policy.t_pf is the number of SMs given to the panel team (default: pool.t_pf); the reference's
    constraint 1 <= t_pf < t holds with t = SM count (lu.py:210-214).
    """
    m, n, ld = _check_tall(a)
    pool = pool or default_pool(a.device.index)
    variant = policy.variant
    b_o, b_i = policy.b.b_outer, policy.b.b_inner
    t_pf = pool.t_pf if policy.t_pf is None else policy.t_pf
    if variant != "lu":
        if pool.t < 2 or not 1 <= t_pf < pool.t:
            raise ValueError(f"policy/pool mismatch: {variant} needs 1 <= t_pf < t, "
                             f"got t_pf={t_pf}, t={pool.t}")
    if n == 0:
        return LuResult(PivotVector(np.empty(0, dtype=np.int64)), 0, False)
    dev_piv = torch.empty(n, dtype=torch.int32, device=a.device)
    cap = n // b_i + 4
    widths = (ctypes.c_int32 * cap)()
    info = _capi.LuInfo()
    _capi.check(_capi.lib().mla_getrf_la_sync(pool.handle, a.data_ptr(), m, n, ld, dev_piv.data_ptr(),
                                              b_o, b_i, _capi.VARIANT_CODES[variant], int(t_pf),
                                              int(policy.q), ctypes.byref(info), widths, cap,
                                              _stream(a)), pool.handle, "lu_la")
    w = tuple(int(x) for x in widths[:min(cap, int(info.n_panels))])
    return LuResult(PivotVector(dev_piv.cpu().numpy(), device=dev_piv), n, bool(info.singular),
                    int(info.et_events), et_widths_from(w, n, b_o, b_i), w, int(info.ws_joins),
                    int(info.sm_pf_peak))


def et_widths_from(widths, n: int, b_o: int, b_i: int) -> tuple:
    """The cut widths among `widths` (reference et_widths), replaying lu.py:318-323."""
    out = []
    if not widths:
        return ()
    b_target, q1 = b_o, widths[0]
    for k_new in widths[1:]:
        w = min(b_target, n - q1)
        if k_new < w:
            out.append(k_new)
            b_target = max(b_i, k_new)
        else:
            b_target = min(b_o, 2 * b_target)
        q1 += k_new
    return tuple(out)


def et_schedule_from(widths, n: int, b_o: int, b_i: int) -> list[int]:
    """Per-iteration 'trip poll' list that makes the CPU oracle replay an ET run: entry it-1 is the
    number of inner blocks after which iteration it's panel was cut (0 = not cut)."""
    out = []
    if not widths:
        return out
    b_target, q1 = b_o, widths[0]
    for k_new in widths[1:]:
        w = min(b_target, n - q1)
        if k_new < w:
            out.append(k_new // b_i)
            b_target = max(b_i, k_new)
        else:
            out.append(0)
            b_target = min(b_o, 2 * b_target)
        q1 += k_new
    return out
