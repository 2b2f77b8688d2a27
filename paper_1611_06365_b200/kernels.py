"""trsm / gemm / row-swap operators of the reference (kernels.py:205-332) over CUDA tensors.

Same names, argument meaning and error behaviour; `team` (a thread team in the reference) is
accepted and ignored -- the kernels are collective over CTAs internally -- and `cfg` (CPU cache
blocking) likewise.  Every call goes through the C ABI in include/mla_b200.h; nothing here computes
on the host.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _capi
from .matrix import PivotVector, _stream, check_colmajor
from .pool import CompletionFlag, default_pool

MAX_PIVOT_BLOCK = 1024  # kMaxPiv in csrc/mla_laswp.cuh


def gemm_malleable(c: torch.Tensor, a: torch.Tensor, b: torch.Tensor, alpha: float = 1.0,
                   beta: float = 1.0, cfg=None, team=None, flag: CompletionFlag | None = None,
                   pool=None, donor_sms: int | None = None) -> None:
    """c := alpha*c + beta*(a @ b) on the FP64 tensor cores (reference kernels.py:205-234).

    `flag`: the reference's worker-sharing entry point.  With a CompletionFlag, `donor_sms` CTAs of
    the persistent grid (default: the pool's t_pf) stay out of the tile queue until the flag is set
    and join it at the next tile boundary.
    """
    m, n, ldc = check_colmajor(c, "c")
    ma, k, lda = check_colmajor(a, "a")
    kb, nb, ldb = check_colmajor(b, "b")
    if ma != m or kb != k or nb != n:
        raise ValueError(f"gemm shapes disagree: c {tuple(c.shape)}, a {tuple(a.shape)}, b {tuple(b.shape)}")
    pool = pool or default_pool(c.device.index)
    fptr, donors = 0, 0
    if flag is not None:
        fptr = flag.ptr
        donors = pool.t_pf if donor_sms is None else int(donor_sms)
    _capi.check(_capi.lib().mla_gemm(pool.handle, c.data_ptr(), m, n, ldc, a.data_ptr(), lda,
                                     b.data_ptr(), ldb, k, float(alpha), float(beta), fptr, donors,
                                     _stream(c)), pool.handle, "gemm_malleable")


def trsm_llu(a11: torch.Tensor, b: torch.Tensor, team=None, pool=None) -> None:
    """Solve trilu(a11) @ x = b in place; unit lower triangle (reference kernels.py:275-293)."""
    nb, nb2, ldl = check_colmajor(a11, "a11")
    if nb != nb2:
        raise ValueError("triangular factor must be square")
    rows, cols, ldb = check_colmajor(b, "b")
    if rows != nb:
        raise ValueError("right-hand side rows disagree with the factor")
    pool = pool or default_pool(b.device.index)
    _capi.check(_capi.lib().mla_trsm_llu(pool.handle, a11.data_ptr(), nb, ldl, b.data_ptr(), cols, ldb,
                                         _stream(b)), pool.handle, "trsm_llu")


def _device_pivots(piv, device) -> torch.Tensor:
    if isinstance(piv, PivotVector):
        return piv.on_device(device)
    if isinstance(piv, torch.Tensor):
        return piv.to(device=device, dtype=torch.int32).contiguous()
    arr = np.asarray(piv, dtype=np.int64)
    if arr.size and (arr.min() < -2 ** 31 or arr.max() >= 2 ** 31):
        raise IndexError("pivot index out of range for this view")
    return torch.from_numpy(arr.astype(np.int32)).to(device)


def laswp(a: torch.Tensor, piv, team=None, reverse: bool = False, pool=None, check: bool = True) -> None:
    """Apply row interchanges k <-> ipiv[k] to every column of a, ascending (descending with
    reverse).  Indices are validated against the view before anything is touched
    (reference kernels.py:316-332)."""
    rows, cols, ld = check_colmajor(a, "a")
    ip = _device_pivots(piv, a.device)
    npiv = int(ip.shape[0])
    if npiv == 0:
        return
    pool = pool or default_pool(a.device.index)
    # pivot vectors longer than one device plan (MAX_PIVOT_BLOCK) are chunked inside the library, after
    # the whole vector was range-checked on the device (nothing is touched on a bad index)
    fn = _capi.lib().mla_laswp if check else _capi.lib().mla_laswp_async   # async: no host sync
    _capi.check(fn(pool.handle, a.data_ptr(), rows, cols, ld, ip.data_ptr(), npiv,
                   int(bool(reverse)), _stream(a)), pool.handle, "laswp")


def apply_panel(panel: torch.Tensor, w: int, target: torch.Tensor, piv, pool=None) -> None:
    """One update step of the block-cyclic driver as a single persistent launch: interchanges, trsm with
    the panel's unit-lower top block and the rank-w update of `target` (rows x cols, same first row as
    the panel) -- laswp + trsm_llu + gemm_malleable of the reference's lu.py:251-253, 280-281 fused."""
    rows, pw, ldp = check_colmajor(panel, "panel")
    trows, cols, ldt = check_colmajor(target, "target")
    if trows != rows or w > pw or w > rows:
        raise ValueError("apply_panel: panel/target shapes disagree")
    ip = _device_pivots(piv, target.device)
    if int(ip.shape[0]) < w:
        raise ValueError("apply_panel: need w pivots")
    pool = pool or default_pool(target.device.index)
    _capi.check(_capi.lib().mla_apply_panel(pool.handle, panel.data_ptr(), rows, w, ldp, target.data_ptr(), cols,
                                            ldt, ip.data_ptr(), _stream(target)), pool.handle, "apply_panel")


def apply_panel_prepare(panel: torch.Tensor, piv, w: int, pool=None, stream=None) -> None:
    """First half of apply_panel (interchange plan, inverted diagonal blocks of the panel's top block, queue,
    tag); see apply_panel_launch."""
    rows, pw, ldp = check_colmajor(panel, "panel")
    if w > pw or w > rows:
        raise ValueError("apply_panel: panel narrower than w")
    device = panel.device
    pool = pool or default_pool(device.index)
    ip = _device_pivots(piv, device)
    if int(ip.shape[0]) < w:
        raise ValueError("apply_panel: need w pivots")
    st = torch.cuda.current_stream(device).cuda_stream if stream is None else stream
    _capi.check(_capi.lib().mla_apply_panel_prepare(pool.handle, panel.data_ptr(), ldp, ip.data_ptr(), w, rows, st),
                pool.handle, "apply_panel_prepare")


def apply_panel_launch(panel: torch.Tensor, w: int, target: torch.Tensor | None, ctas: int = 0, pool=None,
                       skip_cols: int = 0, left: torch.Tensor | None = None) -> None:
    """Second half of apply_panel on the current stream: `ctas` CTAs (0 = all) drain the prepared queue.
    Launching it twice (two streams) makes the second launch join the first one's queue.
    `skip_cols`: leading columns of `target` that already carry the interchanges and their U rows (the
    leftover of an ET-cut panel); `left`: the owned columns left of the panel (same first row), which
    receive the interchanges only."""
    rows, pw, ldp = check_colmajor(panel, "panel")
    cols, ldt, tptr = 0, rows, 0
    if target is not None and target.shape[1] > 0:
        trows, cols, ldt = check_colmajor(target, "target")
        tptr = target.data_ptr()
        if trows != rows:
            raise ValueError("apply_panel: panel/target shapes disagree")
    if w > pw or w > rows:
        raise ValueError("apply_panel: panel/target shapes disagree")
    lcols, ldl, lptr = 0, rows, 0
    if left is not None and left.shape[1] > 0:
        lrows, lcols, ldl = check_colmajor(left, "left")
        lptr = left.data_ptr()
        if lrows != rows:
            raise ValueError("apply_panel: left columns must start at the panel's first row")
    pool = pool or default_pool(panel.device.index)
    _capi.check(_capi.lib().mla_apply_panel_launch(pool.handle, panel.data_ptr(), rows, w, ldp, tptr, cols, ldt,
                                                   int(skip_cols), lptr, lcols, ldl, int(ctas), _stream(panel)),
                pool.handle, "apply_panel_launch")


def step_flag(pool) -> tuple[int, int]:
    """(device address of the pool's step flag, tag of the step prepared last): the flag equals the tag
    once that update step's queue has been drained -- the ET flag for a panel running beside it."""
    import ctypes
    ptr, tag = ctypes.c_void_p(), ctypes.c_uint32()
    _capi.check(_capi.lib().mla_step_flag(pool.handle, ctypes.byref(ptr), ctypes.byref(tag)), pool.handle, "step_flag")
    return int(ptr.value), int(tag.value)


PANEL_HDR_INT32 = 4     # factored width, singular, scheduled width, rows (mla_pack_panel)


def packed_panel_doubles(rows: int, w: int) -> int:
    return int(_capi.lib().mla_packed_panel_doubles(int(rows), int(w)))


def pack_panel(panel: torch.Tensor, piv: torch.Tensor, out: torch.Tensor, pool=None, use_panel_info: bool = True) -> None:
    """Factored panel (rows x w view of the matrix) + int32 pivots + header -> one contiguous broadcast
    buffer (layout: include/mla_b200.h, mla_pack_panel).  Stream-ordered; the factored width comes from the
    device-side record of the pool's last panel kernel."""
    rows, w, ld = check_colmajor(panel, "panel")
    if piv.dtype != torch.int32 or piv.shape[0] < w or out.dtype != torch.float64 or not out.is_contiguous() \
            or out.numel() < packed_panel_doubles(rows, w):
        raise ValueError("pack_panel: need int32 pivots and a contiguous float64 buffer of packed_panel_doubles()")
    pool = pool or default_pool(panel.device.index)
    _capi.check(_capi.lib().mla_pack_panel(pool.handle, panel.data_ptr(), rows, w, ld, piv.data_ptr(),
                                           int(bool(use_panel_info)), out.data_ptr(), _stream(panel)), pool.handle,
                "pack_panel")
