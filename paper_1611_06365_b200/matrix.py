"""Column-major device matrices, seeded fill, pivot bookkeeping, residuals -- the reference's
matrix.py:15-131 on CUDA tensors.

A matrix is a 2-d float64 CUDA tensor with stride (1, ld): the transpose view of a C-contiguous
(cols, ld) allocation, so that sub-matrix views a[i0:i1, j0:j1] keep the parent's leading dimension
exactly like the reference's numpy F-order views.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .pool import default_pool


def alloc_matrix(rows: int, cols: int, ld: int | None = None, device=None) -> torch.Tensor:
    """Zeroed column-major matrix, optionally inside ld x cols storage (matrix.py:15-24)."""
    if rows < 0 or cols < 0:
        raise ValueError("rows and cols must be >= 0")
    if ld is None:
        ld = rows
    if ld < rows:
        raise ValueError("leading dimension smaller than rows")
    buf = torch.zeros((cols, max(ld, 1)), dtype=torch.float64, device=device or "cuda")
    return buf.t()[:rows, :]


def from_numpy(a: np.ndarray, device=None, ld: int | None = None) -> torch.Tensor:
    """Upload a host matrix (any layout) into a fresh column-major device matrix."""
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    out = alloc_matrix(rows, cols, ld, device)
    if rows and cols:
        out.copy_(torch.from_numpy(np.ascontiguousarray(a.T)).t())
    return out


def to_numpy(a: torch.Tensor) -> np.ndarray:
    """Download into a Fortran-order numpy array."""
    return np.asfortranarray(a.detach().cpu().numpy())


def leading_dimension(a: torch.Tensor) -> int:
    if a.ndim != 2:
        raise ValueError("expected a 2-d tensor")
    if a.shape[1] <= 1 and a.shape[0] <= 1:
        return max(a.shape[0], 1)
    if a.shape[1] <= 1:
        return max(a.shape[0], 1)
    return int(a.stride(1))


def check_colmajor(a: torch.Tensor, name: str = "a") -> tuple[int, int, int]:
    """(rows, cols, ld) of a column-major float64 CUDA view, or ValueError."""
    if not isinstance(a, torch.Tensor) or a.ndim != 2 or a.dtype != torch.float64:
        raise ValueError(f"{name}: expected a 2-d float64 tensor")
    if not a.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor (there is no CPU fallback)")
    rows, cols = a.shape
    if rows > 1 and a.stride(0) != 1:
        raise ValueError(f"{name}: expected a column-major view (stride(0) == 1)")
    ld = leading_dimension(a)
    if cols > 1 and ld < rows:
        raise ValueError(f"{name}: leading dimension smaller than rows")
    return rows, cols, max(ld, 1)


def partition_2x2(a: torch.Tensor, i: int, j: int):
    m, n = a.shape
    if not (0 <= i <= m and 0 <= j <= n):
        raise ValueError(f"split ({i}, {j}) out of range for {m} x {n}")
    return a[:i, :j], a[:i, j:], a[i:, :j], a[i:, j:]


def _stream(a: torch.Tensor) -> int:
    return torch.cuda.current_stream(a.device).cuda_stream


def fill_random(a: torch.Tensor, seed: int, scale: float = 1.0, shift: float = 0.0,
                row_scale: torch.Tensor | None = None, col0: int = 0,
                total_rows: int | None = None, pool=None) -> torch.Tensor:
    """SplitMix64 draws in (0,1), bit-identical to the reference's fill_random (matrix.py:44-63);
    scale/shift/row_scale produce the uniform[-1,1] and row-scaled configs on the device."""
    rows, cols, ld = check_colmajor(a)
    pool = pool or default_pool(a.device.index)
    rs = 0 if row_scale is None else row_scale.data_ptr()
    _capi.check(_capi.lib().mla_fill_random(pool.handle, a.data_ptr(), rows, cols, ld,
                                            ctypes.c_uint64(seed & (2 ** 64 - 1)), col0,
                                            total_rows or rows, float(scale), float(shift), rs,
                                            _stream(a)), pool.handle, "fill_random")
    return a


def frobenius_norm(a: torch.Tensor) -> float:
    return float(torch.linalg.norm(a))


@dataclass
class PivotVector:
    """Row-interchange list (reference matrix.py:74-92): step k swapped view rows k and ipiv[k].
    `ipiv` is a host int64 array like the reference's; `device` keeps the int32 device copy."""

    ipiv: np.ndarray
    offset: int = 0
    device: torch.Tensor | None = None

    def __post_init__(self) -> None:
        if isinstance(self.ipiv, torch.Tensor):
            if self.device is None and self.ipiv.is_cuda:
                self.device = self.ipiv.to(torch.int32)
            self.ipiv = self.ipiv.detach().cpu().numpy()
        self.ipiv = np.asarray(self.ipiv, dtype=np.int64)
        if self.ipiv.ndim != 1:
            raise ValueError("ipiv must be 1-d")

    def __len__(self) -> int:
        return int(self.ipiv.shape[0])

    def on_device(self, device) -> torch.Tensor:
        if self.device is None or self.device.device != torch.device(device):
            self.device = torch.from_numpy(self.ipiv.astype(np.int32)).to(device)
        return self.device


def swap_rows(a: torch.Tensor, piv, reverse: bool = False) -> torch.Tensor:
    """Apply interchanges to all columns of a (reference matrix.py:95-113) -- on the device."""
    from .kernels import laswp
    laswp(a, piv, reverse=reverse)
    return a


def split_lu(factors: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Unit-lower L (m x n) and upper U (n x n) from packed factors (matrix.py:107-113)."""
    m, n = factors.shape
    lower = alloc_matrix(m, n, device=factors.device)
    lower.copy_(torch.tril(factors, -1)[:, :n])
    idx = torch.arange(min(m, n), device=factors.device)
    lower[idx, idx] = 1.0
    upper = alloc_matrix(n, n, device=factors.device)
    upper.copy_(torch.triu(factors[:n, :]))
    return lower, upper


def residual_lu(a_orig: torch.Tensor, lower: torch.Tensor, upper: torch.Tensor, piv) -> float:
    """||P A - L U||_F / ||A||_F (matrix.py:116-131), computed on the device with the package's own
    laswp and DMMA gemm."""
    from .kernels import gemm_malleable, laswp
    denom = frobenius_norm(a_orig)
    m, n = a_orig.shape
    pa = alloc_matrix(m, n, device=a_orig.device)
    pa.copy_(a_orig)
    laswp(pa, piv)
    gemm_malleable(pa, lower, upper, 1.0, -1.0)
    num = frobenius_norm(pa)
    return num if denom == 0.0 else num / denom


def residual_packed(a_orig: torch.Tensor, factors: torch.Tensor, piv, block: int = 512) -> float:
    """Same quantity straight from the packed factors, blocked so that no m x n copy of L or U is
    materialised: for each block column kb, R[kb:, kb:] -= Ltri[:, kb] @ Utri[kb, :].
    a_orig is overwritten by the residual matrix."""
    from .kernels import gemm_malleable, laswp
    denom = frobenius_norm(a_orig)
    m, n = a_orig.shape
    laswp(a_orig, piv)
    for k0 in range(0, n, block):
        kw = min(block, n - k0)
        lk = alloc_matrix(m - k0, kw, device=a_orig.device)
        lk.copy_(factors[k0:, k0:k0 + kw])
        lk[:kw, :] = torch.tril(lk[:kw, :], -1)
        idx = torch.arange(kw, device=a_orig.device)
        lk[idx, idx] = 1.0
        uk = alloc_matrix(kw, n - k0, device=a_orig.device)
        uk.copy_(factors[k0:k0 + kw, k0:])
        uk[:, :kw] = torch.triu(uk[:, :kw])
        gemm_malleable(a_orig[k0:, k0:], lk, uk, 1.0, -1.0)
        del lk, uk
    num = frobenius_norm(a_orig)
    return num if denom == 0.0 else num / denom
