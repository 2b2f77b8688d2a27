"""ctypes front end of the CPU oracle (oracle/mla_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module; the product package paper_1611_06365_b200 never does.  Parity status: pinned bit-for-bit
against the unmodified reference through tests/golden/ (see mla_oracle.c header).

All matrices are numpy float64 arrays in Fortran order (or column-major views of one), exactly the
storage of the reference (matrix.py:15-24); pivots are int64 (lu.py:86-89).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (recipe: oracle/Makefile)."""
    src = os.path.join(_HERE, "mla_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "liboracle.so"], check=True, capture_output=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        L.orc_fill_random.argtypes = [_dp, _i64, _i64, _i64, ctypes.c_uint64]
        L.orc_unb_pivoted.argtypes = [_dp, _i64, _i64, _i64, _ip]
        L.orc_unb_pivoted.restype = ctypes.c_int
        L.orc_laswp.argtypes = [_dp, _i64, _i64, _i64, _ip, _i64, ctypes.c_int]
        L.orc_laswp.restype = ctypes.c_int
        L.orc_trsm_llu.argtypes = [_dp, _i64, _i64, _dp, _i64, _i64]
        L.orc_gemm.argtypes = [_dp, _i64, _i64, _i64, _dp, _i64, _dp, _i64, _i64,
                               ctypes.c_double, ctypes.c_double, _i64]
        L.orc_lu_blk_ll.argtypes = [_dp, _i64, _i64, _i64, _i64, _ip, _i64,
                                    ctypes.POINTER(ctypes.c_int), _i64]
        L.orc_lu_blk_ll.restype = _i64
        L.orc_lu_blk_rl.argtypes = [_dp, _i64, _i64, _i64, _i64, _i64, _ip,
                                    ctypes.POINTER(ctypes.c_int), _i64]
        L.orc_lu_la.argtypes = [_dp, _i64, _i64, _i64, _i64, _i64, _ip, _ip, _i64,
                                ctypes.POINTER(ctypes.c_int), _ip, _i64, _ip, _i64]
        L.orc_lu_la.restype = _i64
        L.orc_lu_la_clamped.argtypes = [_dp, _i64, _i64, _i64, _i64, _i64, _ip, _ip, _i64,
                                        ctypes.POINTER(ctypes.c_int), _ip, _i64, _ip, _i64, _i64]
        L.orc_lu_la_clamped.restype = _i64
        L.orc_residual_lu.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _ip]
        L.orc_residual_lu.restype = ctypes.c_double
        _lib = L
    return _lib


def _mat(a: np.ndarray):
    """(pointer, rows, cols, ld) of a column-major float64 view."""
    if a.dtype != np.float64 or a.ndim != 2:
        raise ValueError("expected a 2-d float64 array")
    rows, cols = a.shape
    if rows > 1 and a.strides[0] != 8:
        raise ValueError("expected a column-major (Fortran-order) view")
    if cols > 1:
        ld = a.strides[1] // 8
    else:
        ld = max(rows, 1)
    return a.ctypes.data_as(_dp), rows, cols, max(ld, 1)


def _piv(p: np.ndarray):
    if p.dtype != np.int64 or not p.flags.c_contiguous:
        raise ValueError("pivots must be contiguous int64")
    return p.ctypes.data_as(_ip)


@dataclass
class OracleResult:
    ipiv: np.ndarray
    cols_factored: int
    singular: bool = False
    et_events: int = 0
    widths: tuple = ()


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(t: int) -> None:
    lib().orc_set_num_threads(int(t))


def alloc(rows: int, cols: int, ld: int | None = None) -> np.ndarray:
    ld = rows if ld is None else ld
    return np.zeros((max(ld, 1), cols), dtype=np.float64, order="F")[:rows, :]


def fill_random(a: np.ndarray, seed: int) -> np.ndarray:
    p, r, c, ld = _mat(a)
    lib().orc_fill_random(p, r, c, ld, ctypes.c_uint64(seed & (2 ** 64 - 1)))
    return a


def unb_pivoted(a: np.ndarray) -> OracleResult:
    p, m, n, ld = _mat(a)
    if m < n:
        raise ValueError("need m >= n")
    ipiv = np.zeros(n, dtype=np.int64)
    info = lib().orc_unb_pivoted(p, m, n, ld, _piv(ipiv)) if n else 0
    return OracleResult(ipiv, n, bool(info))


def laswp(a: np.ndarray, ipiv, reverse: bool = False) -> None:
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    p, m, n, ld = _mat(a)
    if lib().orc_laswp(p, m, n, ld, _piv(ipiv), ipiv.shape[0], int(reverse)) != 0:
        raise IndexError("pivot index out of range for this view")


def trsm_llu(a11: np.ndarray, b: np.ndarray) -> None:
    if a11.shape[0] != a11.shape[1]:
        raise ValueError("triangular factor must be square")
    if b.shape[0] != a11.shape[0]:
        raise ValueError("right-hand side rows disagree with the factor")
    lp, w, _, ldl = _mat(a11)
    bp, _, c, ldb = _mat(b)
    lib().orc_trsm_llu(lp, w, ldl, bp, c, ldb)


def gemm(c: np.ndarray, a: np.ndarray, b: np.ndarray, alpha: float = 1.0, beta: float = 1.0,
         k_c: int = 256) -> None:
    m, n = c.shape
    if a.shape[0] != m or b.shape != (a.shape[1], n):
        raise ValueError("gemm shapes disagree")
    cp, _, _, ldc = _mat(c)
    ap, _, k, lda = _mat(a)
    bp, _, _, ldb = _mat(b)
    lib().orc_gemm(cp, m, n, ldc, ap, lda, bp, ldb, k, float(alpha), float(beta), k_c)


def lu_blk_ll(a: np.ndarray, b: int, stop_trip: int = 0, k_c: int = 256) -> OracleResult:
    p, m, n, ld = _mat(a)
    if m < n:
        raise ValueError("need m >= n")
    ipiv = np.zeros(n, dtype=np.int64)
    sing = ctypes.c_int(0)
    cols = lib().orc_lu_blk_ll(p, m, n, ld, b, _piv(ipiv), stop_trip, ctypes.byref(sing), k_c) if n else 0
    return OracleResult(ipiv[:cols].copy(), int(cols), bool(sing.value))


def lu_blk_rl(a: np.ndarray, b: int, inner_b: int | None = None, k_c: int = 256) -> OracleResult:
    p, m, n, ld = _mat(a)
    if m < n:
        raise ValueError("need m >= n")
    ipiv = np.zeros(n, dtype=np.int64)
    sing = ctypes.c_int(0)
    lib().orc_lu_blk_rl(p, m, n, ld, b, inner_b or 0, _piv(ipiv), ctypes.byref(sing), k_c)
    return OracleResult(ipiv, n, bool(sing.value))


def lu_la(a: np.ndarray, b_outer: int, b_inner: int, et_sched=None, k_c: int = 256, clamp: int = 0) -> OracleResult:
    """Serial restatement of lu_la (any non-ET variant); et_sched replays an ET cut schedule.
    clamp > 0: panels never cross a multiple of `clamp` columns (the multi-GPU driver's schedule)."""
    p, m, n, ld = _mat(a)
    if m < n:
        raise ValueError("need m >= n")
    ipiv = np.zeros(n, dtype=np.int64)
    sing = ctypes.c_int(0)
    cap = n // max(b_inner, 1) + 2
    widths = np.zeros(cap, dtype=np.int64)
    nw = np.zeros(1, dtype=np.int64)
    if et_sched is None or len(et_sched) == 0:
        sp, ns = None, 0
    else:
        sched = np.ascontiguousarray(et_sched, dtype=np.int64)
        sp, ns = _piv(sched), sched.shape[0]
    ev = lib().orc_lu_la_clamped(p, m, n, ld, b_outer, b_inner, _piv(ipiv), sp, ns, ctypes.byref(sing),
                                 _piv(widths), cap, _piv(nw), k_c, int(clamp))
    return OracleResult(ipiv, n, bool(sing.value), int(ev), tuple(int(x) for x in widths[:int(nw[0])]))


def residual_lu(a_orig: np.ndarray, lu: np.ndarray, ipiv) -> float:
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    ap, m, n, lda = _mat(a_orig)
    lp, _, _, ldl = _mat(lu)
    return float(lib().orc_residual_lu(ap, lp, m, n, lda, ldl, _piv(ipiv)))
