"""ctypes binding of libmla_b200.so (include/mla_b200.h).  This is the stub a maintainer of the
reference would add to route `mla`'s hot path to the GPU; there is no CPU fallback: a missing or
unloadable library raises immediately."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLA_B200_LIB") or os.path.join(_HERE, "libmla_b200.so")   # override: A/B builds (tools/)

OK, E_INVALID, E_CUDA, E_ABORT, E_INDEX, E_NOMEM = 0, -1, -2, -3, -4, -5
VARIANT_CODES = {"lu": 0, "lu_la": 1, "lu_ws_static": 2, "lu_mb": 3, "lu_et": 4}

_i64, _i32, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p


class LuInfo(ctypes.Structure):
    _fields_ = [("cols_factored", _i32), ("singular", _i32), ("et_events", _i32),
                ("n_panels", _i32), ("ws_joins", _i32), ("sm_pf_peak", _i32), ("reserved", _i32 * 2)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1611_06365_b200.build` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    L.mla_version.restype = ctypes.c_char_p
    L.mla_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
    L.mla_destroy.argtypes = [_vp]
    L.mla_num_sms.argtypes = [_vp]
    L.mla_last_cuda_error.argtypes = [_vp]
    L.mla_gemm.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64,
                           ctypes.c_double, ctypes.c_double, _vp, ctypes.c_int, _vp]
    L.mla_trsm_llu.argtypes = [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp]
    L.mla_laswp.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i64, ctypes.c_int, _vp]
    L.mla_laswp_async.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i64, ctypes.c_int, _vp]
    L.mla_laswp_async.restype = ctypes.c_int
    L.mla_panel_ll.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, _vp, ctypes.c_int,
                               ctypes.c_int, ctypes.POINTER(LuInfo), _vp]
    L.mla_getrf_la.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_int, _vp]
    L.mla_getrf_la_sync.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(LuInfo),
                                    _vp, ctypes.c_int, _vp]
    L.mla_getrf_la_host.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(LuInfo)]
    L.mla_fill_random.argtypes = [_vp, _vp, _i64, _i64, _i64, ctypes.c_uint64, _i64, _i64,
                                  ctypes.c_double, ctypes.c_double, _vp, _vp]
    L.mla_getrf_trace.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.mla_getrf_trace.restype = ctypes.c_int
    L.mla_apply_panel.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp]
    L.mla_apply_panel.restype = ctypes.c_int
    L.mla_panel_ll_async.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                     ctypes.c_uint32, _vp]
    L.mla_panel_ll_async.restype = ctypes.c_int
    L.mla_apply_panel_prepare.argtypes = [_vp, _vp, _i64, _vp, _i64, _i64, _vp]
    L.mla_apply_panel_prepare.restype = ctypes.c_int
    L.mla_apply_panel_launch.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _i64,
                                         ctypes.c_int, _vp]
    L.mla_apply_panel_launch.restype = ctypes.c_int
    L.mla_step_flag.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_uint32)]
    L.mla_step_flag.restype = ctypes.c_int
    L.mla_pack_panel.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, ctypes.c_int, _vp, _vp]
    L.mla_pack_panel.restype = ctypes.c_int
    L.mla_packed_panel_doubles.argtypes = [_i64, _i64]
    L.mla_packed_panel_doubles.restype = _i64
    L.mla_set_trace.argtypes = [_vp, ctypes.c_int]
    L.mla_set_trace.restype = ctypes.c_int
    L.mla_getrf_events.argtypes = [_vp, _vp, ctypes.c_int]
    L.mla_getrf_events.restype = ctypes.c_int
    L.mla_release_host_cache.argtypes = [_vp]
    L.mla_release_host_cache.restype = ctypes.c_int
    L.mla_abort_word.argtypes = [_vp]
    L.mla_abort_word.restype = ctypes.c_int
    L.mla_set_update_sms.argtypes = [_vp, ctypes.c_int]
    L.mla_set_update_sms.restype = ctypes.c_int
    L.mla_set_host_phases.argtypes = [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_int]
    L.mla_set_host_phases.restype = ctypes.c_int
    L.mla_set_panel_sms_max.argtypes = [_vp, ctypes.c_int]
    L.mla_set_panel_sms_max.restype = ctypes.c_int
    L.mla_getrf_debug.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64)]
    L.mla_getrf_debug.restype = ctypes.c_int
    L.mla_panel_profile.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.mla_panel_profile.restype = ctypes.c_int
    for name in ("mla_create", "mla_destroy", "mla_num_sms", "mla_last_cuda_error", "mla_gemm",
                 "mla_trsm_llu", "mla_laswp", "mla_panel_ll", "mla_getrf_la", "mla_getrf_la_sync",
                 "mla_getrf_la_host", "mla_fill_random"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


EXPORTS = ("mla_version", "mla_create", "mla_destroy", "mla_num_sms", "mla_last_cuda_error",
           "mla_gemm", "mla_trsm_llu", "mla_laswp", "mla_panel_ll", "mla_getrf_la",
           "mla_getrf_la_sync", "mla_getrf_la_host", "mla_fill_random", "mla_panel_profile", "mla_getrf_trace", "mla_laswp_async", "mla_getrf_debug",
           "mla_apply_panel", "mla_set_panel_sms_max", "mla_panel_ll_async",
           "mla_set_update_sms", "mla_apply_panel_prepare", "mla_apply_panel_launch", "mla_abort_word",
           "mla_step_flag", "mla_set_trace", "mla_getrf_events", "mla_pack_panel", "mla_packed_panel_doubles", "mla_release_host_cache",
           "mla_set_host_phases")


class MlaError(RuntimeError):
    pass


def check(code: int, handle=None, what: str = "") -> None:
    """Map C return codes onto the reference's exception types."""
    if code == OK:
        return
    if code == E_INVALID:
        raise ValueError(f"{what}: invalid argument")
    if code == E_INDEX:
        raise IndexError("pivot index out of range for this view")
    if code == E_CUDA:
        err = lib().mla_last_cuda_error(handle) if handle else -1
        raise MlaError(f"{what}: CUDA error {err}")
    if code == E_ABORT:
        raise MlaError(f"{what}: device watchdog abort")
    raise MlaError(f"{what}: error {code}")
