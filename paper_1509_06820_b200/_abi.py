"""ctypes binding of librqrcp_b200.so (include/rqrcp_b200.h).

The library is loaded eagerly on first use; a missing library or a missing
GPU raises immediately -- there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RQ_LIB_PATH") or os.path.join(HERE, "librqrcp_b200.so")

RQ_OK, RQ_ERR_INVALID, RQ_ERR_INTERNAL, RQ_ERR_CUDA = 0, -1, -2, -3
RQ_RQRCP, RQ_RSRQRCP, RQ_SSRQRCP, RQ_TRQRCP = 0, 1, 2, 3

OMEGA_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_double))

i64, f64, vp, dp, lp = C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p


class FactorArgs(C.Structure):
    _fields_ = [
        ("m", i64), ("n", i64), ("k", i64), ("block", i64), ("ell", i64),
        ("variant", C.c_int32), ("speculate", C.c_int32),
        ("work", dp), ("ldw", i64), ("Y", dp), ("ldy", i64), ("tau", dp),
        ("W", dp), ("ldW", i64), ("R", dp), ("ldR", i64),
        ("perm", lp), ("swaps", lp), ("swap_cap", i64),
        ("omega0", dp), ("omega_fn", OMEGA_FN), ("omega_user", vp), ("stream", vp),
        ("host_Y", dp), ("ldhY", i64), ("host_R", dp), ("ldhR", i64),
        ("omega_native", C.c_int32), ("omega_threads", C.c_int32),
        ("omega_k0", C.c_uint64), ("omega_k1", C.c_uint64), ("omega_raw", C.c_uint64),
    ]


class FactorResult(C.Structure):
    _fields_ = [("rank", i64), ("nswaps", i64), ("gemm_flops", i64), ("level2_flops", i64),
                ("bytes_touched", i64), ("resamples", i64), ("frob", f64)]


class TuxvArgs(C.Structure):
    _fields_ = [("f", FactorArgs), ("A", dp), ("lda", i64), ("j_max", i64),
                ("U", dp), ("ldu", i64), ("V", dp), ("ldv", i64), ("X", dp), ("ldx", i64)]


class TuxvResult(C.Structure):
    _fields_ = [("f", FactorResult), ("rank", i64), ("x_lower", C.c_int32), ("pad", C.c_int32)]


# name -> (restype, argtypes); every export declared in include/rqrcp_b200.h
SIGNATURES = {
    "rq_version": (C.c_int, []),
    "rq_last_error": (C.c_char_p, []),
    "rq_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "rq_destroy": (C.c_int, [vp]),
    "rq_factor": (C.c_int, [vp, C.POINTER(FactorArgs), C.POINTER(FactorResult)]),
    "rq_tuxv": (C.c_int, [vp, C.POINTER(TuxvArgs), C.POINTER(TuxvResult)]),
    "rq_gemm": (C.c_int, [vp, C.c_int, C.c_int, i64, i64, i64, f64, dp, i64, dp, i64, f64, dp,
                          i64, vp]),
    "rq_sketch": (C.c_int, [vp, i64, i64, i64, dp, i64, dp, i64, dp, i64, vp]),
    "rq_select_pivots": (C.c_int, [vp, i64, i64, i64, dp, i64, dp, i64, lp, dp, i64, dp,
                                   C.POINTER(i64), C.POINTER(i64), vp]),
    "rq_panel_qr": (C.c_int, [vp, i64, i64, dp, i64, dp, i64, dp, dp, i64, f64,
                              C.POINTER(i64), C.POINTER(i64), vp]),
    "rq_t_factor": (C.c_int, [vp, dp, i64, i64, i64, dp, dp, i64, vp]),
    "rq_sample_update": (C.c_int, [vp, i64, i64, i64, dp, i64, dp, dp, i64, f64, dp, i64,
                                   C.POINTER(C.c_int32), vp]),
    "rq_qr_blocked": (C.c_int, [vp, i64, i64, i64, i64, dp, i64, dp, i64, dp, C.POINTER(i64),
                                vp]),
    "rq_q_columns": (C.c_int, [vp, i64, i64, i64, dp, i64, dp, i64, dp, i64, vp]),
    "rq_column_norms": (C.c_int, [vp, dp, i64, i64, i64, C.c_int, dp, vp]),
    "rq_frob_norm": (C.c_int, [vp, dp, i64, i64, i64, dp, vp]),
    "rq_downdate_norms": (C.c_int, [vp, dp, dp, i64, i64, dp, f64, dp, vp, vp]),
    "rq_launch_count": (C.c_int64, []),
    "rq_set_option": (C.c_int, [vp, C.c_char_p, i64]),
    "rq_debug_read": (C.c_int, [vp, C.POINTER(i64), C.c_int]),
    "rq_profile_enable": (C.c_int, [vp, C.c_int]),
    "rq_profile_reset": (C.c_int, [vp]),
    "rq_profile_read": (C.c_int, [vp, C.POINTER(i64), C.POINTER(f64), C.POINTER(f64),
                                  C.POINTER(f64)]),
    "rq_profile_trace": (C.c_int, [vp, i64, C.POINTER(C.c_int32), C.POINTER(f64), C.POINTER(f64),
                                   C.POINTER(i64)]),
    "rq_omega_fill": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, dp, i64, C.c_int,
                                C.POINTER(C.c_uint64)]),
}

PROF_NAMES = ["sketch", "inner", "update", "small_gemm", "select", "panel", "sample_update",
              "swap", "misc"]

_lib = None
_lock = threading.Lock()
_handles: dict[int, C.c_void_p] = {}


def load_library(path: str = LIB_PATH):
    """Load (without touching the GPU) and type every exported symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_1509_06820_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class RqError(RuntimeError):
    pass


def check(rc: int):
    if rc == RQ_OK:
        return
    msg = load_library().rq_last_error().decode(errors="replace")
    if rc == RQ_ERR_INVALID:
        raise ValueError(msg)
    raise RqError(f"librqrcp_b200 error {rc}: {msg}")


def handle(device: int) -> C.c_void_p:
    """Per-device library handle (workspace arena), created on first use."""
    lib = load_library()
    with _lock:
        h = _handles.get(device)
        if h is None:
            h = C.c_void_p()
            check(lib.rq_create(device, C.byref(h)))
            _handles[device] = h
        return h
