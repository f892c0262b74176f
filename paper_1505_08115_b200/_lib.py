"""ctypes binding of librandqr_b200.so (declared in include/randqr_b200.h).

The product path has no fallback: if the CUDA library is missing or no CUDA
device is present, importing the binding raises.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_1505_08115_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RQ_LIB_PATH") or os.path.join(_HERE, "librandqr_b200.so")  # override: tuning builds

RQ_OK, RQ_EDIM, RQ_EVALUE, RQ_ECONV, RQ_ECUDA, RQ_EINTERNAL, RQ_EUNSUPPORTED = range(7)
RQ_PIVOT_PERMUTATION, RQ_PIVOT_REFLECTORS = 0, 1
RQ_SKETCH_FRESH, RQ_SKETCH_DOWNDATE = 0, 1
RQ_FLAG_NO_LOOKAHEAD = 1
RQ_FLAG_TF32_UPDATE = 2


class rq_config(ctypes.Structure):
    _fields_ = [
        ("block", ctypes.c_int32),
        ("oversample", ctypes.c_int32),
        ("power", ctypes.c_int32),
        ("stabilize", ctypes.c_int32),
        ("pivot_kind", ctypes.c_int32),
        ("rrqr", ctypes.c_int32),
        ("sketch_mode", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


PANEL_CB = ctypes.CFUNCTYPE(None, ctypes.c_int32, ctypes.c_void_p)

_i32, _i64, _u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_vp = ctypes.c_void_p
_SIGS = {
    "rq_version": (ctypes.c_char_p, []),
    "rq_last_error": (ctypes.c_char_p, []),
    "rq_ctx_create": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, _vp]),
    "rq_ctx_destroy": (ctypes.c_int, [_vp]),
    "rq_ctx_set_stream": (ctypes.c_int, [_vp, _vp]),
    "rq_ctx_set_inspect": (ctypes.c_int, [_vp, PANEL_CB, _vp]),
    "rq_ctx_set_gemm_cap": (ctypes.c_int, [_vp, _i32]),
    "rq_factorize": (ctypes.c_int, [_vp, ctypes.POINTER(rq_config), _i64, _i64, _vp, _i64, _u64,
                                    ctypes.POINTER(_u64), _vp]),
    "rq_factorize_host": (ctypes.c_int, [_vp, ctypes.POINTER(rq_config), _i64, _i64, _vp, _i64, _u64,
                                         ctypes.POINTER(_u64), _vp, _i64, _vp]),
    "rq_form_q": (ctypes.c_int, [_vp, _i64, _vp, _i64]),
    "rq_form_p": (ctypes.c_int, [_vp, _vp, _i64]),
    "rq_snapshot": (ctypes.c_int, [_vp, _vp, _i64]),
    "rq_snapshot_sketch": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "rq_factors_detach": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "rq_factors_destroy": (ctypes.c_int, [_vp]),
    "rq_factors_form_q": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64]),
    "rq_factors_form_p": (ctypes.c_int, [_vp, _vp, _vp, _i64]),
    "rq_factors_info": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, ctypes.POINTER(_i32)]),
    "rq_apply_q": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i64, _vp, _i64]),
    "rq_apply_p": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i64, _vp, _i64]),
    "rq_householder_sweep": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i32]),
    "rq_gaussian_matrix": (ctypes.c_int, [_vp, _i64, _i64, _u64, _u64, _vp, _i64]),
    "rq_trinv_upper": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _i64]),
    "rq_splitmix_words": (ctypes.c_int, [_vp, _u64, _u64, _i64, _vp]),
    "rq_qr_unpivoted": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i64, _i32]),
    "rq_trailing_frobenius": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp]),
    "rq_trailing_spectral": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _i32, _vp, _vp]),
    "rq_gemm": (ctypes.c_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64,
                               _i64, _i64, _i64, _i64, _vp, _i64, ctypes.c_double, ctypes.c_double]),
    "rq_gemm_f32": (ctypes.c_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64,
                                   _i64, _i64, _i64, _i64, _vp, _i64, ctypes.c_double, ctypes.c_double]),
    "rq_sketch_select": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "rq_panel_factor": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "rq_panel_apply": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i32, _vp, _i64, _i64, _i64,
                                      _i64, _i64, _i64]),
    "rq_test_gemm": (ctypes.c_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64,
                                    _i64, _i64, _i64, _i64, _vp, _i64, ctypes.c_double, ctypes.c_double]),
    "rq_test_sketch_cpqr": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp]),
    "rq_test_leaf_qr": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i32, _vp, _i64, _vp, _i64]),
    "rq_test_wy_update": (ctypes.c_int, [_vp, _i32, _vp, _i64, _i64, _i32, _vp, _i64, _vp, _i64, _i32]),
    "rq_test_debug_timing": (ctypes.c_int, [_i32, _vp, _i32]),
    "rq_launch_count": (_i64, [_vp]),
    "rq_set_profiling": (ctypes.c_int, [_vp, _i32]),
    "rq_profile_read": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(_i64)]),
    "rq_profile_bytes": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(ctypes.c_double)]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load the library (raises if it is missing; there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("RQ_LIB_PATH") and not hasattr(lib, name):
                    continue  # an older tuning build (A/B runs): bind what it exports
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols():
    return list(_SIGS)


def last_error():
    return load().rq_last_error().decode(errors="replace")
