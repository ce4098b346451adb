"""ctypes declarations of libig.so (the C ABI in include/ig.h).  Argument marshalling only."""

from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libig.so")

IG_MAX_HISTORY = 32
IG_PROJ_QR, IG_EXTRAP_LS, IG_PROJ_CLASSIC, IG_EXTRAP_SPARSE = 1, 2, 3, 4
IG_OK, IG_E_ARG, IG_E_OOM, IG_E_CUDA, IG_E_NCCL, IG_E_STATE = 0, 1, 2, 3, 4, 5
STATUS_NAMES = {0: "IG_OK", 1: "IG_E_ARG", 2: "IG_E_OOM", 3: "IG_E_CUDA", 4: "IG_E_NCCL", 5: "IG_E_STATE"}


class ig_stats_t(C.Structure):
    _fields_ = [
        ("d", C.c_int),
        ("admitted", C.c_int),
        ("rho", C.c_double),
        ("norm_Ax", C.c_double),
        ("norm_bt", C.c_double),
        ("launches", C.c_int64),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_SIGS = {
    "ig_create": (_P, [C.c_int64, C.c_int, C.c_int, C.c_int]),
    "ig_create_ext": (_P, [C.c_int64, C.c_int, C.c_int, C.c_int, _P, C.c_size_t]),
    "ig_storage_bytes": (C.c_size_t, [C.c_int64, C.c_int, C.c_int]),
    "ig_destroy": (None, [_P]),
    "ig_reset": (C.c_int, [_P]),
    "ig_last_error": (C.c_char_p, []),
    "ig_set_stream": (C.c_int, [_P, _P]),
    "ig_set_admit_tol": (C.c_int, [_P, C.c_double]),
    "ig_set_schedule": (C.c_int, [_P, C.c_int]),
    "ig_state_bytes": (C.c_size_t, [_P]),
    "ig_save_state": (C.c_int, [_P, _P, C.c_size_t]),
    "ig_load_state": (C.c_int, [_P, _P, C.c_size_t]),
    "ig_form_guess": (C.c_int, [_P, _P, _P]),
    "ig_update": (C.c_int, [_P, _P, _P]),
    "ig_form_guess_host": (C.c_int, [_P, _P, _P]),
    "ig_form_guess_batch": (C.c_int, [C.c_int, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ig_update_batch": (C.c_int, [C.c_int, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ig_update_host": (C.c_int, [_P, _P, _P]),
    "ig_form_guess_batch_host": (C.c_int, [C.c_int, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ig_update_batch_host": (C.c_int, [C.c_int, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ig_next_slot": (_P, [_P]),
    "ig_comm_unique_id": (C.c_int, [_P]),
    "ig_comm_create": (C.c_int, [C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "ig_local_group_create": (_P, [C.c_int]),
    "ig_local_group_destroy": (None, [_P]),
    "ig_comm_create_local": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ig_comm_destroy": (None, [_P]),
    "ig_attach_comm": (C.c_int, [_P, _P]),
    "ig_history_dim": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "ig_weights": (C.c_int, [_P, C.c_int, _D, C.POINTER(C.c_int)]),
    "ig_bytes": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ig_get_stats": (C.c_int, [_P, C.POINTER(ig_stats_t)]),
    "ig_copy_history": (C.c_int, [_P, _P, _P, C.c_int64, _D]),
    "ig_total_launches": (C.c_int64, []),
    "ig_profile": (C.c_int, [_P, C.c_int]),
    "ig_xwin_bytes": (C.c_size_t, []),
    "ig_xwin_export": (C.c_int, [_P, _P]),
    "ig_xwin_ptr": (_P, [_P]),
    "ig_attach_peers": (C.c_int, [_P, C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "ig_set_grid_limit": (C.c_int, [_P, C.c_int]),
    "ig_set_launch": (C.c_int, [_P, C.c_int]),
    "ig_set_watchdog": (C.c_int, [_P, C.c_double]),
    "ig_profile_read": (C.c_int, [_P, C.c_int, _D, C.POINTER(C.c_int64)]),
    "ig_set_device_ring": (C.c_int, [_P, C.c_int]),
    "ig_capture_begin": (C.c_int, [_P]),
    "ig_capture_end": (C.c_int, [_P, C.POINTER(_P)]),
    "ig_graph_launch": (C.c_int, [_P, _P]),
    "ig_graph_destroy": (None, [_P]),
}

KERNELS = ["form_dot", "form_combine", "u1", "u2", "u3", "extrap", "copy", "form_fused", "update_fused"]

_lib = None


def lib() -> C.CDLL:
    """The loaded libig.so.  Fails loudly if it has not been built (there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library with "
                "`python -m paper_2009_10863_b200.build` (there is no CPU fallback)"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
