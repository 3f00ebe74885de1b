"""ctypes binding of libkatsevich.so (include/katsevich.h).  Argument
marshalling only: every step of the reconstruction runs in the library's CUDA
kernels.  There is no CPU fallback — if the shared library is missing the
import fails loudly."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkatsevich.so")

KATS_OK = 0
KATS_WARN_TD_NOT_COVERED = 1
KATS_ERR_NULL = -1
KATS_ERR_INVALID_GEOMETRY = -2
KATS_ERR_NOT_PRECOMPUTED = -3
KATS_ERR_COVERAGE = -4
KATS_ERR_PI_NONCONVERGENCE = -5
KATS_ERR_WORKSPACE = -6
KATS_ERR_CUDA = -7
KATS_ERR_NO_DEVICE = -8
KATS_ERR_ARGUMENT = -9


class KatsevichGeometry(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double), ("D", ctypes.c_double), ("pitch", ctypes.c_double),
        ("lambda0", ctypes.c_double), ("z0", ctypes.c_double), ("r_fov", ctypes.c_double),
        ("n_rows", ctypes.c_int32), ("d_w", ctypes.c_double),
        ("n_cols", ctypes.c_int32), ("d_alpha", ctypes.c_double), ("alpha_offset", ctypes.c_double),
        ("views_per_turn", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
        ("nz_per_pitch", ctypes.c_int32), ("n_psi", ctypes.c_int32), ("flags", ctypes.c_int32),
    ]


class KatsevichStats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 6), ("ms", ctypes.c_double * 6),
                ("busy_ms", ctypes.c_double * 6), ("total_launches", ctypes.c_int64)]


# every symbol include/katsevich.h declares, with (restype, argtypes)
_P = ctypes.c_void_p
_I32, _I64, _SZ = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_PI32, _PI64 = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
_PD, _PSZ = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_size_t)
SIGNATURES = {
    "katsevich_plan_create": (ctypes.c_int, [ctypes.POINTER(KatsevichGeometry), ctypes.c_int, ctypes.POINTER(_P)]),
    "katsevich_precompute": (ctypes.c_int, [_P, _P]),
    "katsevich_pitch_views": (ctypes.c_int, [_P, _I32, _PI64, _PI32]),
    "katsevich_scan_views": (ctypes.c_int, [_P, _I32, _I32, _PI64, _PI64]),
    "katsevich_workspace_bytes": (ctypes.c_int, [_P, _I32, _PSZ]),
    "katsevich_workspace_bytes_host": (ctypes.c_int, [_P, _I32, _PSZ]),
    "katsevich_reconstruct": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _SZ, _P]),
    "katsevich_reconstruct_grouped": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _SZ, _P, _I32,
                                                     ctypes.POINTER(ctypes.c_void_p)]),
    "katsevich_reconstruct_batch": (ctypes.c_int, [_P, _P, _I32, _P, _P, _SZ, _P]),
    "katsevich_workspace_bytes_batch_host": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_SZ)]),
    "katsevich_reconstruct_batch_host": (ctypes.c_int, [_P, _P, _I32, _P, _P, _SZ, _P]),
    "katsevich_reconstruct_host": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _SZ, _P]),
    "katsevich_filter": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _I32, _P, _P, _P, _P]),
    "katsevich_backproject": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _P, _P]),
    "katsevich_table_info": (ctypes.c_int, [_P, _PI32, _PI64, _PI64]),
    "katsevich_hilbert_hk_table": (ctypes.c_int, [_I32, _P, _P, _SZ]),
    "katsevich_export_tables": (ctypes.c_int, [_P, _PI32, _PI32, _PD, _PD, _PI32, _PD, _PI32, _PD]),
    "katsevich_profile_enable": (ctypes.c_int, [_P, ctypes.c_int]),
    "katsevich_profile_read": (ctypes.c_int, [_P, ctypes.POINTER(KatsevichStats), ctypes.c_int]),
    "katsevich_bp_kernel": (ctypes.c_int, [_P]),
    "katsevich_adjoint_workspace_bytes": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_SZ)]),
    "katsevich_adjoint": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _I64, _I64, _P, _SZ, _P]),
    "katsevich_adjoint_batch_workspace_bytes": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_SZ)]),
    "katsevich_adjoint_batch": (ctypes.c_int, [_P, _P, _I32, _P, _P, _SZ, _P]),
    "katsevich_project_ellipsoids": (ctypes.c_int, [_P, _P, _I32, _I64, _I64, _P, _P]),
    "katsevich_project_volume": (ctypes.c_int, [_P, _P, _I32, ctypes.c_double, ctypes.c_double, _I64, _I64, _P,
                                                _PI64, _P]),
    "katsevich_degrade": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_uint64, _I32, _P, _P, _P, _P]),
    "katsevich_destroy": (None, [_P]),
    "katsevich_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "katsevich_last_error_detail": (ctypes.c_char_p, [_P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` or __graft_entry__.build() "
                              "(the CUDA library is required; there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class KatsevichError(RuntimeError):
    def __init__(self, code: int, detail: str = ""):
        self.code = code
        msg = lib().katsevich_error_string(code).decode()
        super().__init__(f"katsevich error {code}: {msg}" + (f" ({detail})" if detail else ""))
