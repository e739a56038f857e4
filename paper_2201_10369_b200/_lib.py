"""ctypes loader for libwino.so (the C ABI of include/wino.h).

There is no fallback: if the library cannot be loaded (or built in-tree with nvcc),
importing the product API raises.  Every step of the hot path runs in libwino's
kernels; Python only marshals arguments.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

_f = ctypes.POINTER(ctypes.c_float)
_d = ctypes.POINTER(ctypes.c_double)
_i = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i64 = ctypes.c_int64

# (name, restype, argtypes) -- mirrors include/wino.h
SIGNATURES = [
    ("wino_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("wino_last_error", ctypes.c_char_p, []),
    ("wino_supported", ctypes.c_int, [ctypes.c_int] * 3),
    ("wino_points_to_matrices", ctypes.c_int, [ctypes.c_int, ctypes.c_int, _d, ctypes.c_int, _d, _d, _d]),
    ("wino_conv2d_workspace_bytes", _sz, [ctypes.c_int] * 8),
    ("wino_conv2d_gemm_tile", ctypes.c_int, [ctypes.c_int] * 8),
    ("wino_conv2d_fp32", ctypes.c_int,
     [_vp, _vp, _vp] + [ctypes.c_int] * 8 + [_d, _vp, _sz, _vp, _vp, _vp]),
    ("wino_conv2d_fp32_ex", ctypes.c_int,
     [_vp, _vp, _vp] + [ctypes.c_int] * 8 + [_d, _vp, _sz, _vp, _vp, ctypes.c_uint, _vp]),
    ("wino_relu_pool_fp32", ctypes.c_int, [_vp, _vp] + [ctypes.c_int] * 5 + [_vp]),
    ("wino_conv2d_relu_pool_fp32", ctypes.c_int,
     [_vp, _vp, _vp, _vp] + [ctypes.c_int] * 8 + [_d, _vp, _sz, _vp, _vp, ctypes.c_int, ctypes.c_uint, _vp]),
    ("wino_error_sweep_workspace_bytes", _sz, [ctypes.c_int] * 4 + [_i64]),
    ("wino_error_sweep", ctypes.c_int,
     [ctypes.c_int] * 3 + [_d, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _i, _vp, _sz, ctypes.c_uint, _vp]),
    ("wino_sweep_outputs", ctypes.c_int,
     [ctypes.c_int] * 3 + [_d, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp, _i, _vp, _sz, ctypes.c_uint, _vp]),
    ("wino_last_launch_count", ctypes.c_int, []),
    ("wino_huffman_jit_mode", ctypes.c_int, [ctypes.c_int]),
    ("wino_huffman_jit_classes", ctypes.c_int, []),
    ("wino_huffman_jit_compile_check", ctypes.c_int,
     [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_size_t)]),
    ("wino_timing_enable", ctypes.c_int, [ctypes.c_int]),
    ("wino_timing_reset", None, []),
    ("wino_timing_read", ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), _i]),
]

_lib = None


def lib_path() -> str:
    return _build.LIB


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if _build.needs_build():
        _build.build()  # raises on failure: no fallback
    L = ctypes.CDLL(_build.LIB)
    for name, res, args in SIGNATURES:
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class WinoError(RuntimeError):
    def __init__(self, status: int, where: str):
        L = load()
        msg = L.wino_last_error().decode(errors="replace")
        name = L.wino_status_string(status).decode()
        super().__init__(f"{where}: {name} ({msg})")
        self.status = status


def check(status: int, where: str) -> None:
    if status != 0:
        raise WinoError(status, where)
