"""ORACLE (test infrastructure only) -- ctypes driver for ``oracle/ref.c``.

``build()`` compiles ref.c with gcc (``-O2 -mfma -ffp-contract=off -fopenmp``);
``__graft_entry__.build()`` calls it so the checker exists on the GPU box.
Functions take/return numpy arrays; fp32 matrices come from ``oracle.r64``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

from . import r64

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ref.c")
_LIB = os.path.join(_HERE, "libwino_oracle.so")
_lib = None

_f = ctypes.POINTER(ctypes.c_float)
_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oref_tile.argtypes = [ctypes.c_int] * 3 + [_f] * 5 + [ctypes.c_int, _f]
        L.oref_direct64_tiles.argtypes = [ctypes.c_int] * 3 + [_i64, _f, _f, _d]
        L.oref_sweep.argtypes = ([ctypes.c_int] * 4 + [_f, _i64, _f, _f, ctypes.c_int, ctypes.c_int,
                                 _d, _d, _i64, _f])
        L.oref_conv2d_wino.argtypes = ([_f, _f, _f] + [ctypes.c_int] * 8 + [_f, _f, _f]
                                       + [ctypes.c_int] * 3)
        L.oref_conv2d_direct64.argtypes = [_f, _f, _d] + [ctypes.c_int] * 9
        L.oref_stats.argtypes = [_f, _d, _i64, _d, _d]
        L.oref_sweep_mixed.argtypes = ([ctypes.c_int] * 4 + [_d, _i64, _f, _f, _d, _d, _i64, _f])
        L.oref_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray], ct):
    if a is None:
        return ctypes.cast(None, ctypes.POINTER(ct))
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def max_threads() -> int:
    return int(lib().oref_max_threads())


def pack_mats(m: int, r: int, point_sets: Sequence[Sequence[float]]) -> np.ndarray:
    """[n_cand, m*n + n*r + n*n] fp32: RN32 of the R64 matrices, per candidate."""
    rows = []
    for pts in point_sets:
        AT, G, BT = r64.build_f32(m, r, pts)
        rows.append(np.concatenate([AT.ravel(), G.ravel(), BT.ravel()]))
    return np.ascontiguousarray(np.stack(rows), dtype=np.float32)


def _mode(nofma, huffman):
    """0: F32-FMA chains, 1: F32-NOFMA chains, 2: Huffman order (NOFMA products)."""
    return 2 if huffman else int(bool(nofma))


def tile(dims, m, r, AT, G, BT, d, g, nofma=False, huffman=False) -> np.ndarray:
    y = np.zeros(m ** dims, dtype=np.float32)
    AT, G, BT, d, g = map(_c32, (AT, G, BT, d, g))
    rc = lib().oref_tile(dims, m, r, _p(AT, ctypes.c_float), _p(G, ctypes.c_float), _p(BT, ctypes.c_float),
                         _p(d, ctypes.c_float), _p(g, ctypes.c_float), _mode(nofma, huffman),
                         _p(y, ctypes.c_float))
    if rc:
        raise ValueError("oref_tile failed")
    return y


def direct64_tiles(dims, m, r, d_tiles, g_tiles) -> np.ndarray:
    d_tiles, g_tiles = _c32(d_tiles), _c32(g_tiles)
    nt = d_tiles.shape[0]
    y = np.zeros((nt, m ** dims), dtype=np.float64)
    lib().oref_direct64_tiles(dims, m, r, nt, _p(d_tiles, ctypes.c_float), _p(g_tiles, ctypes.c_float),
                              _p(y, ctypes.c_double))
    return y


def sweep(dims, m, r, point_sets, d_tiles, g_tiles, nofma=False, n_dump=0, mats=None, huffman=False):
    """O9.  Returns (sums [S,5], maxs [S,2], y_dump [S,n_dump,m^dims] or None).
    huffman=True: transform dot products in Huffman order (reading R21)."""
    if mats is None:
        mats = pack_mats(m, r, point_sets)
    return _sweep(dims, m, r, mats, d_tiles, g_tiles, _mode(nofma, huffman), False, n_dump)


def pack_mats64(m: int, r: int, point_sets: Sequence[Sequence[float]]) -> np.ndarray:
    """[n_cand, m*n + n*r + n*n] fp64: the R64 matrices, per candidate."""
    rows = []
    for pts in point_sets:
        AT, G, BT = r64.build_r64(m, r, pts)
        rows.append(np.concatenate([np.asarray(AT).ravel(), np.asarray(G).ravel(), np.asarray(BT).ravel()]))
    return np.ascontiguousarray(np.stack(rows), dtype=np.float64)


def sweep_mixed(dims, m, r, point_sets, d_tiles, g_tiles, n_dump=0):
    """O9 for the mixed-precision variant (reading R22): fp64 transforms with the R64
    matrices, fp32 U, V and Hadamard product, fp32 output.  Returns (sums, maxs, y_dump)."""
    mats = pack_mats64(m, r, point_sets)
    d_tiles, g_tiles = _c32(d_tiles), _c32(g_tiles)
    S, nt = mats.shape[0], d_tiles.shape[0]
    sums = np.zeros((S, 5))
    maxs = np.zeros((S, 2))
    ydump = np.zeros((S, n_dump, m ** dims), dtype=np.float32) if n_dump else None
    rc = lib().oref_sweep_mixed(dims, m, r, S, _p(mats, ctypes.c_double), nt, _p(d_tiles, ctypes.c_float),
                                _p(g_tiles, ctypes.c_float), _p(sums, ctypes.c_double), _p(maxs, ctypes.c_double),
                                int(n_dump), _p(ydump, ctypes.c_float))
    if rc:
        raise ValueError("oref_sweep_mixed failed")
    return sums, maxs, ydump


def direct32_sweep(dims, m, r, d_tiles, g_tiles, nofma=True):
    """The paper's n = 0 row: fp32 direct correlation scored against fp64."""
    n = m + r - 1
    mats = np.zeros((1, m * n + n * r + n * n), dtype=np.float32)
    s, mx, _ = _sweep(dims, m, r, mats, d_tiles, g_tiles, nofma, True, 0)
    return s[0], mx[0]


def _sweep(dims, m, r, mats, d_tiles, g_tiles, nofma, direct32, n_dump):
    mats, d_tiles, g_tiles = _c32(mats), _c32(d_tiles), _c32(g_tiles)
    S = mats.shape[0]
    nt = d_tiles.shape[0]
    sums = np.zeros((S, 5))
    maxs = np.zeros((S, 2))
    ydump = np.zeros((S, n_dump, m ** dims), dtype=np.float32) if n_dump else None
    rc = lib().oref_sweep(dims, m, r, S, _p(mats, ctypes.c_float), nt, _p(d_tiles, ctypes.c_float),
                          _p(g_tiles, ctypes.c_float), int(nofma), int(direct32),
                          _p(sums, ctypes.c_double), _p(maxs, ctypes.c_double), int(n_dump),
                          _p(ydump, ctypes.c_float))
    if rc:
        raise ValueError("oref_sweep failed")
    return sums, maxs, ydump


def conv2d_wino(x, w, pad, m, points, nofma=False, n_lo=0, n_hi=None, mats=None) -> np.ndarray:
    """O4/O5 fp32 Winograd layer; returns y [N,K,Ho,Wo] (images outside [n_lo,n_hi) are 0)."""
    x, w = _c32(x), _c32(w)
    N, C, H, W = x.shape
    K, C2, r, r2 = w.shape
    assert C2 == C and r2 == r
    if n_hi is None:
        n_hi = N
    if mats is None:
        AT, G, BT = r64.build_f32(m, r, points)
    else:
        AT, G, BT = mats
    AT, G, BT = _c32(AT), _c32(G), _c32(BT)
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    y = np.zeros((N, K, Ho, Wo), dtype=np.float32)
    rc = lib().oref_conv2d_wino(_p(x, ctypes.c_float), _p(w, ctypes.c_float), _p(y, ctypes.c_float),
                                N, C, H, W, K, r, pad, m, _p(AT, ctypes.c_float), _p(G, ctypes.c_float),
                                _p(BT, ctypes.c_float), int(nofma), n_lo, n_hi)
    if rc:
        raise ValueError("oref_conv2d_wino failed")
    return y


def conv2d_direct64(x, w, pad, n_lo=0, n_hi=None) -> np.ndarray:
    x, w = _c32(x), _c32(w)
    N, C, H, W = x.shape
    K, _, r, _ = w.shape
    if n_hi is None:
        n_hi = N
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    y = np.zeros((N, K, Ho, Wo), dtype=np.float64)
    lib().oref_conv2d_direct64(_p(x, ctypes.c_float), _p(w, ctypes.c_float), _p(y, ctypes.c_double),
                               N, C, H, W, K, r, pad, n_lo, n_hi)
    return y


def stats(y32, y64, sums=None, maxs=None):
    """O8 (accumulating).  Returns (sums[5], maxs[2])."""
    y32 = _c32(y32).ravel()
    y64 = np.ascontiguousarray(y64, dtype=np.float64).ravel()
    if sums is None:
        sums = np.zeros(5)
    if maxs is None:
        maxs = np.zeros(2)
    lib().oref_stats(_p(y32, ctypes.c_float), _p(y64, ctypes.c_double), y32.size,
                     _p(sums, ctypes.c_double), _p(maxs, ctypes.c_double))
    return sums, maxs
