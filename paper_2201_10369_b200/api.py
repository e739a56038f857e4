"""Python binding of include/wino.h -- the same names, argument marshalling only.

Device buffers are torch CUDA tensors (PyTorch supplies device memory and streams);
host arrays are numpy.  Nothing here computes any step of the method.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np

from ._lib import check, load

WINO_SUMS = 5
WINO_MAXS = 2
WINO_SWEEP_NOFMA = 1
WINO_SWEEP_HUFFMAN = 2
WINO_SWEEP_MIXED = 4
WINO_CONV_TF32 = 1
WINO_CONV_3XTF32 = 2
WINO_MAX_N = 16

_d = ctypes.POINTER(ctypes.c_double)
_i = ctypes.POINTER(ctypes.c_int)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _np64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def wino_supported(dims: int, m: int, r: int) -> bool:
    """dims 1|2: sweep kernels; dims 0: layer kernels."""
    return bool(load().wino_supported(dims, m, r))


def wino_points_to_matrices(m: int, r: int, points: Sequence[float]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(Aᵀ [m,n], G [n,r], Bᵀ [n,n]) fp64, recipe R64 (host, synchronous)."""
    pts = _np64(points)
    n = pts.size
    AT = np.empty((m, n))
    G = np.empty((n, r))
    BT = np.empty((n, n))
    st = load().wino_points_to_matrices(m, r, pts.ctypes.data_as(_d), n, AT.ctypes.data_as(_d),
                                        G.ctypes.data_as(_d), BT.ctypes.data_as(_d))
    check(st, "wino_points_to_matrices")
    return AT, G, BT


def wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, m) -> int:
    return int(load().wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, m))


def wino_conv2d_fp32(x, w, y, pad: int, m: int, points: Sequence[float], workspace,
                     d_sums=None, d_maxs=None, stream=None, flags: int = 0) -> None:
    """x [N,C,H,W], w [K,C,r,r], y [N,K,Ho,Wo] fp32 CUDA tensors; workspace uint8 CUDA
    tensor; d_sums [5] / d_maxs [2] fp64 CUDA tensors (accumulated) or None.  flags != 0
    calls wino_conv2d_fp32_ex (WINO_CONV_TF32: the tensor-core variant)."""
    N, C, H, W = x.shape
    K, C2, r, r2 = w.shape
    if C2 != C or r2 != r:
        raise ValueError("weight shape mismatch")
    pts = _np64(points)
    args = (_ptr(x), _ptr(w), _ptr(y), N, C, H, W, K, r, pad, m, pts.ctypes.data_as(_d),
            _ptr(workspace), workspace.numel() * workspace.element_size(), _ptr(d_sums), _ptr(d_maxs))
    if flags:
        st = load().wino_conv2d_fp32_ex(*args, flags, _stream_ptr(stream))
        check(st, "wino_conv2d_fp32_ex")
    else:
        st = load().wino_conv2d_fp32(*args, _stream_ptr(stream))
        check(st, "wino_conv2d_fp32")


def wino_relu_pool_fp32(x, y, pool: int, stream=None) -> None:
    """y = maxpool_pool(ReLU(x)); x [N,C,H,W], y [N,C,H/pool,W/pool] fp32 CUDA tensors."""
    N, C, H, W = x.shape
    if tuple(y.shape) != (N, C, H // pool, W // pool):
        raise ValueError("output shape mismatch")
    check(load().wino_relu_pool_fp32(_ptr(x), _ptr(y), N, C, H, W, pool, _stream_ptr(stream)), "wino_relu_pool_fp32")


def wino_error_sweep_workspace_bytes(dims: int, m: int, r: int, n_cand: int, n_tiles: int) -> int:
    return int(load().wino_error_sweep_workspace_bytes(dims, m, r, n_cand, n_tiles))


def wino_error_sweep(dims: int, m: int, r: int, point_sets, d_tiles, g_tiles, d_sums, d_maxs,
                     workspace, flags: int = 0, stream=None) -> np.ndarray:
    """point_sets: host [S, n] fp64; d_tiles/g_tiles: CUDA fp32 [T, n^dims]/[T, r^dims];
    d_sums [S,5] / d_maxs [S,2] CUDA fp64 (accumulated).  Returns per-candidate status."""
    ps = _np64(point_sets)
    S = ps.shape[0] if ps.ndim == 2 else 0
    status = np.zeros(max(S, 1), dtype=np.int32)
    nt = d_tiles.shape[0]
    st = load().wino_error_sweep(dims, m, r, ps.ctypes.data_as(_d), S, _ptr(d_tiles), _ptr(g_tiles), nt,
                                 _ptr(d_sums), _ptr(d_maxs), status.ctypes.data_as(_i), _ptr(workspace),
                                 workspace.numel() * workspace.element_size() if workspace is not None else 0,
                                 flags, _stream_ptr(stream))
    check(st, "wino_error_sweep")
    return status[:S]


def wino_sweep_outputs(dims: int, m: int, r: int, point_sets, d_tiles, g_tiles, d_y, flags: int = 0,
                       stream=None) -> np.ndarray:
    """d_y: CUDA fp32 [S, T, m^dims] (overwritten for accepted candidates)."""
    ps = _np64(point_sets)
    S = ps.shape[0]
    status = np.zeros(max(S, 1), dtype=np.int32)
    st = load().wino_sweep_outputs(dims, m, r, ps.ctypes.data_as(_d), S, _ptr(d_tiles), _ptr(g_tiles),
                                   d_tiles.shape[0], _ptr(d_y), status.ctypes.data_as(_i), flags,
                                   _stream_ptr(stream))
    check(st, "wino_sweep_outputs")
    return status[:S]


def wino_last_launch_count() -> int:
    return int(load().wino_last_launch_count())


def wino_timing_enable(enable: bool) -> bool:
    return bool(load().wino_timing_enable(int(enable)))


def wino_timing_reset() -> None:
    load().wino_timing_reset()


def wino_timing_read(family: str) -> Tuple[float, int]:
    ms = ctypes.c_double(0.0)
    n = ctypes.c_int(0)
    check(load().wino_timing_read(family.encode(), ctypes.byref(ms), ctypes.byref(n)), "wino_timing_read")
    return ms.value, n.value


# ------------------------------------------------------------------ convenience (still marshalling only)

def conv2d(x, w, pad: int, m: int, points, score: bool = False, stream=None, flags: int = 0):
    """Allocate y / workspace with torch and run wino_conv2d_fp32.  Returns (y, sums, maxs)."""
    import torch
    N, C, H, W = x.shape
    K, _, r, _ = w.shape
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    y = torch.empty((N, K, Ho, Wo), dtype=torch.float32, device=x.device)
    ws = torch.empty(wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, m), dtype=torch.uint8, device=x.device)
    sums = maxs = None
    if score:
        sums = torch.zeros(WINO_SUMS, dtype=torch.float64, device=x.device)
        maxs = torch.zeros(WINO_MAXS, dtype=torch.float64, device=x.device)
    wino_conv2d_fp32(x, w, y, pad, m, points, ws, sums, maxs, stream, flags)
    return y, sums, maxs
