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
WINO_CONV_SCORE_PER_IMAGE = 4
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
    import torch
    N, C, H, W = x.shape
    K, C2, r, r2 = w.shape
    if C2 != C or r2 != r:
        raise ValueError("weight shape mismatch")
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    _check_tensor("x", x, torch.float32, (N, C, H, W))
    _check_tensor("w", w, torch.float32, (K, C, r, r))
    _check_tensor("y", y, torch.float32, (N, K, Ho, Wo))
    if (d_sums is None) != (d_maxs is None):
        raise ValueError("d_sums and d_maxs: both or neither")
    if d_sums is not None:
        rows = (N,) if flags & WINO_CONV_SCORE_PER_IMAGE else ()
        _check_tensor("d_sums", d_sums, torch.float64, rows + (WINO_SUMS,))
        _check_tensor("d_maxs", d_maxs, torch.float64, rows + (WINO_MAXS,))
    pts = _np64(points)
    if pts.shape != (m + r - 1,):
        raise ValueError(f"points: expected {m + r - 1} values, got {pts.shape}")
    args = (_ptr(x), _ptr(w), _ptr(y), N, C, H, W, K, r, pad, m, pts.ctypes.data_as(_d),
            _ptr(workspace), workspace.numel() * workspace.element_size(), _ptr(d_sums), _ptr(d_maxs))
    if flags:
        st = load().wino_conv2d_fp32_ex(*args, flags, _stream_ptr(stream))
        check(st, "wino_conv2d_fp32_ex")
    else:
        st = load().wino_conv2d_fp32(*args, _stream_ptr(stream))
        check(st, "wino_conv2d_fp32")


def wino_conv2d_relu_pool_fp32(x, w, y, act, pad: int, m: int, points: Sequence[float], workspace, pool: int,
                               d_sums=None, d_maxs=None, stream=None, flags: int = 0) -> None:
    """The layer with ReLU (+ 2x2 max pool) fused: act [N,K,Ho/pool,Wo/pool] fp32 CUDA tensor;
    y [N,K,Ho,Wo] or None (required when scoring)."""
    import torch
    N, C, H, W = x.shape
    K, C2, r, r2 = w.shape
    if C2 != C or r2 != r:
        raise ValueError("weight shape mismatch")
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    _check_tensor("x", x, torch.float32, (N, C, H, W))
    _check_tensor("w", w, torch.float32, (K, C, r, r))
    if y is not None:
        _check_tensor("y", y, torch.float32, (N, K, Ho, Wo))
    _check_tensor("act", act, torch.float32, (N, K, Ho // pool, Wo // pool))
    if (d_sums is None) != (d_maxs is None):
        raise ValueError("d_sums and d_maxs: both or neither")
    if d_sums is not None:
        rows = (N,) if flags & WINO_CONV_SCORE_PER_IMAGE else ()
        _check_tensor("d_sums", d_sums, torch.float64, rows + (WINO_SUMS,))
        _check_tensor("d_maxs", d_maxs, torch.float64, rows + (WINO_MAXS,))
    pts = _np64(points)
    if pts.shape != (m + r - 1,):
        raise ValueError(f"points: expected {m + r - 1} values, got {pts.shape}")
    st = load().wino_conv2d_relu_pool_fp32(_ptr(x), _ptr(w), _ptr(y), _ptr(act), N, C, H, W, K, r, pad, m,
                                          pts.ctypes.data_as(_d), _ptr(workspace),
                                          workspace.numel() * workspace.element_size(), _ptr(d_sums), _ptr(d_maxs),
                                          pool, flags, _stream_ptr(stream))
    check(st, "wino_conv2d_relu_pool_fp32")


def wino_conv2d_gemm_tile(N: int, C: int, H: int, W: int, K: int, r: int, pad: int, m: int) -> int:
    """Diagnostic: 1000 * k_rows + t_cols of the contraction's CTA tile, 1 for the fused C <= 4 kernel."""
    return int(load().wino_conv2d_gemm_tile(N, C, H, W, K, r, pad, m))


def wino_relu_pool_fp32(x, y, pool: int, stream=None) -> None:
    """y = maxpool_pool(ReLU(x)); x [N,C,H,W], y [N,C,H/pool,W/pool] fp32 CUDA tensors."""
    import torch
    N, C, H, W = x.shape
    _check_tensor("x", x, torch.float32, (N, C, H, W))
    _check_tensor("y", y, torch.float32, (N, C, H // pool, W // pool))
    check(load().wino_relu_pool_fp32(_ptr(x), _ptr(y), N, C, H, W, pool, _stream_ptr(stream)), "wino_relu_pool_fp32")


def wino_error_sweep_workspace_bytes(dims: int, m: int, r: int, n_cand: int, n_tiles: int) -> int:
    return int(load().wino_error_sweep_workspace_bytes(dims, m, r, n_cand, n_tiles))


def _check_tensor(name, t, dtype, shape):
    """Argument validation before a raw pointer crosses the ABI (a wrong dtype or too few
    rows would make the kernels read or write out of bounds)."""
    import torch
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return torch


def _sweep_args(dims, m, r, point_sets, d_tiles, g_tiles):
    import torch
    if dims not in (1, 2):
        raise ValueError("dims must be 1 or 2")
    n = m + r - 1
    ps = _np64(point_sets)
    if ps.size == 0:
        ps = ps.reshape(0, n)
    if ps.ndim != 2 or ps.shape[1] != n:
        raise ValueError(f"point_sets: expected [S, {n}], got {ps.shape}")
    S = ps.shape[0]
    T = d_tiles.shape[0]
    _check_tensor("d_tiles", d_tiles, torch.float32, (T, n ** dims))
    _check_tensor("g_tiles", g_tiles, torch.float32, (T, r ** dims))
    return ps, S, T


def _ws_size(workspace) -> int:
    return workspace.numel() * workspace.element_size() if workspace is not None else 0


def wino_error_sweep(dims: int, m: int, r: int, point_sets, d_tiles, g_tiles, d_sums, d_maxs,
                     workspace, flags: int = 0, stream=None) -> np.ndarray:
    """point_sets: host [S, n] fp64; d_tiles/g_tiles: CUDA fp32 [T, n^dims]/[T, r^dims];
    d_sums [S,5] / d_maxs [S,2] CUDA fp64 (accumulated; NaN rows for rejected candidates).
    Returns the per-candidate status."""
    import torch
    ps, S, T = _sweep_args(dims, m, r, point_sets, d_tiles, g_tiles)
    _check_tensor("d_sums", d_sums, torch.float64, (S, WINO_SUMS))
    _check_tensor("d_maxs", d_maxs, torch.float64, (S, WINO_MAXS))
    status = np.zeros(max(S, 1), dtype=np.int32)
    st = load().wino_error_sweep(dims, m, r, ps.ctypes.data_as(_d), S, _ptr(d_tiles), _ptr(g_tiles), T,
                                 _ptr(d_sums), _ptr(d_maxs), status.ctypes.data_as(_i), _ptr(workspace),
                                 _ws_size(workspace), flags, _stream_ptr(stream))
    check(st, "wino_error_sweep")
    return status[:S]


def wino_sweep_outputs(dims: int, m: int, r: int, point_sets, d_tiles, g_tiles, d_y, workspace=None,
                       d_sums=None, d_maxs=None, flags: int = 0, stream=None) -> np.ndarray:
    """The production sweep kernels with the fp32 outputs written to d_y: CUDA fp32
    [S, T, m^dims] (rows of accepted candidates overwritten).  workspace: uint8 CUDA tensor
    of wino_error_sweep_workspace_bytes (allocated here when None); d_sums/d_maxs as in
    wino_error_sweep, or None."""
    import torch
    ps, S, T = _sweep_args(dims, m, r, point_sets, d_tiles, g_tiles)
    _check_tensor("d_y", d_y, torch.float32, (S, T, m ** dims))
    if (d_sums is None) != (d_maxs is None):
        raise ValueError("d_sums and d_maxs: both or neither")
    if d_sums is not None:
        _check_tensor("d_sums", d_sums, torch.float64, (S, WINO_SUMS))
        _check_tensor("d_maxs", d_maxs, torch.float64, (S, WINO_MAXS))
    if workspace is None:
        workspace = torch.empty(max(1, wino_error_sweep_workspace_bytes(dims, m, r, S, T)), dtype=torch.uint8,
                                device=d_tiles.device)
    status = np.zeros(max(S, 1), dtype=np.int32)
    st = load().wino_sweep_outputs(dims, m, r, ps.ctypes.data_as(_d), S, _ptr(d_tiles), _ptr(g_tiles), T,
                                   _ptr(d_y), _ptr(d_sums), _ptr(d_maxs), status.ctypes.data_as(_i),
                                   _ptr(workspace), _ws_size(workspace), flags, _stream_ptr(stream))
    check(st, "wino_sweep_outputs")
    return status[:S]


def wino_last_launch_count() -> int:
    return int(load().wino_last_launch_count())


def wino_huffman_jit_mode(mode: int) -> int:
    """Huffman-order sweep kernels: 0 auto, 1 run-time specialised always, 2 interpreter
    always (include/wino.h).  Returns the previous mode."""
    return int(load().wino_huffman_jit_mode(int(mode)))


def wino_huffman_jit_classes() -> int:
    return int(load().wino_huffman_jit_classes())


def wino_huffman_jit_compile_check(dims: int, m: int, r: int, points) -> int:
    """Generate and NVRTC-compile (host only) the Huffman-order kernel of one point set's
    class; returns the sm_100a cubin size in bytes."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    out = ctypes.c_size_t(0)
    check(load().wino_huffman_jit_compile_check(int(dims), int(m), int(r),
                                                pts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(out)),
          "wino_huffman_jit_compile_check")
    return int(out.value)


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
