"""configs[4]: the VGG-16 conv stack with every 3x3 convolution as an F(m x m, 3 x 3)
Winograd layer (§6.4 protocol, on synthetic inputs): per layer
wino_conv2d_fp32 (scored against the fp64 direct convolution of the same fp32 input --
the isolated per-layer error, reading R13 of DESIGN.md) with ReLU (+ 2x2 max pool) fused
into its output transform (wino_conv2d_relu_pool_fp32).
Every step runs in libwino's kernels; this module only sequences the calls.

Multi-GPU: one process per GPU, the batch sharded in contiguous image
blocks; each rank runs its images through all layers and scores them PER IMAGE
(WINO_CONV_SCORE_PER_IMAGE) into the rows of a zero-padded global [L][N][7] buffer; one
all_reduce(SUM) of that buffer (every row has exactly one owner, so the sum is exact);
then the per-layer statistics are reduced over images in ascending image order.  Each
image's statistics depend only on that image, so the result is bitwise independent of the
world size.  No activation exchange (the layers are data parallel)."""
from __future__ import annotations

import os
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import api

# (C_in, K_out, H=W, pool_after): VGG-16 "D" convolutions (BASELINE.json configs[4])
VGG16 = [
    (3, 64, 224, False), (64, 64, 224, True),
    (64, 128, 112, False), (128, 128, 112, True),
    (128, 256, 56, False), (256, 256, 56, False), (256, 256, 56, True),
    (256, 512, 28, False), (512, 512, 28, False), (512, 512, 28, True),
    (512, 512, 14, False), (512, 512, 14, False), (512, 512, 14, True),
]


# ResNet-20-shaped plain stack for the CIFAR-sized synthetic networks of NEXT row N4
# (ResNet-20 on CIFAR; widths 16/32/64 at 32/16/8; the stride-2 transitions are
# replaced by 2x2 max pools because the layer is stride 1; no residual adds -- the error
# protocol is per layer)
RESNET20_LIKE = ([(3, 16, 32, False)] + [(16, 16, 32, False)] * 5 + [(16, 16, 32, True)]
                 + [(16, 32, 16, False)] + [(32, 32, 16, False)] * 4 + [(32, 32, 16, True)]
                 + [(32, 64, 8, False)] + [(64, 64, 8, False)] * 5)

# SqueezeNet-shaped CIFAR stack ("SqueezeNet"; 8 of its 26 layers ran as
# Winograd layers): 8 chained 3x3 convolutions with the widths of SqueezeNet's 3x3 expand
# branches (64 at 32x32, 128 at 16x16, 192 / 256 at 8x8) -- the 1x1 squeeze / expand
# convolutions are not Winograd layers and are left out, so each 3x3 layer consumes the
# previous activation directly.  Each entry: (C, K, H, pool_after).
SQUEEZENET_LIKE = [
    (3, 64, 32, False), (64, 64, 32, True),
    (64, 128, 16, False), (128, 128, 16, True),
    (128, 192, 8, False), (192, 192, 8, False), (192, 256, 8, False), (256, 256, 8, False),
]


def vgg16_forward(x, weights: Sequence, points, m: int = 6, score: bool = True, keep: bool = False,
                  stream=None, **kw):
    """x: CUDA [N,3,H,H] fp32; weights: 13 CUDA [K,C,3,3] fp32.  Returns (activation after
    the last pool, sums [13,5] | None, maxs [13,2] | None, conv outputs [13] if keep)."""
    return stack_forward(VGG16, x, weights, points, m, score, keep, stream, **kw)


def shard(n: int, rank: int, world: int):
    """Contiguous block of [0, n) owned by `rank`."""
    return (n * rank) // world, (n * (rank + 1)) // world


def _abi_conv(a, w, y, act, pool, m, points, ws, sums, maxs, stream):
    """One layer: Winograd conv with the ReLU (+ pool) fused into its output transform
    (wino_conv2d_relu_pool_fp32); y (the conv output) is materialised only when given."""
    flags = api.WINO_CONV_SCORE_PER_IMAGE if sums is not None else 0
    api.wino_conv2d_relu_pool_fp32(a, w, y, act, 1, m, points, ws, pool, sums, maxs, stream, flags)


def _abi_ws(N, C, H, K, m):
    return api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m)


def stack_forward(layers, x, weights: Sequence, points, m: int = 6, score: bool = True, keep: bool = False,
                  stream=None, rank: int = 0, world: int = 1, n_global: Optional[int] = None, group=None,
                  conv: Callable = _abi_conv, ws_bytes: Callable = _abi_ws):
    """Generic 3x3 conv stack (C, K, H, pool_after) per layer: Winograd conv (scored) ->
    ReLU (-> 2x2 max pool).

    x: this rank's images [N_r, C, H, H] = images [lo, hi) of the global batch of n_global
    (default: N_r, world 1).  Returns (final activation of the rank's images, sums [L,5],
    maxs [L,2] over ALL images (after the all-reduce when world > 1), conv outputs if keep,
    per-image statistics [L, n_global, 7]).  `conv` / `ws_bytes` are the C-ABI calls; tests
    inject CPU stand-ins to check the sharding and reduction logic.  The conv output y of a
    layer is materialised only when it is scored or kept (otherwise the fused epilogue
    writes just the activation)."""
    import torch
    N, _, H, W = x.shape
    n_global = N if n_global is None else n_global
    lo, hi = shard(n_global, rank, world)
    if hi - lo != N:
        raise ValueError(f"rank {rank} holds {N} images, its shard is [{lo}, {hi})")
    dev = x.device
    L = len(layers)
    wsb = 0
    h = H
    for (C, K, _, pool), w in zip(layers, weights):
        assert tuple(w.shape) == (K, C, 3, 3)
        wsb = max(wsb, ws_bytes(N, C, h, K, m) if N > 0 else 0)
        h = h // 2 if pool else h
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    # one flat zero-padded buffer: [L][n_global][5] sums then [L][n_global][2] maxs
    flat = torch.zeros(L * n_global * 7, dtype=torch.float64, device=dev) if score else None
    sums_img = flat[:L * n_global * 5].view(L, n_global, 5) if score else None
    maxs_img = flat[L * n_global * 5:].view(L, n_global, 2) if score else None
    outs: List = []
    a = x
    for li, ((C, K, _, pool), w) in enumerate(zip(layers, weights)):
        h = a.shape[2]
        y = torch.empty((N, K, h, h), dtype=torch.float32, device=dev) if (score or keep) else None
        p = 2 if pool else 1
        a2 = torch.empty((N, K, h // p, h // p), dtype=torch.float32, device=dev)
        if N > 0:
            conv(a, w, y, a2, p, m, points, ws, sums_img[li, lo:hi] if score else None,
                 maxs_img[li, lo:hi] if score else None, stream)
        if keep:
            outs.append(y)
        a = a2
    if not score:
        return a, None, None, outs, None
    import torch.distributed as dist
    # (WINO_FORCE_COLLECTIVES=1: also with one rank, so a 1-GPU box exercises the NCCL call)
    if world > 1 or (os.environ.get("WINO_FORCE_COLLECTIVES") == "1" and dist.is_initialized()):
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)   # exact: one owner per row
    per_img = np.concatenate([sums_img.cpu().numpy(), maxs_img.cpu().numpy()], axis=2)
    sums, maxs = reduce_images(per_img)
    return a, sums, maxs, outs, per_img


def reduce_images(per_img: np.ndarray):
    """[L, N, 7] per-image statistics -> per-layer sums [L, 5] (Σ over images in ascending
    order) and maxs [L, 2] (max over images)."""
    L, N, _ = per_img.shape
    sums = np.zeros((L, 5))
    maxs = np.zeros((L, 2))
    for i in range(N):
        sums += per_img[:, i, :5]
        maxs = np.maximum(maxs, per_img[:, i, 5:])
    return sums, maxs


def normalized_l1(sums, n_images: int) -> float:
    """Σ_layers Σ_images Σ_elements |e| / (images x layers) (reading R12)."""
    s = sums.cpu().numpy() if hasattr(sums, "cpu") else np.asarray(sums)
    return float(s[:, 0].sum() / (n_images * s.shape[0]))
