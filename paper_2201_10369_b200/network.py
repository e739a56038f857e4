"""configs[4]: the VGG-16 conv stack with every 3x3 convolution as an F(m x m, 3 x 3)
Winograd layer (§6.4 protocol, on synthetic inputs): per layer
wino_conv2d_fp32 (scored against the fp64 direct convolution of the same fp32 input --
the isolated per-layer error, reading R13 of DESIGN.md) then wino_relu_pool_fp32.
Every step runs in libwino's kernels; this module only sequences the calls."""
from __future__ import annotations

from typing import List, Optional, Sequence

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


def vgg16_forward(x, weights: Sequence, points, m: int = 6, score: bool = True, keep: bool = False,
                  stream=None):
    """x: CUDA [N,3,H,H] fp32; weights: 13 CUDA [K,C,3,3] fp32.  Returns (activation after
    the last pool, sums [13,5] | None, maxs [13,2] | None, conv outputs [13] if keep)."""
    return stack_forward(VGG16, x, weights, points, m, score, keep, stream)


def stack_forward(layers, x, weights: Sequence, points, m: int = 6, score: bool = True, keep: bool = False,
                  stream=None):
    """Generic 3x3 conv stack (C, K, H, pool_after) per layer: Winograd conv (scored) ->
    ReLU (-> 2x2 max pool).  Returns (final activation, sums [L,5], maxs [L,2], outputs)."""
    import torch
    N, _, H, W = x.shape
    dev = x.device
    VGG = layers
    wsb = 0
    h = H
    for (C, K, _, pool), w in zip(VGG, weights):
        assert tuple(w.shape) == (K, C, 3, 3)
        wsb = max(wsb, api.wino_conv2d_workspace_bytes(N, C, h, h, K, 3, 1, m))
        h = h // 2 if pool else h
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    sums = torch.zeros((len(VGG), 5), dtype=torch.float64, device=dev) if score else None
    maxs = torch.zeros((len(VGG), 2), dtype=torch.float64, device=dev) if score else None
    outs: List = []
    a = x
    for li, ((C, K, _, pool), w) in enumerate(zip(VGG, weights)):
        h = a.shape[2]
        y = torch.empty((N, K, h, h), dtype=torch.float32, device=dev)
        api.wino_conv2d_fp32(a, w, y, 1, m, points, ws, sums[li] if score else None,
                             maxs[li] if score else None, stream)
        if keep:
            outs.append(y)
        p = 2 if pool else 1
        a2 = torch.empty((N, K, h // p, h // p), dtype=torch.float32, device=dev)
        api.wino_relu_pool_fp32(y, a2, p, stream)
        a = a2
    return a, sums, maxs, outs


def normalized_l1(sums, n_images: int) -> float:
    """Σ_layers Σ_images Σ_elements |e| / (images x layers) (reading R12)."""
    s = sums.cpu().numpy() if hasattr(sums, "cpu") else sums
    return float(s[:, 0].sum() / (n_images * s.shape[0]))
