"""ORACLE (test infrastructure only) -- the configs[4] VGG-16 chain (O10): per layer the
O4/O5 Winograd layer (ref.conv2d_wino), scored against the fp64 direct convolution of the
same fp32 input (isolated per-layer error), then ReLU and 2x2/2 max pool written out in
numpy (exact operations)."""
import numpy as np

from . import ref

VGG16 = [
    (3, 64, 224, False), (64, 64, 224, True),
    (64, 128, 112, False), (128, 128, 112, True),
    (128, 256, 56, False), (256, 256, 56, False), (256, 256, 56, True),
    (256, 512, 28, False), (512, 512, 28, False), (512, 512, 28, True),
    (512, 512, 14, False), (512, 512, 14, False), (512, 512, 14, True),
]


def relu_pool(y: np.ndarray, pool: bool) -> np.ndarray:
    a = np.maximum(y, np.float32(0.0))
    if not pool:
        return a
    N, C, H, W = a.shape
    a = a[:, :, : H // 2 * 2, : W // 2 * 2].reshape(N, C, H // 2, 2, W // 2, 2)
    return a.max(axis=(3, 5))


def vgg16(x, weights, points, m=6, score=True):
    """Returns (conv outputs per layer, sums [13,5], maxs [13,2])."""
    return stack(VGG16, x, weights, points, m, score)


def stack(layers, x, weights, points, m=6, score=True):
    """Generic (C, K, H, pool_after) 3x3 stack; returns (conv outputs, sums [L,5], maxs [L,2])."""
    L = len(layers)
    outs, S, Mx = [], np.zeros((L, 5)), np.zeros((L, 2))
    a = x
    for li, ((C, K, _, pool), w) in enumerate(zip(layers, weights)):
        y = ref.conv2d_wino(a, w, 1, m, points)
        if score:
            y64 = ref.conv2d_direct64(a, w, 1)
            ref.stats(y, y64, S[li], Mx[li])
        outs.append(y)
        a = relu_pool(y, pool)
    return outs, S, Mx
