"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no points, no matrices, no
convolution).  It only draws the data both sides consume, so that the GPU run
and the oracle read byte-identical inputs (SURVEY §8(d) "Synthetic inputs";
DESIGN.md "Input recipe").

Recipe:
  * generator: numpy PCG64 ``default_rng(seed)``; draw float64, round to float32
    (round-to-nearest-even, ``astype(np.float32)``);
  * "uniform" = ``uniform(-1, 1)`` -- the paper's "randomly generated input data"
     read as uniform[-1,1] for input *and* kernel (DESIGN.md
    reading R9, pinned by the T7/T8 n=0 rows P:622);
  * "normal" = ``standard_normal`` (BASELINE.json configs[1] second distribution);
  * "he" = N(0, 2/(C r^2)) weights (configs[2], configs[4]);
  * tiles: d first, then g; layers: x first, then w.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "draw",
    "random_tiles",
    "layer_inputs",
    "integer_layer_inputs",
    "integer_tiles",
    "c_grid",
    "vgg16_inputs",
    "VGG16_CONVS",
]


def draw(rng: np.random.Generator, shape, dist: str, scale: float = 1.0) -> np.ndarray:
    """One fp32 array drawn in fp64 then rounded to nearest fp32."""
    if dist == "uniform":
        a = rng.uniform(-1.0, 1.0, size=shape)
    elif dist == "normal":
        a = rng.standard_normal(size=shape)
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    if scale != 1.0:
        a = a * scale
    return a.astype(np.float32)


def random_tiles(n_tiles: int, dims: int, n: int, r: int, dist: str = "uniform", seed: int = 0):
    """Independent random tiles for the error sweep ("5000 randomly generated
    input data"; BASELINE.json configs[1] uses 100k).

    Returns (d, g): d float32 [n_tiles, n**dims], g float32 [n_tiles, r**dims]
    (row-major n x n / r x r tiles in 2D).
    """
    if dims not in (1, 2):
        raise ValueError("dims must be 1 or 2")
    rng = np.random.default_rng(seed)
    d = draw(rng, (n_tiles, n ** dims), dist)
    g = draw(rng, (n_tiles, r ** dims), dist)
    return np.ascontiguousarray(d), np.ascontiguousarray(g)


def integer_tiles(n_tiles: int, dims: int, n: int, r: int, lo: int = -16, hi: int = 16, seed: int = 0):
    """Integer-valued fp32 tiles (used by the exactness pins)."""
    rng = np.random.default_rng(seed)
    d = rng.integers(lo, hi + 1, size=(n_tiles, n ** dims)).astype(np.float32)
    g = rng.integers(lo, hi + 1, size=(n_tiles, r ** dims)).astype(np.float32)
    return d, g


def layer_inputs(N: int, C: int, H: int, W: int, K: int, r: int,
                 x_dist: str = "uniform", w_dist: str = "uniform", seed: int = 0):
    """x float32 [N,C,H,W] (NCHW), w float32 [K,C,r,r] (KCRS).  Draw x first, then w.
    ``w_dist='he'`` draws N(0, 2/(C r^2)) (He-normal)."""
    rng = np.random.default_rng(seed)
    x = draw(rng, (N, C, H, W), x_dist)
    if w_dist == "he":
        w = draw(rng, (K, C, r, r), "normal", scale=math.sqrt(2.0 / (C * r * r)))
    else:
        w = draw(rng, (K, C, r, r), w_dist)
    return x, w


def integer_layer_inputs(N: int, C: int, H: int, W: int, K: int, r: int,
                         lo: int = -16, hi: int = 16, seed: int = 0):
    rng = np.random.default_rng(seed)
    x = rng.integers(lo, hi + 1, size=(N, C, H, W)).astype(np.float32)
    w = rng.integers(lo, hi + 1, size=(K, C, r, r)).astype(np.float32)
    return x, w


def c_grid(count: int = 4096, lo: float = 0.05, hi: float = 20.0) -> np.ndarray:
    """Log-spaced parameter grid (BASELINE.json configs[1]: "4096 values of c
    log-spaced in [0.05,20]").  c_i = exp(ln lo + i (ln hi - ln lo)/(count-1)) in
    Python float, endpoints forced to lo and hi exactly (reading R15).
    The array is data: both sides receive it, neither recomputes it."""
    if count < 2:
        return np.array([lo], dtype=np.float64)
    a, b = math.log(lo), math.log(hi)
    out = [math.exp(a + i * (b - a) / (count - 1)) for i in range(count)]
    out[0], out[-1] = lo, hi
    return np.array(out, dtype=np.float64)


def vgg16_inputs(N: int, seed: int = 0, H: int = 224):
    """BASELINE.json configs[4]: x [N,3,H,H] ~ N(0,1) (standing in for per-channel
    standardised images), then each layer's He-normal weights [K,C,3,3] in stack order."""
    rng = np.random.default_rng(seed)
    x = draw(rng, (N, 3, H, H), "normal")
    ws = [draw(rng, (K, C, 3, 3), "normal", scale=math.sqrt(2.0 / (C * 9))) for C, K, _, _ in VGG16_CONVS]
    return x, ws


def stack_inputs(layers, N: int, seed: int = 0):
    """Synthetic conv stack inputs: x [N, C0, H0, H0] ~ N(0,1), He-normal weights per layer
    (NEXT row N4: CIFAR-shaped stand-ins, no dataset items, no trained weights)."""
    rng = np.random.default_rng(seed)
    C0, _, H0, _ = layers[0]
    x = draw(rng, (N, C0, H0, H0), "normal")
    ws = [draw(rng, (K, C, 3, 3), "normal", scale=math.sqrt(2.0 / (C * 9))) for C, K, _, _ in layers]
    return x, ws


# VGG-16 conv stack (BASELINE.json configs[4]): (C_in, K_out, H=W, pool_after)
VGG16_CONVS = [
    (3, 64, 224, False), (64, 64, 224, True),
    (64, 128, 112, False), (128, 128, 112, True),
    (128, 256, 56, False), (256, 256, 56, False), (256, 256, 56, True),
    (256, 512, 28, False), (512, 512, 28, False), (512, 512, 28, True),
    (512, 512, 14, False), (512, 512, 14, False), (512, 512, 14, True),
]
