"""NEXT row N3: the tcgen05 kind::tf32 channel contraction (WINO_CONV_TF32), a separately
reported variant WITHOUT the fp32 parity semantics.  Pins: (a) on inputs whose transformed
operands are exactly representable in TF32 (F(2x2,3x3) on {0,-1,1,inf}, small integers) the
layer equals the exact direct correlation, which checks the tensor-core operand layouts,
descriptors, pipeline and epilogue element by element across ragged C/K/T tiles; (b) on the
paper's workloads its error against the fp64 direct convolution stays within the TF32
rounding bound, next to the fp32 FFMA path on the same inputs."""
import math

import numpy as np
import pytest

import synth
from oracle import points as OP, ref

pytestmark = pytest.mark.gpu
INF = math.inf


def _run(x, w, pad, m, pts, flags, score=True):
    import torch
    from paper_2201_10369_b200 import api
    y, s, mx = api.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), pad, m, pts, score=score,
                          flags=flags)
    torch.cuda.synchronize()
    return y.cpu().numpy(), (s.cpu().numpy() if score else None), (mx.cpu().numpy() if score else None)


@pytest.mark.parametrize("N,C,H,W,K", [
    (1, 8, 16, 16, 8),          # one tile in every dimension
    (2, 45, 37, 29, 130),       # C ragged over 32, K over 128, T = 2*19*15 = 570 over 256
    (3, 64, 40, 40, 256),
])
@pytest.mark.parametrize("flags", [1, 2])
def test_tf32_exact_on_representable_operands(N, C, H, W, K, flags):
    """flags 1 = 1xTF32, 2 = 3xTF32 (whose lo planes are then exactly zero)."""
    x, w = synth.integer_layer_inputs(N, C, H, W, K, 3, lo=-3, hi=3, seed=21)
    y64 = ref.conv2d_direct64(x, w, 1)
    assert np.abs(y64).max() < 2 ** 20
    y, s, mx = _run(x, w, 1, 2, OP.f23_c(1.0), flags=flags)
    assert np.array_equal(y.astype(np.float64), y64)
    assert s[0] == 0.0 and mx[0] == 0.0 and s[3] == y64.size


@pytest.mark.parametrize("N,C,H,W,K,r,pad,m,pts", [
    (2, 256, 56, 56, 256, 3, 1, 6, OP.n8_cd(2.0, 1.003)),       # configs[2] shape, 2 images
    (2, 128, 64, 64, 128, 5, 2, 4, OP.n8_c1c2(1.5, 3.1)),       # configs[3] shape, 2 images
    (2, 64, 32, 32, 64, 3, 1, 4, OP.f43_c(1.622)),
])
def test_tf32_error_bound(N, C, H, W, K, r, pad, m, pts):
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=3)
    y32, s32, _ = _run(x, w, pad, m, pts, flags=0)
    ytf, stf, mtf = _run(x, w, pad, m, pts, flags=1)
    assert np.all(np.isfinite(ytf)) and stf[3] == ytf.size and stf[4] == 0
    mae32 = s32[0] / s32[3]
    maetf = stf[0] / stf[3]
    # The variant rounds each GEMM operand to TF32 (round to nearest: unit roundoff 2^-11,
    # against 2^-24 for fp32); rounding errors in U and V are amplified by the output
    # transform exactly as the fp32 rounding errors of the transforms are, so its MAE scales
    # like the fp32 MAE times the roundoff ratio 2^13.  We require the MAE to lie within
    # [2^4, 2^15] x the fp32 path's MAE on the same inputs (the lower end proves the operands
    # were rounded), and the element errors of image 0 against the fp64 direct conv to agree
    # with the scored MAE.
    assert mae32 * 2.0 ** 4 < maetf < mae32 * 2.0 ** 15
    y64 = ref.conv2d_direct64(x[:1], w, pad)
    err0 = np.abs(ytf[:1].astype(np.float64) - y64).mean()
    assert 0.5 < err0 / maetf < 2.0
    print(f"\nm={m} r={r}: MAE fp32 {mae32:.3e}  tf32 {maetf:.3e}  ratio 2^{math.log2(maetf / mae32):.2f}")


@pytest.mark.parametrize("N,C,H,W,K,r,pad,m,pts", [
    (2, 256, 56, 56, 256, 3, 1, 6, OP.n8_cd(2.0, 1.003)),
    (2, 128, 64, 64, 128, 5, 2, 4, OP.n8_c1c2(1.5, 3.1)),
    (1, 45, 29, 37, 130, 3, 1, 4, OP.f43_c(1.622)),          # ragged C, K, T
])
def test_3xtf32_recovers_fp32_accuracy(N, C, H, W, K, r, pad, m, pts):
    """3xTF32 (hi/lo split, three MMAs): the dropped lo*lo term is 2^-22 relative and the
    fp32 accumulation matches the FFMA path's, so its MAE against fp64 direct is the fp32
    path's within a factor 2 (vs 2^10 for 1xTF32), and its outputs stay within a few fp32
    rounding errors of the parity path's."""
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=3)
    y32, s32, _ = _run(x, w, pad, m, pts, flags=0)
    y3, s3, _ = _run(x, w, pad, m, pts, flags=2)
    assert s3[3] == y3.size and s3[4] == 0
    mae32, mae3 = s32[0] / s32[3], s3[0] / s3[3]
    assert 0.5 * mae32 < mae3 < 2.0 * mae32
    assert np.abs(y3 - y32).mean() < 2.0 * mae32
    print(f"\nm={m} r={r}: MAE fp32 {mae32:.3e}  3xtf32 {mae3:.3e}")
