"""GPU parity of the fp32 Winograd layer (wino_conv2d_fp32) against the oracle's O4/O5
layer: outputs bit-identical; scored statistics vs the oracle's fp64 direct convolution
within the north-star tolerance (we assert 1e-9 relative on the MAE)."""
import math

import numpy as np
import pytest

import synth
from oracle import points as OP, ref

pytestmark = pytest.mark.gpu
INF = math.inf


def _run(x, w, pad, m, pts, score=True):
    import torch
    from paper_2201_10369_b200 import api
    y, s, mx = api.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), pad, m, pts, score=score)
    torch.cuda.synchronize()
    return y.cpu().numpy(), (s.cpu().numpy() if score else None), (mx.cpu().numpy() if score else None)


def _oracle_stats(x, w, pad, y_oracle):
    y64 = ref.conv2d_direct64(x, w, pad)
    return ref.stats(y_oracle, y64)


def _check_stats(s, mx, s_ref, m_ref):
    assert s[3] == s_ref[3] and s[4] == s_ref[4]
    assert np.array_equal(mx, m_ref)
    assert abs((s[0] / s[3]) / (s_ref[0] / s_ref[3]) - 1) < 1e-9
    assert abs(s[1] / s_ref[1] - 1) < 1e-9


def test_cfg1_full():
    """BASELINE.json configs[0]: F(2x2,3x3), {0,-1,1,inf}, N=1 C=K=8 16x16 pad 1, U[-1,1] seed 0."""
    x, w = synth.layer_inputs(1, 8, 16, 16, 8, 3, "uniform", "uniform", seed=0)
    pts = OP.f23_c(1.0)
    y, s, mx = _run(x, w, 1, 2, pts)
    y_ref = ref.conv2d_wino(x, w, 1, 2, pts)
    assert np.array_equal(y, y_ref)
    s_ref, m_ref = _oracle_stats(x, w, 1, y_ref)
    _check_stats(s, mx, s_ref, m_ref)
    assert 0 < s_ref[0] / s_ref[3] < 1e-6


def test_cfg1_integer_exact():
    x, w = synth.integer_layer_inputs(1, 8, 16, 16, 8, 3, seed=0)
    y, s, mx = _run(x, w, 1, 2, OP.f23_c(1.0))
    y64 = ref.conv2d_direct64(x, w, 1)
    assert np.array_equal(y.astype(np.float64), y64)
    assert s[0] == 0.0 and mx[0] == 0.0


@pytest.mark.parametrize("N,C,H,W,K,r,pad,m,pts", [
    (2, 13, 19, 23, 37, 3, 1, 6, OP.n8_cd(2.0, 1.003)),      # ragged everything, cfg3 template
    (2, 16, 20, 20, 8, 3, 1, 6, OP.P8),
    (1, 9, 17, 17, 130, 3, 0, 4, OP.f43_c(1.622)),
    (2, 8, 18, 18, 16, 3, 1, 2, OP.f23_c(1.0)),
    (1, 7, 21, 21, 9, 3, 1, 3, [-1.0, 0.0, 0.5, 1.0, INF]),
    (1, 6, 20, 20, 6, 3, 1, 5, [-2.0, -1.0, 0.0, 0.5, 1.0, 2.0, INF]),
    (2, 10, 21, 21, 12, 5, 2, 4, OP.n8_c1c2(1.5, 3.1)),
    (1, 10, 22, 22, 12, 5, 2, 6, OP.n10_c1c2(1.272, 2.099)),
    (1, 3, 9, 9, 4, 5, 2, 2, [-1.0, 0.0, 1.0, 2.0, -2.0, INF][:5] + [INF]),
])
def test_layer_bitexact(N, C, H, W, K, r, pad, m, pts):
    pts = sorted(p for p in pts if p != INF) + [INF]
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=3)
    y, s, mx = _run(x, w, pad, m, pts)
    y_ref = ref.conv2d_wino(x, w, pad, m, pts)
    assert np.array_equal(y, y_ref)
    s_ref, m_ref = _oracle_stats(x, w, pad, y_ref)
    _check_stats(s, mx, s_ref, m_ref)


def test_cfg3_full_size_sampled_images():
    """BASELINE.json configs[2] at full size (N=32, C=K=256, 56x56, F(6x6,3x3), X16 points)
    in the bench's launch configuration; images 0 and 31 recomputed by the oracle."""
    x, w = synth.layer_inputs(32, 256, 56, 56, 256, 3, "normal", "he", seed=0)
    pts = OP.n8_cd(2.0, 1.003)
    y, _, _ = _run(x, w, 1, 6, pts, score=False)
    for img in (0, 31):
        y_ref = ref.conv2d_wino(x, w, 1, 6, pts, n_lo=img, n_hi=img + 1)
        assert np.array_equal(y[img], y_ref[img])


def test_cfg3_shape_scored_two_images():
    x, w = synth.layer_inputs(2, 256, 56, 56, 256, 3, "normal", "he", seed=0)
    pts = OP.n8_cd(2.0, 1.003)
    y, s, mx = _run(x, w, 1, 6, pts)
    y_ref = ref.conv2d_wino(x, w, 1, 6, pts)
    assert np.array_equal(y, y_ref)
    s_ref, m_ref = _oracle_stats(x, w, 1, y_ref)
    _check_stats(s, mx, s_ref, m_ref)


def test_cfg4_full_size_image0():
    """BASELINE.json configs[3] shapes: N=16, C=K=128, 64x64, 5x5, F(4x4) and F(6x6)."""
    x, w = synth.layer_inputs(16, 128, 64, 64, 128, 5, "uniform", "uniform", seed=0)
    for m, pts in ((4, OP.n8_c1c2(1.5, 3.1)), (6, OP.n10_c1c2(1.272, 2.099))):
        y, _, _ = _run(x, w, 2, m, pts, score=False)
        y_ref = ref.conv2d_wino(x, w, 2, m, pts, n_lo=0, n_hi=1)
        assert np.array_equal(y[0], y_ref[0])


def test_layer_errors():
    import torch
    from paper_2201_10369_b200 import api, _lib
    x = torch.zeros((1, 2, 8, 8), device="cuda")
    w = torch.zeros((2, 2, 3, 3), device="cuda")
    y = torch.zeros((1, 2, 8, 8), device="cuda")
    ws = torch.empty(8, dtype=torch.uint8, device="cuda")
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_conv2d_fp32(x, w, y, 1, 2, OP.f23_c(1.0), ws)
    assert ei.value.status == 6
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_conv2d_fp32(x, w, y, 1, 2, [0.0, 0.0, 1.0, INF], ws)
    assert ei.value.status in (3, 6)
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_conv2d_fp32(x, w, y, 1, 9, [float(i) for i in range(10)] + [INF], ws)
    assert ei.value.status == 8


@pytest.mark.parametrize("N,C,H,K,m,pts,pool", [
    (2, 13, 19, 37, 6, OP.n8_cd(2.0, 1.003), 2),     # even m: fused pool, odd H (floor) + ragged tiles
    (2, 8, 16, 16, 6, OP.n8_cd(2.0, 1.003), 1),      # fused ReLU only
    (1, 9, 17, 20, 3, OP.canonical([0.0, 1.0, -1.0, 0.5]), 2),   # odd m: separate pool kernel
    (2, 8, 18, 16, 2, OP.f23_c(1.0), 2),
    (1, 5, 15, 7, 7, OP.chebyshev(9), 2),             # F(7x7,3x3) layer
    (1, 5, 20, 6, 8, OP.P10, 2),                      # F(8x8,3x3) layer
])
def test_fused_relu_pool_equals_separate(N, C, H, K, m, pts, pool):
    _fused_case(N, C, H, K, m, pts, pool)


def _fused_case(N, C, H, K, m, pts, pool):
    """wino_conv2d_relu_pool_fp32: act = maxpool(ReLU(conv)) bit for bit equal to the oracle
    layer followed by the oracle's ReLU / pool; y (when requested) equals the oracle layer;
    scored statistics per image sum to the whole-batch statistics."""
    import torch
    from oracle import network as ON
    from paper_2201_10369_b200 import api
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=7)
    y_ref = ref.conv2d_wino(x, w, 1, m, pts)
    a_ref = ON.relu_pool(y_ref, pool == 2)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m), dtype=torch.uint8, device="cuda")
    act = torch.full(a_ref.shape, float("nan"), dtype=torch.float32, device="cuda")
    y = torch.full(y_ref.shape, float("nan"), dtype=torch.float32, device="cuda")
    sums = torch.zeros((N, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((N, 2), dtype=torch.float64, device="cuda")
    api.wino_conv2d_relu_pool_fp32(xd, wd, y, act, 1, m, pts, ws, pool, sums, maxs,
                                   flags=api.WINO_CONV_SCORE_PER_IMAGE)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_ref)
    assert np.array_equal(act.cpu().numpy(), a_ref)
    s_ref, m_ref = ref.stats(y_ref, ref.conv2d_direct64(x, w, 1))
    s = sums.cpu().numpy().sum(axis=0)
    assert s[3] == s_ref[3] and s[4] == s_ref[4]
    assert abs(s[0] / s_ref[0] - 1) < 1e-9 and np.array_equal(maxs.cpu().numpy().max(axis=0), m_ref)
    if m % 2 == 0 or pool == 1:       # y not materialised: the activation alone
        act2 = torch.full(a_ref.shape, float("nan"), dtype=torch.float32, device="cuda")
        api.wino_conv2d_relu_pool_fp32(xd, wd, None, act2, 1, m, pts, ws, pool)
        torch.cuda.synchronize()
        assert np.array_equal(act2.cpu().numpy(), a_ref)


@pytest.mark.parametrize("N,C,H,K,m,pts,pool", [
    (3, 3, 40, 21, 6, OP.n8_cd(2.0, 1.003), 2),      # RGB, 147 tiles (2 CTAs, ragged), odd K over 2 k-groups
    (2, 3, 35, 16, 6, OP.n8_cd(2.0, 1.003), 1),      # odd H, ReLU only
    (1, 3, 26, 33, 6, OP.chebyshev(8), 2),           # dense (no zero family) F(6x6,3x3), 3 k-groups
    (2, 3, 19, 5, 6, OP.n8_cd(2.0, 1.003), 2),       # odd H with the fused pool (floor), ragged tiles
    (2, 1, 20, 5, 4, OP.f43_c(1.6), 2),              # C = 1
    (1, 3, 21, 6, 4, OP.f43_c(0.7), 2),              # m = 4, odd H, fused pool
    (1, 4, 18, 18, 2, OP.f23_c(1.0), 2),             # C = 4
    (2, 2, 17, 7, 3, OP.canonical([0.0, 1.0, -1.0, 0.5]), 2),   # odd m: separate pool kernel after the fused layer
    (1, 3, 23, 9, 5, [-2.0, -1.0, 0.0, 0.5, 1.0, 2.0, INF], 1),
])
def test_smallc_fused_layer(N, C, H, K, m, pts, pool):
    """C <= 4 layers run K2 + K3 + K4 as one kernel (smallc_kernel): outputs, fused
    activation and statistics equal the oracle's bit for bit, the kernel really is the one
    that ran, and the unfused pipeline (WINO_LAYER_NO_SMALLC=1) gives the same bits."""
    import os
    import torch
    from paper_2201_10369_b200 import api
    api.wino_timing_reset()
    api.wino_timing_enable(True)
    try:
        _fused_case(N, C, H, K, m, pts, pool)
        assert api.wino_timing_read("layer_smallc")[1] >= 1
        assert api.wino_timing_read("layer_gemm")[1] == 0
    finally:
        api.wino_timing_enable(False)
        api.wino_timing_reset()
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=7)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y1, _, _ = api.conv2d(xd, wd, 1, m, pts)
    os.environ["WINO_LAYER_NO_SMALLC"] = "1"
    try:
        y2, _, _ = api.conv2d(xd, wd, 1, m, pts)
    finally:
        del os.environ["WINO_LAYER_NO_SMALLC"]
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


def test_pdl_chain_equals_plain_launches():
    """The unfused layer runs K1 -> K2 -> K3 -> K4 as a programmatic-dependent-launch chain
    (kernels become resident while their predecessor drains and wait before touching its
    output).  At the configs[2] size, with the workspace dirtied between runs, every run of
    the chain gives the same bits as plainly serialised launches (WINO_LAYER_NO_PDL=1)."""
    import os
    import torch
    from paper_2201_10369_b200 import api
    N, C, H, K, m = 32, 256, 56, 256, 6
    pts = OP.n8_cd(2.0, 1.003)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    x = torch.randn((N, C, H, H), device="cuda", generator=g)
    w = torch.randn((K, C, 3, 3), device="cuda", generator=g) * (2.0 / (C * 9)) ** 0.5
    ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m), dtype=torch.uint8, device="cuda")
    y0 = torch.empty((N, K, H, H), device="cuda")
    os.environ["WINO_LAYER_NO_PDL"] = "1"
    try:
        api.wino_conv2d_fp32(x, w, y0, 1, m, pts, ws)
        torch.cuda.synchronize()
    finally:
        del os.environ["WINO_LAYER_NO_PDL"]
    y = torch.empty_like(y0)
    for it in range(6):
        ws.fill_(0xFF)          # NaN patterns: a read before the producer finished would show
        y.fill_(float("nan"))
        api.wino_conv2d_fp32(x, w, y, 1, m, pts, ws)
        if it % 2:              # back-to-back calls: the next chain starts behind this one
            api.wino_conv2d_fp32(x, w, y, 1, m, pts, ws)
        torch.cuda.synchronize()
        assert torch.equal(y, y0)


@pytest.mark.parametrize("N,C,H,K,m,pts,tile", [
    (3, 8, 56, 128, 2, OP.f23_c(1.0), 128064),        # T = 2352: 1 wave of 128 x 64 tiles, 2 of 128 x 128
    (3, 8, 56, 64, 2, OP.f23_c(0.8), 64128),          # K <= 64: 64-row tiles
    (2, 8, 30, 130, 4, OP.f43_c(1.6), 128128),        # Kp = 256
    (2, 3, 30, 130, 4, OP.f43_c(1.6), 1),             # fused C <= 4 kernel
])
def test_every_contraction_kernel_variant(N, C, H, K, m, pts, tile):
    """Each contraction variant the launcher can pick (CTA tile 128 x 128, 64 x 128, 128 x 64,
    the fused C <= 4 kernel) is bit-identical to the oracle layer; wino_conv2d_gemm_tile
    confirms the shape really selects it."""
    from paper_2201_10369_b200 import api
    assert api.wino_conv2d_gemm_tile(N, C, H, H, K, 3, 1, m) == tile
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=9)
    y, s, mx = _run(x, w, 1, m, pts)
    y_ref = ref.conv2d_wino(x, w, 1, m, pts)
    assert np.array_equal(y, y_ref)
    s_ref, m_ref = _oracle_stats(x, w, 1, y_ref)
    _check_stats(s, mx, s_ref, m_ref)


@pytest.mark.parametrize("C,K,H,tile,imgs,pool", [
    (512, 512, 14, 128064, (0, 37, 63), 1),    # conv5_x: T = 576 -> 4 waves of 128 x 64 tiles
    (512, 512, 14, 128064, (11,), 2),          # conv5_3: the same with the fused pool
    (256, 512, 28, 128064, (0, 63), 1),        # conv4_1: T = 1600 -> 11 waves instead of 12
    (3, 64, 224, 1, (63,), 1),                 # conv1_1: the fused C = 3 kernel, 92,416 tiles
    (64, 64, 224, 64128, (5,), 2),             # conv1_2: 64-row GEMM tiles, fused pool
])
def test_vgg_layers_full_batch_sampled_images(C, K, H, tile, imgs, pool):
    """BASELINE.json configs[4] layer shapes at the full batch of 64 in the launch
    configuration the VGG-16 run uses (the narrow GEMM tile / the fused first-layer kernel
    are chosen only at these sizes); sampled images recomputed by the oracle, ReLU
    activation included."""
    import torch
    from oracle import network as ON
    from paper_2201_10369_b200 import api
    N, m = 64, 6
    assert api.wino_conv2d_gemm_tile(N, C, H, H, K, 3, 1, m) == tile
    pts = OP.n8_cd(2.0, 1.003)
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=21)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m), dtype=torch.uint8, device="cuda")
    y = torch.empty((N, K, H, H), dtype=torch.float32, device="cuda")
    act = torch.empty((N, K, H // pool, H // pool), dtype=torch.float32, device="cuda")
    api.wino_conv2d_relu_pool_fp32(xd, wd, y, act, 1, m, pts, ws, pool)
    torch.cuda.synchronize()
    for img in imgs:
        y_ref = ref.conv2d_wino(x, w, 1, m, pts, n_lo=img, n_hi=img + 1)
        assert np.array_equal(y[img].cpu().numpy(), y_ref[img])
        assert np.array_equal(act[img].cpu().numpy(), ON.relu_pool(y_ref[img:img + 1], pool == 2)[0])
