"""BASELINE.json configs[4] (VGG-16 conv stack, every 3x3 conv as F(6x6,3x3) with the
{0,±2,±1/2,-1/1.003,1.003,inf} points) on 2 images at full 224x224 resolution: every
layer's Winograd output bit-identical to the oracle's chain, per-layer statistics vs the
oracle's fp64 direct convolution within 1e-9 relative (north star: 1 %)."""
import numpy as np
import pytest

import synth
from oracle import network as ON, points as OP

pytestmark = pytest.mark.gpu


def test_vgg16_two_images():
    import torch
    from paper_2201_10369_b200 import network
    x, ws = synth.vgg16_inputs(2, seed=0)
    pts = OP.n8_cd(2.0, 1.003)
    dev = torch.device("cuda", 0)
    out, s, mx, ys, _ = network.vgg16_forward(torch.from_numpy(x).to(dev),
                                              [torch.from_numpy(w).to(dev) for w in ws], pts, m=6, score=True,
                                              keep=True)
    torch.cuda.synchronize()
    ys_ref, s_ref, m_ref = ON.vgg16(x, ws, pts, m=6)
    for li in range(13):
        assert np.array_equal(ys[li].cpu().numpy(), ys_ref[li]), li
        assert s[li, 3] == s_ref[li, 3] and s[li, 4] == s_ref[li, 4]
        assert np.array_equal(mx[li], m_ref[li])
        assert abs(s[li, 0] / s_ref[li, 0] - 1) < 1e-9
    assert out.shape == (2, 512, 7, 7)
    final_ref = ON.relu_pool(ys_ref[-1], True)
    assert np.array_equal(out.cpu().numpy(), final_ref)
    assert network.normalized_l1(s, 2) > 0


def test_relu_pool_exact():
    import torch
    from paper_2201_10369_b200 import api
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 9, 7)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    for pool in (1, 2):
        y = torch.empty((2, 3, 9 // pool, 7 // pool), device="cuda")
        api.wino_relu_pool_fp32(xd, y, pool)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), ON.relu_pool(x, pool == 2))


def test_resnet20_like_stack_chebyshev_and_n5():
    """NEXT row N4 stack (CIFAR-shaped synthetic inputs): bit-identical to the oracle chain
    for the Chebyshev nodes (the oracle's own generator) and the n = 5 proposed set, first 8
    layers, 3 images."""
    import torch
    from paper_2201_10369_b200 import network
    layers = network.RESNET20_LIKE[:8]
    x, ws = synth.stack_inputs(layers, 3, seed=1)
    dev = torch.device("cuda", 0)
    for m, pts in ((2, OP.chebyshev(4)), (3, sorted([0.0, 1.0, -1.0, -2.0]) + [float("inf")]),
                   (6, OP.chebyshev(8))):
        _, s, mx, ys, _ = network.stack_forward(layers, torch.from_numpy(x).to(dev),
                                                [torch.from_numpy(w).to(dev) for w in ws], pts, m=m, keep=True)
        torch.cuda.synchronize()
        ys_ref, s_ref, m_ref = ON.stack(layers, x, ws, pts, m=m)
        for li in range(len(layers)):
            assert np.array_equal(ys[li].cpu().numpy(), ys_ref[li]), (m, li)
            assert abs(s[li, 0] / s_ref[li, 0] - 1) < 1e-9
