"""Memory-safety and race checks of our own (compute-sanitizer is closed on this GPU pool,
profiles/r02_sanitizer_unavailable.log): every output / statistics / workspace buffer the
kernels write is embedded in a larger allocation whose guard regions hold a sentinel that
must survive the call (out-of-bounds writes), and repeated launches must give bitwise
identical statistics (a shared-memory race in the fixed-order reductions would not)."""
import numpy as np
import pytest

import synth
from oracle import points as OP

pytestmark = pytest.mark.gpu

SENT = -12345.678


def _guarded(torch, shape, dtype, fill, guard=4096):
    """A contiguous view of `shape` inside a flat buffer with `guard` sentinel elements on
    both sides.  Returns (view, check) -- check() asserts the guards are intact."""
    n = int(np.prod(shape)) if len(shape) else 1
    sent = 0xA5 if dtype == torch.uint8 else SENT
    flat = torch.full((n + 2 * guard,), sent, dtype=dtype, device="cuda")
    view = flat[guard:guard + n].view(*shape)
    view.fill_(fill)

    def check():
        torch.cuda.synchronize()
        g = torch.cat([flat[:guard], flat[guard + n:]]).cpu().numpy()
        assert np.all(g == np.asarray(sent, dtype=g.dtype)), "write outside the buffer"
    return view, check


CASES = [
    (2, 4, 3, [OP.f43_c(c) for c in (0.3, 1.6, 2.4, 1e19)], 0),            # register pairs + careful
    (1, 4, 3, [OP.f43_c(c) for c in (0.3, 1.6, 2.4, 1e19)], 0),            # 1D register pairs
    (2, 4, 5, [OP.n8_c1c2(0.47, 1.04), OP.n8_c1c2(1.5, 3.1)], 0),          # register single tile
    (2, 6, 5, [OP.n10_c1c2(0.39, 0.78)], 0),                               # generic shared-memory
    (2, 2, 3, [OP.f23_c(0.5), OP.f23_c(1.5)], 0),
    (2, 4, 3, [OP.f43_c(1.6), OP.f43_c(0.7)], 2),                          # Huffman order
    (2, 4, 3, [OP.f43_c(1.6), OP.f43_c(0.7), OP.f43_c(1e19)], 2 | 256),    # Huffman, run-time kernels
    (1, 6, 3, [OP.n8_cd(2.0, 1.003)], 2 | 256),                            # (1D)
    (2, 8, 3, [OP.n10_c1c2(1.272, 2.099)], 2 | 256),                       # (n = 10: > 48 KB shared memory)
    (1, 6, 3, [OP.n8_cd(2.0, 1.003)], 4),                                  # mixed precision
    (2, 8, 3, [OP.chebyshev(10)], 0),                                      # dense generic, rolled loops
]
JIT = 256   # test-only marker: force the run-time specialised Huffman kernels


@pytest.mark.parametrize("dims,m,r,sets,flags", CASES)
def test_sweep_writes_stay_in_bounds(dims, m, r, sets, flags):
    import torch
    from paper_2201_10369_b200 import api
    prev = api.wino_huffman_jit_mode(1 if flags & JIT else 2)
    flags &= ~JIT
    n = m + r - 1
    T = 1237
    d, g = synth.random_tiles(T, dims, n, r, "uniform", seed=51)
    dd, check_d = _guarded(torch, d.shape, torch.float32, 0.0)
    gg, check_g = _guarded(torch, g.shape, torch.float32, 0.0)
    dd.copy_(torch.from_numpy(d))
    gg.copy_(torch.from_numpy(g))
    S = len(sets)
    y, check_y = _guarded(torch, (S, T, m ** dims), torch.float32, 0.0)
    sums, check_s = _guarded(torch, (S, 5), torch.float64, 0.0)
    maxs, check_m = _guarded(torch, (S, 2), torch.float64, 0.0)
    wsb = api.wino_error_sweep_workspace_bytes(dims, m, r, S, T)
    ws, check_w = _guarded(torch, (wsb,), torch.uint8, 0, guard=8192)
    try:
        api.wino_sweep_outputs(dims, m, r, np.array(sets), dd, gg, y, ws, sums, maxs, flags=flags)
    finally:
        api.wino_huffman_jit_mode(prev)
    for c in (check_d, check_g, check_y, check_s, check_m, check_w):
        c()


@pytest.mark.parametrize("C", [13, 3])   # C = 3: the fused small-C kernel
def test_layer_writes_stay_in_bounds(C):
    import torch
    from paper_2201_10369_b200 import api
    N, H, K, m = 3, 21, 19, 6
    pts = OP.n8_cd(2.0, 1.003)
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=52)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y, check_y = _guarded(torch, (N, K, H, H), torch.float32, 0.0)
    act, check_a = _guarded(torch, (N, K, H // 2, H // 2), torch.float32, 0.0)
    sums, check_s = _guarded(torch, (N, 5), torch.float64, 0.0)
    maxs, check_m = _guarded(torch, (N, 2), torch.float64, 0.0)
    wsb = api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m)
    ws, check_w = _guarded(torch, (wsb,), torch.uint8, 0, guard=8192)
    api.wino_conv2d_relu_pool_fp32(xd, wd, y, act, 1, m, pts, ws, 2, sums, maxs,
                                   flags=api.WINO_CONV_SCORE_PER_IMAGE)
    for flag in (api.WINO_CONV_TF32, api.WINO_CONV_3XTF32):
        api.wino_conv2d_fp32(xd, wd, y, 1, m, pts, ws, flags=flag)
    for c in (check_y, check_a, check_s, check_m, check_w):
        c()


@pytest.mark.parametrize("dims", [2, 1])
def test_sweep_statistics_deterministic(dims):
    """Five launches of the production configs[1] kernels on the same inputs: bitwise
    identical statistics (fixed-order reductions; no shared-memory race)."""
    import torch
    from paper_2201_10369_b200 import api
    sets = np.array([OP.f43_c(float(c)) for c in synth.c_grid(200)])
    T = 20_011
    d, g = synth.random_tiles(T, dims, 6, 3, "normal", seed=53)
    dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, 4, 3, len(sets), T), dtype=torch.uint8, device="cuda")
    first = None
    for _ in range(5):
        sums = torch.zeros((len(sets), 5), dtype=torch.float64, device="cuda")
        maxs = torch.zeros((len(sets), 2), dtype=torch.float64, device="cuda")
        api.wino_error_sweep(dims, 4, 3, sets, dd, gg, sums, maxs, ws)
        got = np.concatenate([sums.cpu().numpy(), maxs.cpu().numpy()], axis=1)
        if first is None:
            first = got
        else:
            assert np.array_equal(got, first, equal_nan=True)


def test_unaligned_tiles_rejected():
    """The sweep reads tiles with 16-byte vector loads: a misaligned pointer is refused
    (WINO_E_INVALID_ARG) instead of faulting on the device."""
    import torch
    from paper_2201_10369_b200 import _lib, api
    d, g = synth.random_tiles(300, 2, 6, 3, "uniform", seed=54)
    flat = torch.zeros(d.size + 1, dtype=torch.float32, device="cuda")
    dd = flat[1:].view(d.shape)
    dd.copy_(torch.from_numpy(d))
    gg = torch.from_numpy(g).cuda()
    sums = torch.zeros((1, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((1, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(2, 4, 3, 1, 300), dtype=torch.uint8, device="cuda")
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_error_sweep(2, 4, 3, np.array([OP.f43_c(1.6)]), dd, gg, sums, maxs, ws)
    assert ei.value.status == 1
    torch.cuda.synchronize()
