"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): one
launch of every kernel family on BASELINE.json configs[0] and a configs[1] subset, through
the C ABI, with ragged tile counts.  Sizes are tiny because racecheck serialises shared
memory accesses.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --quick
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, points as PP  # noqa: E402


def sweep(dims, m, r, sets, n_tiles, flags=0, outputs=False):
    n = m + r - 1
    d, g = synth.random_tiles(n_tiles, dims, n, r, "uniform", seed=3)
    dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
    S = len(sets)
    sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, m, r, S, n_tiles), dtype=torch.uint8, device="cuda")
    if outputs:
        y = torch.empty((S, n_tiles, m ** dims), dtype=torch.float32, device="cuda")
        api.wino_sweep_outputs(dims, m, r, np.array(sets), dd, gg, y, ws, sums, maxs, flags=flags)
    else:
        api.wino_error_sweep(dims, m, r, np.array(sets), dd, gg, sums, maxs, ws, flags=flags)
    torch.cuda.synchronize()
    return sums.cpu().numpy()


def main():
    quick = "--quick" in sys.argv
    T = 700 if quick else 3001
    cs = [float(c) for c in synth.c_grid(48)][:: (4 if quick else 1)]
    f43 = [PP.family_f43(c) for c in cs if c != 1.0]
    for dims in (1, 2):
        sweep(dims, 4, 3, f43, T)
        sweep(dims, 4, 3, f43[:8], T, outputs=True)
        sweep(dims, 4, 3, f43[:4], T, flags=api.WINO_SWEEP_NOFMA)
        sweep(dims, 4, 3, f43[:3], T, flags=api.WINO_SWEEP_HUFFMAN)
        sweep(dims, 4, 3, f43[:3], T, flags=api.WINO_SWEEP_MIXED)
    # careful path: overflowing candidates between normal ones
    bad = [PP.family_f43(c) for c in (0.7, 1e19, 1.6, 1e12)]
    for dims in (1, 2):
        s = sweep(dims, 4, 3, bad, T, outputs=True)
        assert s[1, 4] > 0 or s[3, 4] > 0
    # other layouts: register single-tile (F(4x4,5x5)), generic shared-memory (F(6x6,5x5))
    sweep(2, 4, 5, [PP.family_n8_c1c2(0.47, 1.04), PP.family_n8_c1c2(1.5, 3.1)], T)
    sweep(2, 6, 5, [PP.family_n10(0.39, 0.78)], 300 if quick else T)
    sweep(2, 2, 3, [PP.family_f23(c) for c in (0.5, 1.5)], T)
    # layers: configs[0] scored, fused ReLU / pool, the tcgen05 variant
    x, w = synth.layer_inputs(1, 8, 16, 16, 8, 3, "uniform", "uniform", seed=0)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    api.conv2d(xd, wd, 1, 2, PP.family_f23(1.0), score=True)
    ws = torch.empty(api.wino_conv2d_workspace_bytes(1, 8, 16, 16, 8, 3, 1, 6), dtype=torch.uint8, device="cuda")
    act = torch.empty((1, 8, 8, 8), dtype=torch.float32, device="cuda")
    y = torch.empty((1, 8, 16, 16), dtype=torch.float32, device="cuda")
    sums = torch.zeros((1, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((1, 2), dtype=torch.float64, device="cuda")
    api.wino_conv2d_relu_pool_fp32(xd, wd, y, act, 1, 6, PP.family_n8_cd(2.0, 1.003), ws, 2, sums, maxs,
                                   flags=api.WINO_CONV_SCORE_PER_IMAGE)
    if not quick:
        x2, w2 = synth.layer_inputs(1, 40, 20, 20, 130, 3, "normal", "he", seed=1)
        api.conv2d(torch.from_numpy(x2).cuda(), torch.from_numpy(w2).cuda(), 1, 2, PP.family_f23(1.0),
                   flags=api.WINO_CONV_TF32)
        api.conv2d(torch.from_numpy(x2).cuda(), torch.from_numpy(w2).cuda(), 1, 4, PP.family_f43(1.622), score=True)
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
