"""Short driver for ncu captures (tools/profile.sh): one configs[1] 2D and 1D sweep at full
size (4096 c x 100k tiles, uniform) and one configs[2] layer, each run twice (warm-up +
captured), through the C ABI."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, points as PP  # noqa: E402
from paper_2201_10369_b200.sweep import cfg2_specs, make_rank_sweep, run_step  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "sweep"):
        specs = cfg2_specs(synth.c_grid(4096), 100_000)
        rs = []
        for sp in (specs[2], specs[0]):
            d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
            rs.append(make_rank_sweep(sp, 0, 1, dev, d, g))
        for _ in range(2):
            run_step(rs)
        torch.cuda.synchronize()
    if what == "cfg4":    # configs[3] grid sweeps, a 24 x 24 sub-grid of (c1, c2) at 100k tiles
        from paper_2201_10369_b200.sweep import SweepSpec
        g = synth.c_grid(24)
        params = np.array([(a, b) for a in g for b in g if a != b], dtype=np.float64)
        rs = []
        for tpl in ("n8_c1c2_r5", "n10_c1c2_r5"):
            sp = SweepSpec("cfg4", 2, tpl, params, "uniform", 100_000, seed=2)
            d, gg = synth.random_tiles(sp.n_tiles, 2, sp.n, sp.r, sp.dist, sp.seed)
            rs.append(make_rank_sweep(sp, 0, 1, dev, d, gg))
        for _ in range(2):
            run_step(rs)
        torch.cuda.synchronize()
    if what == "score":   # the configs[2] layer, scored (the fp64 scorer K5)
        N, C, H, W, K, r, pad, m = 32, 256, 56, 56, 256, 3, 1, 6
        x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=0)
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        pts = PP.family_n8_cd(2.0, 1.003)
        y, s, mx = api.conv2d(xd, wd, pad, m, pts, score=True)
        torch.cuda.synchronize()
    if what == "huff":    # configs[1] 2D uniform Huffman-order sweep, run-time specialised kernels
        sets = np.array([PP.family_f43(float(c)) for c in synth.c_grid(4096)])
        d, g = synth.random_tiles(100_000, 2, 6, 3, "uniform", 0)
        dd, gg = torch.from_numpy(d).to(dev), torch.from_numpy(g).to(dev)
        S, T = len(sets), d.shape[0]
        ws = torch.empty(api.wino_error_sweep_workspace_bytes(2, 4, 3, S, T), dtype=torch.uint8, device=dev)
        sums = torch.zeros((S, 5), dtype=torch.float64, device=dev)
        maxs = torch.zeros((S, 2), dtype=torch.float64, device=dev)
        api.wino_huffman_jit_mode(1)
        for _ in range(2):
            api.wino_error_sweep(2, 4, 3, sets, dd, gg, sums, maxs, ws, flags=api.WINO_SWEEP_HUFFMAN)
        torch.cuda.synchronize()
    if what == "vgg":     # configs[4]: two unscored VGG-16 x64 forwards
        from paper_2201_10369_b200 import network
        x, wts = synth.vgg16_inputs(64, seed=0)
        xd = torch.from_numpy(x).to(dev)
        wd = [torch.from_numpy(w).to(dev) for w in wts]
        for _ in range(2):
            network.vgg16_forward(xd, wd, PP.family_n8_cd(2.0, 1.003), m=6, score=False)
        torch.cuda.synchronize()
    if what in ("all", "layer"):
        N, C, H, W, K, r, pad, m = 32, 256, 56, 56, 256, 3, 1, 6
        x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=0)
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        pts = PP.family_n8_cd(2.0, 1.003)
        y = torch.empty((N, K, H, W), dtype=torch.float32, device=dev)
        ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, m), dtype=torch.uint8, device=dev)
        for _ in range(2):
            api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws)
        torch.cuda.synchronize()
    print("prof_driver ok")


if __name__ == "__main__":
    main()
