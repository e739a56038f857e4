"""BASELINE.json configs[3]: the (c1, c2) grid sweep and the 5x5 layers at its argmin.

    python tools/cfg4_grid.py [--grid 256] [--tiles 100000] [--no-layer]

Sweeps (2D, uniform[-1,1] tiles, seed 2; R18):
  n = 8,  F(4x4,5x5): {0, ±c1, ±1/c1, ±c2, inf}
  n = 10, F(6x6,5x5): {0, ±c1, ±1/c1, ±c2, ±1/c2, inf}
over a grid x grid log-spaced (c1, c2) grid in [0.05, 20]^2 (exact duplicates rejected),
then the layers N=16, C=K=128, 64x64, pad 2 at each argmin, scored against fp64 direct
convolution.  Prints one JSON line (timings from CUDA events)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, points as PP  # noqa: E402
from paper_2201_10369_b200.sweep import SweepSpec, argmin_c, curve, make_rank_sweep, run_step  # noqa: E402


def grid_spec(template, grid, tiles):
    g = synth.c_grid(grid)
    params = np.array([(a, b) for a in g for b in g], dtype=np.float64)
    return SweepSpec(f"cfg4_{template}", 2, template, params, "uniform", tiles, seed=2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--tiles", type=int, default=100_000)
    ap.add_argument("--no-layer", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {"workload": "configs[3]", "grid": args.grid, "tiles": args.tiles, "sweeps": {}, "layers": {}}
    for template in ("n8_c1c2_r5", "n10_c1c2_r5"):
        sp = grid_spec(template, args.grid, args.tiles)
        d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
        rs = make_rank_sweep(sp, 0, 1, dev, d, g)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_step([rs])
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        sums = rs.sums.cpu().numpy()
        mae = curve(sums, rs.status)
        i, best = argmin_c(sp.params, mae)
        evals = int(np.sum(rs.status == 0)) * sp.n_tiles
        out["sweeps"][template] = {
            "m": sp.m, "r": sp.r, "candidates": sp.n_cand, "rejected": int(np.sum(rs.status != 0)),
            "ms": ms, "tile_evals_per_s": evals / (ms * 1e-3), "argmin": sp.params[i].tolist(), "min_mae": best,
        }
        if not args.no_layer:
            N, C, H, W, K, r, pad = 16, 128, 64, 64, 128, 5, 2
            x, w = synth.layer_inputs(N, C, H, W, K, r, "uniform", "uniform", seed=0)
            xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
            pts = PP.TEMPLATES[template][3](*sp.params[i])
            y, s, mx = api.conv2d(xd, wd, pad, sp.m, pts, score=True)   # warm-up + scored stats
            ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, sp.m), dtype=torch.uint8,
                             device=dev)
            times = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                api.wino_conv2d_fp32(xd, wd, y, pad, sp.m, pts, ws)
                b.record()
                b.synchronize()
                times.append(a.elapsed_time(b))
            t = float(np.median(times))
            s = s.cpu().numpy()
            out["layers"][template] = {
                "points": pts[:-1], "ms": t,
                "effective_tflops": 2.0 * N * K * C * H * W * r * r / (t * 1e-3) / 1e12,
                "mae": float(s[0] / s[3]), "max_abs_err": float(mx.cpu().numpy()[0]),
            }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
