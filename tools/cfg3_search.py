"""BASELINE.json configs[2] asks for "the F(6x6,3x3) layer with the best swept c set".
The proposed n = 8 family of the paper (T8 form; R17) is
{0, ±c, ±1/c, -1/d, d, inf}.  This re-derives (c, d) by a 2D F(6x6,3x3) sweep over a
grid x grid log-spaced grid in [0.05, 20]^2 (100k uniform[-1,1] tiles, the paper's error
protocol; exact duplicates rejected), then runs the configs[2] layer (N=32, C=K=256, 56x56,
N(0,1) / He-normal) scored against fp64 direct with the swept argmin, the paper's (2, 1.003)
and the prior-work P8 = {0, ±1, ±1/2, ±2, inf}.  Prints one JSON object.

    python tools/cfg3_search.py [--grid 128] [--tiles 100000]
"""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=128)
    ap.add_argument("--tiles", type=int, default=100_000)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = synth.c_grid(args.grid)
    params = np.array([(a, b) for a in g for b in g], dtype=np.float64)
    sp = SweepSpec("cfg3_cd", 2, "n8_cd", params, "uniform", args.tiles, seed=3)
    d, gt = synth.random_tiles(sp.n_tiles, 2, sp.n, sp.r, sp.dist, sp.seed)
    rs = make_rank_sweep(sp, 0, 1, dev, d, gt)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run_step([rs])
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    mae = curve(rs.sums.cpu().numpy(), rs.status)
    i, best = argmin_c(sp.params, mae)
    out = {"workload": "configs[2] (c, d) sweep, F(6x6,3x3) 2D, {0,±c,±1/c,-1/d,d,inf}", "grid": args.grid,
           "tiles": args.tiles, "candidates": sp.n_cand, "rejected": int(np.sum(rs.status != 0)), "sweep_ms": ms,
           "tile_evals_per_s": int(np.sum(rs.status == 0)) * sp.n_tiles / (ms * 1e-3),
           "argmin": sp.params[i].tolist(), "min_mae": best}
    N, C, H, W, K, r, pad, m = 32, 256, 56, 56, 256, 3, 1, 6
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=0)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    sets = {"swept_argmin": PP.family_n8_cd(*sp.params[i]), "paper_2_1.003": PP.family_n8_cd(2.0, 1.003),
            "prior_P8": list(PP.P8)}
    out["layers"] = {}
    for name, pts in sets.items():
        _, s, mx = api.conv2d(xd, wd, pad, m, pts, score=True)
        s = s.cpu().numpy()
        out["layers"][name] = {"points": [p for p in pts if np.isfinite(p)], "mae": float(s[0] / s[3]),
                               "max_abs_err": float(mx.cpu().numpy()[0])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
