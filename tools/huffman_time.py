"""Time the Huffman-order and mixed-precision sweeps (NEXT row N2) on the configs[1] workload (4096 c x 100k
tiles, uniform) next to the production F32-FMA sweep; prints one JSON object."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from oracle import points as OP
from paper_2201_10369_b200 import api

out = {}
grid = synth.c_grid()
sets = np.array([OP.f43_c(float(c)) for c in grid])
for dims in (1, 2):
    d, g = synth.random_tiles(100_000, dims, 6, 3, "uniform", seed=0)
    dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
    S, T = len(sets), d.shape[0]
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, 4, 3, S, T), dtype=torch.uint8, device="cuda")
    for name, flags, jit in (("fma", 0, 0), ("nofma", 1, 0), ("huffman", 2, 1), ("huffman_interp", 2, 2), ("mixed", 4, 0)):
        api.wino_huffman_jit_mode(jit)
        sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda")
        maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda")
        api.wino_error_sweep(dims, 4, 3, sets, dd, gg, sums, maxs, ws, flags=flags)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            api.wino_error_sweep(dims, 4, 3, sets, dd, gg, sums, maxs, ws, flags=flags)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        s = sums.cpu().numpy()
        mae = s[:, 0] / s[:, 3]
        i = int(np.nanargmin(mae))
        out[f"{dims}d_{name}"] = {"ms": min(ts), "tile_evals_per_s": S * T / (min(ts) * 1e-3),
                                  "argmin_c": float(grid[i]), "min_mae": float(mae[i])}
print(json.dumps(out, indent=1))
