"""Per-rank device time of the configs[1] step when the candidates are sharded over W
ranks, measured on ONE GPU by running rank r's shard alone (no collective; the all-reduce
of 4 x 4096 x 7 fp64 is ~tens of us on NVLink).  Predicts strong-scaling efficiency
t(1) / (W * max_r t_r(W)) before the multi-GPU run."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth
from paper_2201_10369_b200.sweep import cfg2_specs, make_rank_sweep, run_step

dev = torch.device("cuda", 0)
specs = cfg2_specs(synth.c_grid(4096), 100_000)
tiles = {s.name: synth.random_tiles(s.n_tiles, s.dims, s.n, s.r, s.dist, s.seed) for s in specs}
out = {}
for W in (1, 2, 4, 8):
    worst = 0.0
    for r in sorted({0, W - 1}):
        rsw = [make_rank_sweep(s, r, W, dev, *tiles[s.name]) for s in specs]
        for _ in range(3):
            run_step(rsw, reduce=False)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            run_step(rsw, reduce=False)
        b.record()
        b.synchronize()
        worst = max(worst, a.elapsed_time(b) / 5)
        del rsw
    out[W] = worst
eff = {W: out[1] / (W * out[W]) for W in out}
print(json.dumps({"ms_per_step_max_rank": out, "predicted_strong_scaling_efficiency": eff}, indent=1))
