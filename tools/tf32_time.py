"""Time the layer (configs[2] / configs[3] shapes) with the FFMA and the tcgen05 TF32
contraction; per-kernel times from the library's timing hooks."""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from oracle import points as OP
from paper_2201_10369_b200 import api

def run(shape, m, pts, pad, reps=20):
    N, C, H, W, K, r = shape
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=0)
    x, w = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    out = {}
    for flags in (0, 1, 2):
        Ho = H + 2 * pad - r + 1
        y = torch.empty((N, K, Ho, Ho), device="cuda")
        ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, W, K, r, pad, m), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            api.wino_conv2d_fp32(x, w, y, pad, m, pts, ws, flags=flags)
        torch.cuda.synchronize()
        api.wino_timing_enable(1); api.wino_timing_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            api.wino_conv2d_fp32(x, w, y, pad, m, pts, ws, flags=flags)
        e1.record(); torch.cuda.synchronize()
        fam = {f: api.wino_timing_read(f) for f in ("layer_filter", "layer_input", "layer_gemm",
                                                   "layer_gemm_tf32", "layer_gemm_3xtf32", "layer_output")}
        fam = {f: {"ms": v[0], "count": v[1]} for f, v in fam.items() if v[1]}
        api.wino_timing_enable(0)
        n = m + r - 1
        T = N * ((Ho + m - 1) // m) ** 2
        gemm_flop = 2.0 * n * n * C * K * T
        g = fam.get({0: "layer_gemm", 1: "layer_gemm_tf32", 2: "layer_gemm_3xtf32"}[flags])
        out[{0: "fp32", 1: "tf32", 2: "3xtf32"}[flags]] = {"ms": e0.elapsed_time(e1) / reps, "families": fam,
                                            "gemm_tflops": gemm_flop / (g["ms"] / g["count"] * 1e-3) / 1e12 if g else None}
    return out

res = {"cfg3": run((32, 256, 56, 56, 256, 3), 6, OP.n8_cd(2.0, 1.003), 1),
       "cfg4_n8": run((16, 128, 64, 64, 128, 5), 4, OP.n8_c1c2(1.5, 3.1), 2),
       "cfg4_n10": run((16, 128, 64, 64, 128, 5), 6, OP.n10_c1c2(1.272, 2.099), 2)}
print(json.dumps(res, indent=1, default=str))
