"""Time the fp64 scorer (K5) alone on the configs[2] layer: the library's event hook around
layer_score, median of 5 scored calls after a warm-up.    python tools/score_time.py"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, points as PP  # noqa: E402


def main():
    N, C, H, K, m = 32, 256, 56, 256, 6
    x, w = synth.layer_inputs(N, C, H, H, K, 3, "normal", "he", seed=0)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    pts = PP.family_n8_cd(2.0, 1.003)
    y = torch.empty((N, K, H, H), dtype=torch.float32, device="cuda")
    ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, H, K, 3, 1, m), dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(6):
        s = torch.zeros(5, dtype=torch.float64, device="cuda")
        mx = torch.zeros(2, dtype=torch.float64, device="cuda")
        api.wino_timing_reset()
        api.wino_timing_enable(True)
        api.wino_conv2d_fp32(xd, wd, y, 1, m, pts, ws, s, mx)
        torch.cuda.synchronize()
        t = api.wino_timing_read("layer_score")[0]
        api.wino_timing_enable(False)
        if it:
            ts.append(t)
    sv = s.cpu().numpy()
    print(json.dumps({"score_ms": statistics.median(ts), "min": min(ts), "mae": sv[0] / sv[3], "n": sv[3]}))


if __name__ == "__main__":
    main()
