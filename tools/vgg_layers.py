"""Per-layer timing of the configs[4] VGG-16 stack (batch 64, F(6x6,3x3), fused ReLU / pool):
each layer alone on synthetic N(0,1) activations of its shape, CUDA events on the launch
stream (median of 5 after 2 warm-ups), with the per-kernel-family breakdown of the
library's timing hook, the layer roofline t_roof = max(F_alg / P_fp32, B_alg / BW) and the
workspace traffic of the unfused pipeline (V and M round trips).

    python tools/vgg_layers.py [--batch 64]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2201_10369_b200 import api, network, points as PP  # noqa: E402

FAMS = ("layer_filter", "layer_input", "layer_gemm", "layer_output", "layer_smallc")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--only", type=int, default=-1, help="time this layer only (profiling)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    pts = PP.family_n8_cd(2.0, 1.003)
    N, m = args.batch, 6
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    rows = []
    for li, (C, K, h, pool) in enumerate(network.VGG16):
        if args.only >= 0 and li != args.only:
            continue
        x = torch.randn((N, C, h, h), device=dev, generator=g)
        w = torch.randn((K, C, 3, 3), device=dev, generator=g) * (2.0 / (C * 9)) ** 0.5
        p = 2 if pool else 1
        act = torch.empty((N, K, h // p, h // p), device=dev)
        ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, h, h, K, 3, 1, m), dtype=torch.uint8, device=dev)
        times = []
        api.wino_timing_reset()
        for it in range(7):
            if it == 2:
                api.wino_timing_enable(True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            api.wino_conv2d_relu_pool_fp32(x, w, None, act, 1, m, pts, ws, p, None, None, None, 0)
            b.record()
            b.synchronize()
            if it >= 2:
                times.append(a.elapsed_time(b))
        api.wino_timing_enable(False)
        kern = {}
        for f in FAMS:
            ms, cnt = api.wino_timing_read(f)[:2]
            if cnt:
                kern[f] = ms / cnt
        t = statistics.median(times)
        direct = 2.0 * N * K * C * h * h * 9
        th = (h + m - 1) // m
        T = N * th * th
        f_alg = 2.0 * 64 * C * K * T                      # contraction only (the dominant term)
        b_alg = 4.0 * (N * C * h * h + K * C * 9 + N * K * (h // p) ** 2)
        t_roof = max(f_alg / 74.4e12, b_alg / 6458.7e9) * 1e3
        rows.append({"layer": li, "C": C, "K": K, "H": h, "pool": pool, "ms": t, "kernel_ms": kern,
                     "t_roof_ms": t_roof, "frac": t_roof / t, "eff_tflops": direct / (t * 1e-3) / 1e12})
        del x, w, act, ws
    print(json.dumps({"workload": f"configs[4] VGG-16 layers alone, batch {N}", "sum_ms": sum(r["ms"] for r in rows),
                      "layers": rows}))


if __name__ == "__main__":
    main()
