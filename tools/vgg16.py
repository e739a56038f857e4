"""BASELINE.json configs[4]: VGG-16 conv stack forward, batch 64, 224x224x3 N(0,1) inputs,
He-normal weights, every 3x3 conv as F(6x6,3x3) Winograd with the proposed points
{0, ±2, ±1/2, -1/1.003, 1.003, inf} (R17), ReLU + 2x2 maxpool.

    python tools/vgg16.py [--batch 64] [--scored-batch 64]

Reports the unscored forward time (CUDA events, median of 5 after 2 warm-ups) as
effective (direct-equivalent) TFLOP/s, and the per-layer scored statistics (isolated
per-layer error vs fp64 direct convolution, P:673 protocol) on --scored-batch images."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, network, points as PP  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--scored-batch", type=int, default=64)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    pts = PP.family_n8_cd(2.0, 1.003)
    x, ws = synth.vgg16_inputs(args.batch, seed=0)
    xd = torch.from_numpy(x).to(dev)
    wd = [torch.from_numpy(w).to(dev) for w in ws]
    direct_flop = 0.0
    h = 224
    for C, K, _, pool in network.VGG16:
        direct_flop += 2.0 * args.batch * K * C * h * h * 9
        h = h // 2 if pool else h
    # forward time with the library's event hook off (its events would serialise the layers'
    # programmatic-dependent-launch chains); per-kernel totals from 3 more passes with it on
    times = []
    api.wino_timing_reset()
    for it in range(10):
        if it == 7:
            api.wino_timing_enable(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        network.vgg16_forward(xd, wd, pts, m=6, score=False)
        b.record()
        b.synchronize()
        if 2 <= it < 7:
            times.append(a.elapsed_time(b))
    kern = {f: api.wino_timing_read(f)[0] / 3
            for f in ("layer_filter", "layer_input", "layer_gemm", "layer_output", "layer_smallc", "relu_pool")}
    api.wino_timing_enable(False)
    t = statistics.median(times)
    xs = xd[: args.scored_batch].contiguous()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, s, mx, _, _ = network.vgg16_forward(xs, wd, pts, m=6, score=True)
    b.record()
    b.synchronize()
    scored_ms = a.elapsed_time(b)
    print(json.dumps({
        "workload": f"configs[4] VGG-16 conv stack, batch {args.batch}, F(6x6,3x3)", "ms": t,
        "effective_tflops": direct_flop / (t * 1e-3) / 1e12, "kernel_ms": kern,
        "scored_images": args.scored_batch, "scored_ms": scored_ms,
        "per_layer_mae": (s[:, 0] / s[:, 3]).tolist(),
        "normalized_l1": network.normalized_l1(s, args.scored_batch),
    }))


if __name__ == "__main__":
    main()
