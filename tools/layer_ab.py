"""A/B timing of the layer paths with the library's timing hook OFF (the hook's events
serialise the PDL chain): configs[2], the configs[3] layers and the VGG-16 x64 stack, CUDA
events around each call, median of 9 after 3 warm-ups, L2 flushed between runs.

    WINO_LAYER_NO_PDL=1 python tools/layer_ab.py      # plain launches, K1 on a side stream
    python tools/layer_ab.py                          # PDL chain"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, network, points as PP  # noqa: E402


def timed(fn, flush, reps=9, warm=3):
    ts = []
    for it in range(warm + reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if it >= warm:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def main():
    dev = torch.device("cuda", 0)
    fb = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    flush = fb.zero_
    out = {"pdl": os.environ.get("WINO_LAYER_NO_PDL") is None}
    shapes = {"cfg2": (32, 256, 56, 256, 3, 1, 6, PP.family_n8_cd(2.0, 1.003)),
              "cfg3_n8": (16, 128, 64, 128, 5, 2, 4, PP.family_n8_c1c2(1.5, 3.1)),
              "cfg3_n10": (16, 128, 64, 128, 5, 2, 6, PP.family_n10(1.272, 2.099))}
    for name, (N, C, H, K, r, pad, m, pts) in shapes.items():
        x, w = synth.layer_inputs(N, C, H, H, K, r, "normal", "he", seed=0)
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        y = torch.empty((N, K, H, H), dtype=torch.float32, device=dev)
        ws = torch.empty(api.wino_conv2d_workspace_bytes(N, C, H, H, K, r, pad, m), dtype=torch.uint8, device=dev)
        out[name] = timed(lambda: api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws), flush)
        del xd, wd, y, ws
    x, wts = synth.vgg16_inputs(64, seed=0)
    xd = torch.from_numpy(x).to(dev)
    wd = [torch.from_numpy(w).to(dev) for w in wts]
    pts = PP.family_n8_cd(2.0, 1.003)
    out["vgg16_x64"] = timed(lambda: network.vgg16_forward(xd, wd, pts, m=6, score=False), lambda: None, reps=5, warm=2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
