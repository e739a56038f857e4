"""NEXT row N4: the Table tab:win_dcnn protocol on synthetic CIFAR-shaped stacks.

    python tools/synthetic_nets.py [--images 256]

A ResNet-20-shaped and a SqueezeNet-shaped plain 3x3 stack (network.RESNET20_LIKE,
network.SQUEEZENET_LIKE; 32x32x3 N(0,1) inputs, He-normal weights -- stand-ins, no CIFAR
items, no trained weights) are run with every conv as an F(n-2, 3) Winograd layer for
n = 4..10 and the three point families of T9 per n: the prior-work sets, the
paper's proposed sets and the Chebyshev nodes (+inf).  Per layer the isolated error vs
fp64 direct convolution is accumulated; reported as the paper's normalized L1 (Σ|e| over
layers and images / (images x layers), reading R12) and the mean per-element error."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import network, points as P  # noqa: E402


def families():
    c = lambda *v: P._canon(list(v))  # noqa: E731
    return {
        4: {"prior P4": P.P4, "proposed c=1.054": c(0.0, -1 / 1.054, 1 / 1.054), "chebyshev": P.chebyshev(4)},
        5: {"prior P4+{1/2}": c(0.0, -1.0, 1.0, 0.5), "proposed c=2": c(0.0, 1.0, -1.0, -2.0),
            "chebyshev": P.chebyshev(5)},
        6: {"prior P4+{1/2,-2}": c(0.0, -1.0, 1.0, 0.5, -2.0), "proposed c=1.622": P.family_f43(1.622),
            "chebyshev": P.chebyshev(6)},
        7: {"prior P4+{1/2,-2,-1/2}": c(0.0, -1.0, 1.0, 0.5, -2.0, -0.5),
            "proposed c=2,d=1": c(0.0, -0.5, -2.0, 2.0, 0.5, 1.0), "chebyshev": P.chebyshev(7)},
        8: {"prior P8": P.P8, "proposed c=2,d=1.003": P.family_n8_cd(2.0, 1.003), "chebyshev": P.chebyshev(8)},
        9: {"prior P8+{-1/4}": c(0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0, -0.25),
            "proposed c=1.305,d=2.485": c(0.0, -1 / 1.305, -1.305, 1.305, 1 / 1.305, -1 / 2.485, -2.485, 2.485),
            "chebyshev": P.chebyshev(9)},
        10: {"prior P10": P.P10, "proposed c=1.272,d=2.099": P.family_n10(1.272, 2.099), "chebyshev": P.chebyshev(10)},
    }


NETS = {"resnet20": network.RESNET20_LIKE, "squeezenet": network.SQUEEZENET_LIKE}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--nets", default="resnet20,squeezenet")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {"workload": f"synthetic 3x3 stacks, {args.images} synthetic 32x32x3 N(0,1) images, He-normal weights",
           "rows": []}
    for net in args.nets.split(","):
        layers = NETS[net]
        x, ws = synth.stack_inputs(layers, args.images, seed=0)
        xd = torch.from_numpy(x).to(dev)
        wd = [torch.from_numpy(w).to(dev) for w in ws]
        for n, fams in families().items():
            for name, pts in fams.items():
                _, s, _, _, _ = network.stack_forward(layers, xd, wd, pts, m=n - 2, score=True)
                out["rows"].append({"net": net, "n": n, "points": name,
                                    "normalized_l1": network.normalized_l1(s, args.images),
                                    "mean_abs_err": float(s[:, 0].sum() / s[:, 3].sum()),
                                    "nonfinite": int(s[:, 4].sum())})
    # per (net, n): which family is best (the paper's bold entries, T9)
    best = {}
    for r in out["rows"]:
        k = f"{r['net']} n={r['n']}"
        if k not in best or r["normalized_l1"] < best[k][1]:
            best[k] = (r["points"], r["normalized_l1"])
    out["best"] = {k: v[0] for k, v in best.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
