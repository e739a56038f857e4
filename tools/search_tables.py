"""NEXT row N1: reproduce the paper's optimality tables with the template search, in the
paper's Huffman summation order (reading R21; WINO_SWEEP_HUFFMAN) or the sequential
no-FMA order.

    python tools/search_tables.py [--tiles 50000] [--order huffman|nofma]

For each of tab:optimal_f23 / f33 / f43, 1D: sweep c over [1.0, 2.6] in steps of
0.002 for every listed template, report (template, best c, min error) sorted, next to the
paper's best row.  Prints one JSON line."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import search as S  # noqa: E402

PAPER_BEST = {"f23_1d": "{-1,1/c} c=1.028 3.06e-8 (P:511)", "f33_1d": "{0.5,-c,c} c=1.326 4.20e-8 (P:536)",
              "f43_1d": "{-1/c,-c,c,1/c} c=1.829 5.65e-8 (P:552)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=50_000)
    ap.add_argument("--order", choices=["huffman", "nofma"], default="huffman")
    args = ap.parse_args()
    flags = 2 if args.order == "huffman" else 1
    cs = list(np.round(np.arange(1.0, 2.6, 0.002), 6))
    out = {"order": None}
    for key, m in (("f23_1d", 2), ("f33_1d", 3), ("f43_1d", 4)):
        d, g = synth.random_tiles(args.tiles, 1, m + 2, 3, "uniform", seed=0)
        ranking, _, _ = S.run_search(S.PAPER_TABLE_TEMPLATES[key], 1, m, 3, cs, torch.from_numpy(d).cuda(),
                                     torch.from_numpy(g).cuda(), flags=flags)
        out[key] = {"paper_best": PAPER_BEST[key],
                    "ours": [{"template": t.label(), "c": (p[0] if p else None), "mae": e} for t, p, e in ranking]}
    out["order"] = args.order
    print(json.dumps(out))


if __name__ == "__main__":
    main()
