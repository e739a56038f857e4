"""NEXT row N1: reproduce the paper's search experiments with the template search over the
sweep kernels, in the paper's Huffman summation order (reading R21; WINO_SWEEP_HUFFMAN)
or the sequential no-FMA order.

    python tools/search_tables.py [--tiles 5000] [--order huffman|nofma] [--parts optimal,patterns,cd]

* optimal  -- tab:optimal_f23 / f33 / f43, 1D AND 2D columns: every listed
              template swept over c in [1.0, 2.6] step 0.002, ranked by its minimum error.
* patterns -- tab:pattern_1d / pattern_2d: for the base points {0,3,inf},
              {0,-3,inf}, {0,1/2,inf}, {0,1,-1,inf} every subset of {-1/c,-c,c,1/c} completing
              F(3,3) / F(4,3); per base the subset with the lowest minimum error and, per c,
              how often each subset is the best one (the paper's "always reduces the error").
* cd       -- the (c, d) rows of tab:sota_1d / sota_2d for n = 7, 9, 10
              re-derived by a coarse (step 1e-2) then fine (step 1e-3, +-2 coarse cells) grid
              search (our reading of the unstated 2-parameter procedure),
              beside the prior-work sets P4 u {1/2,-3,-1/2} / P8 u {-1/4} / P10.

The paper scores 5000 random inputs per point; --tiles defaults to that.  Prints one
JSON line with the paper's printed values next to ours."""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2201_10369_b200 import api, search as S  # noqa: E402
from paper_2201_10369_b200.sweep import curve  # noqa: E402

INF = math.inf
T = S.Template

# tab:optimal_f23 / f33 / f43: (template, paper c, paper error) per column
OPTIMAL = {
    ("f23", 1): [(T((), ("-1/c", "1/c")), 1.125, 3.11e-8), (T((0.5,), ("-c",)), 1.5, 3.74e-8),
                 (T((3.0,), ("-1/c",)), 1.279, 4.82e-8), (T((-3.0,), ("1/c",)), 1.292, 4.85e-8),
                 (T((1.0,), ("-c",)), 1.016, 3.13e-8), (T((-1.0,), ("1/c",)), 1.028, 3.06e-8)],
    ("f23", 2): [(T((), ("-1/c", "1/c")), 1.054, 9.22e-8), (T((0.5,), ("-c",)), 1.224, 1.31e-7),
                 (T((3.0,), ("-1/c",)), 1.442, 2.02e-7), (T((-3.0,), ("-1/c",)), 1.407, 2.01e-7),
                 (T((1.0,), ("-1/c",)), 1.133, 9.53e-8), (T((-1.0,), ("1/c",)), 1.102, 9.56e-8)],
    ("f33", 1): [(T((), ("-c", "c", "1/c")), 1.64, 5.41e-8), (T((0.5,), ("-c", "c")), 1.326, 4.20e-8),
                 (T((3.0,), ("-1/c", "1/c")), 1.363, 5.34e-8), (T((-3.0,), ("-1/c", "1/c")), 1.298, 5.53e-8),
                 (T((1.0, -1.0), ("c",)), 2.0, 5.04e-8)],
    ("f33", 2): [(T((), ("-1/c", "c", "1/c")), 1.571, 2.27e-7), (T((0.5,), ("-c", "c")), 1.614, 1.89e-7),
                 (T((3.0,), ("-1/c", "1/c")), 1.38, 2.24e-7), (T((-3.0,), ("-1/c", "1/c")), 1.334, 2.32e-7),
                 (T((1.0, -1.0), ("-c",)), 2.0, 1.51e-7)],
    ("f43", 1): [(T((), S.C_MEMBERS), 1.829, 5.65e-8), (T((0.5,), ("-1/c", "-c", "c")), 1.736, 5.81e-8),
                 (T((3.0,), ("-1/c", "-c", "1/c")), 1.613, 6.63e-8),
                 (T((-3.0,), ("-1/c", "c", "1/c")), 1.636, 6.71e-8),   # printed "{-3,-1/c,c,}" (X22)
                 (T((1.0, -1.0), ("-1/c", "c")), 2.431, 6.78e-8)],
    ("f43", 2): [(T((), S.C_MEMBERS), 1.622, 2.37e-7), (T((0.5,), ("-1/c", "-c", "c")), 1.614, 2.52e-7),
                 (T((3.0,), ("-1/c", "-c", "1/c")), 1.567, 3.23e-7),
                 (T((-3.0,), ("-1/c", "-c", "1/c")), 1.578, 3.22e-7),
                 (T((1.0, -1.0), ("-1/c", "c")), 2.125, 3.30e-7)],
}

# tab:pattern_1d / pattern_2d: base -> paper's subset for F(3,3), F(4,3)
PATTERN_BASES = [(3.0,), (-3.0,), (0.5,), (1.0, -1.0)]
PATTERN_PAPER = {
    1: {(3.0,): ("{-1/c,1/c}", "{-1/c,-c,1/c}"), (-3.0,): ("{-1/c,1/c}", "{-1/c,c,1/c}"),
        (0.5,): ("{-c,c}", "{-1/c,-c,c}"), (1.0, -1.0): ("no pattern", "{-1/c,c}")},
    2: {(3.0,): ("{-1/c,1/c}", "{-1/c,-c,1/c}"), (-3.0,): ("{-1/c,1/c}", "{-1/c,-c,1/c}"),
        (0.5,): ("{-c,c}", "{-1/c,-c,c}"), (1.0, -1.0): ("no pattern", "{-1/c,c}")},
}


def _c(*v):
    return sorted(float(x) for x in v) + [INF]


# (c, d) rows of tab:sota_1d / sota_2d: n -> (finite-point maker, prior-work set, paper values)
def _n7(c, d):
    return _c(0.0, -1 / c, -c, c, 1 / c, d)


def _n9(c, d):
    return _c(0.0, -1 / c, -c, c, 1 / c, -1 / d, -d, d)


def _n10(c, d):
    return _c(0.0, -1 / c, -c, c, 1 / c, -1 / d, -d, d, 1 / d)


CD_ROWS = {
    7: (_n7, _c(0.0, -1.0, 1.0, 0.5, -0.5, -3.0), {1: ((2.22, 1.0), 1.07e-7, 9.35e-8), 2: ((2.0, 1.0), 7.72e-7, 6.81e-7)}),
    9: (_n9, _c(0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0, -0.25),
        {1: ((1.313, 2.478), 2.29e-7, 2.34e-7), 2: ((1.305, 2.485), 3.06e-6, 3.71e-6)}),
    10: (_n10, _c(0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0, -0.25, 4.0),
         {1: ((1.953, 1.229), 1.4e-7, 3.46e-7), 2: ((1.272, 2.099), 5.28e-6, 7.35e-6)}),
}
# the prior-work set of the n = 7 2D row differs (P4 u {1/2, -2, -1/2})
CD_PRIOR_2D = {7: _c(0.0, -1.0, 1.0, 0.5, -2.0, -0.5)}


def _tiles(dims, n, r, count, dev):
    d, g = synth.random_tiles(count, dims, n, r, "uniform", seed=0)
    return torch.from_numpy(d).to(dev), torch.from_numpy(g).to(dev)


def _mae_of_sets(dims, m, r, sets, dt, gt, flags):
    sets = np.asarray(sets, dtype=np.float64)
    S_ = sets.shape[0]
    sums = torch.zeros((S_, 5), dtype=torch.float64, device=dt.device)
    maxs = torch.zeros((S_, 2), dtype=torch.float64, device=dt.device)
    ws = torch.empty(max(1, api.wino_error_sweep_workspace_bytes(dims, m, r, S_, dt.shape[0])), dtype=torch.uint8,
                     device=dt.device)
    st = api.wino_error_sweep(dims, m, r, sets, dt, gt, sums, maxs, ws, flags=flags)
    return curve(sums.cpu().numpy(), st)


def part_optimal(args, flags, dev):
    cs = list(np.round(np.arange(1.0, 2.6, 0.002), 6))
    out = {}
    for (fam, dims), rows in OPTIMAL.items():
        m = {"f23": 2, "f33": 3, "f43": 4}[fam]
        dt, gt = _tiles(dims, m + 2, 3, args.tiles, dev)
        templates = [t for t, _, _ in rows]
        ranking, _, _ = S.run_search(templates, dims, m, 3, cs, dt, gt, flags=flags)
        ours = {t.label(): (p[0] if p else None, e) for t, p, e in ranking}
        out[f"{fam}_{dims}d"] = {
            "paper_best": min(rows, key=lambda x: x[2])[0].label(),
            "our_best": ranking[0][0].label(),
            "rows": [{"template": t.label(), "paper_c": pc, "paper_err": pe, "our_c": ours[t.label()][0],
                      "our_err": ours[t.label()][1]} for t, pc, pe in rows],
        }
    return out


def part_patterns(args, flags, dev):
    cs = list(np.round(np.arange(1.1, 2.5, 0.002), 6))
    out = {}
    for dims in (1, 2):
        for m in (3, 4):
            dt, gt = _tiles(dims, m + 2, 3, args.tiles, dev)
            for base in PATTERN_BASES:
                templates = S.enumerate_templates(m + 2, bases=[base])
                ranking, mae, _ = S.run_search(templates, dims, m, 3, cs, dt, gt, flags=flags)
                _, owner, _ = S.candidates(templates, cs)
                # per c: which subset has the lowest error
                per_c = mae.reshape(len(templates), len(cs))
                wins = {}
                for j in range(len(cs)):
                    col = per_c[:, j]
                    if np.all(np.isnan(col)):
                        continue
                    w = templates[int(np.nanargmin(col))].label()
                    wins[w] = wins.get(w, 0) + 1
                tot = sum(wins.values())
                key = f"F({m},3)_{dims}d_base{{0,{','.join(f'{b:g}' for b in base)},inf}}"
                out[key] = {
                    "paper": PATTERN_PAPER[dims][base][m - 3],
                    "best_by_min": ranking[0][0].label(), "best_min_c": ranking[0][1][0], "best_min_err": ranking[0][2],
                    "win_fraction_over_c": {k: v / tot for k, v in sorted(wins.items(), key=lambda kv: -kv[1])},
                    "ranking": [(t.label(), e) for t, _, e in ranking],
                }
    return out


def part_cd(args, flags, dev):
    out = {}
    for n, (maker, prior, paper) in CD_ROWS.items():
        m = n - 2
        for dims in (1, 2):
            if not api.wino_supported(dims, m, 3):
                continue
            dt, gt = _tiles(dims, n, 3, args.tiles, dev)
            t0 = time.time()

            def score(pairs):
                sets = []
                for c, d in pairs:
                    p = maker(c, d)
                    sets.append(p if len(set(p)) == len(p) else [math.nan] * n)
                return _mae_of_sets(dims, m, 3, sets, dt, gt, flags)

            coarse_c = np.round(np.arange(1.0, 2.6 + 1e-9, 0.01), 6)
            coarse_d = np.round(np.arange(0.5, 4.0 + 1e-9, 0.01), 6)
            pairs = [(c, d) for c in coarse_c for d in coarse_d]
            mae = score(pairs)
            i = int(np.nanargmin(mae))
            cc, dc = pairs[i]
            fine_c = np.round(np.arange(cc - 0.02, cc + 0.02 + 1e-9, 0.001), 6)
            fine_d = np.round(np.arange(dc - 0.02, dc + 0.02 + 1e-9, 0.001), 6)
            fpairs = [(c, d) for c in fine_c for d in fine_d if c > 0 and d > 0]
            fmae = score(fpairs)
            j = int(np.nanargmin(fmae))
            prior_set = CD_PRIOR_2D.get(n, prior) if dims == 2 else prior
            prior_err = float(_mae_of_sets(dims, m, 3, [prior_set], dt, gt, flags)[0])
            paper_cd, paper_err, paper_prior = paper[dims]
            paper_set_err = float(score([paper_cd])[0])
            ours = float(fmae[j])
            out[f"n{n}_{dims}d"] = {
                "coarse_argmin": [cc, dc], "coarse_err": float(mae[i]), "fine_argmin": list(fpairs[j]), "fine_err": ours,
                "candidates": len(pairs) + len(fpairs), "seconds": time.time() - t0,
                "prior_err": prior_err, "improvement_pct": 100.0 * (prior_err - ours) / prior_err,
                "paper_cd": list(paper_cd), "paper_err": paper_err, "paper_prior_err": paper_prior,
                "paper_improvement_pct": 100.0 * (paper_prior - paper_err) / paper_prior,
                "our_err_at_paper_cd": paper_set_err,
            }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=5000)
    ap.add_argument("--order", choices=["huffman", "nofma"], default="huffman")
    ap.add_argument("--parts", default="optimal,patterns,cd")
    args = ap.parse_args()
    flags = api.WINO_SWEEP_HUFFMAN if args.order == "huffman" else api.WINO_SWEEP_NOFMA
    dev = torch.device("cuda", 0)
    out = {"order": args.order, "tiles": args.tiles,
           "note": "random uniform[-1,1] tiles (P:465, reading R9); errors are per-element mean |e| vs fp64 direct"}
    parts = args.parts.split(",")
    if "optimal" in parts:
        out["optimal"] = part_optimal(args, flags, dev)
    if "patterns" in parts:
        out["patterns"] = part_patterns(args, flags, dev)
    if "cd" in parts:
        out["cd"] = part_cd(args, flags, dev)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
