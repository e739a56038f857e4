"""NEXT row N1: the paper's template / subset search over the sweep kernel.

A template fixes the base points (always 0 and the formal ∞, plus optional prior-work
points such as 1, -1, 1/2, ±3) and picks members of the symmetric family
{-1/c, -c, c, 1/c} (and, for n > 6, of {-1/d, -d, d, 1/d}):

* eq:ps3: for F(3,3) all 3-element subsets of the c-family;
* eq:subset_points: F(4,3) with base {1, -1} + 2 members, or base {-3} + 3;
* the d-subsets of P:322-327: for F(7,3)-sized sets, all c-members plus 2 d-members;
* the rows of Tables tab:optimal_f23 / f33 / f43.

All templates x all parameter values become one candidate list of explicit point sets
(a1 on the host), scored by ONE wino_error_sweep call per (dims, m) on shared tiles;
templates are ranked by their best (minimum) mean absolute error over the grid.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

INF = math.inf
C_MEMBERS = ("-1/c", "-c", "c", "1/c")
D_MEMBERS = ("-1/d", "-d", "d", "1/d")


def _member(name: str, c: float, d: float) -> float:
    v = {"-1/c": -(1.0 / c), "-c": -c, "c": c, "1/c": 1.0 / c,
         "-1/d": -(1.0 / d), "-d": -d, "d": d, "1/d": 1.0 / d}
    return v[name]


@dataclass(frozen=True)
class Template:
    """Points = {0} ∪ base ∪ chosen family members ∪ {∞}; canonical order."""
    base: Tuple[float, ...]
    members: Tuple[str, ...]

    @property
    def n(self) -> int:
        return 2 + len(self.base) + len(self.members)

    @property
    def n_params(self) -> int:
        return 2 if any("d" in m for m in self.members) else 1

    def points(self, c: float, d: float = 2.0) -> List[float]:
        fin = [0.0, *self.base, *(_member(mm, c, d) for mm in self.members)]
        fin = sorted(float(v) for v in fin)
        return fin + [INF]

    def valid(self, c: float, d: float = 2.0) -> bool:
        p = self.points(c, d)[:-1]
        return all(math.isfinite(v) for v in p) and len(set(p)) == len(p)

    def label(self) -> str:
        b = ",".join(f"{v:g}" for v in self.base)
        return "{" + ",".join([x for x in (b,) if x] + list(self.members)) + "}"


def subsets(members: Sequence[str], k: int) -> List[Tuple[str, ...]]:
    return [tuple(s) for s in itertools.combinations(members, k)]


def enumerate_templates(n: int, bases: Sequence[Tuple[float, ...]] = ((),)) -> List[Template]:
    """Every template with n points: for each base, all subsets of the c-family of the
    size that completes the set (n = 2 + |base| + k); when k > 4 all c-members plus the
    (k-4)-subsets of the d-family."""
    out = []
    for base in bases:
        k = n - 2 - len(base)
        if k < 0:
            continue
        if k <= 4:
            out += [Template(tuple(base), s) for s in subsets(C_MEMBERS, k)]
        elif k <= 8:
            out += [Template(tuple(base), C_MEMBERS + s) for s in subsets(D_MEMBERS, k - 4)]
    return out


# Rows of the paper's optimality tables (the base points + members it lists, 0/∞ implicit)
PAPER_TABLE_TEMPLATES: Dict[str, List[Template]] = {
    # tab:optimal_f23, 1D column
    "f23_1d": [Template((), ("-1/c", "1/c")), Template((0.5,), ("-c",)), Template((3.0,), ("-1/c",)),
               Template((-3.0,), ("1/c",)), Template((1.0,), ("-c",)), Template((-1.0,), ("1/c",))],
    # tab:optimal_f33, 1D column
    "f33_1d": [Template((), ("-c", "c", "1/c")), Template((0.5,), ("-c", "c")), Template((3.0,), ("-1/c", "1/c")),
               Template((-3.0,), ("-1/c", "1/c")), Template((1.0, -1.0), ("c",))],
    # tab:optimal_f43, 1D column (row 4 read as {-3, -1/c, c, 1/c}, reading X22)
    "f43_1d": [Template((), C_MEMBERS), Template((0.5,), ("-1/c", "-c", "c")), Template((3.0,), ("-1/c", "-c", "1/c")),
               Template((-3.0,), ("-1/c", "c", "1/c")), Template((1.0, -1.0), ("-1/c", "c"))],
}


def candidates(templates: Sequence[Template], c_values: Sequence[float], d_values: Sequence[float] = (2.0,)):
    """Explicit point sets for every (template, c[, d]); invalid combinations (duplicate
    points) become NaN rows, rejected per candidate by the library."""
    rows, owner, params = [], [], []
    for ti, t in enumerate(templates):
        ds = d_values if t.n_params == 2 else (2.0,)
        for c in c_values:
            for d in ds:
                rows.append(t.points(c, d) if t.valid(c, d) else [math.nan] * t.n)
                owner.append(ti)
                params.append((c, d))
    return np.array(rows, dtype=np.float64), np.array(owner), np.array(params)


def rank(templates: Sequence[Template], owner: np.ndarray, params: np.ndarray, mae: np.ndarray):
    """Per template: (best parameter, min MAE); sorted by min MAE (NaN last)."""
    res = []
    for ti, t in enumerate(templates):
        idx = np.flatnonzero((owner == ti) & np.isfinite(mae))
        if len(idx) == 0:
            res.append((t, None, math.nan))
            continue
        j = idx[np.argmin(mae[idx])]
        res.append((t, tuple(params[j]), float(mae[j])))
    return sorted(res, key=lambda x: (math.isnan(x[2]), x[2]))


def run_search(templates: Sequence[Template], dims: int, m: int, r: int, c_values, d_tiles, g_tiles,
               flags: int = 0, d_values=(2.0,), stream=None):
    """One wino_error_sweep over every (template, parameter); returns the ranking and the
    per-candidate MAE.  d_tiles / g_tiles: CUDA tensors [T, n^dims] / [T, r^dims]."""
    import torch
    from . import api
    from .sweep import curve
    ps, owner, params = candidates(templates, c_values, d_values)
    S = ps.shape[0]
    dev = d_tiles.device
    sums = torch.zeros((S, 5), dtype=torch.float64, device=dev)
    maxs = torch.zeros((S, 2), dtype=torch.float64, device=dev)
    ws = torch.empty(max(1, api.wino_error_sweep_workspace_bytes(dims, m, r, S, d_tiles.shape[0])), dtype=torch.uint8,
                     device=dev)
    status = api.wino_error_sweep(dims, m, r, ps, d_tiles, g_tiles, sums, maxs, ws, flags=flags, stream=stream)
    mae = curve(sums.cpu().numpy(), status)
    return rank(templates, owner, params, mae), mae, status
