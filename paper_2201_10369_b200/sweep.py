"""c-sweep driver: one process per GPU, candidates sharded in contiguous
blocks over ranks, per-rank stats written into zero-padded global [S,5] / [S,2] fp64
buffers -- views of ONE flat buffer for all the job's sweeps -- then ONE all_reduce(SUM)
(NCCL over NVLink) per step.  Every candidate row has exactly one owner rank and the other
ranks hold zeros, so the SUM is exact for the sums AND the maxs (x + 0 = x; NaN rows of
rejected candidates stay NaN): the reduced statistics are bitwise independent of the world
size.

The per-rank compute is the C ABI (``wino_error_sweep``); a different ``compute`` can be
injected for CPU (gloo) tests of the sharding / reduction logic.
"""
from __future__ import annotations


import math
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import points as P

INF = math.inf


@dataclass
class SweepSpec:
    """One sweep: a point-set template over a parameter list, scored on shared tiles."""
    name: str
    dims: int
    template: str                   # key of points.TEMPLATES
    params: np.ndarray              # [S] or [S, n_params] fp64
    dist: str = "uniform"
    n_tiles: int = 100_000
    seed: int = 0
    flags: int = 0

    @property
    def m(self) -> int:
        return P.TEMPLATES[self.template][0]

    @property
    def r(self) -> int:
        return P.TEMPLATES[self.template][1]

    @property
    def n(self) -> int:
        return self.m + self.r - 1

    @property
    def n_cand(self) -> int:
        return int(self.params.shape[0])

    def point_sets(self, lo: int = 0, hi: Optional[int] = None) -> np.ndarray:
        """a1: instantiate candidates [lo, hi) as explicit fp64 point sets [S, n]."""
        maker = P.TEMPLATES[self.template][3]
        hi = self.n_cand if hi is None else hi
        rows = [tuple(np.atleast_1d(self.params[i]).tolist()) for i in range(lo, hi)]
        sets, _ = P.instantiate(maker, rows)
        return np.array(sets, dtype=np.float64).reshape(hi - lo, self.n)


def cfg2_specs(c_values: np.ndarray, n_tiles: int = 100_000) -> List[SweepSpec]:
    """BASELINE.json configs[1]: F(4,3) / F(4x4,3x3) on {0, ±c, ±1/c, inf}, 1D and 2D, each
    on uniform[-1,1] (seed 0) and N(0,1) (seed 1) tiles."""
    out = []
    for dims in (1, 2):
        for dist, seed in (("uniform", 0), ("normal", 1)):
            out.append(SweepSpec(f"{dims}d_{dist}", dims, "f43_c", np.asarray(c_values, dtype=np.float64),
                                 dist, n_tiles, seed))
    return out


def shard(n: int, rank: int, world: int):
    """Contiguous block of [0, n) owned by `rank`."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


@dataclass
class RankSweep:
    """Device-resident state of one sweep on one rank."""
    spec: SweepSpec
    rank: int
    world: int
    lo: int
    hi: int
    sets: np.ndarray                  # this rank's point sets
    d_tiles: object                   # device tensors
    g_tiles: object
    sums: object                      # global [S,5] / [S,2] (zero padded)
    maxs: object
    workspace: object
    status: np.ndarray = field(default=None)
    launches: int = 0
    flat: object = None               # the flat statistics buffer sums/maxs are views of


def make_rank_sweep(spec: SweepSpec, rank: int, world: int, device, d_host: np.ndarray, g_host: np.ndarray):
    import torch
    from . import api
    lo, hi = shard(spec.n_cand, rank, world)
    sets = spec.point_sets(lo, hi)
    d_t = torch.from_numpy(d_host).to(device)
    g_t = torch.from_numpy(g_host).to(device)
    sums = torch.zeros((spec.n_cand, 5), dtype=torch.float64, device=device)
    maxs = torch.zeros((spec.n_cand, 2), dtype=torch.float64, device=device)
    wsb = api.wino_error_sweep_workspace_bytes(spec.dims, spec.m, spec.r, max(hi - lo, 1), spec.n_tiles)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=device)
    return RankSweep(spec, rank, world, lo, hi, sets, d_t, g_t, sums, maxs, ws)


def pack_stats(rank_sweeps: Sequence[RankSweep]):
    """Rebind every sweep's sums [S,5] / maxs [S,2] to contiguous views of one flat fp64
    buffer (so one collective reduces the whole job).  Returns the buffer."""
    import torch
    total = sum(rs.spec.n_cand * 7 for rs in rank_sweeps)
    flat = torch.zeros(max(total, 1), dtype=torch.float64, device=rank_sweeps[0].sums.device)
    off = 0
    for rs in rank_sweeps:
        S = rs.spec.n_cand
        rs.sums = flat[off:off + 5 * S].view(S, 5)
        off += 5 * S
        rs.maxs = flat[off:off + 2 * S].view(S, 2)
        off += 2 * S
        rs.flat = flat
    return flat


def abi_compute(rs: RankSweep, stream=None) -> None:
    """The product compute: wino_error_sweep on this rank's candidate block, writing into
    the global buffers' [lo, hi) rows."""
    from . import api
    if rs.hi <= rs.lo:
        return
    rs.status = api.wino_error_sweep(rs.spec.dims, rs.spec.m, rs.spec.r, rs.sets, rs.d_tiles, rs.g_tiles,
                                     rs.sums[rs.lo:rs.hi], rs.maxs[rs.lo:rs.hi], rs.workspace,
                                     flags=rs.spec.flags, stream=stream)
    rs.launches = api.wino_last_launch_count()


def run_step(rank_sweeps: Sequence[RankSweep], compute: Callable = abi_compute, group=None,
             reduce: bool = True) -> int:
    """One step: zero the global buffers, compute every sweep's block, ONE all-reduce(SUM)
    of the flat statistics buffer (packed on first use).  Returns the number of library
    kernel launches enqueued."""
    import torch.distributed as dist
    if any(rs.flat is None for rs in rank_sweeps):
        pack_stats(rank_sweeps)
    flats = list({id(rs.flat): rs.flat for rs in rank_sweeps}.values())
    for f in flats:
        f.zero_()
    launches = 0
    for rs in rank_sweeps:
        compute(rs)
        launches += rs.launches
    # (WINO_FORCE_COLLECTIVES=1: also with one rank, so a 1-GPU box exercises the NCCL call)
    if reduce and dist.is_available() and dist.is_initialized() and (
            dist.get_world_size() > 1 or os.environ.get("WINO_FORCE_COLLECTIVES") == "1"):
        for f in flats:
            dist.all_reduce(f, op=dist.ReduceOp.SUM, group=group)
    return launches


def curve(sums: np.ndarray, status: Optional[np.ndarray] = None) -> np.ndarray:
    """Per-candidate mean absolute error Σ|e| / n_scored; NaN where rejected or non-finite."""
    s = np.asarray(sums, dtype=np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        mae = s[:, 0] / s[:, 3]
    bad = (s[:, 3] == 0) | (s[:, 4] > 0)
    if status is not None:
        bad |= np.asarray(status) != 0
    mae[bad] = np.nan
    return mae


def argmin_c(params: np.ndarray, mae: np.ndarray):
    """Argmin ignoring non-finite entries; ties go to the smaller parameter."""
    ok = np.isfinite(mae)
    if not ok.any():
        return None, None
    best = np.nanmin(np.where(ok, mae, np.nan))
    idx = [i for i in range(len(mae)) if ok[i] and mae[i] == best]
    i = min(idx, key=lambda j: tuple(np.atleast_1d(params[j]).tolist()))
    return i, float(best)
