"""The multi-GPU sweep driver's sharding and reduction logic (paper_2201_10369_b200.sweep),
run on CPU with world_size 2 over gloo.  The per-rank compute is injected (the oracle's
sweep on the rank's candidate block) -- the product compute is the C ABI on a GPU; here
we test that contiguous candidate blocks + zero-padded SUM/MAX all-reduces reproduce the
single-process statistics bitwise, for any world size."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import ref
from paper_2201_10369_b200.sweep import RankSweep, SweepSpec, argmin_c, curve, run_step, shard


def _spec():
    cs = synth.c_grid(40)
    cs = np.concatenate([cs, [1.0]])  # c = 1 duplicates points (-1/c == -c): rejected
    return SweepSpec("2d_uniform", 2, "f43_c", cs, "uniform", n_tiles=700, seed=3)


def _oracle_compute(rs: RankSweep):
    d, g = synth.random_tiles(rs.spec.n_tiles, rs.spec.dims, rs.spec.n, rs.spec.r, rs.spec.dist, rs.spec.seed)
    status = np.zeros(rs.hi - rs.lo, dtype=np.int32)
    good = [k for k in range(rs.hi - rs.lo) if not np.any(np.isnan(rs.sets[k])) and len(set(rs.sets[k])) == rs.spec.n]
    status[[k for k in range(rs.hi - rs.lo) if k not in good]] = 3
    if good:
        s, mx, _ = ref.sweep(rs.spec.dims, rs.spec.m, rs.spec.r, [list(rs.sets[k]) for k in good], d, g)
        for j, k in enumerate(good):
            rs.sums[rs.lo + k] += torch.from_numpy(s[j])
            rs.maxs[rs.lo + k] = torch.maximum(rs.maxs[rs.lo + k], torch.from_numpy(mx[j]))
    rs.status = status
    rs.launches = 0


def _make(spec, rank, world):
    lo, hi = shard(spec.n_cand, rank, world)
    sets = spec.point_sets(lo, hi)
    sums = torch.zeros((spec.n_cand, 5), dtype=torch.float64)
    maxs = torch.zeros((spec.n_cand, 2), dtype=torch.float64)
    return RankSweep(spec, rank, world, lo, hi, sets, None, None, sums, maxs, None)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rs = _make(_spec(), rank, world)
    run_step([rs], compute=_oracle_compute)
    if rank == 0:
        np.save(out + "_sums.npy", rs.sums.numpy())
        np.save(out + "_maxs.npy", rs.maxs.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_blocks_cover_exactly():
    for n in (0, 1, 7, 4096, 4097):
        for w in (1, 2, 3, 8):
            blocks = [shard(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_equals_single(tmp_path, world):
    spec = _spec()
    single = _make(spec, 0, 1)
    run_step([single], compute=_oracle_compute)   # no process group: no reduction
    out = str(tmp_path / "w")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    s = np.load(out + "_sums.npy")
    m = np.load(out + "_maxs.npy")
    assert np.array_equal(s, single.sums.numpy())
    assert np.array_equal(m, single.maxs.numpy())
    mae = curve(s)
    assert math.isnan(mae[-1])            # c = 1 rejected, stays zero -> NaN in the curve
    assert np.all(np.isfinite(mae[:-1]))
    i, best = argmin_c(spec.params, mae)
    assert best == np.nanmin(mae) and 0.3 < spec.params[i] < 3.5


def test_argmin_ties_go_to_smaller_parameter():
    params = np.array([3.0, 1.0, 2.0])
    mae = np.array([1e-7, 1e-7, 2e-7])
    assert argmin_c(params, mae) == (1, 1e-7)
    assert argmin_c(params, np.array([np.nan] * 3)) == (None, None)
