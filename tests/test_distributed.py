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
    bad = [k for k in range(rs.hi - rs.lo) if k not in good]
    status[bad] = 3
    for k in bad:                      # the ABI's convention: rejected rows are NaN
        rs.sums[rs.lo + k] = float("nan")
        rs.maxs[rs.lo + k] = float("nan")
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


def _spec1d():
    cs = synth.c_grid(23)
    return SweepSpec("1d_normal", 1, "f43_c", cs, "normal", n_tiles=900, seed=4)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rss = [_make(_spec(), rank, world), _make(_spec1d(), rank, world)]
    run_step(rss, compute=_oracle_compute)      # one packed SUM all-reduce for both sweeps
    assert rss[0].flat is rss[1].flat
    if rank == 0:
        np.save(out + "_sums.npy", rss[0].sums.numpy())
        np.save(out + "_maxs.npy", rss[0].maxs.numpy())
        np.save(out + "_sums1d.npy", rss[1].sums.numpy())
        np.save(out + "_maxs1d.npy", rss[1].maxs.numpy())
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
    assert np.array_equal(s, single.sums.numpy(), equal_nan=True)
    assert np.array_equal(m, single.maxs.numpy(), equal_nan=True)
    single1d = _make(_spec1d(), 0, 1)
    run_step([single1d], compute=_oracle_compute)
    assert np.array_equal(np.load(out + "_sums1d.npy"), single1d.sums.numpy(), equal_nan=True)
    assert np.array_equal(np.load(out + "_maxs1d.npy"), single1d.maxs.numpy(), equal_nan=True)
    mae = curve(s)
    assert math.isnan(mae[-1])            # c = 1 rejected: NaN statistics -> NaN in the curve
    assert np.all(np.isfinite(mae[:-1]))
    i, best = argmin_c(spec.params, mae)
    assert best == np.nanmin(mae) and 0.3 < spec.params[i] < 3.5


def test_argmin_ties_go_to_smaller_parameter():
    params = np.array([3.0, 1.0, 2.0])
    mae = np.array([1e-7, 1e-7, 2e-7])
    assert argmin_c(params, mae) == (1, 1e-7)
    assert argmin_c(params, np.array([np.nan] * 3)) == (None, None)


# ------------------------------------------------------------------ network batch split
# the VGG-style stack sharded by batch; per-image statistics in a
# zero-padded [L][N][7] buffer, one SUM all-reduce, fixed-order reduction over images.
# The per-rank layer compute is the oracle here (CPU); on the GPU it is the C ABI.

_NET = [(3, 8, 16, False), (8, 8, 16, True), (8, 16, 8, False)]
_NET_IMAGES = 5


def _net_inputs():
    return synth.stack_inputs(_NET, _NET_IMAGES, seed=9)


def _oracle_conv(a, w, y, act, pool, m, points, ws, sums, maxs, stream):
    from oracle import network as ON
    x, wt = a.numpy(), w.numpy()
    yy = ref.conv2d_wino(x, wt, 1, m, points)
    y64 = ref.conv2d_direct64(x, wt, 1)
    if y is not None:
        y.copy_(torch.from_numpy(yy))
    act.copy_(torch.from_numpy(ON.relu_pool(yy, pool == 2)))
    for i in range(x.shape[0]):
        si, mi = ref.stats(yy[i], y64[i])
        sums[i] += torch.from_numpy(si)
        maxs[i] = torch.maximum(maxs[i], torch.from_numpy(mi))


def _net_run(rank, world, group=None):
    from oracle import points as OP
    from paper_2201_10369_b200 import network
    x, ws = _net_inputs()
    lo, hi = network.shard(_NET_IMAGES, rank, world)
    return network.stack_forward(_NET, torch.from_numpy(x[lo:hi]), [torch.from_numpy(w) for w in ws],
                                 OP.f23_c(1.0), m=2, rank=rank, world=world, n_global=_NET_IMAGES, group=group,
                                 conv=_oracle_conv, ws_bytes=lambda *a: 1)


def _net_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    act, sums, maxs, _, per_img = _net_run(rank, world)
    np.save(out + f"_act{rank}.npy", act.numpy())
    if rank == 0:
        np.save(out + "_nsums.npy", sums)
        np.save(out + "_nmaxs.npy", maxs)
        np.save(out + "_nper.npy", per_img)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_network_batch_split_equals_single(tmp_path, world):
    from paper_2201_10369_b200 import network
    act1, s1, m1, _, per1 = _net_run(0, 1)
    out = str(tmp_path / "n")
    mp.start_processes(_net_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    assert np.array_equal(np.load(out + "_nsums.npy"), s1)
    assert np.array_equal(np.load(out + "_nmaxs.npy"), m1)
    assert np.array_equal(np.load(out + "_nper.npy"), per1)
    acts = np.concatenate([np.load(out + f"_act{r}.npy") for r in range(world)])
    assert np.array_equal(acts, act1.numpy())
    # the per-layer statistics are the whole-batch statistics of the oracle chain
    from oracle import network as ON, points as OP
    x, ws = _net_inputs()
    _, s_ref, m_ref = ON.stack(_NET, x, ws, OP.f23_c(1.0), m=2)
    assert np.array_equal(s1[:, 3:], s_ref[:, 3:]) and np.array_equal(m1, m_ref)
    assert np.allclose(s1[:, :3], s_ref[:, :3], rtol=1e-12, atol=0)
    assert network.normalized_l1(s1, _NET_IMAGES) > 0
