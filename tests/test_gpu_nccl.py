"""The NCCL calls of the multi-GPU path on ONE GPU: a single-rank NCCL
process group with WINO_FORCE_COLLECTIVES=1, so the packed fp64 SUM all-reduce of the sweep
driver and the [L][N][7] all-reduce of the network stack really go through NCCL on device
buffers.  With one rank the collectives are identities: the results must equal the
undistributed run bit for bit (NaN rows of rejected candidates included).  The sharding
logic itself is covered with world sizes 2 and 3 over gloo in tests/test_distributed.py."""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import points as OP

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture()
def nccl_one_rank():
    import datetime
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0), timeout=datetime.timedelta(seconds=120))
    os.environ["WINO_FORCE_COLLECTIVES"] = "1"
    try:
        yield dist
    finally:
        del os.environ["WINO_FORCE_COLLECTIVES"]
        dist.destroy_process_group()


def _sweep_job(torch):
    from paper_2201_10369_b200.sweep import SweepSpec, make_rank_sweep
    dev = torch.device("cuda", 0)
    cs = np.concatenate([synth.c_grid(50), [1.0]])   # c = 1: duplicate points, rejected (NaN row)
    specs = [SweepSpec("2d_uniform", 2, "f43_c", cs, "uniform", 3000, 3),
             SweepSpec("1d_normal", 1, "f43_c", cs, "normal", 3000, 4)]
    rsw = []
    for sp in specs:
        d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
        rsw.append(make_rank_sweep(sp, 0, 1, dev, d, g))
    return rsw


def test_sweep_step_through_nccl(nccl_one_rank):
    import torch
    from paper_2201_10369_b200.sweep import run_step
    rsw = _sweep_job(torch)
    run_step(rsw, reduce=False)
    torch.cuda.synchronize()
    plain = [(rs.sums.cpu().numpy().copy(), rs.maxs.cpu().numpy().copy()) for rs in rsw]
    run_step(rsw)                      # zeroes, recomputes, all_reduce(SUM) over NCCL
    torch.cuda.synchronize()
    for rs, (s0, m0) in zip(rsw, plain):
        assert np.array_equal(rs.sums.cpu().numpy(), s0, equal_nan=True)
        assert np.array_equal(rs.maxs.cpu().numpy(), m0, equal_nan=True)
        assert np.isnan(s0[-1]).all() and np.isfinite(s0[:-1]).all()


def test_network_stack_through_nccl(nccl_one_rank):
    import torch
    from paper_2201_10369_b200 import network
    layers = [(3, 8, 24, True), (8, 16, 12, False)]
    g = np.random.default_rng(5)
    x = torch.from_numpy(g.standard_normal((3, 3, 24, 24)).astype(np.float32)).cuda()
    ws = [torch.from_numpy((g.standard_normal((K, C, 3, 3)) * (2.0 / (C * 9)) ** 0.5).astype(np.float32)).cuda()
          for C, K, _, _ in layers]
    pts = OP.n8_cd(2.0, 1.003)
    a1, s1, m1, _, p1 = network.stack_forward(layers, x, ws, pts, m=6, score=True)
    del os.environ["WINO_FORCE_COLLECTIVES"]
    try:
        a0, s0, m0, _, p0 = network.stack_forward(layers, x, ws, pts, m=6, score=True)
    finally:
        os.environ["WINO_FORCE_COLLECTIVES"] = "1"
    assert torch.equal(a0, a1)
    assert np.array_equal(s0, s1) and np.array_equal(m0, m1) and np.array_equal(p0, p1)
    assert s1[0, 3] == 3 * 8 * 24 * 24
