"""NEXT row N2: the mixed-precision sweep (WINO_SWEEP_MIXED, reading R22) against the
oracle's oref_sweep_mixed: per-element fp32 outputs bit-identical, statistics to fp64
summation noise, and the flag-combination error."""
import math

import numpy as np
import pytest

import synth
from oracle import points as OP, ref

pytestmark = pytest.mark.gpu
INF = math.inf
MIXED = 4


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


SETS = {
    2: [OP.f23_c(1.0), OP.f23_c(1.7), [-2.0, 0.5, 1.0, INF]],
    4: [OP.f43_c(1.622), OP.f43_c(1.829), OP.f43_c(0.3), [-1.0, 0.0, 0.5, 1.0, 2.0, INF]],
    6: [OP.n8_cd(2.0, 1.003), OP.P8],
}


@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("m", [2, 4, 6])
def test_mixed_outputs_bitexact(dims, m):
    import torch
    from paper_2201_10369_b200 import api
    sets = [sorted(p for p in s if p != INF) + [INF] for s in SETS[m]]
    d, g = synth.random_tiles(1031, dims, m + 2, 3, "normal", seed=41)
    y = torch.full((len(sets), d.shape[0], m ** dims), float("nan"), dtype=torch.float32, device="cuda")
    st = api.wino_sweep_outputs(dims, m, 3, np.array(sets), _dev(d), _dev(g), y, flags=MIXED)
    torch.cuda.synchronize()
    assert np.all(st == 0)
    _, _, y_ref = ref.sweep_mixed(dims, m, 3, sets, d, g, n_dump=d.shape[0])
    assert np.array_equal(y.cpu().numpy(), y_ref)


@pytest.mark.parametrize("dims", [1, 2])
def test_mixed_stats(dims):
    import torch
    from paper_2201_10369_b200 import api
    grid = synth.c_grid()
    sets = [OP.f43_c(float(grid[i])) for i in range(0, 4096, 101)]
    d, g = synth.random_tiles(20_011, dims, 6, 3, "uniform", seed=12)
    S, T = len(sets), d.shape[0]
    sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, 4, 3, S, T), dtype=torch.uint8, device="cuda")
    st = api.wino_error_sweep(dims, 4, 3, np.array(sets), _dev(d), _dev(g), sums, maxs, ws, flags=MIXED)
    torch.cuda.synchronize()
    assert np.all(st == 0)
    s, mx = sums.cpu().numpy(), maxs.cpu().numpy()
    s_ref, m_ref, _ = ref.sweep_mixed(dims, 4, 3, sets, d, g)
    assert np.array_equal(s[:, 3], s_ref[:, 3]) and np.array_equal(mx, m_ref)
    assert np.all(np.abs(s[:, 0] / s_ref[:, 0] - 1) < 1e-12)
    assert np.all(np.abs(s[:, 1] / s_ref[:, 1] - 1) < 1e-12)


def test_mixed_flag_errors():
    import torch
    from paper_2201_10369_b200 import api, _lib
    d, g = synth.random_tiles(100, 2, 6, 3, "uniform", seed=1)
    sums = torch.zeros((1, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((1, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(2, 4, 3, 1, 100), dtype=torch.uint8, device="cuda")
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_error_sweep(2, 4, 3, np.array([OP.f43_c(1.5)]), _dev(d), _dev(g), sums, maxs, ws, flags=MIXED | 2)
    assert ei.value.status == 1
