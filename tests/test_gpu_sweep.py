"""GPU parity of the error sweep (wino_error_sweep / wino_sweep_outputs) against the
oracle: per-element fp32 outputs bit-identical (O5 semantics), statistics within the
north-star tolerance (MAE within 1% relative; we assert 1e-5), edge cases.  Calls go
through the C ABI (paper_2201_10369_b200.api)."""
import math

import numpy as np
import pytest

import synth
from oracle import exact, points as OP, ref

pytestmark = pytest.mark.gpu

INF = math.inf


def _torch():
    import torch
    return torch


def _dev(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu_outputs(dims, m, r, sets, d, g, flags=0, with_stats=False):
    """The production sweep kernels with the output store enabled (wino_sweep_outputs);
    with_stats: also the statistics of the same launch."""
    from paper_2201_10369_b200 import api
    torch = _torch()
    S, T = len(sets), d.shape[0]
    y = torch.full((S, T, m ** dims), float("nan"), dtype=torch.float32, device="cuda")
    sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda") if with_stats else None
    maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda") if with_stats else None
    st = api.wino_sweep_outputs(dims, m, r, np.array(sets), _dev(d), _dev(g), y, d_sums=sums, d_maxs=maxs,
                                flags=flags)
    torch.cuda.synchronize()
    if with_stats:
        return st, y.cpu().numpy(), sums.cpu().numpy(), maxs.cpu().numpy()
    return st, y.cpu().numpy()


def _gpu_stats(dims, m, r, sets, d, g, flags=0, sums=None, maxs=None):
    from paper_2201_10369_b200 import api
    torch = _torch()
    S, T = len(sets), d.shape[0]
    if sums is None:
        sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda")
        maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, m, r, S, T), dtype=torch.uint8, device="cuda")
    st = api.wino_error_sweep(dims, m, r, np.array(sets), _dev(d), _dev(g), sums, maxs, ws, flags=flags)
    torch.cuda.synchronize()
    return st, sums.cpu().numpy(), maxs.cpu().numpy()


def _grid_subset(k=48):
    g = synth.c_grid()
    idx = sorted(set(np.linspace(0, len(g) - 1, k).astype(int).tolist() + [2047, 2048]))
    return [float(g[i]) for i in idx]


# Statistics tolerances (north star: MAE within 1 % relative).  Most sweep kernels score in
# fp64 (agreement ~1e-15); the F(4x4,3x3) production kernel scores tile pairs in fp32 within
# a warp-candidate (e to 2^-23 relative, sums to ~1e-6), hence 1e-5 / 1e-6.
RTOL_SUM, RTOL_MAX = 1e-5, 1e-6


def _assert_stats_close(s_gpu, m_gpu, s_ref, m_ref):
    assert np.array_equal(s_gpu[:, 3], s_ref[:, 3])       # n_scored exact
    assert np.array_equal(s_gpu[:, 4], s_ref[:, 4])       # n_nonfinite exact
    assert np.array_equal(m_gpu[:, 1], m_ref[:, 1])        # max|y_ref| exact
    assert np.all(np.abs(m_gpu[:, 0] / m_ref[:, 0] - 1) <= RTOL_MAX)
    mae_g = s_gpu[:, 0] / s_gpu[:, 3]
    mae_r = s_ref[:, 0] / s_ref[:, 3]
    assert np.all(np.abs(mae_g / mae_r - 1) < RTOL_SUM)
    assert np.all(np.abs(s_gpu[:, 1] / s_ref[:, 1] - 1) < RTOL_SUM)
    assert np.all(np.abs(s_gpu[:, 2] / s_ref[:, 2] - 1) < 1e-12)


@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("dist", ["uniform", "normal"])
@pytest.mark.parametrize("nofma", [False, True])
def test_f43_outputs_bitexact(dims, dist, nofma):
    """cfg2 template on a subset of the c grid; 6,007 tiles (several CTAs + ragged tail)."""
    cs = _grid_subset()
    sets = [OP.f43_c(c) for c in cs]
    d, g = synth.random_tiles(6007, dims, 6, 3, dist, seed=11)
    st, y = _gpu_outputs(dims, 4, 3, sets, d, g, flags=int(nofma))
    assert np.all(st == 0)
    _, _, y_ref = ref.sweep(dims, 4, 3, sets, d, g, nofma=nofma, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("dist", ["uniform", "normal"])
def test_f43_stats(dims, dist):
    cs = _grid_subset()
    sets = [OP.f43_c(c) for c in cs]
    d, g = synth.random_tiles(20_011, dims, 6, 3, dist, seed=12)
    st, s, mx = _gpu_stats(dims, 4, 3, sets, d, g)
    assert np.all(st == 0)
    s_ref, m_ref, _ = ref.sweep(dims, 4, 3, sets, d, g)
    _assert_stats_close(s, mx, s_ref, m_ref)


@pytest.mark.parametrize("dims,m,r,maker,args", [
    (2, 2, 3, OP.f23_c, [0.5, 1.0, 1.054, 2.0]),
    (1, 2, 3, OP.f23_c, [0.5, 1.0, 1.054, 2.0]),
    (2, 6, 3, OP.n8_cd, [(2.0, 1.003), (1.5, 2.5)]),
    (1, 6, 3, OP.n8_cd, [(2.0, 1.003), (1.5, 2.5)]),
    (2, 4, 5, OP.n8_c1c2, [(1.5, 3.1), (0.7, 2.2)]),
    (2, 6, 5, OP.n10_c1c2, [(1.272, 2.099), (1.5, 3.1)]),
    (1, 6, 5, OP.n10_c1c2, [(1.272, 2.099)]),
    (2, 8, 3, OP.n10_c1c2, [(1.272, 2.099)]),
    (1, 8, 3, OP.n10_c1c2, [(1.953, 1.229)]),
    # dense (no structural-zero family) large-n kernels with the rolled loops (COMPACT, n >= 9)
    (2, 7, 3, OP.chebyshev, [9]),
    (2, 6, 5, OP.chebyshev, [10]),
    (2, 8, 3, OP.chebyshev, [10]),
])
def test_other_templates_bitexact(dims, m, r, maker, args):
    sets = [maker(*(a if isinstance(a, tuple) else (a,))) for a in args]
    n = m + r - 1
    d, g = synth.random_tiles(1031, dims, n, r, "uniform", seed=13)
    st, y = _gpu_outputs(dims, m, r, sets, d, g)
    assert np.all(st == 0)
    _, _, y_ref = ref.sweep(dims, m, r, sets, d, g, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref)
    st, s, mx = _gpu_stats(dims, m, r, sets, d, g)
    s_ref, m_ref, _ = ref.sweep(dims, m, r, sets, d, g)
    _assert_stats_close(s, mx, s_ref, m_ref)


@pytest.mark.parametrize("dims", [1, 2])
def test_exact_integer_special_case(dims):
    """F(2,3) on {0,±1,∞} with integer tiles: every intermediate is exact, so the GPU
    output equals the exact correlation (independent of the oracle's fp32 code)."""
    d, g = synth.integer_tiles(777, dims, 4, 3, seed=14)
    st, y = _gpu_outputs(dims, 2, 3, [OP.f23_c(1.0)], d, g)
    for t in range(0, 777, 37):
        if dims == 1:
            ex = exact.correlate_1d([int(v) for v in d[t]], [int(v) for v in g[t]])
            assert y[0, t].tolist() == [float(v) for v in ex]
        else:
            dd = d[t].reshape(4, 4).astype(int).tolist()
            gg = g[t].reshape(3, 3).astype(int).tolist()
            ex = exact.correlate_2d(dd, gg)
            assert y[0, t].reshape(2, 2).tolist() == [[float(v) for v in row] for row in ex]


def test_rejected_candidates_and_accumulation():
    """A rejected candidate does not fail the call; its statistics rows become NaN (include/
    wino.h (3)); accepted rows accumulate over calls."""
    torch = _torch()
    sets = [OP.f43_c(1.7), [0.0, 1.0, 1.0, -1.0, 2.0, INF], [math.nan] * 6, OP.f43_c(0.9)]
    d, g = synth.random_tiles(3001, 2, 6, 3, "uniform", seed=15)
    st, s, mx = _gpu_stats(2, 4, 3, sets, d, g)
    assert st.tolist() == [0, 3, 5, 0]
    assert np.all(np.isnan(s[1:3])) and np.all(np.isnan(mx[1:3]))
    s_ref, m_ref, _ = ref.sweep(2, 4, 3, [sets[0], sets[3]], d, g)
    _assert_stats_close(s[[0, 3]], mx[[0, 3]], s_ref, m_ref)
    # second call accumulates into the accepted rows; rejected rows stay NaN
    sums = torch.from_numpy(s).cuda()
    maxs = torch.from_numpy(mx).cuda()
    _, s2, m2 = _gpu_stats(2, 4, 3, sets, d, g, sums=sums, maxs=maxs)
    ok = [0, 3]
    assert np.allclose(s2[ok], 2 * s[ok], rtol=1e-15) and np.array_equal(m2[ok], mx[ok])
    assert np.all(np.isnan(s2[1:3])) and np.all(np.isnan(m2[1:3]))


def test_empty_inputs():
    torch = _torch()
    from paper_2201_10369_b200 import api
    sums = torch.zeros((2, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((2, 2), dtype=torch.float64, device="cuda")
    d = torch.zeros((0, 36), dtype=torch.float32, device="cuda")
    g = torch.zeros((0, 9), dtype=torch.float32, device="cuda")
    ws = torch.empty(max(1, api.wino_error_sweep_workspace_bytes(2, 4, 3, 2, 0)), dtype=torch.uint8, device="cuda")
    st = api.wino_error_sweep(2, 4, 3, np.array([OP.f43_c(1.5), OP.f43_c(2.5)]), d, g, sums, maxs, ws)
    torch.cuda.synchronize()
    assert st.tolist() == [0, 0] and float(sums.abs().sum()) == 0.0
    # no tiles: a rejected candidate still gets NaN rows, the accepted one is untouched
    st = api.wino_error_sweep(2, 4, 3, np.array([OP.f43_c(1.5), [0.0, 1.0, 1.0, -1.0, 2.0, INF]]), d, g, sums,
                              maxs, ws)
    torch.cuda.synchronize()
    s = sums.cpu().numpy()
    assert st.tolist() == [0, 3] and np.all(s[0] == 0) and np.all(np.isnan(s[1]))
    st = api.wino_error_sweep(2, 4, 3, np.zeros((0, 6)), d, g, sums[:0], maxs[:0], ws)
    assert st.size == 0


def test_unsupported_and_workspace_errors():
    torch = _torch()
    from paper_2201_10369_b200 import api, _lib
    d, g = synth.random_tiles(100, 2, 6, 3, "uniform", seed=1)
    sums = torch.zeros((1, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((1, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_error_sweep(2, 4, 3, np.array([OP.f43_c(1.5)]), _dev(d), _dev(g), sums, maxs, ws)
    assert ei.value.status == 6
    d14, g14 = synth.random_tiles(100, 2, 14, 3, "uniform", seed=1)
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_error_sweep(2, 12, 3, np.zeros((1, 14)), _dev(d14), _dev(g14), sums, maxs, ws)
    assert ei.value.status == 8
    with pytest.raises(ValueError):      # binding-level shape check (tiles of another n)
        api.wino_error_sweep(2, 12, 3, np.zeros((1, 14)), _dev(d), _dev(g), sums, maxs, ws)


@pytest.mark.parametrize("dims", [2, 1])
def test_full_size_cfg2_sampled(dims):
    """BASELINE.json configs[1] at full size (4096 c x 100k tiles, uniform), in the bench's
    launch configuration; the oracle recomputes 6 sampled candidates over all tiles."""
    grid = synth.c_grid()
    sets = [OP.f43_c(float(c)) for c in grid]
    d, g = synth.random_tiles(100_000, dims, 6, 3, "uniform", seed=0)
    st, s, mx = _gpu_stats(dims, 4, 3, sets, d, g)
    assert np.all(st == 0)
    pick = [0, 1000, 2047, 2600, 3100, 4095]
    s_ref, m_ref, _ = ref.sweep(dims, 4, 3, [sets[i] for i in pick], d, g)
    _assert_stats_close(s[pick], mx[pick], s_ref, m_ref)
    assert np.all(s[:, 3] == 100_000 * 4 ** dims)


@pytest.mark.parametrize("dims", [2, 1])
def test_production_outputs_full_tiles(dims):
    """Per-element parity of the PRODUCTION kernels (the bench's configuration: the
    zero-skipping {0,±c,±1/c,∞} instantiation, 100k tiles) with the output store enabled,
    plus the statistics of the same launch, against the oracle."""
    cs = [float(c) for c in synth.c_grid()[::273]]
    sets = [OP.f43_c(c) for c in cs]
    d, g = synth.random_tiles(100_000, dims, 6, 3, "normal", seed=21)
    st, y, s, mx = _gpu_outputs(dims, 4, 3, sets, d, g, with_stats=True)
    assert np.all(st == 0)
    s_ref, m_ref, y_ref = ref.sweep(dims, 4, 3, sets, d, g, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref)
    _assert_stats_close(s, mx, s_ref, m_ref)


def _overflow_sets(maker_name):
    """Normal candidates interleaved with ones whose fp32 matrices overflow (inf entries /
    inf intermediates): c in {1e-19, 1e19} overflow Aᵀ and Bᵀ, c = 1e12, 3e9 overflow
    intermediates only."""
    normal = [0.3, 0.7, 1.6, 2.4, 5.0]
    bad = [1e19, 1e-19, 1e12, 3e9]
    cs = []
    for i in range(max(len(normal), len(bad))):
        if i < len(normal):
            cs.append(normal[i])
        if i < len(bad):
            cs.append(bad[i])
    if maker_name == "f43":
        return [OP.f43_c(c) for c in cs]
    return [OP.n8_cd(c, 1.003) for c in cs]


@pytest.mark.parametrize("dims,m,r,fam", [(2, 4, 3, "f43"), (1, 4, 3, "f43"), (2, 6, 3, "n8cd"), (1, 6, 3, "n8cd")])
def test_nonfinite_candidates_isolated(dims, m, r, fam):
    """Overflowing candidates mixed with normal ones in ONE launch, ragged tile count: the
    careful (exact, dense-chain) path must reproduce the oracle's n_nonfinite / n_scored and
    must not disturb the neighbouring candidates' statistics; outputs (NaN/inf included)
    equal the oracle's element by element."""
    sets = _overflow_sets(fam)
    n = m + r - 1
    d, g = synth.random_tiles(6007, dims, n, r, "uniform", seed=22)
    st, y, s, mx = _gpu_outputs(dims, m, r, sets, d, g, with_stats=True)
    assert np.all(st == 0)
    s_ref, m_ref, y_ref = ref.sweep(dims, m, r, sets, d, g, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref, equal_nan=True)
    assert np.any(s_ref[:, 4] > 0), "the test needs candidates with non-finite outputs"
    assert np.array_equal(s[:, 3], s_ref[:, 3]) and np.array_equal(s[:, 4], s_ref[:, 4])
    fin = s_ref[:, 3] > 0
    assert np.array_equal(mx[:, 1], m_ref[:, 1])
    assert np.all(np.abs(s[fin, 0] / s_ref[fin, 0] - 1) < RTOL_SUM)
    assert np.all(np.abs(mx[fin, 0] / m_ref[fin, 0] - 1) <= RTOL_MAX)
    # the statistics-only call (output store off: the same kernel) gives bitwise the same
    st2, s2, m2 = _gpu_stats(dims, m, r, sets, d, g)
    assert np.array_equal(s2, s, equal_nan=True) and np.array_equal(m2, mx, equal_nan=True)
