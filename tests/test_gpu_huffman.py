"""NEXT row N2: the Huffman-order sweep (WINO_SWEEP_HUFFMAN) against the oracle's Huffman
mode (reading R21): per-element fp32 outputs bit-identical, statistics within the
sweep tolerances, the paper's Huffman-ordered F(4,3) rows reproduced on the GPU path, and
the unsupported-shape error."""
import math

import numpy as np
import pytest

import synth
from oracle import points as OP, ref

pytestmark = pytest.mark.gpu
INF = math.inf
HUFF = 2


@pytest.fixture(autouse=True, params=[2, 1], ids=["interpreter", "jit"])
def huffman_kernel(request):
    """Every test runs on both Huffman kernels: the shared-memory interpreter (mode 2) and
    the run-time specialised register kernels (mode 1, huff_jit.cu)."""
    from paper_2201_10369_b200 import api
    prev = api.wino_huffman_jit_mode(request.param)
    yield request.param
    api.wino_huffman_jit_mode(prev)


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _outputs(dims, m, r, sets, d, g):
    import torch
    from paper_2201_10369_b200 import api
    y = torch.full((len(sets), d.shape[0], m ** dims), float("nan"), dtype=torch.float32, device="cuda")
    st = api.wino_sweep_outputs(dims, m, r, np.array(sets), _dev(d), _dev(g), y, flags=HUFF)
    torch.cuda.synchronize()
    return st, y.cpu().numpy()


def _stats(dims, m, r, sets, d, g):
    import torch
    from paper_2201_10369_b200 import api
    S, T = len(sets), d.shape[0]
    sums = torch.zeros((S, 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((S, 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(dims, m, r, S, T), dtype=torch.uint8, device="cuda")
    st = api.wino_error_sweep(dims, m, r, np.array(sets), _dev(d), _dev(g), sums, maxs, ws, flags=HUFF)
    torch.cuda.synchronize()
    return st, sums.cpu().numpy(), maxs.cpu().numpy()


SETS = {
    2: [OP.f23_c(1.0), OP.f23_c(1.7), [-2.0, 0.5, 1.0, INF]],
    4: [OP.f43_c(1.622), OP.f43_c(1.829), OP.f43_c(0.3), [-1.0, 0.0, 0.5, 1.0, 2.0, INF],
        [-3.0, -1.0, 0.0, 0.5, 1.0, INF]],
    6: [OP.n8_cd(2.0, 1.003), OP.P8],
}


@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("m", [2, 4, 6])
def test_huffman_outputs_bitexact(dims, m):
    sets = [sorted(p for p in s if p != INF) + [INF] for s in SETS[m]]
    d, g = synth.random_tiles(1031, dims, m + 2, 3, "normal", seed=31)
    st, y = _outputs(dims, m, 3, sets, d, g)
    assert np.all(st == 0)
    _, _, y_ref = ref.sweep(dims, m, 3, sets, d, g, huffman=True, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref)
    # and it is a different arithmetic from the sequential NOFMA order
    _, _, y_seq = ref.sweep(dims, m, 3, sets, d, g, nofma=True, n_dump=d.shape[0])
    assert not np.array_equal(y, y_seq)


@pytest.mark.parametrize("dims", [1, 2])
def test_huffman_stats(dims):
    grid = synth.c_grid()
    cs = [float(grid[i]) for i in range(0, 4096, 97)]
    sets = [OP.f43_c(c) for c in cs]
    d, g = synth.random_tiles(20_011, dims, 6, 3, "uniform", seed=12)
    st, s, mx = _stats(dims, 4, 3, sets, d, g)
    assert np.all(st == 0)
    s_ref, m_ref, _ = ref.sweep(dims, 4, 3, sets, d, g, huffman=True)
    assert np.array_equal(s[:, 3], s_ref[:, 3]) and np.array_equal(s[:, 4], s_ref[:, 4])
    assert np.array_equal(mx, m_ref)                       # fp64 scoring: max exact
    assert np.all(np.abs(s[:, 0] / s_ref[:, 0] - 1) < 1e-12)
    assert np.all(np.abs(s[:, 1] / s_ref[:, 1] - 1) < 1e-12)


def test_huffman_jit_classes_compiled(huffman_kernel):
    """The configs[1] c grid falls into a handful of program classes (8 for F(4,3)); the
    JIT mode compiles each once and reuses it."""
    from paper_2201_10369_b200 import api
    if huffman_kernel != 1:
        pytest.skip("JIT only")
    sets = [OP.f43_c(float(c)) for c in synth.c_grid()]
    d, g = synth.random_tiles(3001, 2, 6, 3, "uniform", seed=3)
    before = api.wino_huffman_jit_classes()
    st, s, _ = _stats(2, 4, 3, sets, d, g)
    mid = api.wino_huffman_jit_classes()
    st2, s2, _ = _stats(2, 4, 3, sets, d, g)
    assert np.all(st == 0) and mid - before <= 8 and api.wino_huffman_jit_classes() == mid
    assert np.array_equal(s, s2)
    sub = list(range(0, 4096, 511))
    s_ref, _, _ = ref.sweep(2, 4, 3, [sets[i] for i in sub], d, g, huffman=True)
    assert np.all(np.abs(s[sub, 0] / s_ref[:, 0] - 1) < 1e-12)


def test_huffman_nonfinite_candidates(huffman_kernel):
    """Overflowing candidates between normal ones: outputs bit-identical (NaN / inf
    included), exact non-finite counts, neighbours unaffected."""
    sets = [OP.f43_c(1.3), OP.f43_c(1e19), OP.f43_c(0.7), OP.f43_c(1e-19), OP.f43_c(2.1)]
    d, g = synth.random_tiles(1003, 2, 6, 3, "uniform", seed=8)
    st, y = _outputs(2, 4, 3, sets, d, g)
    _, _, y_ref = ref.sweep(2, 4, 3, sets, d, g, huffman=True, n_dump=d.shape[0])
    assert np.array_equal(y, y_ref, equal_nan=True)
    st, s, mx = _stats(2, 4, 3, sets, d, g)
    s_ref, m_ref, _ = ref.sweep(2, 4, 3, sets, d, g, huffman=True)
    assert np.array_equal(s[:, 3:], s_ref[:, 3:])
    fin = s_ref[:, 4] == 0
    assert np.all(np.abs(s[fin, 0] / s_ref[fin, 0] - 1) < 1e-12)


@pytest.mark.parametrize("dims", [1, 2])
def test_huffman_paper_rows_on_gpu(dims):
    """T7/T8 n=6 through the C ABI: within [-3 %, +5 %] of the paper."""
    import json, os
    paper = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_error_values.json")))
    key = "1d" if dims == 1 else "2d"
    prop, prior = paper[f"f43_proposed_{key}"], paper[f"f43_prior_{key}"]
    base = OP.F43_PRIOR_1D if dims == 1 else OP.F43_PRIOR_2D
    d, g = synth.random_tiles(100_000, dims, 6, 3, "uniform", seed=0)
    st, s, _ = _stats(dims, 4, 3, [OP.f43_c(prop["c"]), base], d, g)
    e = s[:, 0] / s[:, 3]
    assert 0.97 <= e[0] / prop["value"] <= 1.05 and 0.97 <= e[1] / prior["value"] <= 1.05


def test_huffman_unsupported_shape():
    from paper_2201_10369_b200 import _lib
    d, g = synth.random_tiles(100, 2, 8, 5, "uniform", seed=1)
    with pytest.raises(_lib.WinoError) as ei:
        _stats(2, 4, 5, [OP.n8_c1c2(1.5, 3.1)], d, g)
    assert ei.value.status == 8


def _fixture_rows():
    import json, os
    rows = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables_t7_t8.json")))["rows"]
    return rows


def _pts(finite):
    out = []
    for v in finite:
        if isinstance(v, str):
            sign = -1.0 if v.startswith("-") else 1.0
            out.append(sign * (1.0 / float(v.lstrip("-").split("/")[1])))
        else:
            out.append(float(v))
    return sorted(out) + [INF]


@pytest.mark.parametrize("dims", [1, 2])
def test_huffman_all_paper_sizes_bitexact(dims):
    """Every T7/T8 point set (n = 4..10) through the GPU Huffman kernels: outputs
    bit-identical to the oracle on 517 tiles."""
    rows = [r for r in _fixture_rows() if r["dims"] == dims]
    for n in sorted({r["n"] for r in rows}):
        sets = [_pts(r["finite_points"]) for r in rows if r["n"] == n]
        d, g = synth.random_tiles(517, dims, n, 3, "uniform", seed=50 + n)
        st, y = _outputs(dims, n - 2, 3, sets, d, g)
        assert np.all(st == 0)
        _, _, y_ref = ref.sweep(dims, n - 2, 3, sets, d, g, huffman=True, n_dump=d.shape[0])
        assert np.array_equal(y, y_ref), n


@pytest.mark.parametrize("dims", [1, 2])
def test_huffman_paper_tables_on_gpu(dims):
    """The paper's T7/T8 values through the C ABI at 100k tiles (the bench workload size):
    the reproduced rows within [-4 %, +9 %] (1D n=4 P4: +20 %), the two recorded
    non-reproducible rows far above."""
    rows = [r for r in _fixture_rows() if r["dims"] == dims]
    for n in sorted({r["n"] for r in rows}):
        rs = [r for r in rows if r["n"] == n]
        d, g = synth.random_tiles(100_000, dims, n, 3, "uniform", seed=0)
        st, s, _ = _stats(dims, n - 2, 3, [_pts(r["finite_points"]) for r in rs], d, g)
        assert np.all(st == 0)
        for r, row in zip(s, rs):
            rel = r[0] / r[3] / row["value"] - 1
            if "not reproduced" in row.get("note", ""):
                assert rel > 0.3
            elif dims == 1 and n == 4 and row["kind"] == "prior":
                assert -0.04 <= rel <= 0.20
            else:
                assert -0.04 <= rel <= 0.09, (n, row["kind"], rel)


def test_huffman_rejected_candidates(huffman_kernel):
    """Rejected candidates (duplicate / NaN points) between accepted ones: statuses per
    candidate, NaN statistics rows, the accepted rows equal to the oracle's Huffman mode --
    on both kernels (the run-time kernels sort candidates by class; rejected ones have none)."""
    sets = [OP.f43_c(1.7), [0.0, 1.0, 1.0, -1.0, 2.0, INF], [math.nan] * 6, OP.f43_c(0.9), OP.f43_c(1.7)]
    d, g = synth.random_tiles(3001, 2, 6, 3, "uniform", seed=15)
    st, s, mx = _stats(2, 4, 3, sets, d, g)
    assert st.tolist() == [0, 3, 5, 0, 0]
    assert np.all(np.isnan(s[1:3])) and np.all(np.isnan(mx[1:3]))
    s_ref, m_ref, _ = ref.sweep(2, 4, 3, [sets[0], sets[3], sets[4]], d, g, huffman=True)
    ok = [0, 3, 4]
    assert np.array_equal(s[ok, 3:], s_ref[:, 3:]) and np.array_equal(mx[ok], m_ref)
    assert np.all(np.abs(s[ok, 0] / s_ref[:, 0] - 1) < 1e-12)
    assert np.array_equal(s[0], s[4])   # same point set, same class: bitwise equal rows
