"""NEXT row N1: template / subset enumeration (CPU) and the GPU search against the oracle."""
import math

import numpy as np
import pytest

import synth
from oracle import ref
from paper_2201_10369_b200 import search as S


def test_enumeration_matches_paper_counts():
    # eq:ps3: F(3,3) has 4 three-element subsets of {-1/c,-c,c,1/c}
    assert len(S.enumerate_templates(5)) == 4
    # eq:subset_points: base {1,-1} -> 6 pairs; base {-3} -> 4 triples
    assert len(S.enumerate_templates(6, bases=[(1.0, -1.0)])) == 6
    assert len(S.enumerate_templates(6, bases=[(-3.0,)])) == 4
    # F(7,3)-sized (n = 7 + ... ) sets: all c-members + 2 of the d-family = 6
    t = S.enumerate_templates(8)
    assert len(t) == 6 and all(x.n == 8 and x.n_params == 2 for x in t)
    # F(4,3) proposed set = the full family
    assert S.enumerate_templates(6) == [S.Template((), S.C_MEMBERS)]


def test_template_points_and_validity():
    t = S.Template((1.0, -1.0), ("-1/c", "c"))
    p = t.points(2.0)
    assert p == [-1.0, -0.5, 0.0, 1.0, 2.0, math.inf]
    assert not S.Template((), S.C_MEMBERS).valid(1.0)        # ±c == ±1/c
    assert not S.Template((1.0, -1.0), ("c",)).valid(1.0)     # c == 1
    rows, owner, params = S.candidates([t, S.Template((), S.C_MEMBERS)], [1.0, 2.0])
    assert rows.shape == (4, 6) and np.isnan(rows[2]).all() and owner.tolist() == [0, 0, 1, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("dims,m,key", [(1, 2, "f23_1d"), (1, 3, "f33_1d"), (2, 4, "f43_1d"), (1, 4, "f43_1d")])
def test_search_matches_oracle(dims, m, key):
    import torch
    templates = S.PAPER_TABLE_TEMPLATES[key]
    cs = [1.1 + 0.1 * i for i in range(15)]
    n = m + 2
    d, g = synth.random_tiles(4001, dims, n, 3, "uniform", seed=5)
    ranking, mae, status = S.run_search(templates, dims, m, 3, cs, torch.from_numpy(d).cuda(),
                                        torch.from_numpy(g).cuda(), flags=1)
    rows, owner, params = S.candidates(templates, cs)
    ok = np.flatnonzero(status == 0)
    s_ref, _, _ = ref.sweep(dims, m, 3, [list(rows[i]) for i in ok], d, g, nofma=True)
    mae_ref = np.full(len(rows), np.nan)
    mae_ref[ok] = s_ref[:, 0] / s_ref[:, 3]
    assert np.all(np.abs(mae[ok] / mae_ref[ok] - 1) < 1e-5)   # fp32-pair scoring of the 2D F(4,3) kernel
    rank_ref = S.rank(templates, owner, params, mae_ref)
    assert [r[0] for r in ranking] == [r[0] for r in rank_ref]


def _rank_vs_oracle(templates, dims, m, cs, flags, huffman, seed):
    import torch
    n = m + 2
    d, g = synth.random_tiles(1501, dims, n, 3, "uniform", seed=seed)
    ranking, mae, status = S.run_search(templates, dims, m, 3, cs, torch.from_numpy(d).cuda(),
                                        torch.from_numpy(g).cuda(), flags=flags)
    rows, owner, params = S.candidates(templates, cs)
    ok = np.flatnonzero(status == 0)
    s_ref, _, _ = ref.sweep(dims, m, 3, [list(rows[i]) for i in ok], d, g, huffman=huffman, nofma=not huffman)
    mae_ref = np.full(len(rows), np.nan)
    mae_ref[ok] = s_ref[:, 0] / s_ref[:, 3]
    assert np.all(np.abs(mae[ok] / mae_ref[ok] - 1) < 1e-9)   # fp64 scoring of the Huffman / NOFMA kernels
    rank_ref = S.rank(templates, owner, params, mae_ref)
    assert [r[0] for r in ranking] == [r[0] for r in rank_ref]
    assert [r[1] for r in ranking] == [r[1] for r in rank_ref]
    return ranking


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["f23", "f33", "f43"])
def test_optimal_tables_2d_columns_match_oracle(key):
    """The 2D columns of tab:optimal_f23/f33/f43 in the paper's Huffman order:
    the GPU ranking (template order and best c) equals the oracle's."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "search_tables", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "search_tables.py"))
    st = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(st)
    m = {"f23": 2, "f33": 3, "f43": 4}[key]
    templates = [t for t, _, _ in st.OPTIMAL[(key, 2)]]
    _rank_vs_oracle(templates, 2, m, [1.05 + 0.1 * i for i in range(12)], 2, True, seed=41)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,m,base", [(1, 3, (3.0,)), (2, 4, (0.5,)), (1, 4, (1.0, -1.0)), (2, 3, (-3.0,))])
def test_pattern_tables_match_oracle(dims, m, base):
    """tab:pattern_1d / pattern_2d: every subset of the c-family completing the
    base points, ranked on the GPU (Huffman order) exactly as by the oracle."""
    templates = S.enumerate_templates(m + 2, bases=[base])
    k = m + 2 - 2 - len(base)
    assert len(templates) == math.comb(4, k)
    _rank_vs_oracle(templates, dims, m, [1.1 + 0.12 * i for i in range(11)], 2, True, seed=42)


@pytest.mark.gpu
def test_cd_grid_argmin_matches_oracle():
    """(c, d) grid search for the n = 9 template {0,±1/c,±c,-1/d,-d,d}: the
    GPU's argmin over a small grid (Huffman order) is the oracle's."""
    import torch
    from oracle import points as OP  # noqa: F401  (oracle side builds its own sets below)
    from paper_2201_10369_b200 import api
    from paper_2201_10369_b200.sweep import curve
    cs = [1.2, 1.3, 1.4]
    ds = [2.3, 2.5, 2.7]
    sets = [sorted([0.0, -1 / c, -c, c, 1 / c, -1 / d, -d, d]) + [math.inf] for c in cs for d in ds]
    d, g = synth.random_tiles(1201, 1, 9, 3, "uniform", seed=43)
    sums = torch.zeros((len(sets), 5), dtype=torch.float64, device="cuda")
    maxs = torch.zeros((len(sets), 2), dtype=torch.float64, device="cuda")
    ws = torch.empty(api.wino_error_sweep_workspace_bytes(1, 7, 3, len(sets), 1201), dtype=torch.uint8, device="cuda")
    st = api.wino_error_sweep(1, 7, 3, np.array(sets), torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda(),
                              sums, maxs, ws, flags=api.WINO_SWEEP_HUFFMAN)
    mae = curve(sums.cpu().numpy(), st)
    s_ref, _, _ = ref.sweep(1, 7, 3, sets, d, g, huffman=True)
    mae_ref = s_ref[:, 0] / s_ref[:, 3]
    assert int(np.nanargmin(mae)) == int(np.argmin(mae_ref))
    assert np.allclose(mae, mae_ref, rtol=1e-9, atol=0)
