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
