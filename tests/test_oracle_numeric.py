"""Pins of the fp64 recipe R64 (O3) and the C oracle's fp32/fp64 numerics (O5-O9)
against what the paper and the mathematics fix: exact rationals, exactness special
cases, a textbook reduction, power-of-two scaling, SPEC's brute-force example, the
paper's n=0 direct-convolution rows and the F(4,3) ordering (P:625,
P:651), and the c <-> 1/c symmetry of the point family."""
import json
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import synth
from oracle import exact, points as P, r64, ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = float("inf")
PAPER = json.load(open(os.path.join(GOLD, "paper_error_values.json")))


def _cancellation_ok(AT, G, BT, ATx, Gx, BTx, tol_ulp=8):
    """R64 within tol_ulp of exact, exact zeros where exact is zero; entries whose exact
    value is a cancellation (|entry| <= 1e-2 * its largest term) are exempt from the ulp
    bound."""
    worst = 0
    for M, Mx in ((AT, ATx), (G, Gx), (BT, BTx)):
        for i in range(M.shape[0]):
            for j in range(M.shape[1]):
                xv = Mx[i][j]
                if xv == 0:
                    assert M[i, j] == 0.0, (i, j, M[i, j])
                    continue
                u = r64.ulp_distance(M[i, j], float(xv))
                worst = max(worst, u)
    return worst


@pytest.mark.parametrize("m,k,maker,args", [
    (4, 3, P.f43_c, (1.829,)), (4, 3, P.f43_c, (1.622,)), (4, 3, P.f43_c, (0.05,)), (4, 3, P.f43_c, (20.0,)),
    (2, 3, P.f23_c, (1.054,)), (6, 3, lambda: P.P8, ()), (8, 3, lambda: P.P10, ()),
    (8, 3, P.n10_c1c2, (1.953, 1.229)), (6, 5, P.n10_c1c2, (1.272, 2.099)), (4, 5, P.n8_c1c2, (1.5, 3.1)),
])
def test_r64_close_to_exact(m, k, maker, args):
    pts = maker(*args)
    AT, G, BT = r64.build_r64(m, k, pts)
    ATx, Gx, BTx = exact.build_exact(m, k, pts)
    assert _cancellation_ok(AT, G, BT, ATx, Gx, BTx) <= 8


def test_r64_cfg3_set_cancellation_entry():
    """{0,±2,±1/2,-1/1.003,1.003,inf}: the unpaired near-symmetric pair d, -1/d cancels
    (d - 1/d ~ 0.006); the two affected Bᵀ entries (~0.0255) stay within 1e-13 relative
    of exact (112 ulp; a fixed fp64 order cannot do better), every other
    entry within 8 ulp."""
    pts = P.n8_cd(2.0, 1.003)
    AT, G, BT = r64.build_r64(6, 3, pts)
    ATx, Gx, BTx = exact.build_exact(6, 3, pts)
    for M, Mx in ((AT, ATx), (G, Gx), (BT, BTx)):
        for i in range(M.shape[0]):
            for j in range(M.shape[1]):
                xv = float(Mx[i][j])
                if Mx[i][j] == 0:
                    assert M[i, j] == 0.0
                elif r64.ulp_distance(M[i, j], xv) > 8:
                    assert M is BT and abs(M[i, j] - xv) <= 1e-13 * abs(xv), (i, j)


def test_r64_grid_zero_structure():
    """the {±c, ±1/c} family cancels terms exactly.  For every c of the
    4096-point grid except the exact duplicate c=1 (not on the grid), the zero pattern of
    the R64 matrices equals the exact one at a generic c, and Bᵀ's row for point 0 has
    zero odd coefficients."""
    grid = synth.c_grid()
    ATx, Gx, BTx = exact.build_exact(4, 3, P.f43_c(1.7))
    zpat = [np.array([[v == 0 for v in row] for row in Mx]) for Mx in (ATx, Gx, BTx)]
    for c in grid[::7]:
        pts = P.f43_c(float(c))
        mats = r64.build_r64(4, 3, pts)
        for M, z in zip(mats, zpat):
            assert np.array_equal(M == 0.0, z), c
        i0 = pts.index(0.0)
        assert all(mats[2][i0, j] == 0.0 for j in (1, 3, 5))


def test_r64_poly_order_independent():
    rng = np.random.default_rng(0)
    for _ in range(50):
        S = list(rng.uniform(-3, 3, size=6))
        S += [-S[0], -S[2], 0.0]
        a = r64.poly_from_roots_r64(S)
        b = r64.poly_from_roots_r64(list(reversed(S)))
        assert a == b


def test_r64_poly_horner_residual():
    """each root is a root to 1e-12·deg·max|coef|."""
    rng = np.random.default_rng(1)
    for _ in range(50):
        S = list(rng.uniform(-2, 2, size=7))
        p = r64.poly_from_roots_r64(S)
        for x in S:
            v = 0.0
            for c in reversed(p):
                v = v * x + c
            assert abs(v) <= 1e-12 * len(S) * max(abs(c) for c in p)


@pytest.mark.parametrize("bad", [
    [0.0, 1.0, float("nan"), INF], [0.0, INF, 1.0, 2.0], [0.0, 1.0, 2.0, -INF],
    [0.0, -0.0, 1.0, INF], [1.0, 2.0, 1.0, INF], [0.0, 1.0, INF],
])
def test_r64_validation(bad):
    with pytest.raises(ValueError):
        r64.build_r64(2, 3, bad)


# ------------------------------------------------------------------ C oracle (O5-O9)

@pytest.mark.parametrize("pts", [P.f23_c(1.0), P.f23_c(2.0)])
@pytest.mark.parametrize("dims", [1, 2])
def test_exactness_special_case(pts, dims):
    """O5 pin (a): F(2,3) with dyadic sets {0,±1,∞}, {0,±2,∞} and integer inputs in
    [-16,16] keep every fp32 intermediate exact, so y32 == exact correlation bitwise."""
    AT, G, BT = r64.build_f32(2, 3, pts)
    ATx, Gx, BTx = exact.build_exact(2, 3, pts)
    assert np.array_equal(AT, np.array([[float(v) for v in r] for r in ATx], dtype=np.float32))
    d, g = synth.integer_tiles(2000, dims, 4, 3, seed=5)
    for nofma in (False, True):
        su, mx, yd = ref.sweep(dims, 2, 3, [pts], d, g, nofma=nofma, n_dump=2000)
        y64 = ref.direct64_tiles(dims, 2, 3, d, g)
        assert np.array_equal(yd[0].astype(np.float64), y64)
        assert su[0, 0] == 0.0 and mx[0, 0] == 0.0 and su[0, 3] == 2000 * 2 ** dims


def test_two_term_dot_reduction():
    """O5 pin (b): F(1,2) on {0, ∞} is y = RN32(RN32(g0 d0) + RN32(g1 d1)) (a 2-term dot)."""
    d, g = synth.random_tiles(5000, 1, 2, 2, "uniform", seed=3)
    _, _, yd = ref.sweep(1, 1, 2, [[0.0, INF]], d, g, n_dump=5000)
    expect = (g[:, 0] * d[:, 0]) + (g[:, 1] * d[:, 1])  # numpy fp32: each op RN32
    assert np.array_equal(yd[0, :, 0], expect.astype(np.float32))


@pytest.mark.parametrize("dims", [1, 2])
def test_power_of_two_scaling(dims):
    """O5 pin (c): scaling d by 2^k scales y32 exactly (no over/underflow)."""
    d, g = synth.random_tiles(3000, dims, 6, 3, "normal", seed=4)
    pts = P.f43_c(1.7)
    _, _, y1 = ref.sweep(dims, 4, 3, [pts], d, g, n_dump=3000)
    _, _, y2 = ref.sweep(dims, 4, 3, [pts], d * np.float32(8.0), g, n_dump=3000)
    assert np.array_equal(y1 * np.float32(8.0), y2)


def test_fma_mode_differs_from_nofma():
    d, g = synth.random_tiles(2000, 2, 6, 3, "uniform", seed=6)
    _, _, y1 = ref.sweep(2, 4, 3, [P.f43_c(1.7)], d, g, nofma=False, n_dump=2000)
    _, _, y2 = ref.sweep(2, 4, 3, [P.f43_c(1.7)], d, g, nofma=True, n_dump=2000)
    assert not np.array_equal(y1, y2)
    assert np.max(np.abs(y1 - y2)) < 1e-4


def test_direct_spec_example():
    """4x4 ramp ⊛ 3x3 ones = [[54,63],[90,99]] (brute force), through the
    fp64 direct layer and the fp32 Winograd layer (pad 0, F(2x2,3x3), integer-exact)."""
    x = np.arange(1, 17, dtype=np.float32).reshape(1, 1, 4, 4)
    w = np.ones((1, 1, 3, 3), dtype=np.float32)
    y64 = ref.conv2d_direct64(x, w, pad=0)
    assert y64[0, 0].tolist() == [[54.0, 63.0], [90.0, 99.0]]
    y32 = ref.conv2d_wino(x, w, pad=0, m=2, points=P.f23_c(1.0))
    assert y32[0, 0].tolist() == [[54.0, 63.0], [90.0, 99.0]]


def test_layer_integer_exact_cfg1_shape():
    """cfg1 shape (BASELINE.json configs[0]) with integer inputs: Winograd layer ==
    direct layer bitwise (all intermediates dyadic and small)."""
    x, w = synth.integer_layer_inputs(1, 8, 16, 16, 8, 3, seed=0)
    y32 = ref.conv2d_wino(x, w, pad=1, m=2, points=P.f23_c(1.0))
    y64 = ref.conv2d_direct64(x, w, pad=1)
    assert np.array_equal(y32.astype(np.float64), y64)


def test_layer_equals_tiles_c1k1():
    """O4: a C=K=1 layer is the tiled single-tile algorithm (pad 0, exact tiling)."""
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, size=(1, 1, 14, 14)).astype(np.float32)
    w = rng.uniform(-1, 1, size=(1, 1, 3, 3)).astype(np.float32)
    pts = P.f43_c(1.622)
    y = ref.conv2d_wino(x, w, pad=0, m=4, points=pts)  # 12x12 output = 3x3 tiles
    AT, G, BT = r64.build_f32(4, 3, pts)
    for ty in range(3):
        for tx in range(3):
            d = x[0, 0, ty * 4: ty * 4 + 6, tx * 4: tx * 4 + 6].ravel()
            yt = ref.tile(2, 4, 3, AT, G, BT, d, w[0, 0].ravel())
            assert np.array_equal(yt.reshape(4, 4), y[0, 0, ty * 4: ty * 4 + 4, tx * 4: tx * 4 + 4])


def test_layer_close_to_direct():
    x, w = synth.layer_inputs(2, 16, 20, 20, 8, 3, "normal", "he", seed=1)
    pts = P.n8_cd(2.0, 1.003)
    y32 = ref.conv2d_wino(x, w, pad=1, m=6, points=pts)
    y64 = ref.conv2d_direct64(x, w, pad=1)
    assert np.max(np.abs(y32 - y64)) < 1e-4 * np.max(np.abs(y64))
    s, mx = ref.stats(y32, y64)
    assert s[3] == y32.size and s[4] == 0
    assert math.isclose(s[0], float(np.sum(np.abs(y32.astype(np.float64) - y64))), rel_tol=1e-12)


@pytest.mark.parametrize("dims,key", [(1, "n0_direct_1d"), (2, "n0_direct_2d")])
def test_calibration_n0_rows(dims, key):
    """T7/T8 n=0 rows: fp32 direct correlation vs fp64, uniform[-1,1],
    per-element mean |e|, paper arithmetic (no FMA) -> within 2% of the printed value.
    Pins the input distribution (R9), the error norm (R10) and O6."""
    d, g = synth.random_tiles(100_000, dims, 6, 3, "uniform", seed=0)
    s, _ = ref.direct32_sweep(dims, 4, 3, d, g, nofma=True)
    mae = s[0] / s[3]
    assert abs(mae / PAPER[key]["value"] - 1) < 0.02, mae


@pytest.mark.parametrize("dims", [1, 2])
def test_f43_proposed_beats_prior(dims):
    """T7/T8 n=6: the proposed c-family beats the prior-work points, and
    our sequential-order values sit 0-15% above the paper's Huffman-order values."""
    key = "1d" if dims == 1 else "2d"
    prop, prior = PAPER[f"f43_proposed_{key}"], PAPER[f"f43_prior_{key}"]
    base = P.F43_PRIOR_1D if dims == 1 else P.F43_PRIOR_2D
    d, g = synth.random_tiles(50_000, dims, 6, 3, "uniform", seed=0)
    s, _, _ = ref.sweep(dims, 4, 3, [P.f43_c(prop["c"]), base], d, g, nofma=True)
    e = s[:, 0] / s[:, 3]
    assert e[0] < e[1]
    assert 1.0 <= e[0] / prop["value"] <= 1.15
    assert 1.0 <= e[1] / prior["value"] <= 1.15


def test_curve_shape_1d():
    """F(4,3) 1D curve over c in [1.1, 2.5]: interior minimum inside
    [1.45, 1.85] (paper: 1.6-1.8 in Huffman order), endpoints >= 25% higher;
    err(c) == err(1/c) bitwise where 1/(1/c) == c (same point set)."""
    d, g = synth.random_tiles(20_000, 1, 6, 3, "uniform", seed=2)
    cs = [1.1 + 0.05 * i for i in range(29)]
    s, _, _ = ref.sweep(1, 4, 3, [P.f43_c(c) for c in cs], d, g, nofma=True)
    e = s[:, 0] / s[:, 3]
    i = int(np.argmin(e))
    assert 1.45 <= cs[i] <= 1.85
    assert e[0] >= 1.25 * e[i] and e[-1] >= 1.25 * e[i]
    s2, _, _ = ref.sweep(1, 4, 3, [P.f43_c(2.0), P.f43_c(0.5)], d, g, nofma=True)
    assert np.array_equal(s2[0], s2[1])


def test_stats_nonfinite_excluded():
    y32 = np.array([1.0, np.inf, 2.0, np.nan], dtype=np.float32)
    y64 = np.array([1.5, 1.0, 2.0, 0.0])
    s, mx = ref.stats(y32, y64)
    assert s.tolist() == [0.5, 0.25, 4.5, 2.0, 2.0]   # Σ|y_ref| over every output (R16)
    assert mx.tolist() == [0.5, 2.0]


def test_chebyshev_nodes():
    """x_k = cos((2k-1) pi / 2n); our sets use n-1 nodes + inf (reading X24): exactly
    symmetric, the middle node exactly 0, and each node a root of the Chebyshev polynomial."""
    from paper_2201_10369_b200 import points as PP
    for n in range(3, 11):
        p = PP.chebyshev(n)
        assert p[-1] == INF and len(p) == n
        fin = p[:-1]
        assert fin == sorted(-v for v in fin)
        q = n - 1
        for v in fin:
            assert abs(math.cos(q * math.acos(v))) < 1e-12
        if q % 2 == 1:
            assert 0.0 in fin


# ------------------------------------------------------------------ N2: Huffman order (R21)

def test_huffman_tree_order_hand_case():
    """Mode 2 on hand-made matrices (m=3, r=1: U = g, V = d, y_p = Σ_i AT[p][i] d_i).
    Row 0 weights |1|, |1|, |2^-30|: the tree joins term 2 with term 0 first (ties go to the
    lower index), then term 1.  With d = (2^24, -2^24, 2^30): term 2 = 1, and
    RN(2^24 + 1) = 2^24 (ties-to-even), + (-2^24) = 0, while the sequential order gives
    (2^24 - 2^24) + 1 = 1.  Row 1 weights 4, 2, 1 join terms 2 and 1 first:
    2^30 + 2 * (-2^24) = 2^30 - 2^25, then + 4 * 2^24 = 2^30 + 2^25 (all exact).  Row 2 has
    no non-zero coefficient: +0."""
    AT = np.array([[1.0, 1.0, 2.0 ** -30], [4.0, 2.0, 1.0], [0.0, 0.0, 0.0]], dtype=np.float32)
    G = np.ones((3, 1), dtype=np.float32)
    BT = np.eye(3, dtype=np.float32)
    d = np.array([2.0 ** 24, -2.0 ** 24, 2.0 ** 30], dtype=np.float32)
    g = np.array([1.0], dtype=np.float32)
    yh = ref.tile(1, 3, 1, AT, G, BT, d, g, huffman=True)
    ys = ref.tile(1, 3, 1, AT, G, BT, d, g, nofma=True)
    assert yh[0] == 0.0 and ys[0] == 1.0
    assert yh[1] == np.float32(2.0 ** 30 - 2.0 ** 25 + 2.0 ** 26)
    assert yh[2] == 0.0 and not np.signbit(yh[2])     # no terms -> +0


def test_huffman_exact_special_case():
    """Huffman order changes only the rounding: on the exactness special case (F(2,3)
    {0,±1,∞}, integer data) it still reproduces the exact correlation."""
    d, g = synth.integer_tiles(300, 2, 4, 3, seed=4)
    for t in range(0, 300, 29):
        y = ref.tile(2, 2, 3, *r64.build_f32(2, 3, P.f23_c(1.0)), d[t], g[t], huffman=True)
        ex = exact.correlate_2d(d[t].reshape(4, 4).astype(int).tolist(), g[t].reshape(3, 3).astype(int).tolist())
        assert y.reshape(2, 2).tolist() == [[float(v) for v in row] for row in ex]


@pytest.mark.parametrize("dims", [1, 2])
def test_huffman_reproduces_paper_f43_rows(dims):
    """T7/T8 n=6 rows are Huffman-ordered.  With the Huffman reading
    R21 the oracle lands within [-3 %, +5 %] of all four printed values (the paper averages
    5000 inputs), and closer to each than the sequential order (which sits 6-9 % above)."""
    key = "1d" if dims == 1 else "2d"
    prop, prior = PAPER[f"f43_proposed_{key}"], PAPER[f"f43_prior_{key}"]
    base = P.F43_PRIOR_1D if dims == 1 else P.F43_PRIOR_2D
    d, g = synth.random_tiles(100_000, dims, 6, 3, "uniform", seed=0)
    sets = [P.f43_c(prop["c"]), base]
    sh, _, _ = ref.sweep(dims, 4, 3, sets, d, g, huffman=True)
    ss, _, _ = ref.sweep(dims, 4, 3, sets, d, g, nofma=True)
    eh = sh[:, 0] / sh[:, 3]
    es = ss[:, 0] / ss[:, 3]
    for j, paper in enumerate((prop["value"], prior["value"])):
        assert 0.97 <= eh[j] / paper <= 1.05, (j, eh[j], paper)
        assert abs(eh[j] / paper - 1) < abs(es[j] / paper - 1)
    assert eh[0] < eh[1]


# ------------------------------------------------------------------ N2: mixed precision (R22)

def test_mixed_exact_special_case():
    """fp64 transforms on integer tiles with F(2,3) {0,±1,∞}: every value is exact, so the
    mixed-precision output is the exact correlation."""
    d, g = synth.integer_tiles(200, 2, 4, 3, seed=6)
    _, _, y = ref.sweep_mixed(2, 2, 3, [P.f23_c(1.0)], d, g, n_dump=200)
    for t in range(0, 200, 23):
        ex = exact.correlate_2d(d[t].reshape(4, 4).astype(int).tolist(), g[t].reshape(3, 3).astype(int).tolist())
        assert y[0, t].reshape(2, 2).tolist() == [[float(v) for v in row] for row in ex]


@pytest.mark.parametrize("dims", [1, 2])
def test_mixed_error_bound(dims):
    """R22 leaves three fp32 roundings per Winograd-domain term (U, V, U*V) and one on the
    output: |y - y64| <= u|y64| + 3.01 u Σ|A||A| |U V| (+ fp64 noise), u = 2^-24, with U, V
    the exact-transform values (fp64 from the R64 matrices); the bound holds for every
    output, and the mixed mode beats the all-fp32 mode on average."""
    c = 1.829 if dims == 1 else 1.622
    pts = P.f43_c(c)
    d, g = synth.random_tiles(2000, dims, 6, 3, "uniform", seed=8)
    _, _, ym = ref.sweep_mixed(dims, 4, 3, [pts], d, g, n_dump=2000)
    _, _, yf = ref.sweep(dims, 4, 3, [pts], d, g, n_dump=2000)
    y64 = ref.direct64_tiles(dims, 4, 3, d, g)
    AT, G, BT = (np.asarray(M_, dtype=np.float64) for M_ in r64.build_r64(4, 3, pts))
    u = 2.0 ** -24
    if dims == 1:
        U = g.astype(np.float64) @ G.T
        V = d.astype(np.float64) @ BT.T
        bound = u * np.abs(y64) + 3.01 * u * (np.abs(U * V) @ np.abs(AT).T) + 1e-12
    else:
        gg = g.reshape(-1, 3, 3).astype(np.float64)
        dd = d.reshape(-1, 6, 6).astype(np.float64)
        U = G @ gg @ G.T
        V = BT @ dd @ BT.T
        W_ = np.abs(U * V)
        bound = (u * np.abs(y64).reshape(-1, 4, 4) + 3.01 * u * (np.abs(AT) @ W_ @ np.abs(AT).T) + 1e-12)
        bound = bound.reshape(-1, 16)
    em = np.abs(ym[0].astype(np.float64) - y64)
    ef = np.abs(yf[0].astype(np.float64) - y64)
    assert np.all(em <= bound)
    assert em.mean() < ef.mean()


@pytest.mark.parametrize("dims", [1, 2])
def test_mixed_reduces_to_rounded_exact_transforms(dims):
    """With F(2,3) on {0,±1,∞} every fp64 transform of fp32 data is exact (coefficients 0,
    ±1/2, ±1; at most 16 terms), so R22 reduces to: U, V = RN32(exact transforms),
    M = RN32(U V), y = RN32(exact Aᵀ M A) -- three library roundings, computed here with
    numpy float32 / float64 on the exact rational matrices of O2."""
    pts = P.f23_c(1.0)
    AT, G, BT = (np.asarray(M_, dtype=np.float64) for M_ in r64.build_r64(2, 3, pts))
    for M_ in (AT, G, BT):                      # dyadic: the fp64 matrices are the exact ones
        assert np.all(M_ * 2 == np.round(M_ * 2))
    d, g = synth.random_tiles(3000, dims, 4, 3, "uniform", seed=9)
    _, _, ym = ref.sweep_mixed(dims, 2, 3, [pts], d, g, n_dump=3000)
    _, _, yf = ref.sweep(dims, 2, 3, [pts], d, g, n_dump=3000)
    if dims == 1:
        U = (g.astype(np.float64) @ G.T).astype(np.float32)
        V = (d.astype(np.float64) @ BT.T).astype(np.float32)
        y = ((U * V).astype(np.float64) @ AT.T).astype(np.float32)
    else:
        U = (G @ g.reshape(-1, 3, 3).astype(np.float64) @ G.T).astype(np.float32)
        V = (BT @ d.reshape(-1, 4, 4).astype(np.float64) @ BT.T).astype(np.float32)
        y = (AT @ (U * V).astype(np.float64) @ AT.T).astype(np.float32).reshape(-1, 4)
    assert np.array_equal(ym[0], y)
    assert not np.array_equal(yf[0], y)


@pytest.mark.parametrize("dims,lo,hi", [(1, 1.6, 1.85), (2, 1.55, 1.8)])
def test_huffman_curve_minimum_region(dims, lo, hi):
    """with Huffman-ordered summation (R21) the F(4,3) error-vs-c curve of the
    {0,±c,±1/c,inf} family has its minimum for c in 1.6-1.8, rising on either side.  On a
    0.025 grid over [1.1, 2.5] the oracle's argmin lies in that region (1D: 1.825, next to
    T4's 1.829; 2D: within one grid step below it, the curve being jagged at the
    1e-3 level), and both ends are >= 25 % above the minimum."""
    cs = [1.1 + 0.025 * i for i in range(57)]
    d, g = synth.random_tiles(50_000 if dims == 1 else 20_000, dims, 6, 3, "uniform", seed=2)
    s, _, _ = ref.sweep(dims, 4, 3, [P.f43_c(c) for c in cs], d, g, huffman=True)
    e = s[:, 0] / s[:, 3]
    i = int(np.argmin(e))
    assert lo <= cs[i] <= hi, cs[i]
    assert e[0] >= 1.25 * e[i] and e[-1] >= 1.25 * e[i]


def _fixture_points(finite):
    pts = []
    for v in finite:
        if isinstance(v, str):
            sign = -1.0 if v.startswith("-") else 1.0
            pts.append(sign * (1.0 / float(v.lstrip("-").split("/")[1])))
        else:
            pts.append(float(v))
    return sorted(pts) + [INF]


T78 = json.load(open(os.path.join(GOLD, "paper_tables_t7_t8.json")))["rows"]


@pytest.mark.parametrize("row", T78, ids=[f"{r['dims']}d-n{r['n']}-{r['kind']}" for r in T78])
def test_huffman_reproduces_paper_tables(row):
    """Every T7/T8 row, kernel size 3, n = 4..10: the Huffman-mode oracle
    (R21, the paper's order) lands within [-4 %, +9 %] of the printed error (the
    paper averages 5000 inputs; we use 100k 1D / 20k 2D uniform[-1,1] tiles, R9).  Rows the
    fixture marks "not reproduced" (a printed set that evaluates far from its value in every
    summation order) are asserted to stay far, so a change of reading shows up.  The
    1D n=4 P4 row sits at +14.5 % in every order (F(2,3) has too few terms for the order to
    matter) and is held to +20 %."""
    dims, n = row["dims"], row["n"]
    pts = _fixture_points(row["finite_points"])
    assert len(pts) == n
    d, g = synth.random_tiles(100_000 if dims == 1 else 20_000, dims, n, 3, "uniform", seed=0)
    s, _, _ = ref.sweep(dims, n - 2, 3, [pts], d, g, huffman=True)
    rel = s[0, 0] / s[0, 3] / row["value"] - 1
    if "not reproduced" in row.get("note", ""):
        assert rel > 0.3
    elif dims == 1 and n == 4 and row["kind"] == "prior":
        assert -0.04 <= rel <= 0.20
    else:
        assert -0.04 <= rel <= 0.09, rel
