"""Pins of the exact-rational oracle against what PAPER.md fixes:
its worked closed-form matrices, the canonical F(2,3) matrices, Table 1,
and the mathematical identity "Winograd == valid cross-correlation" checked by brute
force on tiny rational inputs."""
import json
import os
import random
from fractions import Fraction as Fr

import pytest

from oracle import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = float("inf")


def _rand_fr(rng, lo=-9, hi=9, den=7):
    while True:
        v = Fr(rng.randint(lo * den, hi * den), rng.randint(1, den))
        if v != 0:
            return v


def test_f23_canonical_golden():
    gold = json.load(open(os.path.join(GOLD, "f23_points_m1_0_1_inf.json")))
    pts = [p if p != "inf" else INF for p in gold["points"]]
    AT, G, BT = exact.build_exact(2, 3, pts)
    assert AT == [[Fr(x) for x in row] for row in gold["AT"]]
    assert G == [[Fr(x) for x in row] for row in gold["G"]]
    assert BT == [[Fr(x) for x in row] for row in gold["BT"]]


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_f23a_pm_c(seed):
    """eq:f2_3a: points in the paper's row order (-c, 0, c, inf)."""
    c = abs(_rand_fr(random.Random(seed)))
    _, G, BT = exact.build_exact(2, 3, [-c, Fr(0), c, INF])
    BT_paper = [[0, -c, 1, 0], [-c * c, 0, 1, 0], [0, c, 1, 0], [0, -c * c, 0, 1]]
    G_paper = [[1 / (2 * c * c), -1 / (2 * c), Fr(1, 2)], [-1 / (c * c), 0, 0],
               [1 / (2 * c * c), 1 / (2 * c), Fr(1, 2)], [0, 0, 1]]
    assert BT == [[Fr(x) for x in r] for r in BT_paper]
    assert G == [[Fr(x) for x in r] for r in G_paper]


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_f23b_generic(seed):
    """eq:f2_3b: points (0, a, b, inf)."""
    rng = random.Random(100 + seed)
    a = _rand_fr(rng)
    b = _rand_fr(rng)
    while b == a:
        b = _rand_fr(rng)
    _, G, BT = exact.build_exact(2, 3, [Fr(0), a, b, INF])
    BT_paper = [[a * b, -a - b, 1, 0], [0, -b, 1, 0], [0, -a, 1, 0], [0, a * b, -a - b, 1]]
    G_paper = [[1 / (a * b), 0, 0],
               [1 / (a * (a - b)), 1 / (a - b), a / (a - b)],
               [-1 / (b * (a - b)), -1 / (a - b), -b / (a - b)],
               [0, 0, 1]]
    assert BT == [[Fr(x) for x in r] for r in BT_paper]
    assert G == [[Fr(x) for x in r] for r in G_paper]


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_f43a_symmetric(seed):
    """eq:f4_3a: points (-1/c, -c, 0, c, 1/c, inf); "1/2(c^4-1)" read as
    1/(2(c^4-1))."""
    c = abs(_rand_fr(random.Random(200 + seed)))
    if c == 1:
        c = Fr(3, 2)
    _, G, BT = exact.build_exact(4, 3, [-1 / c, -c, Fr(0), c, 1 / c, INF])
    c2, c4 = c * c, c ** 4
    q = (c4 + 1) / c2
    BT_paper = [[0, c, -c2, -1 / c, 1, 0],
                [0, 1 / c, -1 / c2, -c, 1, 0],
                [1, 0, -q, 0, 1, 0],
                [0, -1 / c, -1 / c2, c, 1, 0],
                [0, -c, -c2, 1 / c, 1, 0],
                [0, 1, 0, -q, 0, 1]]
    D = 2 * c4 - 2
    G_paper = [[-c4 / D, c ** 3 / D, -c2 / D],
               [1 / D, -c / D, c2 / D],
               [1, 0, 0],
               [1 / D, c / D, c2 / D],
               [-c4 / D, -c ** 3 / D, -c2 / D],
               [0, 0, 1]]
    assert BT == [[Fr(x) for x in r] for r in BT_paper]
    assert G == [[Fr(x) for x in r] for r in G_paper]


def _f43_generic_paper(a, b, c, d, typo=False):
    """eq:f4_3b-d transcribed; `typo=True` keeps the printed
    "-ab(c+d)-cd(a-b)" of P:432 (reading R6 corrects it to -cd(a+b))."""
    e2_bcd = b * (c + d) + c * d
    B00 = [[a * b * c * d, -a * b * (c + d) - c * d * (a + b), a * (b + c + d) + b * (c + d) + c * d],
           [0, -b * c * d, e2_bcd],
           [0, -a * c * d, a * (c + d) + c * d]]
    B03 = [[-a - b - c - d, 1, 0], [-b - c - d, 1, 0], [-a - c - d, 1, 0]]
    last = -a * b * (c + d) - c * d * (a - b) if typo else -a * b * (c + d) - c * d * (a + b)
    B30 = [[0, -a * b * d, a * (b + d) + b * d], [0, -a * b * c, a * (b + c) + b * c], [0, a * b * c * d, last]]
    B33 = [[-a - b - d, 1, 0], [-a - b - c, 1, 0], [a * (b + c + d) + b * (c + d) + c * d, -a - b - c - d, 1]]
    BT = [B00[i] + B03[i] for i in range(3)] + [B30[i] + B33[i] for i in range(3)]
    G = [[1 / (a * b * c * d), 0, 0],
         [1 / (a * (a - b) * (a - c) * (a - d)), 1 / ((a - b) * (a - c) * (a - d)), a / ((a - b) * (a - c) * (a - d))],
         [-1 / (b * (a - b) * (b - c) * (b - d)), -1 / ((a - b) * (b - c) * (b - d)), -b / ((a - b) * (b - c) * (b - d))],
         [1 / (c * (a - c) * (b - c) * (c - d)), 1 / ((a - c) * (b - c) * (c - d)), c / ((a - c) * (b - c) * (c - d))],
         [-1 / (d * (a - d) * (b - d) * (c - d)), -1 / ((a - d) * (b - d) * (c - d)), -d / ((a - d) * (b - d) * (c - d))],
         [0, 0, 1]]
    return [[Fr(x) for x in r] for r in BT], [[Fr(x) for x in r] for r in G]


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_f43_generic(seed):
    rng = random.Random(300 + seed)
    vals = []
    while len(vals) < 4:
        v = _rand_fr(rng)
        if v not in vals:
            vals.append(v)
    a, b, c, d = vals
    _, G, BT = exact.build_exact(4, 3, [Fr(0), a, b, c, d, INF])
    BT_p, G_p = _f43_generic_paper(a, b, c, d)
    assert BT == BT_p
    assert G == G_p
    # the printed entry of P:432 differs whenever cd·b != 0 (typo, reading R6)
    BT_typo, _ = _f43_generic_paper(a, b, c, d, typo=True)
    assert BT_typo[5][2] != BT[5][2]


def _distinct_points(rng, count):
    pts = []
    while len(pts) < count:
        v = Fr(rng.randint(-40, 40), rng.randint(1, 8))
        if v not in pts:
            pts.append(v)
    return pts


@pytest.mark.parametrize("k", [2, 3, 5])
@pytest.mark.parametrize("modified", [True, False])
def test_identity_1d(k, modified):
    """Aᵀ[(Gg) ⊙ (Bᵀd)] == valid correlation, exactly, for n = k..10 (brute force)."""
    rng = random.Random(k * 10 + modified)
    for n in range(k, 11):
        m = n - k + 1
        nf = n - 1 if modified else n
        pts = _distinct_points(rng, nf) + ([INF] if modified else [])
        AT, G, BT = exact.build_exact(m, k, pts)
        for _ in range(3):
            d = [Fr(rng.randint(-50, 50), rng.randint(1, 9)) for _ in range(n)]
            g = [Fr(rng.randint(-50, 50), rng.randint(1, 9)) for _ in range(k)]
            assert exact.winograd_1d(AT, G, BT, d, g) == exact.correlate_1d(d, g)


@pytest.mark.parametrize("m,k", [(2, 3), (4, 3), (6, 3), (8, 3), (4, 5), (6, 5)])
@pytest.mark.parametrize("modified", [True, False])
def test_identity_2d(m, k, modified):
    rng = random.Random(1000 + 10 * m + k + modified)
    n = m + k - 1
    nf = n - 1 if modified else n
    pts = _distinct_points(rng, nf) + ([INF] if modified else [])
    AT, G, BT = exact.build_exact(m, k, pts)
    d = [[Fr(rng.randint(-20, 20), rng.randint(1, 5)) for _ in range(n)] for _ in range(n)]
    g = [[Fr(rng.randint(-20, 20), rng.randint(1, 5)) for _ in range(k)] for _ in range(k)]
    assert exact.winograd_2d(AT, G, BT, d, g) == exact.correlate_2d(d, g)


def test_identity_catches_convolution_convention():
    """The transposed algorithm is cross-correlation, not convolution (reading R3):
    a flipped kernel gives a different result."""
    AT, G, BT = exact.build_exact(2, 3, [Fr(-1), Fr(0), Fr(1), INF])
    d = [Fr(1), Fr(2), Fr(3), Fr(4)]
    g = [Fr(1), Fr(2), Fr(5)]
    y = exact.winograd_1d(AT, G, BT, d, g)
    assert y == exact.correlate_1d(d, g)
    assert y != exact.correlate_1d(d, g[::-1])


def test_infinity_structure():
    """Modified algorithm block form."""
    rng = random.Random(7)
    for m, k in [(2, 3), (4, 3), (6, 3), (4, 5)]:
        n = m + k - 1
        pts = _distinct_points(rng, n - 1)
        AT, G, BT = exact.build_exact(m, k, pts + [INF])
        assert G[n - 1] == [0] * (k - 1) + [1]
        assert [AT[p][n - 1] for p in range(m)] == [0] * (m - 1) + [1]
        assert [BT[i][n - 1] for i in range(n)] == [0] * (n - 1) + [1]
        assert BT[n - 1] == exact.poly_from_roots(pts)


def test_poly_from_roots_spec_examples():
    """SPEC S:60-62 ("M(x) = x(x-1)(x+1)")."""
    assert exact.poly_from_roots([]) == [1]
    assert exact.poly_from_roots([Fr(0), Fr(1), Fr(-1)]) == [0, -1, 0, 1]
    assert exact.poly_from_roots([Fr(2), Fr(-2)]) == [-4, 0, 1]


def test_multiplies_per_output_table1():
    gold = json.load(open(os.path.join(GOLD, "paper_error_values.json")))["multiplies_per_output"]
    for kk, key in ((3, "k3"), (5, "k5")):
        for n, v in gold[key].items():
            val = float(exact.multiplies_per_output(int(n), kk, 2))
            assert round(val, 2) == v, (n, kk, val)


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8, 9, 10, 11])
def test_chebyshev_nodes_are_roots_of_Tq(n):
    """Oracle Chebyshev generator (reading X24): the n - 1 finite nodes are the roots
    of the Chebyshev polynomial T_{n-1} (three-term recurrence, a textbook fact independent
    of the cosine formula), distinct, exactly symmetric (x and -x both present, 0 for odd
    counts), within 4 ulp of 1 of cos((2k-1) pi / (2q)) (the mirrored half differs from the
    direct formula only by the rounding of its argument), and inf last."""
    import math
    from oracle import points as OP
    pts = OP.chebyshev(n)
    assert len(pts) == n and pts[-1] == math.inf
    fin = pts[:-1]
    q = n - 1
    assert len(set(fin)) == q and fin == sorted(fin)
    assert sorted(-v for v in fin) == fin
    for x in fin:
        t0, t1 = 1.0, x
        for _ in range(q - 1):
            t0, t1 = t1, 2 * x * t1 - t0
        assert abs(t1) < 1e-12 * q
    direct = sorted(math.cos((2 * k - 1) * math.pi / (2 * q)) for k in range(1, q + 1))
    for a, b in zip(fin, direct):
        assert abs(a - b) <= 4 * math.ulp(1.0)


def test_chebyshev_product_template_matches_oracle():
    """The product's template (paper_2201_10369_b200.points.chebyshev) and the oracle's
    generator agree bit for bit (GPU tests feed the oracle's sets to both sides)."""
    from oracle import points as OP
    from paper_2201_10369_b200 import points as PP
    for n in range(3, 12):
        assert PP.chebyshev(n) == OP.chebyshev(n)
