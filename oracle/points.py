"""ORACLE (test infrastructure only) -- the paper's point families.

Each family returns an ordered fp64 list in canonical order (finite ascending,
+inf last; reading R7).  1/c is one fp64 division (RN); negation is exact,
so ±c and ±1/c cancel exactly in the matrix recipe.
"""
from __future__ import annotations

from typing import List

INF = float("inf")


def canonical(finite: List[float], inf: bool = True) -> List[float]:
    pts = sorted(float(p) for p in finite)
    return pts + ([INF] if inf else [])


def f23_c(c: float) -> List[float]:
    """{0, -c, c, ∞} for F(2,3)  (eq:ps0)."""
    return canonical([0.0, -c, c])


def f43_c(c: float) -> List[float]:
    """{0, -1/c, -c, c, 1/c, ∞} for F(4,3)  (eq:ps1)."""
    q = 1.0 / c
    return canonical([0.0, -q, -c, c, q])


def n8_cd(c: float, d: float) -> List[float]:
    """{0, ±1/c, ±c, -1/d, d, ∞}: the 2D n=8 row of T8."""
    q, e = 1.0 / c, 1.0 / d
    return canonical([0.0, -q, -c, c, q, -e, d])


def n8_c1c2(c1: float, c2: float) -> List[float]:
    """{0, ±c1, ±1/c1, ±c2, ∞}: c-family plus the ±d pair (T7 n=8 form)."""
    q = 1.0 / c1
    return canonical([0.0, -q, -c1, c1, q, -c2, c2])


def n10_c1c2(c1: float, c2: float) -> List[float]:
    """{0, ±c1, ±1/c1, ±c2, ±1/c2, ∞} (eq:ps2; T7/T8 n=10)."""
    q1, q2 = 1.0 / c1, 1.0 / c2
    return canonical([0.0, -q1, -c1, c1, q1, -q2, -c2, c2, q2])


def chebyshev(n: int) -> List[float]:
    """Chebyshev nodes for n points ("Chebyshev nodes"): the q = n - 1 roots of T_q,
    x_k = cos((2k - 1) pi / (2q)), k = 1..q, plus the formal inf (modified algorithm).
    Reading X24: the set is made exactly symmetric -- node q + 1 - k is the
    negation of node k (cos(pi - t) = -cos(t)) and the middle node of an odd q is exactly 0 --
    so the +-x cancellations of the paper's symmetric sets hold for it too."""
    import math
    q = n - 1
    x = [math.cos((2 * k - 1) * math.pi / (2 * q)) for k in range(1, q + 1)]
    for k in range(1, q + 1):
        if 2 * k > q + 1:
            x[k - 1] = -x[q - k]        # mirror of node q + 1 - k
        elif 2 * k == q + 1:
            x[k - 1] = 0.0
    return canonical(x)


# prior-work ("Barabasz et al.") sets of P:291, P:623-633, P:649-659 (∞ implicit)
P4 = canonical([0.0, -1.0, 1.0])
P8 = canonical([0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0])
P10 = canonical([0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0, -0.25, 4.0])
F43_PRIOR_1D = canonical([0.0, -1.0, 1.0, 0.5, -3.0])   # T7 n=6
F43_PRIOR_2D = canonical([0.0, -1.0, 1.0, 0.5, -2.0])   # T8 n=6
