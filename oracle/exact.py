"""ORACLE (test infrastructure only) -- exact-rational Toom-Cook construction.

Every fp64 value is a dyadic rational, so ``Fraction(x)`` is exact.  This module
writes out PAPER.md §4.1-4.2 literally:

* Aᵀ (m x n): column i = [1, αᵢ, …, αᵢ^{m-1}]ᵀ  (Vandermonde);
* G  (n x k): row i = [1, αᵢ, …, αᵢ^{k-1}] / Nᵢ, Nᵢ = ∏_{j≠i}(αᵢ-αⱼ)
  ("scaling factor … embedded into the matrix G"; divided, as every concrete
  G of P:354-359, P:372-377, P:397-404, P:443-450 shows -- DESIGN.md reading R1);
* Bᵀ (n x n): row i = ascending coefficients of Mᵢ(x) = ∏_{j≠i}(x-αⱼ);
* modified algorithm: the points are n-1 finite αⱼ plus the formal ∞;
  G gets the row [0,…,0,1], Aᵀ the column [0,…,0,1]ᵀ,
  Bᵀ the row of M′(x) = ∏_j(x-αⱼ) coefficients ending in 1 and the column
  [0,…,0,1]ᵀ (reading R4).

Winograd (P:174 eq:conv_1d, P:181 eq:conv_2d) and valid cross-correlation
(eq:conv P:112, reading R3) are evaluated exactly.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence, Tuple

INF = float("inf")

Matrix = List[List[Fraction]]


def _is_inf(p) -> bool:
    return isinstance(p, float) and p == INF or (isinstance(p, str) and p == "inf")


def split_points(points: Sequence) -> Tuple[List[Fraction], bool]:
    """(finite points as Fractions in caller order, has_inf).  ∞ must be last."""
    pts = list(points)
    has_inf = len(pts) > 0 and _is_inf(pts[-1])
    fin = pts[:-1] if has_inf else pts
    if any(_is_inf(p) for p in fin):
        raise ValueError("inf allowed only as the last point")
    F = [p if isinstance(p, Fraction) else Fraction(p) for p in fin]
    if len(set(F)) != len(F):
        raise ValueError("duplicate points")
    return F, has_inf


def poly_from_roots(roots: Sequence[Fraction]) -> List[Fraction]:
    """Ascending coefficients of ∏(x - r) ("M(x) = (x-α₀)…(x-α_{n-1})")."""
    p = [Fraction(1)]
    for r in roots:
        q = [Fraction(0)] * (len(p) + 1)
        for j, c in enumerate(p):
            q[j + 1] += c
            q[j] -= r * c
        p = q
    return p


def scaling_factor(F: Sequence[Fraction], i: int) -> Fraction:
    """Nᵢ = ∏_{j≠i}(αᵢ - αⱼ) over the finite points."""
    N = Fraction(1)
    for j, a in enumerate(F):
        if j != i:
            N *= F[i] - a
    return N


def build_exact(m: int, k: int, points: Sequence) -> Tuple[Matrix, Matrix, Matrix]:
    """Exact (Aᵀ, G, Bᵀ) for F(m, k) on ``points`` (n = m + k - 1 of them, the
    last may be ∞ = modified Toom-Cook).  Row/column i belongs to points[i]."""
    n = m + k - 1
    if len(points) != n:
        raise ValueError(f"need n = m + k - 1 = {n} points, got {len(points)}")
    F, has_inf = split_points(points)
    nf = len(F)
    AT = [[Fraction(0)] * n for _ in range(m)]
    G = [[Fraction(0)] * k for _ in range(n)]
    BT = [[Fraction(0)] * n for _ in range(n)]
    for i, a in enumerate(F):
        Ni = scaling_factor(F, i)
        for p in range(m):
            AT[p][i] = a ** p
        for q in range(k):
            G[i][q] = a ** q / Ni
        Mi = poly_from_roots([b for j, b in enumerate(F) if j != i])
        for j, c in enumerate(Mi):
            BT[i][j] = c
    if has_inf:
        AT[m - 1][nf] = Fraction(1)
        G[nf][k - 1] = Fraction(1)
        Mp = poly_from_roots(F)  # M'(x), degree n-1, leading coefficient 1
        for j, c in enumerate(Mp):
            BT[nf][j] = c
    return AT, G, BT


# ---------------------------------------------------------------- exact evaluation

def matvec(A: Matrix, x: Sequence[Fraction]) -> List[Fraction]:
    return [sum((a * b for a, b in zip(row, x)), Fraction(0)) for row in A]


def matmul(A: Matrix, B: Matrix) -> Matrix:
    return [[sum((A[i][t] * B[t][j] for t in range(len(B))), Fraction(0))
             for j in range(len(B[0]))] for i in range(len(A))]


def transpose(A: Matrix) -> Matrix:
    return [list(r) for r in zip(*A)]


def winograd_1d(AT, G, BT, d, g) -> List[Fraction]:
    """Y = Aᵀ[(Gg) ⊙ (Bᵀd)] (eq:conv_1d)."""
    U = matvec(G, g)
    V = matvec(BT, d)
    return matvec(AT, [u * v for u, v in zip(U, V)])


def winograd_2d(AT, G, BT, d, g) -> Matrix:
    """Y = Aᵀ[(G g Gᵀ) ⊙ (Bᵀ d B)]A (eq:conv_2d)."""
    U = matmul(matmul(G, g), transpose(G))
    V = matmul(matmul(BT, d), transpose(BT))
    Mh = [[U[i][j] * V[i][j] for j in range(len(U[0]))] for i in range(len(U))]
    return matmul(matmul(AT, Mh), transpose(AT))


def correlate_1d(d, g) -> List[Fraction]:
    """Valid cross-correlation y_i = Σ_j g_j d_{i+j} (brute force)."""
    k = len(g)
    return [sum((g[j] * d[i + j] for j in range(k)), Fraction(0)) for i in range(len(d) - k + 1)]


def correlate_2d(d, g) -> Matrix:
    """Valid 2D cross-correlation y[p][s] = Σ_u Σ_v g[u][v] d[p+u][s+v] (eq:conv P:112)."""
    r = len(g)
    H = len(d) - r + 1
    W = len(d[0]) - len(g[0]) + 1
    return [[sum((g[u][v] * d[p + u][s + v] for u in range(r) for v in range(len(g[0]))), Fraction(0))
             for s in range(W)] for p in range(H)]


def multiplies_per_output(n: int, k: int, dims: int) -> Fraction:
    """Table 1: n^d / (n-k+1)^d Hadamard multiplies per output."""
    m = n - k + 1
    if m < 1:
        raise ValueError("input block smaller than kernel")
    return Fraction(n ** dims, m ** dims)
