"""ORACLE (test infrastructure only) -- fp64 matrix recipe "R64".

The paper builds the transform matrices "from the point values" in floating
point (the cancellations of §5, "manifest"
only if ±c terms cancel exactly).  The paper does not fix an fp64 operation
order; reading R5 fixes this one, and it is the bit-exact contract of
``wino_points_to_matrices``.  Python floats are IEEE binary64, every operation
below is one correctly-rounded op (RN-even), with no contraction.

(i)  root products ∏(x - r) over a set S of finite roots:
     p = [1.0];
     for each a > 0 with -a ∈ S, ascending a:  s = a*a;
         p'_j = p_{j-2} - s*p_j            (factor x² - s)
     for each remaining non-zero root r, ascending:
         p'_j = p_{j-1} - r*p_j            (factor x - r)
     out-of-range p_j read as +0.0;  if 0 ∈ S: prepend +0.0 (factor x).
(ii) Nᵢ: acc = 1.0; for j in caller index order, j ≠ i: acc = acc * (αᵢ - αⱼ).
(iii) powers pw_0 = 1.0, pw_{p+1} = pw_p * αᵢ.
(iv) G[i][q] = pw_q / Nᵢ;  Aᵀ[p][i] = pw_p.
(v)  Bᵀ row i = (i) over F∖{αᵢ} padded with +0.0;  ∞ row = (i) over F;
     ∞ column/row structure as in ``oracle.exact``.
fp32 matrices = RN32 of these (numpy ``astype(np.float32)``).
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

INF = float("inf")


def validate(m: int, k: int, points: Sequence[float]) -> None:
    n = m + k - 1
    if m < 1 or k < 1:
        raise ValueError("m, k >= 1")
    if len(points) != n:
        raise ValueError("n != m + k - 1")
    for i, p in enumerate(points):
        if math.isnan(p):
            raise ValueError("NaN point")
        if math.isinf(p) and (p < 0 or i != n - 1):
            raise ValueError("inf must be +inf and last")
    fin = [p for p in points if not math.isinf(p)]
    for i in range(len(fin)):
        for j in range(i):
            if fin[i] == fin[j]:
                raise ValueError("duplicate points")


def poly_from_roots_r64(S: Sequence[float]) -> List[float]:
    """Recipe (i).  Result depends only on the set S, not its order."""
    S = [float(x) for x in S]
    has_zero = any(x == 0.0 for x in S)
    nz = [x for x in S if x != 0.0]
    pos = sorted(a for a in nz if a > 0.0 and (-a) in nz)
    paired = set(pos) | set(-a for a in pos)
    lin = sorted(x for x in nz if x not in paired)
    p = [1.0]
    for a in pos:
        s = a * a
        q = []
        for j in range(len(p) + 2):
            pj2 = p[j - 2] if 0 <= j - 2 < len(p) else 0.0
            pj = p[j] if j < len(p) else 0.0
            q.append(pj2 - s * pj)
        p = q
    for r in lin:
        q = []
        for j in range(len(p) + 1):
            pj1 = p[j - 1] if 0 <= j - 1 < len(p) else 0.0
            pj = p[j] if j < len(p) else 0.0
            q.append(pj1 - r * pj)
        p = q
    if has_zero:
        p = [0.0] + p
    return p


def build_r64(m: int, k: int, points: Sequence[float]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(Aᵀ [m,n], G [n,k], Bᵀ [n,n]) as float64 arrays, recipe R64."""
    points = [float(p) for p in points]
    validate(m, k, points)
    n = m + k - 1
    has_inf = math.isinf(points[-1])
    F = points[:-1] if has_inf else points
    nf = len(F)
    AT = np.zeros((m, n))
    G = np.zeros((n, k))
    BT = np.zeros((n, n))
    for i, a in enumerate(F):
        Ni = 1.0
        for j, b in enumerate(F):
            if j != i:
                Ni = Ni * (a - b)
        pw = [1.0]
        for _ in range(max(m, k) - 1):
            pw.append(pw[-1] * a)
        for p in range(m):
            AT[p, i] = pw[p]
        for q in range(k):
            G[i, q] = pw[q] / Ni
        Mi = poly_from_roots_r64([b for j, b in enumerate(F) if j != i])
        BT[i, : len(Mi)] = Mi
    if has_inf:
        AT[m - 1, nf] = 1.0
        G[nf, k - 1] = 1.0
        Mp = poly_from_roots_r64(F)
        BT[nf, : len(Mp)] = Mp
    return AT, G, BT


def build_f32(m: int, k: int, points: Sequence[float]):
    """fp32 copies (RN) of the R64 matrices."""
    AT, G, BT = build_r64(m, k, points)
    return AT.astype(np.float32), G.astype(np.float32), BT.astype(np.float32)


def ulp_distance(a: float, b: float) -> int:
    """Number of fp64 values between a and b (0 if equal)."""
    if a == b:
        return 0
    ia = np.array([a]).view(np.int64)[0]
    ib = np.array([b]).view(np.int64)[0]
    ia = ia if ia >= 0 else -(ia & 0x7FFFFFFFFFFFFFFF)
    ib = ib if ib >= 0 else -(ib & 0x7FFFFFFFFFFFFFFF)
    return int(abs(int(ia) - int(ib)))
