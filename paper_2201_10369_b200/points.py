"""Point-set instantiation (§8(a) row a1): the paper's families as explicit fp64 point
lists in canonical order (finite ascending, +inf last; reading R7).

{0, -c, c, inf} for F(2,3) (eq:ps0); {0, ±c, ±1/c, inf} for F(4,3)
(eq:ps1); {0, ±c, ±1/c, ±d, ±1/d, inf} for F(8,3) (eq:ps2) and
the n = 7..9 subsets of P:322-327; the n = 8 2D row {0, ±1/c, ±c, -1/d, d, inf}
(P:654-655).  1/c is one fp64 division; negation is exact.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Sequence

INF = math.inf


class TemplateError(ValueError):
    """Template-level rejection raised before the ABI (SPEC NonPositiveC / DegenerateFamily)."""


def _canon(finite: Sequence[float]) -> List[float]:
    fin = sorted(float(v) for v in finite)
    for a, b in zip(fin, fin[1:]):
        if a == b:
            raise TemplateError(f"degenerate family: duplicate point {a!r}")
    return fin + [INF]


def _pos(*cs: float) -> None:
    for c in cs:
        if not (c > 0 and math.isfinite(c)):
            raise TemplateError("family parameters must be finite and > 0")


def family_f23(c: float) -> List[float]:
    _pos(c)
    return _canon([0.0, -c, c])


def family_f43(c: float) -> List[float]:
    _pos(c)
    q = 1.0 / c
    return _canon([0.0, -c, c, -q, q])


def family_n8_cd(c: float, d: float) -> List[float]:
    _pos(c, d)
    q, e = 1.0 / c, 1.0 / d
    return _canon([0.0, -q, -c, c, q, -e, d])


def family_n8_c1c2(c1: float, c2: float) -> List[float]:
    _pos(c1, c2)
    q = 1.0 / c1
    return _canon([0.0, -q, -c1, c1, q, -c2, c2])


def family_n10(c1: float, c2: float) -> List[float]:
    _pos(c1, c2)
    q1, q2 = 1.0 / c1, 1.0 / c2
    return _canon([0.0, -q1, -c1, c1, q1, -q2, -c2, c2, q2])


# name -> (m, r, n_params, maker)
TEMPLATES: Dict[str, tuple] = {
    "f23_c": (2, 3, 1, family_f23),
    "f43_c": (4, 3, 1, family_f43),
    "n8_cd": (6, 3, 2, family_n8_cd),
    "n8_c1c2_r5": (4, 5, 2, family_n8_c1c2),
    "n10_c1c2_r5": (6, 5, 2, family_n10),
    "n10_c1c2": (8, 3, 2, family_n10),
}

# Prior-work sets (∞ implicit)
P4 = _canon([0.0, -1.0, 1.0])
P8 = _canon([0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0])
P10 = _canon([0.0, -1.0, 1.0, 0.5, -0.5, 2.0, -2.0, -0.25, 4.0])


def chebyshev(n: int) -> List[float]:
    """n - 1 Chebyshev nodes x_k = cos((2k - 1) pi / (2(n - 1))), k = 1..n-1, plus
    the formal ∞ (modified algorithm).  Computed for k <= ceil((n-1)/2) and mirrored by
    negation, so the set is exactly symmetric and the middle node of an odd count is
    exactly 0 (reading X24)."""
    q = n - 1
    if q < 1:
        raise TemplateError("n >= 2")
    half = []
    for k in range(1, (q + 1) // 2 + 1):
        half.append(math.cos((2 * k - 1) * math.pi / (2 * q)))
    nodes = [v for v in half if not (q % 2 == 1 and v == half[-1])] if q % 2 == 1 else half
    fin = nodes + [-v for v in nodes] + ([0.0] if q % 2 == 1 else [])
    return _canon(fin)


def instantiate(maker: Callable[..., List[float]], params) -> tuple:
    """Instantiate a template over parameter tuples.  Returns (point_sets [S][n] as a list,
    ok flags): a degenerate parameter gives a row of NaNs (rejected by the ABI as
    WINO_E_NONFINITE_POINT) instead of aborting the sweep."""
    sets, ok = [], []
    n = None
    for p in params:
        p = p if isinstance(p, tuple) else (p,)
        try:
            s = maker(*p)
            n = len(s)
            sets.append(s)
            ok.append(True)
        except TemplateError:
            sets.append(None)
            ok.append(False)
    n = n or 0
    return [s if s is not None else [math.nan] * n for s in sets], ok
