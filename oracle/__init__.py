"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the hot path of
arXiv 2201.10369 computes, written from PAPER.md (cited ``P:<line>``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything here.  The
product package ``paper_2201_10369_b200`` never imports it and shares no code
with it (no kernels, headers, helpers, constant generators or pre/post
processing).  Only ``synth`` (seeded input generators, no method arithmetic)
serves both sides.

Modules
  exact   -- exact-rational (fractions.Fraction) matrices, Winograd and correlation
             (SURVEY §8(c) O2).  Pinned: closed forms of P:346-452, brute force.
  r64     -- the fp64 matrix recipe R64 (O3), Python floats (IEEE binary64, RN,
             no contraction).  Pinned: within a few ulp of ``exact``, exact zeros.
  points  -- the paper's point families {0, +-c, +-1/c, ..., inf}.
  ref     -- ctypes driver for ref.c: canonical fp32 Winograd (O5/O6), fp64 direct
             correlation (O7), error statistics (O8), sweep (O9), layer (O4).
             Pinned: exactness special cases, T7/T8 n=0 rows, SPEC examples.

Parity status of each function is listed in DESIGN.md §4 ("parity pins").
"""
