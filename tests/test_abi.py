"""C-ABI library: loads, exports every symbol include/wino.h declares, and its host
matrix builder (wino_points_to_matrices) is bit-identical to the oracle's R64 recipe
on every point set the configs use plus random sets.  CPU only (no device calls)."""
import math
import os
import re

import numpy as np
import pytest

import synth
from oracle import points as OP, r64
from paper_2201_10369_b200 import _lib, api, points as PP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INF = math.inf


def _header_functions():
    src = open(os.path.join(ROOT, "include", "wino.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wino_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    L = _lib.load()
    names = _header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(L, n), n
    declared = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == declared


def test_status_strings():
    L = _lib.load()
    for s in range(9):
        assert L.wino_status_string(s).decode().startswith("WINO_")


def _same_bits(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def _check(m, r, pts):
    got = api.wino_points_to_matrices(m, r, pts)
    exp = r64.build_r64(m, r, pts)
    for g, e in zip(got, exp):
        assert _same_bits(g, e), (m, r, pts)


def test_builder_bitexact_cfg1_cfg3_sets():
    _check(2, 3, [-1.0, 0.0, 1.0, INF])
    _check(6, 3, PP.family_n8_cd(2.0, 1.003))
    _check(6, 3, PP.P8)
    _check(8, 3, PP.P10)


def test_builder_bitexact_cfg2_grid():
    for c in synth.c_grid():
        _check(4, 3, PP.family_f43(float(c)))


def test_builder_bitexact_cfg4_full_grid():
    """BASELINE.json configs[3]: every one of the 256 x 256 (c1, c2) point sets of BOTH
    templates (n = 8 and n = 10, r = 5), memcmp of all three fp64 matrices against the
    oracle's R64 (SURVEY §8(c) acceptance table).  The points come from the oracle's own
    template makers; degenerate cells (c1 == c2, c1 == 1/c2, ...) must be rejected by both."""
    from oracle import points as OP
    g = [float(c) for c in synth.c_grid(256)]
    n_checked = n_rejected = 0
    for c1 in g:
        for c2 in g:
            for m, maker in ((4, OP.n8_c1c2), (6, OP.n10_c1c2)):
                pts = maker(c1, c2)
                if len(set(pts)) != len(pts):
                    with pytest.raises(_lib.WinoError):
                        api.wino_points_to_matrices(m, 5, pts)
                    n_rejected += 1
                    continue
                _check(m, 5, pts)
                n_checked += 1
    assert n_checked + n_rejected == 2 * 256 * 256 and n_checked > 2 * 65000


def test_zero_masks_header_rederived():
    """csrc/zero_masks.h (the structural zeros the sweep kernels skip at compile time) is
    exactly what libwino's own builder gives over the configs' grids (tools/gen_zero_masks.py);
    and each family's mask is a true zero pattern of the oracle's R64 matrices at sampled
    parameters (an independent check that no skipped entry is ever non-zero)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_zero_masks", os.path.join(ROOT, "tools", "gen_zero_masks.py"))
    gz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gz)
    text = open(gz.HEADER).read()
    assert gz.parse(text) == gz.derive(step2=1)
    assert gz.render(gz.derive(step2=1)) == text
    from oracle import points as OP
    makers = {"f23_c": OP.f23_c, "f43_c": OP.f43_c, "n8_cd": OP.n8_cd, "n8_c1c2_r5": OP.n8_c1c2,
              "n10_c1c2_r5": OP.n10_c1c2, "n10_c1c2": OP.n10_c1c2}
    masks = gz.parse(text)
    rng = np.random.default_rng(5)
    for fid, name, m, r, _, npar, _ in gz.FAMILIES:
        for _ in range(25):
            p = tuple(float(v) for v in np.exp(rng.uniform(np.log(0.05), np.log(20), npar)))
            pts = makers[name](*p)
            if len(set(pts)) != len(pts):
                continue
            for z, M in zip(masks[fid], r64.build_r64(m, r, pts)):
                flat = np.asarray(M).ravel()
                skipped = [k for k in range(flat.size) if (z >> k) & 1]
                assert np.all(flat[skipped] == 0.0), (name, p)


def test_builder_bitexact_random_sets():
    rng = np.random.default_rng(0)
    for trial in range(3000):
        r = int(rng.choice([2, 3, 5]))
        n = int(rng.integers(r, 13))
        m = n - r + 1
        modified = bool(rng.integers(0, 2))
        nf = n - 1 if modified else n
        vals = list(np.unique(rng.standard_normal(nf) * rng.choice([0.1, 1.0, 10.0])))
        if len(vals) != nf:
            continue
        if rng.integers(0, 3) == 0 and nf >= 3:  # symmetric pairs
            vals[1] = -vals[0]
            if len(set(vals)) != nf:
                continue
        pts = [float(v) for v in rng.permutation(vals)] + ([INF] if modified else [])
        _check(m, r, pts)


def test_templates_match_oracle_templates():
    for c in synth.c_grid()[::17]:
        assert PP.family_f43(float(c)) == OP.f43_c(float(c))
        assert PP.family_f23(float(c)) == OP.f23_c(float(c))
    assert PP.family_n8_cd(2.0, 1.003) == OP.n8_cd(2.0, 1.003)
    assert PP.P8 == OP.P8 and PP.P10 == OP.P10


@pytest.mark.parametrize("m,r,pts,status", [
    (2, 3, [-1.0, 0.0, 1.0], 2),
    (2, 3, [-1.0, 0.0, 0.0, INF], 3),
    (2, 3, [-1.0, 0.0, -0.0, INF], 3),
    (2, 3, [-1.0, INF, 1.0, 2.0], 4),
    (2, 3, [-1.0, 0.0, 1.0, -INF], 4),
    (2, 3, [-1.0, math.nan, 1.0, INF], 5),
    (0, 3, [0.0, 1.0], 1),
    (10, 8, [float(i) for i in range(17)], 8),
])
def test_builder_errors(m, r, pts, status):
    with pytest.raises(_lib.WinoError) as ei:
        api.wino_points_to_matrices(m, r, pts)
    assert ei.value.status == status


def test_supported_table():
    assert api.wino_supported(2, 4, 3) and api.wino_supported(1, 4, 3) and api.wino_supported(2, 3, 3)
    assert api.wino_supported(0, 6, 3) and api.wino_supported(0, 2, 3)
    assert not api.wino_supported(3, 4, 3)


def test_workspace_sizes():
    assert api.wino_error_sweep_workspace_bytes(2, 4, 3, 4096, 100_000) > 100_000 * 16 * 8
    b = api.wino_conv2d_workspace_bytes(32, 256, 56, 56, 256, 3, 1, 6)
    assert b > 3 * 64 * 256 * 3200 * 4 // 2
    assert api.wino_conv2d_workspace_bytes(1, 1, 1, 1, 1, 3, 0, 2) == 0


def test_layer_empty_batch_and_validation_without_device():
    """Host-side paths of wino_conv2d_fp32 that enqueue nothing: N == 0 / K == 0 are
    successful no-ops (dummy, never dereferenced pointers); validation errors are reported
    before any device call."""
    import ctypes
    L = _lib.load()
    buf = (ctypes.c_float * 16)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    pts = np.array(OP.f23_c(1.0), dtype=np.float64)
    pp = pts.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    for N, K in ((0, 8), (2, 0)):
        st = L.wino_conv2d_fp32(p, p, p, N, 8, 16, 16, K, 3, 1, 2, pp, None, 0, None, None, None)
        assert st == 0, st
        assert L.wino_last_launch_count() == 0
    st = L.wino_conv2d_fp32(p, p, p, -1, 8, 16, 16, 8, 3, 1, 2, pp, None, 0, None, None, None)
    assert st == 1
    bad = np.array([0.0, 0.0, 1.0, INF])
    st = L.wino_conv2d_fp32(p, p, p, 0, 8, 16, 16, 8, 3, 1, 2, bad.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            None, 0, None, None, None)
    assert st == 3                                   # point validation still applies
    st = L.wino_conv2d_fp32_ex(p, p, p, 0, 8, 16, 16, 8, 3, 1, 2, pp, None, 0, None, None, 8, None)
    assert st == 1                                   # unknown flag


def test_contraction_kernel_choice_vgg_shapes():
    """wino_conv2d_gemm_tile (host only): the configs[4] VGG-16 x64 layers pick the fused
    first-layer kernel, 64-row tiles for K = 64, and the 128 x 64 tile exactly where it saves
    a wave (28 x 28: 11 waves instead of 12; 14 x 14: 4 instead of 5)."""
    from paper_2201_10369_b200 import api
    t = lambda C, K, H: api.wino_conv2d_gemm_tile(64, C, H, H, K, 3, 1, 6)
    assert t(3, 64, 224) == 1
    assert t(64, 64, 224) == 64128
    assert t(64, 128, 112) == 128128 and t(256, 256, 56) == 128128
    assert t(256, 512, 28) == 128064 and t(512, 512, 14) == 128064
    assert api.wino_conv2d_gemm_tile(32, 256, 56, 56, 256, 3, 1, 6) == 128128   # configs[2]
    assert api.wino_conv2d_gemm_tile(0, 3, 8, 8, 8, 3, 1, 6) == 0 and t(8, 8, 9) != 0
    assert api.wino_conv2d_gemm_tile(1, 8, 8, 8, 8, 4, 1, 6) == 0               # no F(6,4) layer kernel
