"""Host-side checks of the run-time specialised Huffman-order kernels (huff_jit.cu, reading
R21): the generated source of every T7/T8 shape (F(m,3), m = 2..8, 1D and 2D) compiles with
NVRTC for sm_100a -- no GPU needed -- and point sets with the same coefficient order share
one class.  GPU parity (bit-identical outputs vs the oracle's Huffman mode) is in
tests/test_gpu_huffman.py, which runs every test on both Huffman kernels."""
import math

import pytest

from oracle import points as OP

INF = math.inf


@pytest.mark.parametrize("dims", [1, 2])
def test_generated_kernels_compile(dims):
    from paper_2201_10369_b200 import api
    for m in range(2, 9):
        n = m + 2
        finite = [0.0] + [s * v for v in (0.5, 1.0, 2.0, 3.0, 1 / 3.0, 4.0, 0.25) for s in (-1, 1)]
        pts = sorted(finite[:n - 1]) + [INF]
        assert api.wino_huffman_jit_compile_check(dims, m, 3, pts) > 10_000, m


def test_compile_check_rejects_bad_points():
    from paper_2201_10369_b200 import api, _lib
    with pytest.raises(_lib.WinoError):
        api.wino_huffman_jit_compile_check(2, 4, 3, [0.0, 1.0, 1.0, -1.0, 2.0, INF])


def test_jit_mode_roundtrip():
    from paper_2201_10369_b200 import api
    prev = api.wino_huffman_jit_mode(2)
    assert api.wino_huffman_jit_mode(1) == 2
    assert api.wino_huffman_jit_mode(prev) == 1
