// Huffman-order 2D F(7x7,3x3) sweep kernels (own translation unit: compile time).
#include "sweep_huff.cuh"

namespace wino {
HuffCfg huff_cfg_2d_7_3() { return make_huff_cfg<2, 7, 3>(); }
}  // namespace wino
