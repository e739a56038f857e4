// Huffman-order 2D F(8x8,3x3) sweep kernels (own translation unit: compile time).
#include "sweep_huff.cuh"

namespace wino {
HuffCfg huff_cfg_2d_8_3() { return make_huff_cfg<2, 8, 3>(); }
}  // namespace wino
