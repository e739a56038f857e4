// Huffman-order sweep kernels for F(6,3), F(7,3), F(8,3) in 1D and F(6,3) in 2D; the 2D
// F(7,3) / F(8,3) kernels (the slowest to compile) live in their own translation units.
#include "sweep_huff.cuh"

namespace wino {

HuffCfg huff_cfg_2d_7_3();
HuffCfg huff_cfg_2d_8_3();

std::vector<HuffCfg> sweep_huff_cfgs_large() {
  return {
      make_huff_cfg<1, 6, 3>(), make_huff_cfg<1, 7, 3>(), make_huff_cfg<1, 8, 3>(),
      make_huff_cfg<2, 6, 3>(), huff_cfg_2d_7_3(),        huff_cfg_2d_8_3(),
  };
}

}  // namespace wino
