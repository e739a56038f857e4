// Huffman-order sweep kernels for F(6,3), F(7,3), F(8,3) (n = 8..10), 1D and 2D.
#include "sweep_huff.cuh"

namespace wino {

std::vector<HuffCfg> sweep_huff_cfgs_large() {
  return {
      make_huff_cfg<1, 6, 3>(), make_huff_cfg<1, 7, 3>(), make_huff_cfg<1, 8, 3>(),
      make_huff_cfg<2, 6, 3>(), make_huff_cfg<2, 7, 3>(), make_huff_cfg<2, 8, 3>(),
  };
}

}  // namespace wino
