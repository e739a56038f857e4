// Huffman-order sweep kernels (NEXT row N2, sweep_huff.cuh) for the paper's F(m,3) tables:
// F(2,3), F(4,3), F(6,3) in 1D and 2D.
#include "sweep_huff.cuh"

namespace wino {

std::vector<HuffCfg> sweep_huff_cfgs() {
  return {
      make_huff_cfg<1, 2, 3>(), make_huff_cfg<1, 4, 3>(), make_huff_cfg<1, 6, 3>(),
      make_huff_cfg<2, 2, 3>(), make_huff_cfg<2, 4, 3>(), make_huff_cfg<2, 6, 3>(),
  };
}

}  // namespace wino
