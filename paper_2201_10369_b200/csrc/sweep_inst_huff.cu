// Huffman-order sweep kernels (NEXT row N2, sweep_huff.cuh) for the paper's F(m,3) tables
// (T7/T8, n = m + 2 = 4..10): the small shapes here, the large ones in
// sweep_inst_huff_large.cu (parallel compilation units).
#include "sweep_huff.cuh"

namespace wino {

std::vector<HuffCfg> sweep_huff_cfgs_large();

std::vector<HuffCfg> sweep_huff_cfgs() {
  std::vector<HuffCfg> v = {
      make_huff_cfg<1, 2, 3>(), make_huff_cfg<1, 3, 3>(), make_huff_cfg<1, 4, 3>(), make_huff_cfg<1, 5, 3>(),
      make_huff_cfg<2, 2, 3>(), make_huff_cfg<2, 3, 3>(), make_huff_cfg<2, 4, 3>(), make_huff_cfg<2, 5, 3>(),
  };
  for (auto& h : sweep_huff_cfgs_large()) v.push_back(h);
  return v;
}

}  // namespace wino
