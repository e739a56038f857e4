// Mixed-precision sweep kernels (NEXT row N2, sweep_mixed.cuh): F(2,3), F(4,3), F(6,3),
// 1D and 2D.
#include "sweep_mixed.cuh"

namespace wino {

std::vector<HuffCfg> sweep_mixed_cfgs() {
  return {
      make_mixed_cfg<1, 2, 3>(), make_mixed_cfg<1, 4, 3>(), make_mixed_cfg<1, 6, 3>(),
      make_mixed_cfg<2, 2, 3>(), make_mixed_cfg<2, 4, 3>(), make_mixed_cfg<2, 6, 3>(),
  };
}

}  // namespace wino
