// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.  2D, n = 7..8: one tile per thread,
// held in registers (TSINGLE_REG, packed inputs), no shared-memory staging.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_2d_mid() {
  return {
      make_cfg<2, 5, 3, TSINGLE_REG>(),
      make_cfg<2, 6, 3, TSINGLE_REG>({make_variant<2, 6, 3, TSINGLE_REG, kZ_N8_CD>()}),
      make_cfg<2, 4, 5, TSINGLE_REG>({make_variant<2, 4, 5, TSINGLE_REG, kZ_N8_C1C2_R5>()}),
  };
}

}  // namespace wino
