// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_1d_large() {
  return {
      make_cfg<1, 6, 3, TPAIR_REG>({make_variant<1, 6, 3, TPAIR_REG, kZ_N8_CD>()}),
      make_cfg<1, 7, 3, TPAIR_REG>(),
      make_cfg<1, 8, 3, TPAIR_REG>({make_variant<1, 8, 3, TPAIR_REG, kZ_N10_C1C2>()}),
      make_cfg<1, 6, 5, TPAIR_REG>({make_variant<1, 6, 5, TPAIR_REG, kZ_N10_C1C2_R5>()}),
  };
}

}  // namespace wino
