// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_1d() {
  return {
      make_cfg<1, 1, 2, TPAIR_REG>(),
      make_cfg<1, 2, 3, TPAIR_REG>({make_variant<1, 2, 3, TPAIR_REG, kZ_F23_C>()}),
      make_cfg<1, 3, 3, TPAIR_REG>(),
      make_cfg<1, 4, 3, TPAIR_REG>({make_variant<1, 4, 3, TPAIR_REG, kZ_F43_C>()}),
      make_cfg<1, 5, 3, TPAIR_REG>(),
  };
}

}  // namespace wino
