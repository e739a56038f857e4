// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_2d_small() {
  return {
      make_cfg<2, 1, 2, TPAIR_REG>(),
      make_cfg<2, 2, 3, TPAIR_REG>({make_variant<2, 2, 3, TPAIR_REG, kZ_F23_C>()}),
      make_cfg<2, 3, 3, TPAIR_REG>(),
  };
}

}  // namespace wino
