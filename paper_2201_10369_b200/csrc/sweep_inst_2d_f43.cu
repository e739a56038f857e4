// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_2d_f43() {
  return {make_cfg<2, 4, 3, TPAIR_REG>({make_variant<2, 4, 3, TPAIR_REG, kZ_F43_C>()})};
}

}  // namespace wino
