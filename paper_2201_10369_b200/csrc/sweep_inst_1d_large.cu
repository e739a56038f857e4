// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_1d_large() {
  return {
      make_cfg<1, 6, 3, TPAIR>(), make_cfg<1, 7, 3, TPAIR>(), make_cfg<1, 8, 3, TPAIR>(), make_cfg<1, 6, 5, TPAIR>(),
  };
}

}  // namespace wino
