// Kernel instantiations for the sweep registry (see sweep_kernels.cuh); split across
// translation units so nvcc compiles them in parallel.  2D, n >= 9: one tile per thread,
// tiles and T2 staged in shared memory (a tile does not fit in registers).
#include "sweep_kernels.cuh"

namespace wino {

std::vector<SweepCfg> sweep_cfgs_2d_large() {
  return {
      make_cfg<2, 6, 5, TSINGLE>({make_variant<2, 6, 5, TSINGLE, kZ_N10_C1C2_R5>()}),
      make_cfg<2, 7, 3, TSINGLE>(),
      make_cfg<2, 8, 3, TSINGLE>({make_variant<2, 8, 3, TSINGLE, kZ_N10_C1C2>()}),
  };
}

}  // namespace wino
