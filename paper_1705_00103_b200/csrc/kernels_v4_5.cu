// Warp-tiled sweep kernels of the 5-point stencil.
#include "kernels_v4.cuh"

namespace cjm {

KernelFn pick_sweep_v4_5(int variant, int K, int mode, int nw) {
#ifdef CJM_EXPERIMENT_9PT_V7
  if (5 != 9) return nullptr;
#endif
  return pick_variant_v4<5>(variant, K, mode, nw);
}

}  // namespace cjm
