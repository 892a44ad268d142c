// Warp-tiled sweep kernels of the 17-point stencil.
#include "kernels_v4.cuh"

namespace cjm {

KernelFn pick_sweep_v4_17(int variant, int K, int mode, int nw) {
#ifdef CJM_EXPERIMENT_9PT_V7
  if (17 != 9) return nullptr;
#endif
  return pick_variant_v4<17>(variant, K, mode, nw);
}

}  // namespace cjm
