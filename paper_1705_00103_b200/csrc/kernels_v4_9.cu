// Warp-tiled sweep kernels of the 9-point stencil.
#include "kernels_v4.cuh"

namespace cjm {

KernelFn pick_sweep_v4_9(int variant, int K, int mode, int nw) {
#ifdef CJM_EXPERIMENT_9PT_V7
  if (9 != 9) return nullptr;
#endif
  return pick_variant_v4<9>(variant, K, mode, nw);
}

}  // namespace cjm
