// Warp-tiled sweep kernels of the 5-point stencil.
#include "kernels_v4.cuh"

namespace cjm {

KernelFn pick_sweep_v4_5(int K, int mode, int nw) { return pick_variant_v4<5>(K, mode, nw); }

}  // namespace cjm
