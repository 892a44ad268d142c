// Warp-tiled sweep kernels of the 17-point stencil.
#include "kernels_v4.cuh"

namespace cjm {

KernelFn pick_sweep_v4_17(int K, int mode, int nw) { return pick_variant_v4<17>(K, mode, nw); }

}  // namespace cjm
