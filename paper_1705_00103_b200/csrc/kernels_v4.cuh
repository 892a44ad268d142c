// Instantiation helpers of the warp-tiled sweep kernels (sweep_v4.cuh),
// included by kernels_v4_{5,9,17}.cu.
#pragma once

#include "kernels.h"
#include "sweep_v4.cuh"

namespace cjm {

// warp-tiled kernel (sweep_v4.cuh): NW consumer warps, C columns per lane,
// RPS input rows per TMA ring stage
template <int ST, int K, int C, int RPS, int NW = 4>
KernelFn pick_mode_v4(int mode) {
  switch (mode) {
    case MODE_HOT: return cjm_sweep_kernel_v4<ST, NW, K, C, false, true, RPS>;
    case MODE_CHECK: return cjm_sweep_kernel_v4<ST, NW, K, C, true, true, RPS>;
    default: return cjm_sweep_kernel_v4<ST, NW, 1, C, true, false, RPS>;
  }
}

// the 17-point warp-tiled kernel with 4 columns per lane and K >= 2 does not
// fit the register file (5-row rings of 4 columns x 3 arrays per level), nor
// with 2 columns beyond K = 2 (one row per stage) / K = 3 (2r+1 rows per
// stage, 255 registers): not instantiated, the plan uses the shared-line
// variant there
template <int ST, int C, int RPS, int NW = 4>
KernelFn pick_k_v4(int K, int mode) {
  if constexpr (ST == 17 && C == 4) {
    return K == 1 ? pick_mode_v4<ST, 1, C, RPS, NW>(mode) : nullptr;
  } else if constexpr (ST == 17 && RPS > 1) {   // variant 7: up to K = 3
    return K == 1 ? pick_mode_v4<ST, 1, C, RPS, NW>(mode)
           : K == 2 ? pick_mode_v4<ST, 2, C, RPS, NW>(mode)
           : K == 3 ? pick_mode_v4<ST, 3, C, RPS, NW>(mode) : nullptr;
  } else if constexpr (ST == 17) {
    return K == 1 ? pick_mode_v4<ST, 1, C, RPS, NW>(mode)
                  : K == 2 ? pick_mode_v4<ST, 2, C, RPS, NW>(mode) : nullptr;
  } else {
    switch (K) {
      case 1: return pick_mode_v4<ST, 1, C, RPS, NW>(mode);
      case 2: return pick_mode_v4<ST, 2, C, RPS, NW>(mode);
      case 3: return pick_mode_v4<ST, 3, C, RPS, NW>(mode);
      default: return pick_mode_v4<ST, 4, C, RPS, NW>(mode);
    }
  }
}

// variant -> (columns per lane, rows per stage), nw -> consumer warps
template <int ST>
KernelFn pick_variant_v4(int variant, int K, int mode, int nw) {
  constexpr int RPS = 2 * Point<ST>::R + 1;
#ifdef CJM_EXPERIMENT_9PT_V7
  if (ST != 9 || variant != 7) return nullptr;
#else
  switch (variant) {      // 4 / 2 columns per lane, 1 / 2r+1 rows per stage
    case 4: return pick_k_v4<ST, 4, 1>(K, mode);
    case 5: return pick_k_v4<ST, 2, 1>(K, mode);
    case 6: return pick_k_v4<ST, 4, RPS>(K, mode);
    default: break;
  }
#endif
  if constexpr (Point<ST>::R == 1) {   // one CTA of 11 consumer warps per SM (K = 4)
    if (nw == 11)   // K = 4, and K = 1 for remainder sweeps and residuals
      return K == 4 ? pick_mode_v4<ST, 4, 2, RPS, 11>(mode)
           : K == 1 ? pick_mode_v4<ST, 1, 2, RPS, 11>(mode) : nullptr;
  }
  return nw == 5 ? pick_k_v4<ST, 2, RPS, 5>(K, mode)
       : nw == 7 ? pick_k_v4<ST, 2, RPS, 7>(K, mode) : pick_k_v4<ST, 2, RPS, 4>(K, mode);
}

}  // namespace cjm
