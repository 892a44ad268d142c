// Instantiation helpers of the warp-tiled sweep kernel (sweep_v4.cuh,
// "variant 7": 2 columns per lane, 2r+1 input rows per TMA ring stage),
// included by kernels_v4_{5,9,17}.cu.
#pragma once

#include "kernels.h"
#include "sweep_v4.cuh"

namespace cjm {

template <int ST, int K, int NW>
KernelFn pick_mode_v4(int mode) {
  constexpr int RPS = 2 * Point<ST>::R + 1;
  switch (mode) {
    case MODE_HOT: return cjm_sweep_kernel_v4<ST, NW, K, 2, false, true, RPS>;
    case MODE_CHECK: return cjm_sweep_kernel_v4<ST, NW, K, 2, true, true, RPS>;
    default: return cjm_sweep_kernel_v4<ST, NW, 1, 2, true, false, RPS>;
  }
}

// K = 1..4 (5/9-point) or 1..3 (17-point: a fourth level of 5-row register
// rings does not fit the register file; the plan runs the shared-line kernel,
// variant 3, for a 17-point temporal_k = 4)
template <int ST, int NW>
KernelFn pick_k_v4(int K, int mode) {
  switch (K) {
    case 1: return pick_mode_v4<ST, 1, NW>(mode);
    case 2: return pick_mode_v4<ST, 2, NW>(mode);
    case 3: return pick_mode_v4<ST, 3, NW>(mode);
    default:
      if constexpr (Point<ST>::R == 2) return nullptr;
      else return pick_mode_v4<ST, 4, NW>(mode);
  }
}

// nw = consumer warps per CTA: 4, 5, 7, or 11 (one CTA per SM; 5/9-point at
// K = 4, plus its K = 1 remainder / residual launches)
template <int ST>
KernelFn pick_variant_v4(int K, int mode, int nw) {
  if constexpr (Point<ST>::R == 1) {
    if (nw == 11)
      return K == 4 ? pick_mode_v4<ST, 4, 11>(mode) : K == 1 ? pick_mode_v4<ST, 1, 11>(mode) : nullptr;
  }
  switch (nw) {
    case 4: return pick_k_v4<ST, 4>(K, mode);
    case 5: return pick_k_v4<ST, 5>(K, mode);
    case 7: return pick_k_v4<ST, 7>(K, mode);
    default: return nullptr;
  }
}

}  // namespace cjm
