// Instantiations of the shared-line sweep kernel (variant 3, sweep.cuh).
#include "kernels.h"

namespace cjm {
namespace {

template <int ST, int NT, int K>
KernelFn pick_mode(int mode) {
  switch (mode) {
    case MODE_HOT: return cjm_sweep_kernel<ST, NT, K, false, true>;
    case MODE_CHECK: return cjm_sweep_kernel<ST, NT, K, true, true>;
    default: return cjm_sweep_kernel<ST, NT, 1, true, false>;
  }
}

template <int ST, int NT>
KernelFn pick_k(int K, int mode) {
  switch (K) {
    case 1: return pick_mode<ST, NT, 1>(mode);
    case 2: return pick_mode<ST, NT, 2>(mode);
    case 3: return pick_mode<ST, NT, 3>(mode);
    default: return pick_mode<ST, NT, 4>(mode);
  }
}

template <int ST>
KernelFn pick_nt(int NT, int K, int mode) {
  return NT == 256 ? pick_k<ST, 256>(K, mode) : pick_k<ST, 128>(K, mode);
}

}  // namespace

KernelFn pick_sweep_v3(int stencil, int NT, int K, int mode) {
  switch (stencil) {
    case 5: return pick_nt<5>(NT, K, mode);
    case 9: return pick_nt<9>(NT, K, mode);
    default: return pick_nt<17>(NT, K, mode);
  }
}

}  // namespace cjm
