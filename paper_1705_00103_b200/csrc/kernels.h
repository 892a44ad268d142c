// Sweep-kernel selection (internal).  The template instantiations of the
// sweep kernels are spread over kernels_*.cu so that the library compiles in
// parallel; each returns the kernel for (variant, K, mode, warps) or nullptr
// when that combination is not instantiated.
#pragma once

#include "sweep.cuh"

namespace cjm {

enum Mode { MODE_HOT = 0, MODE_CHECK = 1, MODE_RESID = 2 };

using KernelFn = void (*)(const SweepParams);

// shared-line kernel (variant 3, sweep.cuh), NT = 128 or 256 threads
KernelFn pick_sweep_v3(int stencil, int NT, int K, int mode);
// warp-tiled kernel (variant 7, sweep_v4.cuh), one file per stencil; nw =
// consumer warps per CTA
KernelFn pick_sweep_v4_5(int K, int mode, int nw);
KernelFn pick_sweep_v4_9(int K, int mode, int nw);
KernelFn pick_sweep_v4_17(int K, int mode, int nw);

}  // namespace cjm
