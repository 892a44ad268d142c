// sm_100a fp64 CJM sweep kernel.
//
// One sweep of u_{n+1} = u_n + w_n D^{-1}(b - A u_n) for the 5-,
// 9- or 17-point Laplacian, optionally fused
// with the residual reduction sum(d^2), max|d| of the INPUT iterate
// (d = D^{-1} r).
//
// Design:
//  * HBM-bound (24 B per lattice update: read u, read g, write u'), no tensor
//    cores -- this is not a contraction.
//  * Persistent grid: num_SMs x ctas_per_sm CTAs.  The interior is cut into
//    column strips of W columns; the (strip, row) pairs are split into equal
//    contiguous ranges, one per CTA, so every CTA streams the same number of
//    rows (no tail wave) and re-reads only 2r halo rows per range.
//  * One producer warp per CTA issues a 1-D TMA bulk copy
//    (cp.async.bulk ... mbarrier::complete_tx) per input row: the u row
//    segment [i0-2, i0+W+2) and the g row of the output row, into a ring of
//    `stages` shared-memory slots guarded by full/empty mbarriers.  W
//    consumer threads (one column each) read the newest row from shared
//    memory, keep the vertical window of centre values and horizontal pair
//    sums in registers (the association of DESIGN R6 makes each pair sum
//    computed once and reused for three output rows), and store the output
//    row coalesced.
//  * The sweep index n lives in device memory: every sweep kernel reads it,
//    picks w = w[n mod P] and the ping-pong buffers by the parity of n, and
//    the last CTA to finish (atomic ticket) advances it.  All sweep launches
//    therefore have identical parameters and a whole cycle is replayed from
//    a few CUDA graphs.  The last CTA also finishes the residual reduction in
//    a fixed order (deterministic, no floating-point atomics).
#pragma once

#include <cstdint>

#include "internal.h"

namespace cjm {

struct SweepParams {
  const double* buf0;          // iterate buffer read when n is even
  const double* buf1;          // iterate buffer read when n is odd
  const double* g;             // g = D^-1 b, interior rows, same pitch / PADL
  const double* w;             // weights in application order, P entries
  unsigned long long* ctr;     // sweep index n (device)
  unsigned int* ticket;        // CTA completion counter (device, 0 between sweeps)
  double* partials;            // 2 doubles per CTA (REDUCE)
  double* result;              // sum d^2, max |d| (REDUCE)
  long long P;                 // weights per cycle
  long long ld;                // pitch of every internal buffer, doubles
  long long units;             // nstrips * rows
  int nx;                      // interior columns
  int rows;                    // interior rows handled by this launch
  int row0;                    // first interior row of this launch
  int stages;                  // TMA ring depth
  int advance;                 // 1: last CTA advances *ctr
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).  Streaming data: L2 evict-first policy.
__device__ __forceinline__ void tma_row_load(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ double nan_max(double a, double b) {
  // max that propagates NaN (divergence must reach the host)
  return (b > a || b != b) ? b : a;
}

// ------------------------------------------------------- per-point arithmetic
// The fixed association of DESIGN R6; __dadd_rn / __fma_rn forbid any other
// contraction.  h1 = horizontal pair sum at distance 1 (uW + uE) of a row,
// h2 the same at distance 2; uc = centre values; index R = the output row.
template <int STENCIL>
struct Point;

template <>
struct Point<5> {
  static constexpr int R = 1;
  __device__ static __forceinline__ double jacobi_target(const double* uc, const double* h1,
                                                        const double*, double g) {
    const double S1 = __dadd_rn(h1[1], __dadd_rn(uc[0], uc[2]));
    return __fma_rn(0.25, S1, g);
  }
};

template <>
struct Point<9> {
  static constexpr int R = 1;
  __device__ static __forceinline__ double jacobi_target(const double* uc, const double* h1,
                                                        const double*, double g) {
    const double S1 = __dadd_rn(h1[1], __dadd_rn(uc[0], uc[2]));
    const double S2 = __dadd_rn(h1[0], h1[2]);
    return __fma_rn(0.2, S1, __fma_rn(0.05, S2, g));
  }
};

template <>
struct Point<17> {
  static constexpr int R = 2;
  __device__ static __forceinline__ double jacobi_target(const double* uc, const double* h1,
                                                        const double* h2, double g) {
    const double S1 = __dadd_rn(h1[2], __dadd_rn(uc[1], uc[3]));
    const double S2 = __dadd_rn(h2[2], __dadd_rn(uc[0], uc[4]));
    const double S3 = __dadd_rn(h1[1], h1[3]);
    const double S4 = __dadd_rn(h2[0], h2[4]);
    return __fma_rn(64.0 / 300.0, S1,
           __fma_rn(-4.0 / 300.0, S2,
           __fma_rn(16.0 / 300.0, S3,
           __fma_rn(-1.0 / 300.0, S4, g))));
  }
};

// ------------------------------------------------------------------- kernel
template <int STENCIL, int W, bool REDUCE, bool STORE>
__global__ void __launch_bounds__(W + 32)
cjm_sweep_kernel(const SweepParams p) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int UROW = W + 8;          // >= W + 4 columns, 64-byte multiple
  constexpr int NWARP = W / 32;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* su = reinterpret_cast<double*>(smem_raw);
  double* sg = su + (size_t)p.stages * UROW;
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + (size_t)p.stages * W);
  uint64_t* empty = full + p.stages;
  __shared__ double red_s[NWARP], red_m[NWARP];
  __shared__ int is_last;

  const int tid = threadIdx.x;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const unsigned long long n = __ldcg(p.ctr);
  const double* src = (n & 1ull) ? p.buf1 : p.buf0;
  double* dst = const_cast<double*>((n & 1ull) ? p.buf0 : p.buf1);
  const long long ld = p.ld;
  const long long u_begin = (long long)blockIdx.x * p.units / gridDim.x;
  const long long u_end = (long long)(blockIdx.x + 1) * p.units / gridDim.x;

  double acc_s = 0.0, acc_m = 0.0;

  if (tid >= W) {
    // ------------------------------------------------ producer warp (lane 0)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      long long used = 0;
      for (long long uu = u_begin; uu < u_end;) {
        const int strip = (int)(uu / p.rows);
        const int ja = (int)(uu - (long long)strip * p.rows) + p.row0;
        const long long seg_end = min(u_end, (long long)(strip + 1) * p.rows);
        const int jb = ja + (int)(seg_end - uu);
        const int i0 = strip * W;
        const int wc = min(W, p.nx - i0);
        const uint32_t ubytes = (uint32_t)(((wc + 4 + 1) & ~1) * 8);
        const uint32_t gbytes = (uint32_t)(((wc + 1) & ~1) * 8);
        const int nin = jb - ja + 2 * R;
        for (int k = 0; k < nin; ++k) {
          if (used >= p.stages) mbar_wait(&empty[stage], phase ^ 1u);
          const int row = ja - R + k;                 // interior row of the u row
          const bool hasg = k >= 2 * R;
          mbar_arrive_expect_tx(&full[stage], ubytes + (hasg ? gbytes : 0u));
          tma_row_load(su + (size_t)stage * UROW,
                       src + (long long)(row + R) * ld + (PADL - 2) + i0, ubytes,
                       &full[stage], pol);
          if (hasg)
            tma_row_load(sg + (size_t)stage * W,
                         p.g + (long long)(row - R) * ld + PADL + i0, gbytes,
                         &full[stage], pol);
          ++used;
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
        }
        uu = seg_end;
      }
    }
  } else {
    // ---------------------------------------------- consumer threads (W)
    const double w = __ldg(p.w + (long long)(n % (unsigned long long)p.P));
    int stage = 0;
    uint32_t phase = 0;
    for (long long uu = u_begin; uu < u_end;) {
      const int strip = (int)(uu / p.rows);
      const int ja = (int)(uu - (long long)strip * p.rows) + p.row0;
      const long long seg_end = min(u_end, (long long)(strip + 1) * p.rows);
      const int jb = ja + (int)(seg_end - uu);
      const int i = strip * W + tid;
      const bool active = i < p.nx;
      const int nin = jb - ja + 2 * R;
      double uc[2 * R + 1], h1[2 * R + 1], h2[2 * R + 1];
#pragma unroll
      for (int q = 0; q < 2 * R + 1; ++q) { uc[q] = 0.0; h1[q] = 0.0; h2[q] = 0.0; }
      double* out = dst + (long long)(ja + R) * ld + PADL + i;
      for (int k = 0; k < nin; ++k) {
        mbar_wait(&full[stage], phase);
        const double* rp = su + (size_t)stage * UROW + 2 + tid;   // column i
        const double c = rp[0];
        const double e1 = __dadd_rn(rp[-1], rp[1]);
        double e2 = 0.0;
        if (R == 2) e2 = __dadd_rn(rp[-2], rp[2]);
        double gv = 0.0;
        if (k >= 2 * R) gv = sg[(size_t)stage * W + tid];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
#pragma unroll
        for (int q = 0; q < 2 * R; ++q) { uc[q] = uc[q + 1]; h1[q] = h1[q + 1]; h2[q] = h2[q + 1]; }
        uc[2 * R] = c; h1[2 * R] = e1; h2[2 * R] = e2;
        if (k >= 2 * R) {
          const double J = Point<STENCIL>::jacobi_target(uc, h1, h2, gv);
          const double d = __dsub_rn(J, uc[R]);
          if (active) {
            if (STORE) *out = __fma_rn(w, d, uc[R]);
            if (REDUCE) { acc_s = __fma_rn(d, d, acc_s); acc_m = nan_max(acc_m, fabs(d)); }
          }
          out += ld;
        }
        if (++stage == p.stages) { stage = 0; phase ^= 1u; }
      }
      uu = seg_end;
    }
  }

  if (REDUCE) {
    if (tid < W) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc_s = __dadd_rn(acc_s, __shfl_xor_sync(0xffffffffu, acc_s, o));
        acc_m = nan_max(acc_m, __shfl_xor_sync(0xffffffffu, acc_m, o));
      }
      if (lane == 0) { red_s[tid >> 5] = acc_s; red_m[tid >> 5] = acc_m; }
    }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0, m = 0.0;
      for (int q = 0; q < NWARP; ++q) { s = __dadd_rn(s, red_s[q]); m = nan_max(m, red_m[q]); }
      p.partials[2 * blockIdx.x] = s;
      p.partials[2 * blockIdx.x + 1] = m;
    }
  }

  // ---- completion ticket: the last CTA finishes the reduction and advances n
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(p.ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (REDUCE) {
      double s = 0.0, m = 0.0;
      if (tid < W) {
        for (int b = tid; b < (int)gridDim.x; b += W) {
          s = __dadd_rn(s, __ldcg(p.partials + 2 * b));
          m = nan_max(m, __ldcg(p.partials + 2 * b + 1));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
          m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
        }
        if (lane == 0) { red_s[tid >> 5] = s; red_m[tid >> 5] = m; }
      }
      __syncthreads();
      if (tid == 0) {
        s = 0.0; m = 0.0;
        for (int q = 0; q < NWARP; ++q) { s = __dadd_rn(s, red_s[q]); m = nan_max(m, red_m[q]); }
        p.result[0] = s;
        p.result[1] = m;
      }
    }
    if (tid == 0) {
      if (p.advance) *p.ctr = n + 1ull;
      *p.ticket = 0u;
      __threadfence();
    }
  }
}

// g = gscale * b in place on the interior of the internal g buffer (row a5).
__global__ void cjm_scale_kernel(double* g, long long ld, int nx, int rows, double gscale) {
  const long long total = (long long)nx * rows;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / nx, i = e - j * nx;
    double* q = g + j * ld + PADL + i;
    *q = __dmul_rn(gscale, *q);
  }
}

}  // namespace cjm
