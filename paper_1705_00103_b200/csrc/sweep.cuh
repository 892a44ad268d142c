// sm_100a fp64 CJM sweep kernel (NEXT-1).
//
// One launch applies K consecutive sweeps of u_{n+1} = u_n + w_n D^{-1}(b - A u_n)
// for the 5-, 9- or 17-point Laplacian (P:95-99, P:118-125,
// P:342-349), each sweep with its own weight w_{n+l} ("strictly
// different weights at each iteration"), optionally fused with the residual
// reduction sum(d^2), max|d| of the INPUT iterate (d = D^{-1} r).
//
// Design:
//  * HBM-bound (24 B per lattice update per launch: read u, read g, write u'),
//    no tensor cores -- this is not a contraction.  K > 1 (temporal blocking)
//    keeps the K-1 intermediate iterates on chip, so a launch moves 24 B per
//    node for K lattice updates.
//  * Persistent grid: num_SMs x ctas_per_sm CTAs.  The interior is cut into
//    column strips of TOUT = 2*NT - 2E owned columns (E = halo lost by the
//    K-1 on-chip levels, rounded to keep 16-byte alignment); the
//    (strip, row) pairs are split into equal contiguous ranges, one per CTA,
//    so every CTA streams the same number of rows (no tail wave).
//  * One producer warp issues a 1-D TMA bulk copy (cp.async.bulk ...
//    mbarrier::complete_tx) per input row: the u row segment of the tile plus
//    2 halo columns each side, and the g row of the level-1 output row, into a
//    ring of `stages` shared-memory slots guarded by full/empty mbarriers.
//  * NT consumer threads own 2 adjacent columns each (LDS.128 / STG.128).
//    Per level they keep the vertical window of centre values and horizontal
//    pair sums in registers (the association of DESIGN R6 computes each pair
//    sum once and reuses it for 2r+1 output rows).  A level's output row is
//    handed to the next level through a double-buffered shared-memory line;
//    one named barrier per row serves all levels (levels are skewed by one
//    row-step each).  Ghost nodes are pass-through at every level.
//  * The sweep index n and the current buffer live in device memory: every
//    launch reads them, takes w[(n+l) mod P], reads buffer `cur` and writes
//    buffer cur^1; the last CTA to finish (atomic ticket) advances n by K and
//    flips cur.  All launches of a plan therefore have identical parameters
//    and the hot loop is replayed from CUDA graphs.  The last CTA also
//    finishes the residual reduction in a fixed order (deterministic, no
//    floating-point atomics).
#pragma once

#include <cstdint>

#include "internal.h"

namespace cjm {

struct SweepState {
  unsigned long long n;        // global sweep index of the input iterate
  unsigned int cur;            // buffer holding the input iterate
  unsigned int ticket;         // CTA completion counter (0 between launches)
};

struct SweepParams {
  double* buf[2];              // iterate buffers (ghost rings included)
  const double* g;             // g = D^-1 b, interior rows, same pitch / PADL
  const double* w;             // weights in application order, P entries
  SweepState* state;           // device-resident n / cur / ticket
  double* partials;            // 2 doubles per CTA (REDUCE)
  double* result;              // sum d^2, max |d| (REDUCE)
  long long P;                 // weights per cycle
  long long ld;                // pitch of every internal buffer, doubles
  long long units;             // nstrips * rows
  int nx;                      // interior columns
  int rows;                    // interior rows of this (slab) buffer
  int stages;                  // TMA ring depth
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

// named barrier for the NT consumer threads only (the producer warp never joins)
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ double nan_max(double a, double b) {
  // max that propagates NaN (divergence must reach the host)
  return (b > a || b != b) ? b : a;
}

// ------------------------------------------------------- per-point arithmetic
// The fixed association of DESIGN R6; __dadd_rn / __fma_rn forbid any other
// contraction.  Window index R is the output row; uc = centre values, h1 =
// horizontal pair sums at distance 1 (uW + uE), h2 at distance 2.
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

// Per-level register window of one thread (its 2 columns a, b).
template <int R>
struct Window {
  double ua[2 * R + 1], ub[2 * R + 1];
  double h1a[2 * R + 1], h1b[2 * R + 1];
  double h2a[2 * R + 1], h2b[2 * R + 1];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int q = 0; q < 2 * R + 1; ++q) ua[q] = ub[q] = h1a[q] = h1b[q] = h2a[q] = h2b[q] = 0.0;
  }
  // Push the newest row: centre values ca, cb and neighbours l2, l1 (columns
  // a-2, a-1) and r1, r2 (columns b+1, b+2).  Pair sums are (west + east).
  __device__ __forceinline__ void push(double ca, double cb, double l2, double l1, double r1,
                                       double r2) {
#pragma unroll
    for (int q = 0; q < 2 * R; ++q) {
      ua[q] = ua[q + 1]; ub[q] = ub[q + 1];
      h1a[q] = h1a[q + 1]; h1b[q] = h1b[q + 1];
      if (R == 2) { h2a[q] = h2a[q + 1]; h2b[q] = h2b[q + 1]; }
    }
    ua[2 * R] = ca; ub[2 * R] = cb;
    h1a[2 * R] = __dadd_rn(l1, cb);     // u(a-1) + u(a+1)
    h1b[2 * R] = __dadd_rn(ca, r1);     // u(b-1) + u(b+1)
    if (R == 2) {
      h2a[2 * R] = __dadd_rn(l2, r1);   // u(a-2) + u(a+2)
      h2b[2 * R] = __dadd_rn(l1, r2);   // u(b-2) + u(b+2)
    }
  }
};

// Read centre (ca, cb) and neighbours of thread t's columns from a shared row
// whose index 0 is column c0 - 2 (thread t's columns at 2t+2, 2t+3).
template <int R>
__device__ __forceinline__ void read_row(const double* row, int t, double& ca, double& cb,
                                         double& l2, double& l1, double& r1, double& r2) {
  const double2 c = *reinterpret_cast<const double2*>(row + 2 * t + 2);
  ca = c.x; cb = c.y;
  if (R == 2) {
    const double2 lft = *reinterpret_cast<const double2*>(row + 2 * t);
    const double2 rgt = *reinterpret_cast<const double2*>(row + 2 * t + 4);
    l2 = lft.x; l1 = lft.y; r1 = rgt.x; r2 = rgt.y;
  } else {
    l2 = 0.0; r2 = 0.0;
    l1 = row[2 * t + 1];
    r1 = row[2 * t + 4];
  }
}

template <int R>
__device__ __forceinline__ void read_nbrs(const double* row, int t, double& l2, double& l1,
                                          double& r1, double& r2) {
  if (R == 2) {
    const double2 lft = *reinterpret_cast<const double2*>(row + 2 * t);
    const double2 rgt = *reinterpret_cast<const double2*>(row + 2 * t + 4);
    l2 = lft.x; l1 = lft.y; r1 = rgt.x; r2 = rgt.y;
  } else {
    l2 = 0.0; r2 = 0.0;
    l1 = row[2 * t + 1];
    r1 = row[2 * t + 4];
  }
}

template <int R, int K>
struct TileGeom {
  // columns lost per side by the K-1 on-chip levels, rounded up to even so
  // that tile origins stay 16-byte aligned
  static constexpr int E = (K == 1) ? 0 : ((R * (K - 1) + 1) & ~1);
};

// ------------------------------------------------------------------- kernel
template <int STENCIL, int NT, int K, bool REDUCE, bool STORE>
__global__ void __launch_bounds__(NT + 32)
cjm_sweep_kernel(const SweepParams p) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int T = 2 * NT;                 // tile columns (every level)
  constexpr int E = TileGeom<R, K>::E;
  constexpr int TOUT = T - 2 * E;           // owned output columns per strip
  constexpr int ROW = T + 8;                // shared row stride, >= T + 4
  constexpr int NWARP = NT / 32;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* su = reinterpret_cast<double*>(smem_raw);
  double* sg = su + (size_t)p.stages * ROW;
  double* lb = sg + (size_t)p.stages * T;                       // (K-1) x 2 rows
  uint64_t* full = reinterpret_cast<uint64_t*>(lb + (size_t)(K - 1) * 2 * ROW);
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
  if (K > 1)
    for (int e = tid; e < (K - 1) * 2 * ROW; e += blockDim.x) lb[e] = 0.0;
  __syncthreads();

  const unsigned long long n = __ldcg(&p.state->n);
  const unsigned int cur = __ldcg(&p.state->cur);
  // select, not p.buf[cur]: a dynamic index would copy the parameters to local memory
  const double* src = (cur & 1u) ? p.buf[1] : p.buf[0];
  double* dst = (cur & 1u) ? p.buf[0] : p.buf[1];
  const long long ld = p.ld;
  const int rows = p.rows;
  const long long u_begin = (long long)blockIdx.x * p.units / gridDim.x;
  const long long u_end = (long long)(blockIdx.x + 1) * p.units / gridDim.x;

  double acc_s = 0.0, acc_m = 0.0;

  if (tid >= NT) {
    // ------------------------------------------------ producer warp (lane 0)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      long long used = 0;
      for (long long uu = u_begin; uu < u_end;) {
        const int strip = (int)(uu / rows);
        const int ja = (int)(uu - (long long)strip * rows);
        const long long seg_end = min(u_end, (long long)(strip + 1) * rows);
        const int jb = ja + (int)(seg_end - uu);
        const int c0 = strip * TOUT - E;
        // u columns [c0-2, min(c0+T+2, nx+R+2)), g columns [c0, min(c0+T, nx))
        const int ucols = min(T + 4, p.nx + R + 2 - c0);
        const uint32_t ubytes = (uint32_t)(((ucols + 1) & ~1) * 8);
        const int gc0 = max(c0, 0);
        const int gcols = min(c0 + T, p.nx) - gc0;
        const uint32_t gbytes = gcols > 0 ? (uint32_t)(((gcols + 1) & ~1) * 8) : 0u;
        const int nin = jb - ja + 2 * K * R;
        for (int k = 0; k < nin; ++k) {
          if (used >= p.stages) mbar_wait(&empty[stage], phase ^ 1u);
          const int gin = ja - K * R + k;          // global row of the u row
          const bool hasu = gin >= -R && gin < rows + R;
          const int g1 = gin - R;                   // level-1 output row
          const bool hasg = k >= 2 * R && g1 >= 0 && g1 < rows && gbytes;
          mbar_arrive_expect_tx(&full[stage], (hasu ? ubytes : 0u) + (hasg ? gbytes : 0u));
          if (hasu)
            tma_row_load(su + (size_t)stage * ROW,
                         src + (long long)(gin + R) * ld + (PADL - 2) + c0, ubytes,
                         &full[stage], pol);
          if (hasg)
            tma_row_load(sg + (size_t)stage * T + (gc0 - c0),
                         p.g + (long long)g1 * ld + PADL + gc0, gbytes, &full[stage], pol);
          ++used;
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
        }
        uu = seg_end;
      }
    }
  } else {
    // ---------------------------------------------- consumer threads (NT)
    double wl[K];
#pragma unroll
    for (int l = 0; l < K; ++l) wl[l] = __ldg(p.w + (long long)((n + l) % (unsigned long long)p.P));
    int stage = 0;
    uint32_t phase = 0;
    Window<R> win[K];
    double gf[K][R + 1][2];   // g handed from level l-1 to level l, delayed R+1 steps
    for (long long uu = u_begin; uu < u_end;) {
      const int strip = (int)(uu / rows);
      const int ja = (int)(uu - (long long)strip * rows);
      const long long seg_end = min(u_end, (long long)(strip + 1) * rows);
      const int jb = ja + (int)(seg_end - uu);
      const int c0 = strip * TOUT - E;
      const int ca = c0 + 2 * tid, cb = ca + 1;
      const bool ina = ca >= 0 && ca < p.nx, inb = cb >= 0 && cb < p.nx;
      const bool owna = ina && ca >= c0 + E && ca < c0 + T - E;
      const bool ownb = inb && cb >= c0 + E && cb < c0 + T - E;
      const int nin = jb - ja + 2 * K * R;
      const int nsteps = nin + K - 1;
#pragma unroll
      for (int l = 0; l < K; ++l) {
        win[l].clear();
#pragma unroll
        for (int q = 0; q <= R; ++q) { gf[l][q][0] = 0.0; gf[l][q][1] = 0.0; }
      }
      for (int k = 0; k < nsteps; ++k) {
        // ---- level 1 input: the TMA row
        double g1a = 0.0, g1b = 0.0;
        if (k < nin) {
          mbar_wait(&full[stage], phase);
          double ca_, cb_, l2, l1, r1, r2;
          read_row<R>(su + (size_t)stage * ROW, tid, ca_, cb_, l2, l1, r1, r2);
          if (k >= 2 * R) {
            const double2 gv = *reinterpret_cast<const double2*>(sg + (size_t)stage * T + 2 * tid);
            g1a = gv.x; g1b = gv.y;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
          win[0].push(ca_, cb_, l2, l1, r1, r2);
        }
        // ---- levels 2..K input: previous step's output line of level l-1
#pragma unroll
        for (int l = 1; l < K; ++l) {
          // level l-1 (0-based) produced a row at step k-1 ?
          const int lo = 2 * l * R + l - 1;        // first active step of level l-1 (0-based l-1)
          if (k - 1 >= lo && k - 1 < nin + l - 1) {
            const double* row = lb + (size_t)((l - 1) * 2 + ((k - 1) & 1)) * ROW;
            double l2, l1, r1, r2;
            read_nbrs<R>(row, tid, l2, l1, r1, r2);
            // own centre values: what this thread wrote at step k-1
            const double2 c = *reinterpret_cast<const double2*>(row + 2 * tid + 2);
            win[l].push(c.x, c.y, l2, l1, r1, r2);
          }
        }
        // ---- compute every active level
        double gcur[K][2];
#pragma unroll
        for (int l = 0; l < K; ++l) {
          // g of this level's row: level 0 from the TMA slot, level l from the
          // FIFO fed by level l-1 (R+1 steps earlier)
          const double ga = (l == 0) ? g1a : gf[l][R][0];
          const double gb = (l == 0) ? g1b : gf[l][R][1];
          gcur[l][0] = ga;
          gcur[l][1] = gb;
          const int first = 2 * (l + 1) * R + l;   // first active step of level l (0-based)
          if (k >= first && k < nin + l) {
            const int q = k - (l + 1) * R - l;      // segment row index of the output
            const int G = ja - K * R + q;           // global row
            const bool rowin = G >= 0 && G < rows;
            const Window<R>& wv = win[l];
            const double Ja = Point<STENCIL>::jacobi_target(wv.ua, wv.h1a, wv.h2a, ga);
            const double Jb = Point<STENCIL>::jacobi_target(wv.ub, wv.h1b, wv.h2b, gb);
            const double da = __dsub_rn(Ja, wv.ua[R]);
            const double db = __dsub_rn(Jb, wv.ub[R]);
            const double oa = (rowin && ina) ? __fma_rn(wl[l], da, wv.ua[R]) : wv.ua[R];
            const double ob = (rowin && inb) ? __fma_rn(wl[l], db, wv.ub[R]) : wv.ub[R];
            if (REDUCE && l == 0 && G >= ja && G < jb) {
              if (owna) { acc_s = __fma_rn(da, da, acc_s); acc_m = nan_max(acc_m, fabs(da)); }
              if (ownb) { acc_s = __fma_rn(db, db, acc_s); acc_m = nan_max(acc_m, fabs(db)); }
            }
            if (l < K - 1) {
              double* row = lb + (size_t)(l * 2 + (k & 1)) * ROW;
              *reinterpret_cast<double2*>(row + 2 * tid + 2) = make_double2(oa, ob);
            } else if (STORE) {
              double* o = dst + (long long)(G + R) * ld + PADL + ca;
              if (owna && ownb) *reinterpret_cast<double2*>(o) = make_double2(oa, ob);
              else if (owna) o[0] = oa;
              else if (ownb) o[1] = ob;
            }
          }
        }
        // feed the g FIFOs (every step, so FIFO positions count steps):
        // level l reads gf[l][R] = level l-1's g from step k-1-R
#pragma unroll
        for (int l = 1; l < K; ++l) {
#pragma unroll
          for (int q = R; q > 0; --q) { gf[l][q][0] = gf[l][q - 1][0]; gf[l][q][1] = gf[l][q - 1][1]; }
          gf[l][0][0] = gcur[l - 1][0];
          gf[l][0][1] = gcur[l - 1][1];
        }
        if (K > 1) consumer_bar(NT);
      }
      uu = seg_end;
    }
  }

  if (REDUCE) {
    if (tid < NT) {
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
    const unsigned int t = atomicAdd(&p.state->ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (REDUCE) {
      double s = 0.0, m = 0.0;
      if (tid < NT) {
        for (int b = tid; b < (int)gridDim.x; b += NT) {
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
      if (STORE) {
        p.state->n = n + (unsigned long long)K;
        p.state->cur = cur ^ 1u;
      }
      p.state->ticket = 0u;
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
