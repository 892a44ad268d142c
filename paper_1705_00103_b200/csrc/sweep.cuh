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
  unsigned int next_chunk;     // dynamic work counter of the warp-tiled kernel (0 between launches)
  unsigned int pad_;
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
  long long units;             // nstrips * nrows
  int nx;                      // interior columns
  int rows;                    // interior rows of this (slab) buffer
  int H;                       // ghost rows stored above / below the slab (buf and g)
  int row_lo, row_hi;          // local rows that are interior in the GLOBAL grid
                               // (others are Dirichlet ghosts: pass-through)
  int row0, nrows;             // the band of output rows of this launch
  int stages;                  // TMA ring depth
  int advance;                 // the last CTA advances n / flips cur (last launch of a sweep)
  int chunk_rows;              // warp-tiled kernel: 0 = one contiguous range of (strip, row)
                               // units per CTA; > 0 = units [0, units_static) in static
                               // per-CTA ranges, the rest in chunk_rows-unit work items taken
                               // from a device counter (dynamic balancing)
  long long units_static;
  // bounds of the buffers (CJM_DEBUG_CHECKS builds check every TMA copy, ring
  // read and store against them and count violations in dbg[0], the first
  // violation's code in dbg[1]; dbg is NULL in product builds)
  long long buf_elems;         // doubles per iterate / g buffer
  unsigned long long* dbg;
};

// Device-side bounds checks of the CJM_DEBUG_CHECKS build (compute-sanitizer
// is closed on this GPU pool): a violated condition is counted, never
// trapped, and the library turns a non-zero count into CJM_ERR_CUDA.
#ifdef CJM_DEBUG_CHECKS
#define CJM_CHECK(p, cond, code)                                                  \
  do {                                                                            \
    if (!(cond) && (p).dbg) {                                                     \
      atomicAdd((p).dbg, 1ull);                                                   \
      atomicCAS((p).dbg + 1, 0ull, (unsigned long long)(code));                   \
    }                                                                             \
  } while (0)
#else
#define CJM_CHECK(p, cond, code) \
  do {                           \
  } while (0)
#endif
enum CheckCode {
  CHK_TMA_U = 1,       // TMA u row source outside the iterate buffer
  CHK_TMA_G = 2,       // TMA g row source outside the g buffer
  CHK_TMA_DST = 3,     // TMA destination outside the ring
  CHK_TMA_ALIGN = 4,   // TMA address / size not 16-byte aligned
  CHK_STORE = 5,       // store outside the interior of the output buffer
  CHK_RING_READ = 6,   // consumer ring read outside the ring
  CHK_TX = 7,          // expected transaction bytes above one stage
  CHK_DESC = 8         // segment descriptor outside the launch's band
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

__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  // the retry loop lives inside the asm block: no C-level divergent loop, so
  // the compiler emits no convergence barrier around it
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "CJM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CJM_WAIT_%=;\n\t}"
      ::"r"(a), "r"(parity) : "memory");
}

// Order this thread's generic-proxy reads of a ring slot before the async-proxy
// (TMA) writes that will refill it once the slot is released (cross-proxy WAR).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
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
// The a_k = -c_k/c_C live in the constant bank so DFMA reads them directly
// (the same doubles as the literals of DESIGN R6).
__constant__ double c_coef[7] = {0.25, 0.2, 0.05, 64.0 / 300.0, -4.0 / 300.0, 16.0 / 300.0,
                                 -1.0 / 300.0};

template <int STENCIL>
struct Point;

template <>
struct Point<5> {
  static constexpr int R = 1;
  __device__ static __forceinline__ double jacobi_target(const double* uc, const double* h1,
                                                        const double*, double g) {
    const double S1 = __dadd_rn(h1[1], __dadd_rn(uc[0], uc[2]));
    return __fma_rn(c_coef[0], S1, g);
  }
};

template <>
struct Point<9> {
  static constexpr int R = 1;
  __device__ static __forceinline__ double jacobi_target(const double* uc, const double* h1,
                                                        const double*, double g) {
    const double S1 = __dadd_rn(h1[1], __dadd_rn(uc[0], uc[2]));
    const double S2 = __dadd_rn(h1[0], h1[2]);
    return __fma_rn(c_coef[1], S1, __fma_rn(c_coef[2], S2, g));
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
    return __fma_rn(c_coef[3], S1,
           __fma_rn(c_coef[4], S2,
           __fma_rn(c_coef[5], S3,
           __fma_rn(c_coef[6], S4, g))));
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


// Register state of one consumer thread, carried across the segments of a CTA.
template <int R, int K>
struct ConsumerState {
  static constexpr int P = 2 * R + 1;
  // level l (0-based; applies sweep n+l): the last P rows of level l-1 values
  // (level 0: the input iterate) for the thread's columns a, b, in a ring of
  // P slots (the row pushed at step kk sits in slot kk mod P), and the g of
  // level l-1 pushed at step kk (used R+1 steps later by level l)
  double ua[K][P], ub[K][P], h1a[K][P], h1b[K][P], h2a[K][P], h2b[K][P];
  double gra[K][P], grb[K][P];
  double wl[K];
  int stage;
  uint32_t phase;
  uint32_t full_a, empty_a;   // shared addresses of the mbarrier arrays
  __device__ __forceinline__ void init(const SweepParams& p, unsigned long long n, uint64_t* full,
                                       uint64_t* empty) {
#pragma unroll
    for (int l = 0; l < K; ++l) {
      wl[l] = __ldg(p.w + (long long)((n + l) % (unsigned long long)p.P));
#pragma unroll
      for (int q = 0; q < P; ++q) {
        ua[l][q] = ub[l][q] = h1a[l][q] = h1b[l][q] = h2a[l][q] = h2b[l][q] = 0.0;
        gra[l][q] = grb[l][q] = 0.0;
      }
    }
    stage = 0;
    phase = 0;
    full_a = smem_addr(full);
    empty_a = smem_addr(empty);
  }
};

// One segment (rows [ja, jb) of the strip whose tile starts at column c0) of
// the consumer loop.  The step loop is unrolled by P = 2R+1 so every ring
// slot index is a compile-time constant (no register moves for the sliding
// windows).  Levels are skewed by one step each: level l reads the line
// level l-1 wrote at the previous step, so one named barrier per step serves
// all levels.
template <int STENCIL, int NT, int K, bool REDUCE, bool STORE, bool FAST>
__device__ __forceinline__ void consumer_segment(ConsumerState<Point<STENCIL>::R, K>& cs,
                                                 const SweepParams& p, const double* su,
                                                 const double* sg, double* lb, double* dst,
                                                 int ja, int jb, int c0, int tid, int lane,
                                                 double& acc_s, double& acc_m) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int P = 2 * R + 1;
  constexpr int T = 2 * NT;
  constexpr int E = TileGeom<R, K>::E;
  constexpr int ROW = T + 8;
  const long long ld = p.ld;
      const int ca = c0 + 2 * tid, cb = ca + 1;
      const bool ina = ca >= 0 && ca < p.nx, inb = cb >= 0 && cb < p.nx;
      const bool owna = ina && ca >= c0 + E && ca < c0 + T - E;
      const bool ownb = inb && cb >= c0 + E && cb < c0 + T - E;
      const int nin = jb - ja + 2 * K * R;
      const int nsteps = nin + K - 1;
      const int row_base = ja - K * R;               // global row of input step 0
      double* outp = dst + (long long)(ja + p.H) * ld + PADL + ca;
      for (int k0 = 0; k0 < nsteps; k0 += P) {
#pragma unroll
        for (int ph = 0; ph < P; ++ph) {
          const int kk = k0 + ph;
          if (kk < nsteps) {
            // ---- level 0 input: the TMA row of step kk (slot ph)
            double g0a = 0.0, g0b = 0.0;
            if (kk < nin) {
              mbar_wait_a(cs.full_a + 8u * cs.stage, cs.phase);
              double c_a, c_b, l2, l1, r1, r2;
              read_row<R>(su + (size_t)cs.stage * ROW, tid, c_a, c_b, l2, l1, r1, r2);
              if (kk >= 2 * R) {
                const double2 gv = *reinterpret_cast<const double2*>(sg + (size_t)cs.stage * T + 2 * tid);
                g0a = gv.x;
                g0b = gv.y;
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) mbar_arrive_a(cs.empty_a + 8u * cs.stage);
              if (++cs.stage == p.stages) { cs.stage = 0; cs.phase ^= 1u; }
              cs.ua[0][ph] = c_a;
              cs.ub[0][ph] = c_b;
              cs.h1a[0][ph] = __dadd_rn(l1, c_b);      // u(a-1) + u(a+1)
              cs.h1b[0][ph] = __dadd_rn(c_a, r1);      // u(b-1) + u(b+1)
              if (R == 2) {
                cs.h2a[0][ph] = __dadd_rn(l2, r1);     // u(a-2) + u(a+2)
                cs.h2b[0][ph] = __dadd_rn(l1, r2);     // u(b-2) + u(b+2)
              }
            }
            // ---- levels 1..K-1 input: level l-1's line of step kk-1
#pragma unroll
            for (int l = 1; l < K; ++l) {
              const int lo = 2 * l * R + l - 1;     // first active step of level l-1
              if (kk - 1 >= lo && kk - 1 < nin + l - 1) {
                const double* row = lb + (size_t)((l - 1) * P + (ph + P - 1) % P) * ROW;
                double l2, l1, r1, r2;
                read_nbrs<R>(row, tid, l2, l1, r1, r2);
                const double2 c = *reinterpret_cast<const double2*>(row + 2 * tid + 2);
                cs.ua[l][ph] = c.x;
                cs.ub[l][ph] = c.y;
                cs.h1a[l][ph] = __dadd_rn(l1, c.y);
                cs.h1b[l][ph] = __dadd_rn(c.x, r1);
                if (R == 2) {
                  cs.h2a[l][ph] = __dadd_rn(l2, r1);
                  cs.h2b[l][ph] = __dadd_rn(l1, r2);
                }
              }
            }
            // ---- compute every active level
#pragma unroll
            for (int l = 0; l < K; ++l) {
              const double ga = (l == 0) ? g0a : cs.gra[l][(ph + P - R - 1) % P];
              const double gb = (l == 0) ? g0b : cs.grb[l][(ph + P - R - 1) % P];
              if (l + 1 < K) { cs.gra[l + 1][ph] = ga; cs.grb[l + 1][ph] = gb; }
              const int first = 2 * (l + 1) * R + l;   // first active step of level l
              if (kk >= first && kk < nin + l) {
                double wa[P], wb[P], xa[P], xb[P], ya[P], yb[P];
#pragma unroll
                for (int q = 0; q < P; ++q) {          // logical row q -> slot (ph+1+q) mod P
                  const int sl = (ph + 1 + q) % P;
                  wa[q] = cs.ua[l][sl]; wb[q] = cs.ub[l][sl];
                  xa[q] = cs.h1a[l][sl]; xb[q] = cs.h1b[l][sl];
                  ya[q] = cs.h2a[l][sl]; yb[q] = cs.h2b[l][sl];
                }
                const int G = row_base + kk - (l + 1) * R - l;   // global row of the output
                const bool rowin = G >= p.row_lo && G < p.row_hi;
                const double Ja = Point<STENCIL>::jacobi_target(wa, xa, ya, ga);
                const double Jb = Point<STENCIL>::jacobi_target(wb, xb, yb, gb);
                const double da = __dsub_rn(Ja, wa[R]);
                const double db = __dsub_rn(Jb, wb[R]);
                const double oa = (FAST || (rowin && ina)) ? __fma_rn(cs.wl[l], da, wa[R]) : wa[R];
                const double ob = (FAST || (rowin && inb)) ? __fma_rn(cs.wl[l], db, wb[R]) : wb[R];
                if (REDUCE && l == 0 && (unsigned)(G - ja) < (unsigned)(jb - ja)) {
                  if (owna) { acc_s = __fma_rn(da, da, acc_s); acc_m = nan_max(acc_m, fabs(da)); }
                  if (ownb) { acc_s = __fma_rn(db, db, acc_s); acc_m = nan_max(acc_m, fabs(db)); }
                }
                if (l < K - 1) {
                  double* row = lb + (size_t)(l * P + ph) * ROW;
                  *reinterpret_cast<double2*>(row + 2 * tid + 2) = make_double2(oa, ob);
                } else {
                  if (STORE) {
                    if (FAST ? (tid >= E / 2 && tid < NT - E / 2) : (owna && ownb))
                      *reinterpret_cast<double2*>(outp) = make_double2(oa, ob);
                    else if (owna) outp[0] = oa;
                    else if (ownb) outp[1] = ob;
                  }
                  outp += ld;
                }
              }
            }
            if (K > 1) consumer_bar(NT);
          }
        }
      }
}

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
  double* lb = sg + (size_t)p.stages * T;                       // (K-1) x (2R+1) rows
  uint64_t* full = reinterpret_cast<uint64_t*>(lb + (size_t)(K - 1) * (2 * R + 1) * ROW);
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
    for (int e = tid; e < (K - 1) * (2 * R + 1) * ROW; e += blockDim.x) lb[e] = 0.0;
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
        const int strip = (int)(uu / p.nrows);
        const int ja = p.row0 + (int)(uu - (long long)strip * p.nrows);
        const long long seg_end = min(u_end, (long long)(strip + 1) * p.nrows);
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
          if (used >= p.stages) mbar_wait_a(smem_addr(&empty[stage]), phase ^ 1u);
          const int gin = ja - K * R + k;          // global row of the u row
          const bool hasu = gin >= -p.H && gin < rows + p.H;
          const int g1 = gin - R;                   // level-1 output row
          const bool hasg = k >= 2 * R && g1 >= p.row_lo && g1 < p.row_hi && gbytes;
          mbar_arrive_expect_tx(&full[stage], (hasu ? ubytes : 0u) + (hasg ? gbytes : 0u));
          if (hasu)
            tma_row_load(su + (size_t)stage * ROW,
                         src + (long long)(gin + p.H) * ld + (PADL - 2) + c0, ubytes,
                         &full[stage], pol);
          if (hasg)
            tma_row_load(sg + (size_t)stage * T + (gc0 - c0),
                         p.g + (long long)(g1 + p.H) * ld + PADL + gc0, gbytes, &full[stage], pol);
          ++used;
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
        }
        uu = seg_end;
      }
    }
  } else {
    // ---------------------------------------------- consumer threads (NT)
    ConsumerState<R, K> cs;
    cs.init(p, n, full, empty);
    for (long long uu = u_begin; uu < u_end;) {
      const int strip = (int)(uu / p.nrows);
      const int ja = p.row0 + (int)(uu - (long long)strip * p.nrows);
      const long long seg_end = min(u_end, (long long)(strip + 1) * p.nrows);
      const int jb = ja + (int)(seg_end - uu);
      const int c0 = strip * TOUT - E;
      // FAST: every row the segment touches is interior and the tile holds no
      // ghost / padding column, so no node of it is pass-through
      const bool fast = ja - K * R >= p.row_lo && jb + K * R <= p.row_hi && c0 >= 0 && c0 + T <= p.nx;
      if (fast)
        consumer_segment<STENCIL, NT, K, REDUCE, STORE, true>(cs, p, su, sg, lb, dst, ja, jb, c0,
                                                               tid, lane, acc_s, acc_m);
      else
        consumer_segment<STENCIL, NT, K, REDUCE, STORE, false>(cs, p, su, sg, lb, dst, ja, jb, c0,
                                                                tid, lane, acc_s, acc_m);
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
      if (STORE && p.advance) {
        p.state->n = n + (unsigned long long)K;
        p.state->cur = cur ^ 1u;
      }
      p.state->ticket = 0u;
      __threadfence();
    }
  }
}

}  // namespace cjm
