// sm_100a fp64 CJM sweep kernel, warp-tiled variant (
// NEXT-1 temporal blocking).
//
// Same contract, state machine, producer and reduction as cjm_sweep_kernel
// (sweep.cuh); the consumer side is organised around independent WARP tiles:
//  * each lane owns CPL = 4 adjacent columns (LDS.128 / STG.128), a warp spans
//    128 columns at every level;
//  * the K on-chip levels hand their rows to the next level IN REGISTERS:
//    the horizontal neighbours a level needs come from the adjacent lanes
//    (__shfl_up / __shfl_down), so there is no shared-memory line, no named
//    barrier and no level skew -- the warps of a CTA only meet at the TMA
//    ring's mbarriers;
//  * the price is a lost halo of E = r(K-1) (rounded up to even) columns per
//    side per WARP (instead of per CTA): a warp owns 128 - 2E output columns
//    and adjacent warp windows overlap by 2E columns.
//  * a TMA ring stage holds RPS consecutive input rows (RPS = 1, or 2r+1 for
//    variants 6 / 7): one mbarrier wait, one cross-proxy fence and one
//    release per RPS rows, and the RPS rows of a stage are independent
//    dependency chains at every level, which the compiler interleaves (the
//    kernel is latency-bound: few warps per SM, long fp64 chains per row).
//  * work distribution: the producer warp decides the CTA's segments (a column
//    strip and a row range) and hands each one to the consumer warps in a
//    per-stage descriptor guarded by the stage's full barrier.  Hot launches
//    take chunk_rows-row segments from a device counter (CTAs on slower SMs
//    or with boundary work simply take fewer); launches that reduce keep one
//    static contiguous range per CTA so that the per-CTA partial sums, and
//    the residual, are bitwise reproducible.
// Everything else (pass-through ghosts, the FAST instantiations, the fixed
// association of DESIGN R6, device-side n / cur, ticket, fixed-order
// reduction) is as in sweep.cuh.
#pragma once

#include "sweep.cuh"

namespace cjm {

template <int R, int K, int C>
struct WarpGeom {
  static constexpr int CPL = C;                               // columns per lane (2 or 4)
  static constexpr int WSPAN = 32 * CPL;                      // warp window
  static constexpr int E = (K == 1) ? 0 : ((R * (K - 1) + 1) & ~1);
  static constexpr int WOUT = WSPAN - 2 * E;                  // owned per warp
};

template <int R, int K, int NW, int C>
struct TileV4 {
  using WG = WarpGeom<R, K, C>;
  static constexpr int TOUT = NW * WG::WOUT;                  // owned per CTA strip
  static constexpr int TG = (NW - 1) * WG::WOUT + WG::WSPAN;  // g columns loaded
  static constexpr int TLOAD = TG + 4;                        // u columns loaded
  static constexpr int ROW = ((TLOAD + 7) / 8) * 8;           // shared row stride
  static constexpr int GROW = ((TG + 7) / 8) * 8;
};

template <int R, int K, int C>
struct WarpState {
  static constexpr int P = 2 * R + 1;
  double u[K][P][C], h1[K][P][C], h2[K][P][C];   // ring slot = step mod P
  double wl[K];
  int stage;
  uint32_t phase;
  uint32_t full_a, empty_a;
};

// Push one row of level values (C centre values + neighbours: l2, l1 west of
// column 0, r1, r2 east of column C-1) into slot `sl` of the level's ring:
// centre values and pair sums (west + east).
template <int R, int K, int C>
__device__ __forceinline__ void push_row(WarpState<R, K, C>& ws, int l, int sl, const double (&c)[C],
                                         double l2, double l1, double r1, double r2) {
#pragma unroll
  for (int j = 0; j < C; ++j) {
    ws.u[l][sl][j] = c[j];
    const double w1 = j == 0 ? l1 : c[j - 1];
    const double e1 = j == C - 1 ? r1 : c[j + 1];
    ws.h1[l][sl][j] = __dadd_rn(w1, e1);
    if (R == 2) {
      const double w2 = j == 0 ? l2 : (j == 1 ? l1 : c[j - 2]);
      const double e2 = j == C - 1 ? r2 : (j == C - 2 ? r1 : c[j + 2]);
      ws.h2[l][sl][j] = __dadd_rn(w2, e2);
    }
  }
}

// Per-segment constants of one lane.
template <int C>
struct LaneSeg {
  bool in[C], own[C];
  int ja, jb, row_base, uoff;
  double* outp;
#ifdef CJM_DEBUG_CHECKS
  const double* out_base;   // the output buffer (bounds checks)
#endif
};

// One input row kk (row RI of the ring stage `st`; ring slot ph = kk mod P) of
// a lane, the stage already waited for: read the TMA row, run every level
// (unconditionally: a level computes garbage until its window is full, which
// is never stored), store the last level when it is active.  RI and PH are
// compile-time, so every register-ring slot and every stage offset folds.
// FM (fast mode): 2 = the warp window holds no ghost / padding column and the
// segment no ghost row (no checks); 1 = no ghost column, ghost rows possible
// (one uniform row test per level); 0 = every node checked.
template <int STENCIL, int NW, int K, int C, int RPS, int RI, int PH, bool REDUCE, bool STORE,
          int FM, bool STEADY = false>
__device__ __forceinline__ void warp_row(WarpState<Point<STENCIL>::R, K, C>& ws, LaneSeg<C>& ls,
                                         const SweepParams& p, const double* su, const double* sg,
                                         int st, const double* ucur, const double* gcur,
                                         const double* gprev, int kk, int lane, double& acc_s,
                                         double& acc_m) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int P = 2 * R + 1;
  constexpr int ph = PH;
  using WG = WarpGeom<R, K, C>;
  using TG_ = TileV4<R, K, NW, C>;
  constexpr int E = WG::E;
  // ---- level 0 input: row RI of stage st
  // A stage stays held until level K-1 has read the g rows of all its rows,
  // R(K-1) rows later (level l reads the g row that arrived with input row
  // kk - lR), so g needs no register ring.
  {
    const double* row = ucur + RI * TG_::ROW;   // row[2 + j] = column j
    CJM_CHECK(p, row >= su && row + 2 + C + 2 <= su + (size_t)p.stages * RPS * TG_::ROW, CHK_RING_READ);
    double cc[C];
#pragma unroll
    for (int j = 0; j < C; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(row + 2 + j);
      cc[j] = v.x;
      cc[j + 1] = v.y;
    }
    double l2 = 0.0, l1, r1, r2 = 0.0;
    if (R == 2) {
      const double2 lft = *reinterpret_cast<const double2*>(row);
      const double2 rgt = *reinterpret_cast<const double2*>(row + 2 + C);
      l2 = lft.x; l1 = lft.y; r1 = rgt.x; r2 = rgt.y;
    } else {
      l1 = row[1];
      r1 = row[2 + C];
    }
    push_row<R, K, C>(ws, 0, ph, cc, l2, l1, r1, r2);
  }
  // ---- levels, in order; level l hands its row to level l+1 in registers
#pragma unroll
  for (int l = 0; l < K; ++l) {
    // g of level l's output row: arrived with the u row of step kk - lR
    // (stale during a level's warm-up: never stored then)
    double g[C];
    {
      // input row kk - lR: row GR of the stage GB stages back (compile-time)
      const int GB = (l * R - RI + RPS - 1) / RPS;  // l R <= RI: 0 (folds: l unrolled)
      const int GR = RI - l * R + GB * RPS;
      const double* grow;
      if (RPS > 1 && GB <= 1) {            // this or the previous stage: per-stage bases
        grow = (GB == 0 ? gcur : gprev) + GR * TG_::GROW;
      } else {
        int gs = st - GB;
        if (gs < 0) gs += p.stages;
        grow = sg + ((size_t)gs * RPS + GR) * TG_::GROW + ls.uoff;
      }
      CJM_CHECK(p, grow >= sg && grow + C <= sg + (size_t)p.stages * RPS * TG_::GROW, CHK_RING_READ);
#pragma unroll
      for (int j = 0; j < C; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(grow + j);
        g[j] = v.x;
        g[j + 1] = v.y;
      }
    }
    const int G = ls.row_base + kk - (l + 1) * R;           // global row of the output
    // one predicate per node, evaluated without short-circuit branches (the
    // nested form compiled to three FSEL pairs per node)
    const bool rowin = (G >= p.row_lo) & (G < p.row_hi);
    double o[C], dd[C];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      double uw[P], x1[P], x2[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {                      // logical row q -> ring slot
        const int sl = (ph + 1 + q) % P;
        uw[q] = ws.u[l][sl][j];
        x1[q] = ws.h1[l][sl][j];
        x2[q] = ws.h2[l][sl][j];
      }
      const double J = Point<STENCIL>::jacobi_target(uw, x1, x2, g[j]);
      dd[j] = __dsub_rn(J, uw[R]);
      const bool upd = FM == 2 || (FM == 1 ? rowin : (ls.in[j] & rowin));
      o[j] = upd ? __fma_rn(ws.wl[l], dd[j], uw[R]) : uw[R];
    }
    const bool active = STEADY || kk >= 2 * (l + 1) * R;   // STEADY: past every warm-up
    if (REDUCE && l == 0 && active && (unsigned)(G - ls.ja) < (unsigned)(ls.jb - ls.ja)) {
#pragma unroll
      for (int j = 0; j < C; ++j)
        if (ls.own[j]) { acc_s = __fma_rn(dd[j], dd[j], acc_s); acc_m = nan_max(acc_m, fabs(dd[j])); }
    }
    if (l + 1 < K) {
      // neighbours of this lane's columns at level l: adjacent lanes (the two
      // warp-edge lanes get their own values: garbage inside the lost halo)
      const double l1 = __shfl_up_sync(0xffffffffu, o[C - 1], 1);
      const double r1 = __shfl_down_sync(0xffffffffu, o[0], 1);
      double l2 = 0.0, r2 = 0.0;
      if (R == 2) {
        l2 = __shfl_up_sync(0xffffffffu, o[C - 2], 1);
        r2 = __shfl_down_sync(0xffffffffu, o[1], 1);
      }
      push_row<R, K, C>(ws, l + 1, ph, o, l2, l1, r1, r2);
    } else if (active) {
#ifdef CJM_DEBUG_CHECKS
      if (STORE) {   // every column this lane may store: interior of a band row
        const long long off = ls.outp - ls.out_base;
        const long long orow = off / p.ld, ocol = off - orow * p.ld;
        for (int j = 0; j < C; ++j)
          if (FM >= 1 ? (C * lane + j >= E && C * lane + j < WG::WSPAN - E) : ls.own[j])
            CJM_CHECK(p, off >= 0 && orow >= p.H + p.row0 && orow < p.H + p.row0 + p.nrows &&
                             ocol + j >= PADL && ocol + j < PADL + p.nx &&
                             off + j < p.buf_elems, CHK_STORE);
      }
#endif
      if (STORE) {
#pragma unroll
        for (int j = 0; j < C; j += 2) {
          // FAST: every column is interior, ownership depends on the lane only
          // (E even: both columns of a pair are owned or neither).  (Stores
          // predicated inside inline PTX instead of branches measured slower:
          // 32.2 vs 31.4 us per sweep, profiles/r01_v7_tune.jsonl.)
          const bool ownp = FM >= 1 ? (C * lane + j >= E && C * lane + j + 2 <= WG::WSPAN - E)
                                    : (ls.own[j] && ls.own[j + 1]);
          if (ownp) *reinterpret_cast<double2*>(ls.outp + j) = make_double2(o[j], o[j + 1]);
          else if (FM == 0) {
            if (ls.own[j]) ls.outp[j] = o[j];
            if (ls.own[j + 1]) ls.outp[j + 1] = o[j + 1];
          }
        }
      }
      ls.outp += p.ld;
    }
  }
}

// Process ring stage `st` (input rows kk0 .. kk0 + RPS - 1; ring slot of row
// kk0 is PH0): wait for it, run its rows (rows >= nin only in a segment's
// last stage, when GUARD), then release the stage whose rows level K-1 has
// now read for the last time.
template <int STENCIL, int NW, int K, int C, int RPS, int PH0, bool GUARD, bool REDUCE,
          bool STORE, int FM, bool STEADY = false>
__device__ __forceinline__ void warp_stage(WarpState<Point<STENCIL>::R, K, C>& ws, LaneSeg<C>& ls,
                                           const SweepParams& p, const double* su,
                                           const double* sg, int s, int kk0, int nin, int lane,
                                           double& acc_s, double& acc_m) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int P = 2 * R + 1;
  constexpr int HS = ((K - 1) * R + RPS - 1) / RPS;   // stages held after processing
  const int st = ws.stage;
#ifndef CJM_DIAG_NOWAIT   // diagnostic builds only: consumers do not wait for their data
  mbar_wait_a(ws.full_a + 8u * st, ws.phase);
#endif
  if (++ws.stage == p.stages) { ws.stage = 0; ws.phase ^= 1u; }
  using TG_ = TileV4<R, K, NW, C>;
  const double* ucur = su + (size_t)st * RPS * TG_::ROW + ls.uoff;
  const double* gcur = sg + (size_t)st * RPS * TG_::GROW + ls.uoff;
  const double* gprev = sg + (size_t)(st == 0 ? p.stages - 1 : st - 1) * RPS * TG_::GROW + ls.uoff;
#define CJM_V4_ROW(RI)                                                                         \
  if (RI < RPS && (!GUARD || kk0 + RI < nin))                                                  \
    warp_row<STENCIL, NW, K, C, RPS, (RI < RPS ? RI : 0), (PH0 + RI) % P, REDUCE, STORE, FM,    \
             STEADY>(                                                                          \
        ws, ls, p, su, sg, st, ucur, gcur, gprev, kk0 + RI, lane, acc_s, acc_m);
  CJM_V4_ROW(0) CJM_V4_ROW(1) CJM_V4_ROW(2) CJM_V4_ROW(3) CJM_V4_ROW(4)
#undef CJM_V4_ROW
  static_assert(RPS <= 5, "rows per stage <= 5");
  // ---- release stage s - HS: level K-1 has read its last g row
  if (s >= HS) {
    int rel = st - HS;
    if (rel < 0) rel += p.stages;
    fence_proxy_async_smem();   // my reads of the slot before its TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive_a(ws.empty_a + 8u * rel);
  }
}

template <int STENCIL, int NW, int K, int C, int RPS, bool REDUCE, bool STORE, int FM>
__device__ __forceinline__ void warp_segment(WarpState<Point<STENCIL>::R, K, C>& ws,
                                             const SweepParams& p, const double* su,
                                             const double* sg, double* dst, int ja, int jb,
                                             int c0, int warp, int lane, double& acc_s,
                                             double& acc_m) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int P = 2 * R + 1;
  using WG = WarpGeom<R, K, C>;
  constexpr int E = WG::E;
  const int wbase = warp * WG::WOUT;                 // warp window offset in the tile
  const int cl = c0 + wbase + C * lane;              // first column of this lane
  LaneSeg<C> ls;
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int c = cl + j;
    ls.in[j] = c >= 0 && c < p.nx;
    ls.own[j] = ls.in[j] && (C * lane + j) >= E && (C * lane + j) < WG::WSPAN - E;
  }
  ls.ja = ja;
  ls.jb = jb;
  ls.row_base = ja - K * R;
  ls.uoff = wbase + C * lane;                        // shared index of column cl - 2
  ls.outp = dst + (long long)(ja + p.H) * p.ld + PADL + cl;
#ifdef CJM_DEBUG_CHECKS
  ls.out_base = dst;
#endif
  const int nin = jb - ja + 2 * K * R;
  const int nst = (nin + RPS - 1) / RPS;             // ring stages of the segment
  if (c0 + wbase >= p.nx + R) {
    // the whole warp window lies right of the last ghost column (ragged last
    // strip): nothing to compute, keep the TMA ring in step
    for (int s = 0; s < nst; ++s) {
      mbar_wait_a(ws.full_a + 8u * ws.stage, ws.phase);
      __syncwarp();
      if (lane == 0) mbar_arrive_a(ws.empty_a + 8u * ws.stage);
      if (++ws.stage == p.stages) { ws.stage = 0; ws.phase ^= 1u; }
    }
    return;
  }
  // U stages make a whole number of register-ring periods (U RPS = 0 mod P),
  // so the ring slot of every row is compile-time inside a period
  constexpr int U = (RPS % P == 0) ? 1 : P;
  constexpr int UR = U * RPS;
  int s0 = 0;
  // full periods, no guards: first those holding a level's warm-up rows
  // (input rows < 2 K r), then the steady ones (every level active)
#define CJM_V4_STAGE_FM(u, FMX)                                                             \
  if (u < U)                                                                                \
    warp_stage<STENCIL, NW, K, C, RPS, ((u < U ? u : 0) * RPS) % P, false, REDUCE, STORE,     \
               (FM == 1 ? FMX : FM), true>(ws, ls, p, su, sg, s0 + u, (s0 + u) * RPS, nin,   \
                                           lane, acc_s, acc_m);
#define CJM_V4_STAGE(u, STEADY)                                                             \
  if (u < U)                                                                                \
    warp_stage<STENCIL, NW, K, C, RPS, ((u < U ? u : 0) * RPS) % P, false, REDUCE, STORE, FM, \
               STEADY>(ws, ls, p, su, sg, s0 + u, (s0 + u) * RPS, nin, lane, acc_s, acc_m);
  for (; (s0 + U) * RPS <= nin && s0 * RPS < 2 * K * R; s0 += U) {
    CJM_V4_STAGE(0, false) CJM_V4_STAGE(1, false) CJM_V4_STAGE(2, false) CJM_V4_STAGE(3, false)
    CJM_V4_STAGE(4, false)
  }
  for (; (s0 + U) * RPS <= nin; s0 += U) {
    if (FM == 1) {
      // a segment that touches ghost rows (FM 1: one row test per level)
      // needs the test only near them: periods whose output rows at every
      // level (row_base + kk - (l+1) r) are interior run without it
      const int glo = ls.row_base + s0 * RPS - K * R;
      const int ghi = ls.row_base + (s0 + U) * RPS - 1 - R;
      if (glo >= p.row_lo && ghi < p.row_hi) {
        CJM_V4_STAGE_FM(0, 2) CJM_V4_STAGE_FM(1, 2) CJM_V4_STAGE_FM(2, 2) CJM_V4_STAGE_FM(3, 2)
        CJM_V4_STAGE_FM(4, 2)
        continue;
      }
    }
    CJM_V4_STAGE(0, true) CJM_V4_STAGE(1, true) CJM_V4_STAGE(2, true) CJM_V4_STAGE(3, true)
    CJM_V4_STAGE(4, true)
  }
#undef CJM_V4_STAGE
#undef CJM_V4_STAGE_FM
  static_assert(U <= 5, "stages per period <= 5");
  // tail: fewer than UR rows left, in at most U stages (rows >= nin guarded)
#define CJM_V4_TAIL(u)                                                                     \
  if (u < U && s0 + u < nst)                                                               \
    warp_stage<STENCIL, NW, K, C, RPS, ((u < U ? u : 0) * RPS) % P, true, REDUCE, STORE,   \
               FM>(ws, ls, p, su, sg, s0 + u, (s0 + u) * RPS, nin, lane, acc_s, acc_m);
  CJM_V4_TAIL(0) CJM_V4_TAIL(1) CJM_V4_TAIL(2) CJM_V4_TAIL(3) CJM_V4_TAIL(4)
#undef CJM_V4_TAIL
  (void)UR;
  // the last HS stages of the segment were still held: release them
  constexpr int HS = ((K - 1) * R + RPS - 1) / RPS;
  if (HS > 0) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int i = HS; i > 0; --i) {
        int rel = ws.stage - i;
        if (rel < 0) rel += p.stages;
        mbar_arrive_a(ws.empty_a + 8u * rel);
      }
    }
  }
}

// Register cap.  The register file is split between the 4 SM sub-partitions
// (16 K registers each), so 2 resident CTAs of 5 warps (3 warps on some
// sub-partition) need <= 168 registers per thread: 172 registers (one more
// live value) silently halve the occupancy of the K = 2 kernel (58 vs 38 us
// per sweep at 4096^2, ncu occupancy_limit_registers = 1).  Kernels whose
// natural count is far above 168 (4 columns per lane with K >= 3, the
// 17-point) keep one CTA per SM and are not capped.
template <int STENCIL, int K, int C>
struct V4Regs {
  static constexpr int value =
      Point<STENCIL>::R == 1 ? ((C == 2 || K <= 2) ? 168 : 255) : ((C == 2 && K == 1) ? 168 : 255);
};

template <int STENCIL, int NW, int K, int C, bool REDUCE, bool STORE, int RPS = 1>
__global__ void __maxnreg__((V4Regs<STENCIL, K, C>::value)) cjm_sweep_kernel_v4(const SweepParams p) {
  constexpr int R = Point<STENCIL>::R;
  using WG = WarpGeom<R, K, C>;
  using TG_ = TileV4<R, K, NW, C>;
  constexpr int E = WG::E;
  constexpr int NT = 32 * NW;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* su = reinterpret_cast<double*>(smem_raw);            // stages x RPS u rows
  double* sg = su + (size_t)p.stages * RPS * TG_::ROW;          // stages x RPS g rows
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + (size_t)p.stages * RPS * TG_::GROW);
  uint64_t* empty = full + p.stages;
  __shared__ double red_s[NW], red_m[NW];
  __shared__ int is_last;
  __shared__ int4 seg_desc[32];   // per ring stage: (strip, ja, jb, valid) of a segment's first stage

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
#ifdef CJM_DIAG_TIMES
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif

  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);        // one arrival per consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  const unsigned long long n = __ldcg(&p.state->n);
  const unsigned int cur = __ldcg(&p.state->cur);
  const double* src = (cur & 1u) ? p.buf[1] : p.buf[0];
  double* dst = (cur & 1u) ? p.buf[0] : p.buf[1];
  const long long ld = p.ld;
  const int rows = p.rows;
  // static part of the (strip, row) units: one contiguous range per CTA; the
  // rest [units_static, units) goes out in chunk_rows-unit items (hot launches)
  const long long ustat = p.chunk_rows > 0 ? p.units_static : p.units;
  const long long u_begin = (long long)blockIdx.x * ustat / gridDim.x;
  const long long u_end = (long long)(blockIdx.x + 1) * ustat / gridDim.x;

  double acc_s = 0.0, acc_m = 0.0;

  if (tid >= NT) {
    // ------------------------------------------------ producer warp (lane 0)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      long long used = 0;
      const uint32_t full_a = smem_addr(full), empty_a = smem_addr(empty);
      long long uu = u_begin, ue = u_end;    // current unit range
      for (;;) {
        // ---- next segment: (strip, rows [ja, jb)), or the end marker.  A
        // range that spans a strip boundary yields two segments.
        if (uu >= ue && p.chunk_rows > 0) {
          const long long c = atomicAdd(&p.state->next_chunk, 1u);
          uu = p.units_static + c * p.chunk_rows;
          ue = min(uu + p.chunk_rows, p.units);
        }
        const bool more = uu < ue;
        int strip = 0, ja = 0, jb = 0;
        if (more) {
          strip = (int)(uu / p.nrows);
          ja = p.row0 + (int)(uu - (long long)strip * p.nrows);
          const long long seg_end = min(ue, (long long)(strip + 1) * p.nrows);
          jb = ja + (int)(seg_end - uu);
          uu = seg_end;
        }
        if (!more) {   // end marker: a stage without data
          if (used >= p.stages) mbar_wait_a(empty_a + 8u * stage, phase ^ 1u);
          seg_desc[stage] = make_int4(0, 0, 0, 0);
          mbar_arrive_expect_tx(&full[stage], 0u);
          break;
        }
        const int c0 = strip * TG_::TOUT - E;
        const int ucols = min(TG_::TLOAD, p.nx + R + 2 - c0);
        const uint32_t ubytes = (uint32_t)(((ucols + 1) & ~1) * 8);
        const int gc0 = max(c0, 0);
        const int gcols = min(c0 + TG_::TG, p.nx) - gc0;
        const uint32_t gbytes = gcols > 0 ? (uint32_t)(((gcols + 1) & ~1) * 8) : 0u;
        const int nin = jb - ja + 2 * K * R;
        for (int k0 = 0; k0 < nin; k0 += RPS) {       // one ring stage: rows k0 .. k0+RPS-1
          if (used >= p.stages) mbar_wait_a(empty_a + 8u * stage, phase ^ 1u);
          uint32_t tx = 0;
#pragma unroll
          for (int r = 0; r < RPS; ++r) {
            const int k = k0 + r;
            const int gin = ja - K * R + k;
            const int g1 = gin - R;
            const bool hasu = k < nin && gin >= -p.H && gin < rows + p.H;
            const bool hasg = k < nin && k >= 2 * R && g1 >= p.row_lo && g1 < p.row_hi && gbytes;
            tx += (hasu ? ubytes : 0u) + (hasg ? gbytes : 0u);
          }
#ifdef CJM_DIAG_NOTMA      // diagnostic builds only: no HBM reads, the stage completes at once
          tx = 0;
#endif
          if (k0 == 0) seg_desc[stage] = make_int4(strip, ja, jb, 1);   // released by the arrive
          CJM_CHECK(p, tx <= (uint32_t)(RPS * (TG_::ROW + TG_::GROW) * 8), CHK_TX);
          CJM_CHECK(p, ja >= p.row0 && jb <= p.row0 + p.nrows && ja < jb, CHK_DESC);
          mbar_arrive_expect_tx(&full[stage], tx);
#pragma unroll
          for (int r = 0; r < RPS; ++r) {
            const int k = k0 + r;
            const int gin = ja - K * R + k;
            const int g1 = gin - R;
            const bool hasu = k < nin && gin >= -p.H && gin < rows + p.H;
            const bool hasg = k < nin && k >= 2 * R && g1 >= p.row_lo && g1 < p.row_hi && gbytes;
#ifdef CJM_DIAG_NOTMA
            continue;
#endif
#ifdef CJM_DEBUG_CHECKS
            if (hasu) {
              const long long so = (long long)(gin + p.H) * ld + (PADL - 2) + c0;
              const long long dso = ((long long)stage * RPS + r) * TG_::ROW;
              CJM_CHECK(p, so >= 0 && so + ubytes / 8 <= p.buf_elems &&
                               (PADL - 2) + c0 + (long long)(ubytes / 8) <= ld, CHK_TMA_U);
              CJM_CHECK(p, dso >= 0 && dso + ubytes / 8 <= (long long)p.stages * RPS * TG_::ROW,
                        CHK_TMA_DST);
              CJM_CHECK(p, (so % 2) == 0 && (ubytes % 16) == 0, CHK_TMA_ALIGN);
            }
            if (hasg) {
              const long long so = (long long)(g1 + p.H) * ld + PADL + gc0;
              const long long dso = ((long long)stage * RPS + r) * TG_::GROW + (gc0 - c0);
              CJM_CHECK(p, so >= 0 && so + gbytes / 8 <= p.buf_elems && PADL + gc0 + gbytes / 8 <= ld,
                        CHK_TMA_G);
              CJM_CHECK(p, dso >= 0 && dso + gbytes / 8 <= (long long)p.stages * RPS * TG_::GROW,
                        CHK_TMA_DST);
              CJM_CHECK(p, (so % 2) == 0 && (dso % 2) == 0 && (gbytes % 16) == 0, CHK_TMA_ALIGN);
            }
#endif
            if (hasu)
              tma_row_load(su + ((size_t)stage * RPS + r) * TG_::ROW,
                           src + (long long)(gin + p.H) * ld + (PADL - 2) + c0, ubytes, &full[stage],
                           pol);
            if (hasg)
              tma_row_load(sg + ((size_t)stage * RPS + r) * TG_::GROW + (gc0 - c0),
                           p.g + (long long)(g1 + p.H) * ld + PADL + gc0, gbytes, &full[stage], pol);
          }
          ++used;
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else {
    // ---------------------------------------------- consumer warps
    WarpState<R, K, C> ws;
#pragma unroll
    for (int l = 0; l < K; ++l) {
      ws.wl[l] = __ldg(p.w + (long long)((n + l) % (unsigned long long)p.P));
#pragma unroll
      for (int q = 0; q < 2 * R + 1; ++q)
#pragma unroll
        for (int j = 0; j < C; ++j) ws.u[l][q][j] = ws.h1[l][q][j] = ws.h2[l][q][j] = 0.0;
    }
    ws.stage = 0;
    ws.phase = 0;
    ws.full_a = smem_addr(full);
    ws.empty_a = smem_addr(empty);
    for (;;) {
      // the next segment's descriptor arrives with its first stage
      mbar_wait_a(ws.full_a + 8u * ws.stage, ws.phase);
      const int4 d = seg_desc[ws.stage];
      if (!d.w) break;
      const int strip = d.x, ja = d.y, jb = d.z;
      const int c0 = strip * TG_::TOUT - E;
      // fast mode per warp (FM above): no ghost / padding column in its window
      // (2 if the segment also touches no ghost row, else 1), or 0.  A CTA
      // whose range starts at the top or ends at the bottom of a strip (every
      // CTA that crosses a strip boundary) thus checks rows, not nodes: with
      // node checks such CTAs ran 28% longer than the rest
      // (profiles/r01_v7_cta_times.jsonl).
      const int cw = c0 + warp * WG::WOUT;
      const bool fastc = cw >= 0 && cw + WG::WSPAN <= p.nx;
      const bool fastr = ja - K * R >= p.row_lo && jb + K * R <= p.row_hi;
      if (fastc && fastr)
        warp_segment<STENCIL, NW, K, C, RPS, REDUCE, STORE, 2>(ws, p, su, sg, dst, ja, jb, c0, warp,
                                                               lane, acc_s, acc_m);
      else if (fastc)
        warp_segment<STENCIL, NW, K, C, RPS, REDUCE, STORE, 1>(ws, p, su, sg, dst, ja, jb, c0, warp,
                                                               lane, acc_s, acc_m);
      else
        warp_segment<STENCIL, NW, K, C, RPS, REDUCE, STORE, 0>(ws, p, su, sg, dst, ja, jb, c0, warp,
                                                               lane, acc_s, acc_m);
    }
  }

  if (REDUCE) {
    if (tid < NT) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc_s = __dadd_rn(acc_s, __shfl_xor_sync(0xffffffffu, acc_s, o));
        acc_m = nan_max(acc_m, __shfl_xor_sync(0xffffffffu, acc_m, o));
      }
      if (lane == 0) { red_s[warp] = acc_s; red_m[warp] = acc_m; }
    }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0, m = 0.0;
      for (int q = 0; q < NW; ++q) { s = __dadd_rn(s, red_s[q]); m = nan_max(m, red_m[q]); }
      p.partials[2 * blockIdx.x] = s;
      p.partials[2 * blockIdx.x + 1] = m;
    }
  }

  __syncthreads();
#ifdef CJM_DIAG_TIMES
  if (!REDUCE && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    reinterpret_cast<unsigned long long*>(p.partials)[2 * blockIdx.x] = t_start;
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const long long useg = u_begin, ueg = u_end;
    const unsigned long long nseg = (unsigned long long)((ueg - 1) / p.nrows - useg / p.nrows + 1);
    reinterpret_cast<unsigned long long*>(p.partials)[2 * blockIdx.x + 1] =
        (t_end - t_start) | ((unsigned long long)smid << 40) | (nseg << 52);
  }
#endif
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
        if (lane == 0) { red_s[warp] = s; red_m[warp] = m; }
      }
      __syncthreads();
      if (tid == 0) {
        s = 0.0; m = 0.0;
        for (int q = 0; q < NW; ++q) { s = __dadd_rn(s, red_s[q]); m = nan_max(m, red_m[q]); }
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
      p.state->next_chunk = 0u;
      __threadfence();
    }
  }
}

}  // namespace cjm
