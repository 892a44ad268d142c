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
// Everything else (pass-through ghosts, the FAST instantiation, the fixed
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
};

// One step (input row kk, ring slot ph = kk mod P) of a lane: read the TMA row,
// run every level (unconditionally: a level computes garbage until its window
// is full, which is never stored), store the last level when it is active.
template <int STENCIL, int NW, int K, int C, bool REDUCE, bool STORE, bool FAST>
__device__ __forceinline__ void warp_step(WarpState<Point<STENCIL>::R, K, C>& ws, LaneSeg<C>& ls,
                                          const SweepParams& p, const double* su, const double* sg,
                                          int kk, int ph, int lane, double& acc_s, double& acc_m) {
  constexpr int R = Point<STENCIL>::R;
  constexpr int P = 2 * R + 1;
  using WG = WarpGeom<R, K, C>;
  using TG_ = TileV4<R, K, NW, C>;
  constexpr int E = WG::E;
  // ---- level 0 input: the TMA row of step kk (slot rs)
  // The slot of step kk stays held until level K-1 has read its g row, R(K-1)
  // steps later (level l reads the g row that arrived with step kk - lR), so
  // g needs no register ring.
  const int rs = ws.stage;
  {
    mbar_wait_a(ws.full_a + 8u * rs, ws.phase);
    const double* row = su + (size_t)rs * TG_::ROW + ls.uoff;   // row[2 + j] = column j
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
    if (++ws.stage == p.stages) { ws.stage = 0; ws.phase ^= 1u; }
    push_row<R, K, C>(ws, 0, ph, cc, l2, l1, r1, r2);
  }
  // ---- levels, in order; level l hands its row to level l+1 in registers
#pragma unroll
  for (int l = 0; l < K; ++l) {
    // g of level l's output row: arrived with the u row of step kk - lR
    // (stale during a level's warm-up: never stored then)
    double g[C];
    {
      int gs = rs - l * R;
      if (gs < 0) gs += p.stages;
      const double* grow = sg + (size_t)gs * TG_::GROW + ls.uoff;
#pragma unroll
      for (int j = 0; j < C; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(grow + j);
        g[j] = v.x;
        g[j + 1] = v.y;
      }
    }
    const int G = ls.row_base + kk - (l + 1) * R;           // global row of the output
    const bool rowin = G >= p.row_lo && G < p.row_hi;
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
      o[j] = (FAST || (rowin && ls.in[j])) ? __fma_rn(ws.wl[l], dd[j], uw[R]) : uw[R];
    }
    const bool active = kk >= 2 * (l + 1) * R;
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
      if (STORE) {
#pragma unroll
        for (int j = 0; j < C; j += 2) {
          // FAST: every column is interior, ownership depends on the lane only
          // (E even: both columns of a pair are owned or neither)
          const bool ownp = FAST ? (C * lane + j >= E && C * lane + j + 2 <= WG::WSPAN - E)
                                 : (ls.own[j] && ls.own[j + 1]);
          if (ownp) *reinterpret_cast<double2*>(ls.outp + j) = make_double2(o[j], o[j + 1]);
          else if (!FAST) {
            if (ls.own[j]) ls.outp[j] = o[j];
            if (ls.own[j + 1]) ls.outp[j + 1] = o[j + 1];
          }
        }
      }
      ls.outp += p.ld;
    }
  }
  // ---- release the slot whose last reader (level K-1's g) was this step
  if (kk >= (K - 1) * R) {
    int rel = rs - (K - 1) * R;
    if (rel < 0) rel += p.stages;
    fence_proxy_async_smem();   // my reads of the slot before its TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive_a(ws.empty_a + 8u * rel);
  }
}

template <int STENCIL, int NW, int K, int C, bool REDUCE, bool STORE, bool FAST>
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
  const int nin = jb - ja + 2 * K * R;
  if (c0 + wbase >= p.nx + R) {
    // the whole warp window lies right of the last ghost column (ragged last
    // strip): nothing to compute, keep the TMA ring in step
    for (int kk = 0; kk < nin; ++kk) {
      mbar_wait_a(ws.full_a + 8u * ws.stage, ws.phase);
      __syncwarp();
      if (lane == 0) mbar_arrive_a(ws.empty_a + 8u * ws.stage);
      if (++ws.stage == p.stages) { ws.stage = 0; ws.phase ^= 1u; }
    }
    return;
  }
  int k0 = 0;
  for (; k0 + P <= nin; k0 += P) {                  // full periods: no guards
#pragma unroll
    for (int ph = 0; ph < P; ++ph)
      warp_step<STENCIL, NW, K, C, REDUCE, STORE, FAST>(ws, ls, p, su, sg, k0 + ph, ph, lane, acc_s,
                                                        acc_m);
  }
#pragma unroll
  for (int ph = 0; ph < P - 1; ++ph)                 // tail
    if (k0 + ph < nin)
      warp_step<STENCIL, NW, K, C, REDUCE, STORE, FAST>(ws, ls, p, su, sg, k0 + ph, ph, lane, acc_s,
                                                        acc_m);
  // the last R(K-1) slots of the segment were still held: release them
  if (K > 1) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int i = (K - 1) * R; i > 0; --i) {
        int rel = ws.stage - i;
        if (rel < 0) rel += p.stages;
        mbar_arrive_a(ws.empty_a + 8u * rel);
      }
    }
  }
}

// K = 2 is register-limited to 2 CTAs (10 warps) per SM at its natural 168
// registers; asking for 3 resident CTAs caps it at 136 (V4_MIN_BLOCKS_K2).
#ifndef V4_MIN_BLOCKS_K2
#define V4_MIN_BLOCKS_K2 1
#endif
template <int STENCIL, int NW, int K, int C, bool REDUCE, bool STORE>
__global__ void __launch_bounds__(32 * NW + 32, (K == 2 && C == 4 ? V4_MIN_BLOCKS_K2 : 1))
cjm_sweep_kernel_v4(const SweepParams p) {
  constexpr int R = Point<STENCIL>::R;
  using WG = WarpGeom<R, K, C>;
  using TG_ = TileV4<R, K, NW, C>;
  constexpr int E = WG::E;
  constexpr int NT = 32 * NW;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* su = reinterpret_cast<double*>(smem_raw);
  double* sg = su + (size_t)p.stages * TG_::ROW;
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + (size_t)p.stages * TG_::GROW);
  uint64_t* empty = full + p.stages;
  __shared__ double red_s[NW], red_m[NW];
  __shared__ int is_last;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

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
      const uint32_t full_a = smem_addr(full), empty_a = smem_addr(empty);
      for (long long uu = u_begin; uu < u_end;) {
        const int strip = (int)(uu / p.nrows);
        const int ja = p.row0 + (int)(uu - (long long)strip * p.nrows);
        const long long seg_end = min(u_end, (long long)(strip + 1) * p.nrows);
        const int jb = ja + (int)(seg_end - uu);
        const int c0 = strip * TG_::TOUT - E;
        const int ucols = min(TG_::TLOAD, p.nx + R + 2 - c0);
        const uint32_t ubytes = (uint32_t)(((ucols + 1) & ~1) * 8);
        const int gc0 = max(c0, 0);
        const int gcols = min(c0 + TG_::TG, p.nx) - gc0;
        const uint32_t gbytes = gcols > 0 ? (uint32_t)(((gcols + 1) & ~1) * 8) : 0u;
        const int nin = jb - ja + 2 * K * R;
        for (int k = 0; k < nin; ++k) {
          if (used >= p.stages) mbar_wait_a(empty_a + 8u * stage, phase ^ 1u);
          const int gin = ja - K * R + k;
          const bool hasu = gin >= -p.H && gin < rows + p.H;
          const int g1 = gin - R;
          const bool hasg = k >= 2 * R && g1 >= p.row_lo && g1 < p.row_hi && gbytes;
          mbar_arrive_expect_tx(&full[stage], (hasu ? ubytes : 0u) + (hasg ? gbytes : 0u));
          if (hasu)
            tma_row_load(su + (size_t)stage * TG_::ROW,
                         src + (long long)(gin + p.H) * ld + (PADL - 2) + c0, ubytes, &full[stage], pol);
          if (hasg)
            tma_row_load(sg + (size_t)stage * TG_::GROW + (gc0 - c0),
                         p.g + (long long)(g1 + p.H) * ld + PADL + gc0, gbytes, &full[stage], pol);
          ++used;
          if (++stage == p.stages) { stage = 0; phase ^= 1u; }
        }
        uu = seg_end;
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
    for (long long uu = u_begin; uu < u_end;) {
      const int strip = (int)(uu / p.nrows);
      const int ja = p.row0 + (int)(uu - (long long)strip * p.nrows);
      const long long seg_end = min(u_end, (long long)(strip + 1) * p.nrows);
      const int jb = ja + (int)(seg_end - uu);
      const int c0 = strip * TG_::TOUT - E;
      // FAST per warp: its window holds no ghost / padding column and the
      // segment touches no ghost row
      const int cw = c0 + warp * WG::WOUT;
      const bool fast = ja - K * R >= p.row_lo && jb + K * R <= p.row_hi && cw >= 0 &&
                        cw + WG::WSPAN <= p.nx;
      if (fast)
        warp_segment<STENCIL, NW, K, C, REDUCE, STORE, true>(ws, p, su, sg, dst, ja, jb, c0, warp,
                                                             lane, acc_s, acc_m);
      else
        warp_segment<STENCIL, NW, K, C, REDUCE, STORE, false>(ws, p, su, sg, dst, ja, jb, c0, warp,
                                                              lane, acc_s, acc_m);
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
      __threadfence();
    }
  }
}

}  // namespace cjm
