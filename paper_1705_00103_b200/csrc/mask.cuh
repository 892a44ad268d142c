// sm_100a fp64 CJM sweeps with generic masks (
// P:380-418, tab:ste1, tab:ste2): the 5-point mask kernel below, and the
// (2m+1)^2 square-mask kernel (cjm_maskn_kernel, m = 1, 2) further down.
//
// The paper's code takes the Laplacian as a per-node mask of coefficient
// functions (f_W, f_E, f_S, f_N, f_C) so that any orthogonal coordinate system
// (polar, bipolar, ...) runs through the same Jacobi kernel.  Here
// the mask is stored once per plan, already divided by the centre
// coefficient:  a_q = -c_q / c_C (q = W, E, S, N), plus c_C itself for the
// residual, and g = b / c_C replaces b.  One sweep is then, per node,
//     J  = fma(aW, uW, fma(aE, uE, fma(aS, uS, fma(aN, uN, g))))   (DESIGN R10)
//     d  = J - uC,   u' = fma(w, d, uC)
// and the residual of a check launch is r = c_C d (PDE units).
//
// Memory-bound streaming kernel: per node and sweep it reads u (8 B, the four
// neighbours come from L1 / registers), the four a planes and g (40 B) and
// writes u' (8 B): 56 B/LUP (64 B/LUP in check launches, + c_C).  Temporal
// blocking would only save the 16 B of u traffic of the 56 (the coefficients
// must be re-read every sweep), so the kernel runs one sweep per launch.
// Each CTA owns one 256-column strip and a contiguous band of rows (grid =
// strips x bands sized to the persistent CTA count): a thread walks down its
// column keeping uS / uC / uN in registers; the W / E neighbours are loads of
// the same row that the neighbouring lanes also issue (L1 hits).  Same
// device-side n / cur / ticket protocol and fixed-order reduction as the
// Cartesian kernels (sweep.cuh), so it runs inside the same CUDA graphs.
#pragma once

#include "sweep.cuh"

namespace cjm {

struct MaskParams {
  double* buf[2];              // iterate buffers, one ghost ring (H = 1)
  const double* g;             // g = b / c_C, same layout as buf
  const double* a;             // planes aW, aE, aS, aN, cC: node (i, j) at q * plane + j * ld + PADL + i
  long long plane;             // elements per plane
  const double* w;             // weights in application order, P entries
  SweepState* state;
  double* partials;            // 2 doubles per CTA (REDUCE)
  double* result;              // sum r^2, max |r|
  long long P, ld;
  int nx, rows;                // interior columns / rows
  int bands;                   // row bands per column strip
  unsigned int present;        // square masks: bit q set = neighbour plane q present
};

constexpr int MASK_NT = 256;

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Fixed-order reduction of a check launch and the device-side n / cur /
// ticket protocol, common to the mask kernels.
template <bool REDUCE, bool STORE>
__device__ __forceinline__ void mask_finish(const MaskParams& p, unsigned long long n,
                                            unsigned int cur, double acc_s, double acc_m,
                                            double* red_s, double* red_m, int& is_last, int tid,
                                            int lane, int warp) {
  constexpr int NW = MASK_NT / 32;
  if (REDUCE) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc_s = __dadd_rn(acc_s, __shfl_xor_sync(0xffffffffu, acc_s, o));
      acc_m = nan_max(acc_m, __shfl_xor_sync(0xffffffffu, acc_m, o));
    }
    if (lane == 0) { red_s[warp] = acc_s; red_m[warp] = acc_m; }
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
      for (int b = tid; b < (int)gridDim.x; b += MASK_NT) {
        s = __dadd_rn(s, __ldcg(p.partials + 2 * b));
        m = nan_max(m, __ldcg(p.partials + 2 * b + 1));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
        m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
      }
      if (lane == 0) { red_s[warp] = s; red_m[warp] = m; }
      __syncthreads();
      if (tid == 0) {
        s = 0.0; m = 0.0;
        for (int q = 0; q < NW; ++q) { s = __dadd_rn(s, red_s[q]); m = nan_max(m, red_m[q]); }
        p.result[0] = s;
        p.result[1] = m;
      }
    }
    if (tid == 0) {
      if (STORE) {
        p.state->n = n + 1ull;
        p.state->cur = cur ^ 1u;
      }
      p.state->ticket = 0u;
      __threadfence();
    }
  }
}

template <bool REDUCE, bool STORE>
__global__ void __launch_bounds__(MASK_NT) cjm_mask_kernel(const MaskParams p) {
  constexpr int NW = MASK_NT / 32;
  __shared__ double red_s[NW], red_m[NW];
  __shared__ int is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = __ldcg(&p.state->n);
  const unsigned int cur = __ldcg(&p.state->cur);
  const double* src = (cur & 1u) ? p.buf[1] : p.buf[0];
  double* dst = (cur & 1u) ? p.buf[0] : p.buf[1];
  const double w = __ldg(p.w + (long long)(n % (unsigned long long)p.P));
  const long long ld = p.ld;
  double acc_s = 0.0, acc_m = 0.0;

  const int strips = (p.nx + MASK_NT - 1) / MASK_NT;
  const long long units = (long long)strips * p.bands;
  for (long long uu = blockIdx.x; uu < units; uu += gridDim.x) {
    const int strip = (int)(uu % strips), band = (int)(uu / strips);
    const int i = strip * MASK_NT + tid;
    const int ja = (int)((long long)band * p.rows / p.bands);
    const int jb = (int)((long long)(band + 1) * p.rows / p.bands);
    if (i >= p.nx || ja >= jb) continue;
    long long c = (long long)(ja + 1) * ld + PADL + i;   // buf / g index of node (i, ja)
    const double* ak = p.a + (long long)ja * ld + PADL + i;
    double uS = __ldg(src + c - ld), uC = __ldg(src + c);
#pragma unroll 4
    for (int j = ja; j < jb; ++j) {
      const double uN = __ldg(src + c + ld);
      const double uW = __ldg(src + c - 1), uE = __ldg(src + c + 1);
      const double aW = ld_stream(ak), aE = ld_stream(ak + p.plane);
      const double aS = ld_stream(ak + 2 * p.plane), aN = ld_stream(ak + 3 * p.plane);
      const double g = ld_stream(p.g + c);
      const double J = __fma_rn(aW, uW, __fma_rn(aE, uE, __fma_rn(aS, uS, __fma_rn(aN, uN, g))));
      const double d = __dsub_rn(J, uC);
      if (STORE) dst[c] = __fma_rn(w, d, uC);
      if (REDUCE) {
        const double r = __dmul_rn(ld_stream(ak + 4 * p.plane), d);
        acc_s = __fma_rn(r, r, acc_s);
        acc_m = nan_max(acc_m, fabs(r));
      }
      uS = uC;
      uC = uN;
      c += ld;
      ak += ld;
    }
  }

  mask_finish<REDUCE, STORE>(p, n, cur, acc_s, acc_m, red_s, red_m, is_last, tid, lane, warp);
}

// Generic (2MR+1) x (2MR+1) masks (MR = 1: up to 9 points, MR = 2: the most
// generic case of up to 24 neighbours, tab:ste1 / P:385-395).  Planes in mask
// order q = (dy+MR)(2MR+1) + (dx+MR) hold a_q = -c_q / c_C, the centre plane
// holds c_C; absent neighbours (bit q of `present` clear) are neither read nor
// added.  Per node (DESIGN R11):
//   J = fma(a_0, u_0, fma(a_1, u_1, ... fma(a_{Q-1}, u_{Q-1}, g))) over the
//   present q (innermost = largest q),  d = J - uC,  u' = fma(w, d, uC).
// Same streaming organisation as the 5-point kernel: a thread walks down its
// column keeping the (2MR+1) x (2MR+1) window of u in registers (one new row
// of 2MR+1 values per step; the columns of the neighbouring lanes are L1
// hits), the coefficient planes and g are streamed once (HBM-bound:
// 8 (2 + present) + 8 bytes per lattice update).
template <int MR, bool REDUCE, bool STORE>
__global__ void __launch_bounds__(MASK_NT) cjm_maskn_kernel(const MaskParams p) {
  constexpr int NW = MASK_NT / 32;
  constexpr int S = 2 * MR + 1;
  constexpr int QC = MR * S + MR;
  __shared__ double red_s[NW], red_m[NW];
  __shared__ int is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = __ldcg(&p.state->n);
  const unsigned int cur = __ldcg(&p.state->cur);
  const double* src = (cur & 1u) ? p.buf[1] : p.buf[0];
  double* dst = (cur & 1u) ? p.buf[0] : p.buf[1];
  const double w = __ldg(p.w + (long long)(n % (unsigned long long)p.P));
  const long long ld = p.ld;
  const unsigned int present = p.present;
  double acc_s = 0.0, acc_m = 0.0;

  const int strips = (p.nx + MASK_NT - 1) / MASK_NT;
  const long long units = (long long)strips * p.bands;
  for (long long uu = blockIdx.x; uu < units; uu += gridDim.x) {
    const int strip = (int)(uu % strips), band = (int)(uu / strips);
    const int i = strip * MASK_NT + tid;
    const int ja = (int)((long long)band * p.rows / p.bands);
    const int jb = (int)((long long)(band + 1) * p.rows / p.bands);
    if (i >= p.nx || ja >= jb) continue;
    long long c = (long long)(ja + MR) * ld + PADL + i;   // buf / g index of node (i, ja)
    const double* ak = p.a + (long long)ja * ld + PADL + i;
    double win[S][S];                                     // win[dy + MR][dx + MR]
#pragma unroll
    for (int r = 0; r < S - 1; ++r)
#pragma unroll
      for (int x = 0; x < S; ++x) win[r][x] = __ldg(src + c + (long long)(r - MR) * ld + (x - MR));
    for (int j = ja; j < jb; ++j) {
#pragma unroll
      for (int x = 0; x < S; ++x) win[S - 1][x] = __ldg(src + c + (long long)MR * ld + (x - MR));
      // issue every present plane's load before the chain (a load under a
      // branch cannot be hoisted: the loads would serialise on HBM latency)
      double a[S * S];
#pragma unroll
      for (int q = 0; q < S * S; ++q)
        a[q] = (q != QC && (present & (1u << q))) ? ld_stream(ak + q * p.plane) : 0.0;
      double J = ld_stream(p.g + c);
#pragma unroll
      for (int q = S * S - 1; q >= 0; --q) {
        if (q == QC) continue;
        const double t = __fma_rn(a[q], win[q / S][q % S], J);
        J = (present & (1u << q)) ? t : J;
      }
      const double uC = win[MR][MR];
      const double d = __dsub_rn(J, uC);
      if (STORE) dst[c] = __fma_rn(w, d, uC);
      if (REDUCE) {
        const double r = __dmul_rn(ld_stream(ak + QC * p.plane), d);
        acc_s = __fma_rn(r, r, acc_s);
        acc_m = nan_max(acc_m, fabs(r));
      }
#pragma unroll
      for (int r = 0; r < S - 1; ++r)
#pragma unroll
        for (int x = 0; x < S; ++x) win[r][x] = win[r + 1][x];
      c += ld;
      ak += ld;
    }
  }
  mask_finish<REDUCE, STORE>(p, n, cur, acc_s, acc_m, red_s, red_m, is_last, tid, lane, warp);
}

// a_q = -c_q / c_C and c_C into the plan's planes (cjm_mask_set).  The user's
// coefficient arrays are ny x nx of pitch ldc.
__global__ void cjm_mask_prepare_kernel(double* a, long long plane, long long ld, const double* cW,
                                        const double* cE, const double* cS, const double* cN,
                                        const double* cC, long long ldc, int nx, int rows) {
  const long long total = (long long)nx * rows;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / nx, i = e - j * nx;
    const long long k = j * ldc + i;
    const double cc = cC[k];
    double* q = a + j * ld + PADL + i;
    q[0] = __ddiv_rn(-cW[k], cc);
    q[plane] = __ddiv_rn(-cE[k], cc);
    q[2 * plane] = __ddiv_rn(-cS[k], cc);
    q[3 * plane] = __ddiv_rn(-cN[k], cc);
    q[4 * plane] = cc;
  }
}

// Square masks: a_q = -c_q / c_C for the present neighbour planes, c_C into
// the centre plane (cjm_mask_set_n).  User arrays ny x nx of pitch ldc.
struct MaskPlanes {
  const double* c[25];
};

__global__ void cjm_maskn_prepare_kernel(double* a, long long plane, long long ld, MaskPlanes m,
                                         int nplanes, int qc, long long ldc, int nx, int rows) {
  const long long total = (long long)nx * rows;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / nx, i = e - j * nx;
    const long long k = j * ldc + i;
    const double cc = m.c[qc][k];
    double* q = a + j * ld + PADL + i;
    for (int t = 0; t < nplanes; ++t) {
      if (t == qc) q[t * plane] = cc;
      else if (m.c[t]) q[t * plane] = __ddiv_rn(-m.c[t][k], cc);
    }
  }
}

// g = b / c_C in place on the interior of the internal g buffer (row a5 for masks).
__global__ void cjm_mask_scale_kernel(double* g, long long ld, int nx, int rows, const double* cC) {
  const long long total = (long long)nx * rows;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / nx, i = e - j * nx;
    double* q = g + j * ld + PADL + i;
    *q = __ddiv_rn(*q, cC[j * ld + PADL + i]);
  }
}

}  // namespace cjm
