// libcjm: plan, executor and C ABI of the B200-native CJM (include/cjm.h).
//
// Executor (SURVEY section 3 "New build"):
//   setup (row a5)      : u -> both iterate buffers (cudaMemcpy2DAsync into the
//                         pitched, 32-byte aligned internal layout), rhs -> g,
//                         g *= h^2/c_C (cjm_scale_kernel), n = 0
//   sweep 0 + reduction : ||r_0|| (check kernel, one 16-byte D2H, one sync)
//   hot loop            : sweeps 1..P-1 of each cycle replayed from CUDA graphs
//                         of identical sweep launches (each kernel reads n)
//   check sweep n = cP  : fused reduction of u_{cP}, one D2H + sync per cycle,
//                         host stop decision (row a8, DESIGN R4)
//   multi-GPU           : NCCL halo exchange of r rows after every sweep (a9)
//                         and sum/max allreduce of the reduction (a10)
//   generic masks       : cjm_plan_mask + cjm_mask_set (NEXT-4): the same
//                         executor with the per-node mask kernel (mask.cuh)
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "cjm.h"   // include/ (-I)
#include "internal.h"
#include "kernels.h"
#include "resident.cuh"
#include "mask.cuh"

namespace cjm {

// max |u - u_ref| over the interior of an iterate buffer (the paper's "real
// error"), NaN-propagating.  The maximum of non-negative doubles is
// the maximum of their bit patterns, so one atomicMax per warp on the bits is
// exact and order-free.
__global__ void cjm_error_kernel(const double* buf, long long ld, int H, const double* ref,
                                 long long ld_ref, int nx, int rows, unsigned long long* out_bits) {
  const long long total = (long long)nx * rows;
  double m = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / nx, i = e - j * nx;
    const double d = fabs(__dsub_rn(buf[(j + H) * ld + PADL + i], ref[j * ld_ref + i]));
    m = nan_max(m, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(m));
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

// 17-point odd-reflection closure (cjm_options.closure, DESIGN R12): the
// outer ghost ring of the INPUT iterate (buffer state->cur) from the boundary
// nodes and the interior, before every sweep.  0-based interior (i, j) at
// row j + H, column PADL + i; boundary i = -1, nx / j = -1, ny; outer ring
// i = -2, nx+1 / j = -2, ny+1.  Columns (rows -1..ny) first, then rows (all
// columns; the four outer corners reflect the reflected columns, recomputed
// inline with the same operations):  u(mirror) = (2 u_b) - u, 2 u_b exact.
__global__ void cjm_odd_closure_kernel(double* buf0, double* buf1, const SweepState* st,
                                       long long ld, int H, int nx, int ny) {
  double* u = (__ldcg(&st->cur) & 1u) ? buf1 : buf0;
  auto at = [&](int i, int j) -> double& { return u[(long long)(j + H) * ld + PADL + i]; };
  auto refl = [](double ub, double v) { return __dsub_rn(__dmul_rn(2.0, ub), v); };
  const int ncol = ny + 2;            // column phase: rows -1..ny, both sides
  const int nrow = nx + 4;            // row phase: columns -2..nx+1, both sides
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * (ncol + nrow); t += gridDim.x * blockDim.x) {
    if (t < 2 * ncol) {
      const int j = t / 2 - 1;
      if (t & 1) at(nx + 1, j) = refl(at(nx, j), at(nx - 1, j));
      else at(-2, j) = refl(at(-1, j), at(0, j));
    } else {
      const int q = t - 2 * ncol, i = q / 2 - 2;
      const bool bot = q & 1;
      const int jb = bot ? ny : -1, jm = bot ? ny - 1 : 0, jo = bot ? ny + 1 : -2;
      double ub, v;
      if (i == -2) {                  // corner: the column reflection of rows jb and jm
        ub = refl(at(-1, jb), at(0, jb));
        v = refl(at(-1, jm), at(0, jm));
      } else if (i == nx + 1) {
        ub = refl(at(nx, jb), at(nx - 1, jb));
        v = refl(at(nx, jm), at(nx - 1, jm));
      } else {
        ub = at(i, jb);
        v = at(i, jm);
      }
      at(i, jo) = refl(ub, v);
    }
  }
}

}  // namespace cjm

namespace {

thread_local std::string g_last_error;

// CJM_TRACE=1 in the environment: host-side phase timings on stderr
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("CJM_TRACE");
    return e && *e && *e != '0';
  }();
  return on;
}

struct TraceTimer {
  const char* scope;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit TraceTimer(const char* s) : scope(s) {}
  void mark(const char* what) {
    if (!trace_on()) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cjm] %s %-24s %9.3f ms\n", scope, what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

void set_error(const char* what, const char* msg) {
  g_last_error = std::string(what) + ": " + msg;
}

#define CUDA_TRY(expr)                                            \
  do {                                                            \
    cudaError_t e_ = (expr);                                      \
    if (e_ != cudaSuccess) {                                      \
      set_error(#expr, cudaGetErrorString(e_));                   \
      return e_ == cudaErrorMemoryAllocation ? CJM_ERR_OOM : CJM_ERR_CUDA; \
    }                                                             \
  } while (0)

#define NCCL_TRY(expr)                                            \
  do {                                                            \
    ncclResult_t r_ = (expr);                                     \
    if (r_ != ncclSuccess) {                                      \
      set_error(#expr, ncclGetErrorString(r_));                   \
      return CJM_ERR_NCCL;                                        \
    }                                                             \
  } while (0)

#define STATUS_TRY(expr)                  \
  do {                                    \
    cjm_status s_ = (expr);               \
    if (s_ != CJM_OK) return s_;          \
  } while (0)

using cjm::MODE_HOT;
using cjm::MODE_CHECK;
using cjm::MODE_RESID;
using cjm::KernelFn;

// variant 7: the warp-tiled kernel, nw consumer warps per CTA (4, 5, 7 or
// 11); variant 3: the shared-line kernel, NT threads.  The instantiations
// live in kernels_*.cu (compiled in parallel); nullptr = not instantiated.
KernelFn pick_kernel(int stencil, int variant, int NT, int K, int mode, int nw = 4) {
  if (variant == 7) {
    switch (stencil) {
      case 5: return cjm::pick_sweep_v4_5(K, mode, nw);
      case 9: return cjm::pick_sweep_v4_9(K, mode, nw);
      default: return cjm::pick_sweep_v4_17(K, mode, nw);
    }
  }
  return cjm::pick_sweep_v3(stencil, NT, K, mode);
}

// halo columns lost per side by K-1 on-chip levels (mirror of TileGeom::E)
int tile_e(int R, int K) { return K == 1 ? 0 : ((R * (K - 1) + 1) & ~1); }

__global__ void set_state_kernel(cjm::SweepState* st, unsigned long long n) {
  st->n = n;
  st->cur = 0u;
  st->ticket = 0u;
  st->next_chunk = 0u;
}

}  // namespace

// NCCL communicator cache: plans created repeatedly with the same unique id
// (one plan per solve, as bench.py does) reuse the communicator instead of
// paying ncclCommInitRank each time.  cjm_pool_trim destroys them.
namespace {
struct CommKey {
  unsigned char id[128];
  int world, rank, device;
  bool operator<(const CommKey& o) const {
    if (world != o.world) return world < o.world;
    if (rank != o.rank) return rank < o.rank;
    if (device != o.device) return device < o.device;
    return std::memcmp(id, o.id, sizeof(id)) < 0;
  }
};
std::mutex g_comm_mu;
std::map<CommKey, std::pair<ncclComm_t, int>> g_comms;   // comm, plans using it
}  // namespace

struct cjm_plan_s {
  // problem
  int stencil = 9, R = 1, nx = 0, ny = 0, y0 = 0, ny_local = 0;
  // ghost rows: H stored above / below the slab in buf and G (r, or K r for
  // multi-GPU deep halos); Hu of them in the user's u, Hr in the user's rhs;
  // local rows [row_lo, row_hi) are interior rows of the global grid
  int H = 1, Hu = 1, Hr = 0, row_lo = 0, row_hi = 0;
  double h = 0, tol = 0, gscale = 0;
  int method = CJM_METHOD_CHEBYSHEV, max_cycles = 8;
  cjm::Schedule sched;
  long long P = 0;
  // distribution
  int world = 1, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  // device memory
  long long ld = 0;
  size_t buf_elems = 0, g_elems = 0;
  double* buf[2] = {nullptr, nullptr};
  double* G = nullptr;
  double* w_dev = nullptr;
  // generic 5-point mask (NEXT-4): planes aW, aE, aS, aN, cC of ny x ld
  double* A = nullptr;
  size_t a_elems = 0;
  int mask_ready = 0, bands = 1;
  int mask_r = 0;              // 0: 5-point cross (cjm_plan_mask); 1, 2: (2m+1)^2 masks
  int nplanes = 5;             // coefficient planes stored (a_q ..., c_C)
  int mask_qc = 4;             // plane holding c_C
  unsigned int present = 0;    // square masks: neighbour planes present
  double* partials = nullptr;
  double* result = nullptr;
  double* result_host = nullptr;  // pinned, 2 doubles
  cjm::SweepState* state = nullptr;
  unsigned long long* err_bits = nullptr;   // real-error reduction (cjm_solve_ref)
  unsigned long long* dbg = nullptr;        // CJM_DEBUG_CHECKS: violation count, first code
  void* small_block = nullptr;              // partials | result | state | err_bits
  size_t small_bytes = 0;
  // launch configuration
  int NT = 128, K = 1, stages = 8, nctas = 0, ctas_per_sm = 2, graph_chunk = 64;
  int variant = 7;   // 3: shared-line levels (sweep.cuh), 7: warp-tiled (sweep_v4.cuh)
  int nw = 4;        // consumer warps per CTA (warp-tiled)
  int chunk_rows = -1;  // warp-tiled hot launches: rows per dynamically scheduled work item
                        // (0: static ranges, -1: chosen per launch)
  int dyn_pct = 20;     // percent of the units scheduled dynamically (CJM_DYN_PCT)
  int band_split = 0;  // split hot sweeps into boundary / interior bands even without NCCL
  int closure = CJM_CLOSURE_DIRICHLET;   // 17-point outer ghost ring (DESIGN R12)
  // resident (whole grid in shared memory) hot path
  int resident = 0, res_ctas = 0, res_rows = 0;
  size_t res_smem = 0;
  double* res_halo = nullptr;
  unsigned int* res_flags = nullptr;
  size_t res_halo_bytes = 0;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t comm_stream = nullptr;               // multi-GPU halo exchange
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::map<std::pair<long long, int>, cudaGraphExec_t> graphs;
  std::map<std::pair<long long, int>, long long> graph_kernels;   // kernels per graph
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double plan_s = 0;
  // host mirror of the device state during a call
  int host_cur = 0;
  long long launches = 0;
};

namespace {

// warp-tiled kernel: 2 columns per lane, 2r+1 input rows per TMA ring stage
constexpr int V4_CPL = 2;
int v4_rps(int R) { return 2 * R + 1; }

int v4_tout(int R, int K, int C, int nw) {   // owned columns per CTA strip, warp-tiled variant
  const int E = K == 1 ? 0 : ((R * (K - 1) + 1) & ~1);
  return nw * (32 * C - 2 * E);
}

int tile_out(const cjm_plan_s* pl, int K) {
  if (pl->variant == 7) return v4_tout(pl->R, K, V4_CPL, pl->nw);
  return 2 * pl->NT - 2 * tile_e(pl->R, K);
}

size_t smem_bytes(const cjm_plan_s* pl, int K) {
  if (pl->variant == 7) {
    const int C = V4_CPL;
    const int E = K == 1 ? 0 : ((pl->R * (K - 1) + 1) & ~1);
    const int WOUT = 32 * C - 2 * E;
    const int TG = (pl->nw - 1) * WOUT + 32 * C;
    const int ROW = (TG + 4 + 7) / 8 * 8, GROW = (TG + 7) / 8 * 8;
    return (size_t)pl->stages * v4_rps(pl->R) * (ROW + GROW) * sizeof(double) +
           2 * (size_t)pl->stages * sizeof(uint64_t);
  }
  const int T = 2 * pl->NT, ROW = T + 8;
  return (size_t)pl->stages * (ROW + T) * sizeof(double) +
         (size_t)(K - 1) * (2 * pl->R + 1) * ROW * sizeof(double) +
         2 * (size_t)pl->stages * sizeof(uint64_t);
}

int block_threads(const cjm_plan_s* pl) { return pl->variant == 7 ? pl->nw * 32 + 32 : pl->NT + 32; }

// One sweep-kernel launch of K fused sweeps reading buffer host_cur.
// One sweep-kernel launch of K fused sweeps reading buffer host_cur, over the
// output rows [row0, row0 + nrows) of the slab (default: all of them).  Only
// a launch with advance = 1 moves the device-side n / cur (the last launch of
// a sweep that is split into bands).
template <int MR>
void launch_maskn(int mode, int grid, cudaStream_t st, const cjm::MaskParams& mp) {
  switch (mode) {
    case MODE_HOT: cjm::cjm_maskn_kernel<MR, false, true><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
    case MODE_CHECK: cjm::cjm_maskn_kernel<MR, true, true><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
    default: cjm::cjm_maskn_kernel<MR, true, false><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
  }
}

cjm_status launch_mask(cjm_plan_s* pl, int mode, cudaStream_t st) {
  cjm::MaskParams mp;
  mp.buf[0] = pl->buf[0];
  mp.buf[1] = pl->buf[1];
  mp.g = pl->G;
  mp.a = pl->A;
  mp.plane = (long long)pl->a_elems / pl->nplanes;
  mp.present = pl->present;
  mp.w = pl->w_dev;
  mp.state = pl->state;
  mp.partials = pl->partials;
  mp.result = pl->result;
  mp.P = pl->P;
  mp.ld = pl->ld;
  mp.nx = pl->nx;
  mp.rows = pl->ny_local;
  mp.bands = pl->bands;
  const long long strips = (pl->nx + cjm::MASK_NT - 1) / cjm::MASK_NT;
  const int grid = (int)std::min<long long>(pl->nctas, strips * pl->bands);
switch (pl->mask_r) {
    case 1: launch_maskn<1>(mode, grid, st, mp); break;
    case 2: launch_maskn<2>(mode, grid, st, mp); break;
    default:
      switch (mode) {
        case MODE_HOT: cjm::cjm_mask_kernel<false, true><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
        case MODE_CHECK: cjm::cjm_mask_kernel<true, true><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
        default: cjm::cjm_mask_kernel<true, false><<<grid, cjm::MASK_NT, 0, st>>>(mp); break;
      }
  }
  CUDA_TRY(cudaGetLastError());
  pl->launches += 1;
  if (mode != MODE_RESID) pl->host_cur ^= 1;
  return CJM_OK;
}

cjm_status launch_sweep(cjm_plan_s* pl, int mode, int K, cudaStream_t st, int row0 = 0,
                        int nrows = -1, int advance = 1) {
  if (pl->stencil == CJM_STENCIL_MASK) return launch_mask(pl, mode, st);   // K = 1, one band
  if (pl->closure == CJM_CLOSURE_ODD) {   // K = 1, one band, one GPU: reflect the input's outer ring
    const int n = 2 * (pl->ny + 2) + 2 * (pl->nx + 4);
    cjm::cjm_odd_closure_kernel<<<(n + 255) / 256, 256, 0, st>>>(pl->buf[0], pl->buf[1], pl->state,
                                                                 pl->ld, pl->H, pl->nx, pl->ny);
    CUDA_TRY(cudaGetLastError());
    pl->launches += 1;
  }
  if (nrows < 0) nrows = pl->ny_local;
  cjm::SweepParams sp;
  sp.buf[0] = pl->buf[0];
  sp.buf[1] = pl->buf[1];
  sp.g = pl->G;
  sp.w = pl->w_dev;
  sp.state = pl->state;
  sp.partials = pl->partials;
  sp.result = pl->result;
  sp.P = pl->P;
  sp.ld = pl->ld;
  sp.nx = pl->nx;
  sp.rows = pl->ny_local;
  sp.H = pl->H;
  sp.row_lo = pl->row_lo;
  sp.row_hi = pl->row_hi;
  sp.row0 = row0;
  sp.nrows = nrows;
  sp.stages = pl->stages;
  sp.advance = advance;
  const int tout = tile_out(pl, K);
  const long long nstrips = (pl->nx + tout - 1) / tout;
  sp.units = nstrips * nrows;
  const int grid = (int)std::min<long long>(pl->nctas, sp.units);
  // Dynamic balancing for hot launches of the warp-tiled kernels only (a
  // reducing launch keeps static per-CTA ranges: bitwise-reproducible sums):
  // a static per-CTA range over the first 80% of the units, the last 20% in
  // work items of 1/8 of a CTA's share (16..128 units) from a device counter
  // -- the CTAs on faster SMs take more of them.  Each item re-reads and
  // recomputes 2 K r halo rows.  Measured (profiles/r01_v7_chunks.jsonl): 9-pt
  // K=4 at 4096^2 24.0 vs 26.6 us per sweep static, 16384^2 325 vs 425.
  int chunk = 0;
  long long ustat = sp.units;
  const long long per_cta = sp.units / std::max(grid, 1);
  if (mode == MODE_HOT && pl->variant == 7 &&
      (pl->chunk_rows > 0 || (pl->chunk_rows < 0 && per_cta >= 64))) {
    // (auto: small grids, e.g. 1024^2 with 14 rows per CTA, stay static --
    // 21.3 vs 27.7 ms per 9-point solve)
    chunk = pl->chunk_rows > 0 ? pl->chunk_rows
                               : (int)std::max<long long>(16, std::min<long long>(128, per_cta / 8));
    ustat = sp.units - sp.units * pl->dyn_pct / 100;
  }
  sp.chunk_rows = chunk;
  sp.units_static = ustat;
  sp.buf_elems = (long long)pl->buf_elems;
#ifdef CJM_DEBUG_CHECKS
  sp.dbg = pl->dbg;
  // negative control of the checks: CJM_DEBUG_INJECT=1 understates the buffer
  // size, so the TMA bounds checks must fire (scripts/sanitize_cases.py --inject)
  static const bool inject = std::getenv("CJM_DEBUG_INJECT") != nullptr;
  if (inject) sp.buf_elems /= 2;
#else
  sp.dbg = nullptr;
#endif
  KernelFn k = pick_kernel(pl->stencil, pl->variant, pl->NT, K, mode, pl->nw);
  k<<<grid, block_threads(pl), smem_bytes(pl, K), st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  pl->launches += 1;
  if (mode != MODE_RESID && advance) pl->host_cur ^= 1;
  return CJM_OK;
}

// Halo exchange of the iterate buffer `b` (row a9), one grouped NCCL
// send/recv per neighbour as laid out by cjm_halo_plan.  Rows are contiguous
// (r rows x ld doubles, ghost columns included: they hold the same Dirichlet
// data on both ranks).
cjm_status halo_exchange(cjm_plan_s* pl, double* b, cudaStream_t st) {
  if (!pl->comm) return CJM_OK;   // single GPU, or external_halo: the caller moves them
  // the element-level transfer list of cjm_halo_xfers, executed verbatim (a
  // one-rank communicator has none: an empty NCCL group)
  cjm_halo_xfer xs[2];
  int nx_ = 0;
  long long ld = 0;
  if (pl->world > 1) STATUS_TRY(cjm_halo_xfers(pl->nx, pl->ny, pl->H, pl->world, pl->rank, xs, &nx_, &ld));
  NCCL_TRY(ncclGroupStart());
  for (int k = 0; k < nx_; ++k) {
    NCCL_TRY(ncclSend(b + xs[k].send_off, (size_t)xs[k].count, ncclDouble, xs[k].peer, pl->comm, st));
    NCCL_TRY(ncclRecv(b + xs[k].recv_off, (size_t)xs[k].count, ncclDouble, xs[k].peer, pl->comm, st));
  }
  NCCL_TRY(ncclGroupEnd());
  return CJM_OK;
}

// A sweep launch followed by the halo exchange of its output (multi-GPU).
// Hot sweeps with a communicator overlap the exchange with the interior
// (SURVEY 8(e)): the 2r boundary rows are computed first (two small band
// launches), the NCCL exchange of those rows runs on the plan's comm stream
// while the interior band runs on the main stream, and the main stream waits
// for the exchange before the next sweep.  The interior launch is the one
// that advances n / cur.  Check sweeps (the reduction must cover every row of
// one launch) are not split.
cjm_status sweep_and_exchange(cjm_plan_s* pl, int mode, int K, cudaStream_t st) {
  const int Hh = pl->H, nyl = pl->ny_local;
  if (mode == MODE_HOT && (pl->comm || pl->band_split) && nyl > 4 * Hh) {
    // the neighbours need my first / last H rows (H = K r: the deep halo of a
    // K-fused launch)
    STATUS_TRY(launch_sweep(pl, mode, K, st, 0, Hh, 0));
    STATUS_TRY(launch_sweep(pl, mode, K, st, nyl - Hh, Hh, 0));
    double* out = pl->buf[pl->host_cur ^ 1];    // the buffer this sweep writes
    CUDA_TRY(cudaEventRecord(pl->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(pl->comm_stream, pl->ev_fork, 0));
    STATUS_TRY(halo_exchange(pl, out, pl->comm_stream));
    CUDA_TRY(cudaEventRecord(pl->ev_join, pl->comm_stream));
    STATUS_TRY(launch_sweep(pl, mode, K, st, Hh, nyl - 2 * Hh, 1));
    CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_join, 0));
    return CJM_OK;
  }
  STATUS_TRY(launch_sweep(pl, mode, K, st));
  return halo_exchange(pl, pl->buf[pl->host_cur], st);
}

// Graph of `len` hot launches of K sweeps each.  Single GPU: every launch has
// identical parameters (buffers resolved on the device), one graph per length.
// Multi-GPU: the NCCL buffers depend on the starting buffer parity.
cjm_status get_graph(cjm_plan_s* pl, long long len, int K, cudaGraphExec_t* out,
                     long long* kernels) {
  const int par = pl->comm ? pl->host_cur : 0;
  const std::pair<long long, int> key{len * 8 + K, par};
  auto it = pl->graphs.find(key);
  if (it != pl->graphs.end()) {
    *out = it->second;
    *kernels = pl->graph_kernels[key];
    return CJM_OK;
  }
  const int saved_cur = pl->host_cur;
  const long long saved_launches = pl->launches;
  TraceTimer tt("graph");
  cudaGraph_t graph = nullptr;
  CUDA_TRY(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
  cjm_status s = CJM_OK;
  for (long long k = 0; k < len && s == CJM_OK; ++k) s = sweep_and_exchange(pl, MODE_HOT, K, pl->cap_stream);
  cudaError_t e = cudaStreamEndCapture(pl->cap_stream, &graph);
  pl->host_cur = saved_cur;
  const long long captured = pl->launches - saved_launches;
  pl->launches = saved_launches;
  if (s != CJM_OK) { if (graph) cudaGraphDestroy(graph); return s; }
  CUDA_TRY(e);
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CUDA_TRY(e);
  pl->graphs[key] = exec;
  pl->graph_kernels[key] = captured;
  tt.mark("capture+instantiate");
  *out = exec;
  *kernels = captured;
  return CJM_OK;
}

// Run `count` hot sweeps: blocks of K fused sweeps from CUDA graphs, the
// remainder (< K) as single-sweep launches.  Returns the hot launch count.
using ResidentFn = void (*)(const cjm::ResidentParams);

ResidentFn pick_resident(int stencil) {
  switch (stencil) {
    case 5: return cjm::cjm_resident_kernel<5>;
    case 9: return cjm::cjm_resident_kernel<9>;
    default: return cjm::cjm_resident_kernel<17>;
  }
}

// `count` sweeps in ONE cooperative launch with the grid resident in shared
// memory (resident.cuh); reads buffer host_cur, writes host_cur ^ 1.
cjm_status run_resident(cjm_plan_s* pl, long long count, cudaStream_t st) {
  cjm::ResidentParams rp;
  rp.buf[0] = pl->buf[0];
  rp.buf[1] = pl->buf[1];
  rp.g = pl->G;
  rp.w = pl->w_dev;
  rp.state = pl->state;
  rp.halo = pl->res_halo;
  rp.flags = pl->res_flags;
  rp.P = pl->P;
  rp.ld = pl->ld;
  rp.nx = pl->nx;
  rp.rows = pl->ny_local;
  rp.count = (int)count;
  rp.rows_per_cta = pl->res_rows;
  rp.buf_elems = (long long)pl->buf_elems;
  rp.halo_elems = (long long)(pl->res_halo_bytes / sizeof(double));
#ifdef CJM_DEBUG_CHECKS
  rp.dbg = pl->dbg;
#else
  rp.dbg = nullptr;
#endif
  CUDA_TRY(cudaMemsetAsync(pl->res_flags, 0, (size_t)pl->res_ctas * sizeof(unsigned int), st));
  void* args[] = {&rp};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)pick_resident(pl->stencil), dim3(pl->res_ctas),
                                       dim3(512), args, pl->res_smem, st));
  pl->launches += 1;
  pl->host_cur ^= 1;
  return CJM_OK;
}

// Run `count` hot sweeps: blocks of K fused sweeps from CUDA graphs, the
// remainder (< K) as single-sweep launches -- or, for grids resident in
// shared memory, one cooperative launch.  Counts hot launches.
cjm_status run_hot(cjm_plan_s* pl, long long count, cudaStream_t st, long long* hot_launches) {
  if (pl->resident && count >= 8 && count < (1LL << 31)) {
    STATUS_TRY(run_resident(pl, count, st));
    *hot_launches += 1;
    return CJM_OK;
  }
  const int K = pl->K;
  long long blocks = count / K;
  const long long rem = count % K;
  while (blocks > 0) {
    const long long len = std::min<long long>(pl->graph_chunk, blocks);
    cudaGraphExec_t ex;
    long long kernels = 0;
    STATUS_TRY(get_graph(pl, len, K, &ex, &kernels));
    CUDA_TRY(cudaGraphLaunch(ex, st));
    pl->host_cur ^= (int)(len & 1);
    pl->launches += kernels;
    *hot_launches += len;
    blocks -= len;
  }
  for (long long r = 0; r < rem; ++r) {
    STATUS_TRY(sweep_and_exchange(pl, MODE_HOT, 1, st));
    *hot_launches += 1;
  }
  return CJM_OK;
}

// Sum / max over ranks of the reduction result and D2H of the two scalars.
cjm_status fetch_result(cjm_plan_s* pl, cudaStream_t st, double* s, double* m) {
  if (pl->comm) {
    NCCL_TRY(ncclGroupStart());
    NCCL_TRY(ncclAllReduce(pl->result, pl->result, 1, ncclDouble, ncclSum, pl->comm, st));
    NCCL_TRY(ncclAllReduce(pl->result + 1, pl->result + 1, 1, ncclDouble, ncclMax, pl->comm, st));
    NCCL_TRY(ncclGroupEnd());
  }
  CUDA_TRY(cudaMemcpyAsync(pl->result_host, pl->result, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *s = pl->result_host[0];
  *m = pl->result_host[1];
  return CJM_OK;
}

// max |u_which - u_ref| over the (global) interior.
cjm_status real_error(cjm_plan_s* pl, int which, const double* ref, long long ld_ref,
                      cudaStream_t st, double* err) {
  CUDA_TRY(cudaMemsetAsync(pl->err_bits, 0, sizeof(unsigned long long), st));
  const long long total = (long long)pl->nx * pl->ny_local;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
  cjm::cjm_error_kernel<<<blocks, 256, 0, st>>>(pl->buf[which], pl->ld, pl->H, ref, ld_ref, pl->nx,
                                                pl->ny_local, pl->err_bits);
  CUDA_TRY(cudaGetLastError());
  pl->launches += 1;
  if (pl->comm) {
    double* d = reinterpret_cast<double*>(pl->err_bits);
    NCCL_TRY(ncclAllReduce(d, d, 1, ncclDouble, ncclMax, pl->comm, st));
  }
  CUDA_TRY(cudaMemcpyAsync(pl->result_host, pl->err_bits, sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *err = pl->result_host[0];
  return CJM_OK;
}

cjm_status set_state(cjm_plan_s* pl, unsigned long long n, cudaStream_t st) {
  set_state_kernel<<<1, 1, 0, st>>>(pl->state, n);
  CUDA_TRY(cudaGetLastError());
  pl->host_cur = 0;
  pl->launches += 1;
  return CJM_OK;
}

// Row a5: user layout -> internal buffers.  kind = H2D or D2D.  The user's u
// carries Hu ghost rows (r, or K r for external-halo deep halos) and r ghost
// columns; rhs carries Hr extra rows (0, or H for external-halo deep halos).
cjm_status stage_in(cjm_plan_s* pl, const double* rhs, long long ld_rhs, const double* u,
                    long long ld_u, bool both, cudaMemcpyKind kind, cudaStream_t st) {
  const int R = pl->R;
  const size_t upitch = (size_t)pl->ld * sizeof(double);
  CUDA_TRY(cudaMemcpy2DAsync(pl->buf[0] + (long long)(pl->H - pl->Hu) * pl->ld + (cjm::PADL - R), upitch,
                             u, (size_t)ld_u * sizeof(double),
                             (size_t)(pl->nx + 2 * R) * sizeof(double),
                             (size_t)(pl->ny_local + 2 * pl->Hu), kind, st));
  if (both)
    CUDA_TRY(cudaMemcpyAsync(pl->buf[1], pl->buf[0], pl->buf_elems * sizeof(double),
                             cudaMemcpyDeviceToDevice, st));
  if (rhs) {
    double* g0 = pl->G + (long long)(pl->H - pl->Hr) * pl->ld;
    const int grows = pl->ny_local + 2 * pl->Hr;
    CUDA_TRY(cudaMemcpy2DAsync(g0 + cjm::PADL, upitch, rhs, (size_t)ld_rhs * sizeof(double),
                               (size_t)pl->nx * sizeof(double), (size_t)grows, kind, st));
    const long long total = (long long)pl->nx * grows;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    if (pl->stencil == CJM_STENCIL_MASK)   // g = b / c_C
      cjm::cjm_mask_scale_kernel<<<blocks, 256, 0, st>>>(
          g0, pl->ld, pl->nx, grows, pl->A + pl->mask_qc * (pl->a_elems / pl->nplanes));
    else
      cjm::cjm_scale_kernel<<<blocks, 256, 0, st>>>(g0, pl->ld, pl->nx, grows, pl->gscale);
    CUDA_TRY(cudaGetLastError());
    pl->launches += 1;
    // NCCL plans with deep halos: the neighbours' g rows (once per solve)
    if (pl->comm && pl->H > pl->R) STATUS_TRY(halo_exchange(pl, pl->G, st));
  }
  return CJM_OK;
}

cjm_status stage_out(cjm_plan_s* pl, int which, double* u, long long ld_u, cudaMemcpyKind kind,
                     cudaStream_t st) {
  const int R = pl->R;
  CUDA_TRY(cudaMemcpy2DAsync(u + (long long)pl->Hu * ld_u + R, (size_t)ld_u * sizeof(double),
                             pl->buf[which] + (long long)pl->H * pl->ld + cjm::PADL,
                             (size_t)pl->ld * sizeof(double), (size_t)pl->nx * sizeof(double),
                             (size_t)pl->ny_local, kind, st));
  return CJM_OK;
}

bool check_layout(const cjm_plan_s* pl, const void* rhs, long long ld_rhs, const void* u,
                  long long ld_u) {
  return pl && u && ld_u >= pl->nx + 2 * pl->R && (!rhs || ld_rhs >= pl->nx) &&
         (pl->stencil != CJM_STENCIL_MASK || pl->mask_ready);   // cjm_mask_set first
}

// CJM_DEBUG_CHECKS builds: a non-zero device violation count (bounds checks
// of the sweep kernel, sweep.cuh CheckCode) fails the call.
cjm_status debug_verify(cjm_plan_s* pl) {
#ifdef CJM_DEBUG_CHECKS
  unsigned long long h[2] = {0, 0};
  CUDA_TRY(cudaMemcpy(h, pl->dbg, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[0]) {
    char msg[128];
    std::snprintf(msg, sizeof(msg), "%llu bounds-check violations, first code %llu", h[0], h[1]);
    set_error("CJM_DEBUG_CHECKS", msg);
    return CJM_ERR_CUDA;
  }
#else
  (void)pl;
#endif
  return CJM_OK;
}

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e-3;
}

void fill_static(const cjm_plan_s* pl, cjm_report* r) {
  std::memset(r, 0, sizeof(*r));
  r->cycle_len = pl->P;
  r->m_min = pl->sched.m_min;
  r->kappa_min = pl->sched.kmin;
  r->kappa_max = pl->sched.kmax;
  r->plan_s = pl->plan_s;
  r->temporal_k = pl->K;
  r->resident = pl->resident;
  r->variant = pl->variant;
  r->warps = pl->variant == 7 ? pl->nw : pl->NT / 32;
  r->stages = pl->stages;
  r->ctas = pl->nctas;
  r->ghost_rows = pl->Hu;
  r->rhs_ghost_rows = pl->Hr;
  if (pl->comm) {
    ncclCommCount(pl->comm, &r->comm_nranks);
    ncclCommUserRank(pl->comm, &r->comm_rank);
  } else {
    r->comm_nranks = 0;
    r->comm_rank = -1;
  }
}

// The whole solve (rows a5-a10); `kin` / `kout` select device or host user buffers.
cjm_status solve_impl(cjm_plan_s* pl, const double* rhs, long long ld_rhs, double* u,
                      long long ld_u, cudaMemcpyKind kin, cudaMemcpyKind kout, void* stream,
                      cjm_report* rep_out, const double* ref = nullptr, long long ld_ref = 0,
                      double real_tol = 0.0) {
  if (!check_layout(pl, rhs, ld_rhs, u, ld_u) || !rhs ||
      (ref && (ld_ref < pl->nx || !(real_tol > 0.0)))) {
    set_error("cjm_solve", "invalid pointer or pitch");
    return CJM_ERR_INVALID_ARG;
  }
  if (pl->world > 1 && !pl->comm) {
    set_error("cjm_solve", "external_halo plans run cjm_sweeps / cjm_residual only");
    return CJM_ERR_UNSUPPORTED;
  }
  CUDA_TRY(cudaSetDevice(pl->device));
  cudaStream_t st = (cudaStream_t)stream;
  cjm_report rep;
  fill_static(pl, &rep);
  const double sc = std::fabs(pl->gscale);
  pl->launches = 0;
  // the check launch fuses Kc sweeps (K, or 1 when a cycle is shorter than K:
  // only K and 1 are configured launches); the hot part of a cycle is P - Kc
  const int Kc = pl->P >= pl->K ? pl->K : 1;

  CUDA_TRY(cudaEventRecord(pl->ev[0], st));
  STATUS_TRY(stage_in(pl, rhs, ld_rhs, u, ld_u, true, kin, st));
  if (kin == cudaMemcpyHostToDevice) {
    rep.h2d_bytes = (double)(pl->ny_local + 2 * pl->Hu) * (pl->nx + 2 * pl->R) * 8.0 +
                    (double)(pl->ny_local + 2 * pl->Hr) * pl->nx * 8.0;
  }
  STATUS_TRY(set_state(pl, 0ull, st));
  STATUS_TRY(halo_exchange(pl, pl->buf[0], st));

  double s, m;
  int check_in = pl->host_cur;           // buffer holding u_0
  STATUS_TRY(sweep_and_exchange(pl, MODE_CHECK, Kc, st));
  STATUS_TRY(fetch_result(pl, st, &s, &m));
  rep.r0_l2 = std::sqrt(s) / sc;
  rep.r0_linf = m / sc;
  rep.r_l2 = rep.r0_l2;
  rep.r_linf = rep.r0_linf;
  double err = 0.0;
  if (ref) {
    STATUS_TRY(real_error(pl, check_in, ref, ld_ref, st, &err));
    rep.real_error = err;
  }

  int status = CJM_ERR_NOT_CONVERGED;
  int out_buf = check_in;                 // buffer of the exported iterate
  if (ref ? err <= real_tol : rep.r0_l2 == 0.0) {
    status = CJM_OK;
  } else if (!std::isfinite(rep.r0_l2)) {
    status = CJM_ERR_DIVERGED;
  } else {
    double rho_prev = rep.r0_l2;
    for (int c = 1; c <= pl->max_cycles; ++c) {
      CUDA_TRY(cudaEventRecord(pl->ev[2], st));
      STATUS_TRY(run_hot(pl, pl->P - Kc, st, &rep.hot_launches));
      CUDA_TRY(cudaEventRecord(pl->ev[3], st));
      check_in = pl->host_cur;            // holds u_{cP}
      STATUS_TRY(sweep_and_exchange(pl, MODE_CHECK, Kc, st));
      STATUS_TRY(fetch_result(pl, st, &s, &m));
      rep.sweep_s += elapsed_s(pl->ev[2], pl->ev[3]);
      rep.sweeps_timed += pl->P - Kc;
      const double rho = std::sqrt(s) / sc;
      rep.cycles = c;
      rep.iterations = (long long)c * pl->P;
      rep.r_l2 = rho;
      rep.r_linf = m / sc;
      out_buf = check_in;
      if (!std::isfinite(rho)) { status = CJM_ERR_DIVERGED; break; }
      if (ref) {   // the paper's real-error stop, checked per cycle
        STATUS_TRY(real_error(pl, check_in, ref, ld_ref, st, &err));
        rep.real_error = err;
        if (err <= real_tol) { status = CJM_OK; break; }
      } else if (rho <= pl->tol * rep.r0_l2) {
        status = CJM_OK;
        break;
      }
      if (pl->method == CJM_METHOD_CHEBYSHEV && rho > 0.5 * rho_prev) {
        status = CJM_ERR_STAGNATED;
        break;
      }
      rho_prev = rho;
    }
  }
  STATUS_TRY(stage_out(pl, out_buf, u, ld_u, kout, st));
  if (kout == cudaMemcpyDeviceToHost) rep.d2h_bytes = (double)pl->ny_local * pl->nx * 8.0;
  CUDA_TRY(cudaEventRecord(pl->ev[1], st));
  CUDA_TRY(cudaEventSynchronize(pl->ev[1]));
  rep.solve_s = elapsed_s(pl->ev[0], pl->ev[1]);
  rep.kernel_launches = pl->launches;
  rep.status = status;
  if (rep_out) *rep_out = rep;
  STATUS_TRY(debug_verify(pl));
  return (cjm_status)status;
}

}  // namespace

// =========================================================================
// C ABI
// =========================================================================
extern "C" {

void cjm_default_options(cjm_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->max_cycles = 0;   // method-dependent default
  o->order = CJM_ORDER_LEBEDEV23;
  o->method = CJM_METHOD_CHEBYSHEV;
  o->jacobi_check = 1024;
  o->world_size = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->device = -1;
}

cjm_status cjm_schedule(int stencil, int nx, int ny, double tol, int order, double* kappa_min,
                        double* kappa_max, long long* m_min, long long* cycle_len,
                        long long* t_out, double* w_out, long long capacity) {
  if (!cjm::stencil_reach(stencil) || nx < 4 || ny < 4 || !(tol > 0.0 && tol < 1.0) ||
      (order != CJM_ORDER_LEBEDEV23 && order != CJM_ORDER_ASCENDING && order != CJM_ORDER_LEBEDEV2)) {
    set_error("cjm_schedule", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  cjm::Schedule s;
  if (!cjm::build_schedule(stencil, nx, ny, tol, order, &s)) return CJM_ERR_INVALID_ARG;
  if (kappa_min) *kappa_min = s.kmin;
  if (kappa_max) *kappa_max = s.kmax;
  if (m_min) *m_min = s.m_min;
  if (cycle_len) *cycle_len = s.P;
  if (t_out || w_out) {
    if (capacity < s.P) {
      set_error("cjm_schedule", "capacity < cycle length");
      return CJM_ERR_INVALID_ARG;
    }
    for (long long k = 0; k < s.P; ++k) {
      if (t_out) t_out[k] = s.t[k];
      if (w_out) w_out[k] = s.w[k];
    }
  }
  return CJM_OK;
}

cjm_status cjm_slab(int ny, int world_size, int rank, int* y0, int* ny_local) {
  if (ny < 1 || world_size < 1 || rank < 0 || rank >= world_size) return CJM_ERR_INVALID_ARG;
  const long long a = (long long)rank * ny / world_size;
  const long long b = (long long)(rank + 1) * ny / world_size;
  if (y0) *y0 = (int)a;
  if (ny_local) *ny_local = (int)(b - a);
  return CJM_OK;
}

cjm_status cjm_halo_plan(int ny, int r, int world_size, int rank, cjm_halo_msg* msgs,
                         int* nmsgs) {
  int y0 = 0, nyl = 0;
  if (!msgs || !nmsgs || r < 1 || r > 16 || cjm_slab(ny, world_size, rank, &y0, &nyl) != CJM_OK ||
      (world_size > 1 && nyl < 2 * r + 1)) {
    set_error("cjm_halo_plan", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  int n = 0;
  if (rank > 0) {                    // neighbour above: lower global rows
    msgs[n].peer = rank - 1;
    msgs[n].send_row = r;            // my first r interior rows
    msgs[n].recv_row = 0;            // into my first r ghost rows
    msgs[n].rows = r;
    ++n;
  }
  if (rank < world_size - 1) {       // neighbour below: higher global rows
    msgs[n].peer = rank + 1;
    msgs[n].send_row = nyl;          // my last r interior rows (r + nyl - r)
    msgs[n].recv_row = nyl + r;      // into my last r ghost rows
    msgs[n].rows = r;
    ++n;
  }
  *nmsgs = n;
  return CJM_OK;
}

cjm_status cjm_buffer_layout(int nx, long long* ld, int* col0) {
  if (nx < 1) return CJM_ERR_INVALID_ARG;
  if (ld) *ld = ((long long)nx + 2 * cjm::PADL + 31) / 32 * 32;
  if (col0) *col0 = cjm::PADL;
  return CJM_OK;
}

cjm_status cjm_halo_xfers(int nx, int ny, int depth, int world_size, int rank, cjm_halo_xfer* xfers,
                          int* nxfers, long long* ld_out) {
  cjm_halo_msg msgs[2];
  int nm = 0;
  long long ld = 0;
  if (!xfers || !nxfers || cjm_buffer_layout(nx, &ld, nullptr) != CJM_OK) {
    set_error("cjm_halo_xfers", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  STATUS_TRY(cjm_halo_plan(ny, depth, world_size, rank, msgs, &nm));
  for (int k = 0; k < nm; ++k) {
    xfers[k].peer = msgs[k].peer;
    xfers[k].send_off = (long long)msgs[k].send_row * ld;
    xfers[k].recv_off = (long long)msgs[k].recv_row * ld;
    xfers[k].count = (long long)msgs[k].rows * ld;   // whole rows, ghost columns included
  }
  *nxfers = nm;
  if (ld_out) *ld_out = ld;
  return CJM_OK;
}

cjm_status cjm_get_nccl_id(void* out128) {
  if (!out128) return CJM_ERR_INVALID_ARG;
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return CJM_OK;
}

cjm_status cjm_plan_destroy(cjm_plan_t p) {
  if (!p) return CJM_OK;
  TraceTimer tt("destroy");
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  tt.mark("device sync");
  for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
  p->graphs.clear();
  p->graph_kernels.clear();
  tt.mark("graph exec destroy");
  for (auto& e : p->ev) if (e) cudaEventDestroy(e);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->comm_stream) cudaStreamDestroy(p->comm_stream);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  cjm::pool_free(p->device, p->buf_elems * sizeof(double), p->buf[0]);
  cjm::pool_free(p->device, p->buf_elems * sizeof(double), p->buf[1]);
  cjm::pool_free(p->device, p->g_elems * sizeof(double), p->G);
  cjm::pool_free(p->device, (size_t)p->P * sizeof(double), p->w_dev);
  if (p->A) cjm::pool_free(p->device, p->a_elems * sizeof(double), p->A);
  cjm::pool_free(p->device, p->small_bytes, p->small_block);
  if (p->res_halo) cjm::pool_free(p->device, p->res_halo_bytes, p->res_halo);
  if (p->res_flags) cjm::pool_free(p->device, (size_t)p->res_ctas * sizeof(unsigned int), p->res_flags);
  cjm::pool_free_host(2 * sizeof(double), p->result_host);
  if (p->comm) {   // back to the communicator cache (destroyed by cjm_pool_trim)
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (auto& kv : g_comms)
      if (kv.second.first == p->comm) kv.second.second -= 1;
  }
  tt.mark("free");
  delete p;
  return CJM_OK;
}

// cjm_plan / cjm_plan_mask.  bounds = {kappa_min, kappa_max} for masks.
static cjm_status plan_create(cjm_plan_t* out, int stencil, int nx, int ny, double h, int bc,
                              double tol, const cjm_options* opt_in, const double* bounds,
                              int mask_r = 0) {
  if (!out) return CJM_ERR_INVALID_ARG;
  *out = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cjm_options opt;
  cjm_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (bc != CJM_BC_DIRICHLET) {
    set_error("cjm_plan", "only Dirichlet boundary conditions are supported");
    return CJM_ERR_UNSUPPORTED;
  }
  const bool mask = stencil == CJM_STENCIL_MASK;
  // NCCL data plane: world_size > 1 without external_halo, or a one-rank
  // communicator requested by passing an id with world_size = 1 (runs the
  // multi-GPU schedule -- comm stream, band split, NCCL groups, allreduce --
  // on one GPU)
  const bool use_nccl = !mask && ((opt.world_size > 1 && !opt.external_halo) ||
                                  (opt.world_size == 1 && opt.nccl_id));
  if (mask && opt.world_size != 1) {
    set_error("cjm_plan_mask", "generic-mask plans are single-GPU");
    return CJM_ERR_UNSUPPORTED;
  }
  const int R = mask ? std::max(1, mask_r) : cjm::stencil_reach(stencil);
  if (!R || nx < 4 || ny < 4 || !(h > 0.0) || !std::isfinite(h) || !(tol > 0.0 && tol < 1.0) ||
      opt.world_size < 1 || opt.rank < 0 || opt.rank >= opt.world_size ||
      (opt.world_size > 1 && !opt.nccl_id && !opt.external_halo) ||
      (opt.method != CJM_METHOD_CHEBYSHEV && opt.method != CJM_METHOD_JACOBI) ||
      (opt.tile_w != 0 && opt.tile_w != 256 && opt.tile_w != 512) || opt.stages < 0 ||
      opt.temporal_k < 0 || opt.temporal_k > 4 ||
      (opt.variant != 0 && opt.variant != 3 && opt.variant != 7) ||
      opt.stages > 32 || opt.ctas_per_sm < 0 || opt.graph_chunk < 0 || opt.max_cycles < 0 ||
      opt.jacobi_check < 0 || (opt.closure != CJM_CLOSURE_DIRICHLET && opt.closure != CJM_CLOSURE_ODD)) {
    set_error("cjm_plan", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  if (opt.closure == CJM_CLOSURE_ODD &&
      (stencil != CJM_STENCIL_17 || opt.world_size != 1 || opt.nccl_id || opt.temporal_k > 1 ||
       opt.resident == 1 || opt.band_split)) {
    set_error("cjm_plan", "closure=ODD: 17-point, single GPU, temporal_k 1, no resident kernel");
    return CJM_ERR_INVALID_ARG;
  }
  int y0 = 0, nyl = 0;
  cjm_slab(ny, opt.world_size, opt.rank, &y0, &nyl);
  if (opt.world_size > 1 && nyl < 2 * R + 1) {
    set_error("cjm_plan", "slab thinner than 2r+1 rows");
    return CJM_ERR_INVALID_ARG;
  }

  cjm_plan_s* pl = new cjm_plan_s;
  pl->stencil = stencil;
  pl->R = R;
  pl->nx = nx;
  pl->ny = ny;
  pl->y0 = y0;
  pl->ny_local = nyl;
  pl->h = h;
  pl->tol = tol;
  // g = (h^2 / c_C) b, c_C = -4, -20/6, -300/72 (DESIGN R6)
  // (masks: g = b / c_C per node, the residual r = c_C d is already in PDE units)
  pl->gscale = mask ? -1.0 : stencil == 5 ? -(h * h) * 0.25 : stencil == 9 ? -(h * h) * 0.3
                                                                      : -(h * h) * (72.0 / 300.0);
  pl->method = opt.method;
  pl->closure = opt.closure;
  pl->world = opt.world_size;
  pl->rank = opt.rank;

  if (mask ? !cjm::build_schedule_bounds(bounds[0], bounds[1], tol, opt.order, &pl->sched)
           : !cjm::build_schedule(stencil, nx, ny, tol, opt.order, &pl->sched)) {
    delete pl;
    set_error("cjm_plan", mask ? "invalid order or kappa bounds" : "invalid order");
    return CJM_ERR_INVALID_ARG;
  }
  if (opt.method == CJM_METHOD_JACOBI) {
    pl->P = opt.jacobi_check > 0 ? opt.jacobi_check : 1024;
    pl->sched.w.assign(pl->P, 1.0);
    pl->sched.t.assign(pl->P, 0);
    pl->max_cycles = opt.max_cycles > 0 ? opt.max_cycles : 100000;
  } else {
    pl->P = pl->sched.P;
    pl->max_cycles = opt.max_cycles > 0 ? opt.max_cycles : 8;
  }

  auto fail = [&](cjm_status s) { cjm_plan_destroy(pl); return s; };
#define PLAN_CUDA(expr)                                                  \
  do {                                                                   \
    cudaError_t e_ = (expr);                                             \
    if (e_ != cudaSuccess) {                                             \
      set_error(#expr, cudaGetErrorString(e_));                          \
      return fail(e_ == cudaErrorMemoryAllocation ? CJM_ERR_OOM : CJM_ERR_CUDA); \
    }                                                                    \
  } while (0)

  TraceTimer tt("plan");
  int dev = opt.device;
  if (dev < 0) PLAN_CUDA(cudaGetDevice(&dev));
  pl->device = dev;
  PLAN_CUDA(cudaSetDevice(dev));
  int nsm = 0;
  PLAN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));

  int smem_optin = 0;
  PLAN_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (mask) {
    // one sweep per launch, 256-column strips x row bands, up to 8 CTAs / SM
    pl->variant = 0;
    pl->K = 1;
    pl->NT = cjm::MASK_NT;
    pl->graph_chunk = opt.graph_chunk > 0 ? opt.graph_chunk : 64;
  pl->chunk_rows = opt.chunk_rows > 0 ? opt.chunk_rows : (opt.chunk_rows < 0 ? 0 : -1);   // -1: auto
  if (const char* e = std::getenv("CJM_DYN_PCT")) pl->dyn_pct = std::max(0, std::min(100, std::atoi(e)));
    pl->ctas_per_sm = opt.ctas_per_sm > 0 ? opt.ctas_per_sm : 8;
    int occ = 0;
    PLAN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, (const void*)cjm::cjm_mask_kernel<true, true>, cjm::MASK_NT, 0));
    if (occ < 1) {
      set_error("cjm_plan_mask", "mask kernel does not fit on an SM");
      return fail(CJM_ERR_INVALID_ARG);
    }
    pl->nctas = nsm * std::min(occ, pl->ctas_per_sm);
    const int strips = (nx + cjm::MASK_NT - 1) / cjm::MASK_NT;
    pl->bands = std::max(1, std::min(nyl, pl->nctas / strips));
  } else {
  // ---- launch configuration
  // up to 4 CTAs/SM (the register file usually allows 2); multi-GPU: one CTA
  // slot per SM left free so the NCCL exchange kernels can run next to the
  // persistent interior kernel
  pl->ctas_per_sm = opt.ctas_per_sm > 0 ? opt.ctas_per_sm : (opt.world_size > 1 ? 3 : 4);
  // Default: the warp-tiled kernel with 2 columns per lane and 2r+1 rows per
  // TMA stage (variant 7), consumer warps per CTA chosen below.  5/9-point:
  // four sweeps per launch from 4096^2 up, three below; 17-point: three from
  // 4096^2 up, two below (profiles/r01_v7_tune.jsonl: 27.3 us per 9-point
  // sweep at 4096^2 vs 37.9 for variant 4 at K = 2; 404 vs 599 at 16384^2;
  // 17-point at 8192^2: 139 us at K = 3, 155 at K = 2, 290 for variant 3 at
  // K = 1).  An explicit tile_w selects the shared-line kernel (variant 3).
  const bool wide = stencil == 17;
  pl->NT = opt.tile_w == 512 || (opt.tile_w == 0 && wide) ? 256 : 128;
  pl->variant = opt.variant ? opt.variant : (opt.tile_w ? 3 : 7);
  pl->band_split = opt.band_split;
  pl->K = opt.temporal_k > 0 ? opt.temporal_k
                             : ((long long)nx * ny >= 4096LL * 4096LL ? (wide ? 3 : 4) : (wide ? 2 : 3));
  if (opt.closure == CJM_CLOSURE_ODD) pl->K = 1;   // the outer ring is reflected before every sweep
  // multi-GPU: K-fused launches need H = K r deep halos, exchanged after every
  // launch; the slab must stay thicker than 2H + 1 rows (else fall back to K=1)
  if (pl->world > 1 && nyl < 2 * pl->K * R + 1) pl->K = 1;
  if (stencil == 17 && pl->K > 3 && pl->variant == 7) {
    // the warp-tiled kernel runs the 17-point with temporal_k <= 3 (register
    // rings); temporal_k = 4 is the shared-line kernel's
    if (opt.variant == 7) {
      set_error("cjm_plan", "variant 7 runs the 17-point with temporal_k <= 3 only");
      return fail(CJM_ERR_INVALID_ARG);
    }
    pl->variant = 3;
  }
  pl->stages = opt.stages > 0 ? opt.stages
                              : (pl->variant == 7 ? (R == 1 ? 6 : 4) : (pl->NT == 256 ? 12 : 4));
  pl->graph_chunk = opt.graph_chunk > 0 ? opt.graph_chunk : 64;
  pl->chunk_rows = opt.chunk_rows > 0 ? opt.chunk_rows : (opt.chunk_rows < 0 ? 0 : -1);   // -1: auto
  if (const char* e = std::getenv("CJM_DYN_PCT")) pl->dyn_pct = std::max(0, std::min(100, std::atoi(e)));
  // The grid is sized for the hot kernel (persistent: ctas_per_sm per SM, all
  // resident).  Check / residual / remainder kernels may need more registers;
  // they then run the same grid in more than one wave, which is correct
  // because no CTA ever waits for another.
  if ((opt.warps != 0 &&
       (pl->variant != 7 ||
        (opt.warps != 4 && opt.warps != 5 && opt.warps != 7 &&
         !(opt.warps == 11 && R == 1 && pl->K == 4)))) ||
      opt.warps < 0) {
    set_error("cjm_plan", "warps must be 4, 5 or 7 (or 11 for the 5/9-point at K = 4), with variant 7");
    return fail(CJM_ERR_INVALID_ARG);
  }
  if (pl->variant == 7) {
    // Consumer warps per CTA and ring depth: the pair that keeps the most
    // consumer warps resident per SM (registers are split between the SM's
    // 4 sub-partitions, shared memory holds stages x (2r+1) rows per CTA);
    // ties: the deeper ring, then fewer warps.
    // (11 warps: one CTA per SM, 5/9-point at K = 4 only -- 23.7 vs 24.0 us
    // per sweep at 4096^2, 328 vs 346 at 16384^2, profiles/r01_v7_tune.jsonl)
    const int nws[4] = {4, 5, 7, 11};
    constexpr int NNW = 4;
    const int st_hi = opt.stages > 0 ? opt.stages : (R == 1 ? 6 : 4);
    const int st_lo = opt.stages > 0 ? opt.stages : 4;
    int best = -1, best_nw = 4, best_st = st_hi;
    for (int i = 0; i < NNW; ++i) {
      if (opt.warps && nws[i] != opt.warps) continue;
      if (nws[i] == 11 && !(R == 1 && pl->K == 4)) continue;
      for (int stg = st_hi; stg >= st_lo; --stg) {
        pl->nw = nws[i];
        pl->stages = stg;
        const size_t sm = smem_bytes(pl, pl->K);
        if (sm > (size_t)smem_optin - 2048) continue;
        KernelFn k = pick_kernel(stencil, 7, pl->NT, pl->K, MODE_HOT, pl->nw);
        if (!k) continue;                       // (nw, K) not instantiated
        PLAN_CUDA(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm));
        int occ = 0;
        PLAN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k,
                                                                block_threads(pl), sm));
        const int score = std::min(occ, pl->ctas_per_sm) * pl->nw;
        if (score > best) { best = score; best_nw = pl->nw; best_st = stg; }
      }
    }
    pl->nw = best_nw;
    pl->stages = best_st;
  }
  if (pl->variant == 7 && pl->stages < ((pl->K - 1) * R + v4_rps(R) - 1) / v4_rps(R) + 2) {
    // the warp-tiled kernel holds a stage until level K-1 has read the g rows
    // of its rows, R(K-1) rows later
    set_error("cjm_plan", "stages must be >= ceil(r(temporal_k-1) / rows_per_stage) + 2 for the "
                          "warp-tiled kernel");
    return fail(CJM_ERR_INVALID_ARG);
  }
  if (smem_bytes(pl, pl->K) > (size_t)smem_optin - 2048) {
    set_error("cjm_plan", "TMA ring too deep for shared memory (lower stages)");
    return fail(CJM_ERR_INVALID_ARG);
  }
  int occ_min = 1 << 30;
  for (int K = 1; K <= pl->K; ++K) {
    if (K != 1 && K != pl->K) continue;
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == MODE_RESID && K != 1) continue;
      KernelFn k = pick_kernel(stencil, pl->variant, pl->NT, K, mode, pl->nw);
      if (!k) {   // every launch the executor can issue must be instantiated
        set_error("cjm_plan", "no sweep kernel instantiated for this (stencil, temporal_k, warps)");
        return fail(CJM_ERR_INVALID_ARG);
      }
      const size_t sm = smem_bytes(pl, K);
      PLAN_CUDA(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
      if (K == pl->K && mode == MODE_HOT) {
        PLAN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_min, (const void*)k,
                                                                block_threads(pl), sm));
      }
    }
  }
  if (occ_min < 1) {
    set_error("cjm_plan", "sweep kernel does not fit on an SM with these options");
    return fail(CJM_ERR_INVALID_ARG);
  }
  // multi-GPU with NCCL: two SMs are left to the NCCL kernels of the halo
  // exchange, which overlaps the interior band launch (a persistent grid on
  // every SM would leave them no slot: the warp-tiled kernels fill the
  // register file); the dynamic work items absorb the lost SMs
  const int reserve = (use_nccl && nsm > 8) ? 2 : 0;
  pl->nctas = (nsm - reserve) * std::min(occ_min, pl->ctas_per_sm);
  }

  // ---- resident (shared-memory) hot path: single GPU, whole grid fits in the
  // SMs' shared memory with at least 16 rows per CTA
  if (pl->world == 1 && !use_nccl && opt.resident >= 0 && !mask && opt.closure == CJM_CLOSURE_DIRICHLET) {
    const int ldS = nx + 2 * R;
    auto smem_for = [&](int rows) {
      return ((size_t)2 * (rows + 2 * R) * ldS + (size_t)rows * nx) * sizeof(double);
    };
    // at least 16 rows per CTA for small grids (fewer handshakes), else the
    // minimum slab height that spreads the grid over all SMs
    const int rows_min = (nyl + nsm - 1) / nsm;
    // (every CTA but the last must own >= R rows: a CTA publishes its first /
    // last R rows to its neighbours, and a thinner slab would publish one of
    // its own ghost rows, a stale copy of the neighbour's data)
    int rows = std::max(rows_min, std::min(16, nyl));
    if (smem_for(rows) + 1024 > (size_t)smem_optin) rows = rows_min;
    rows = std::max(rows, std::min(R, nyl));
    // the whole grid in ONE CTA when it fits: no handshakes at all
    if (smem_for(nyl) + 1024 <= (size_t)smem_optin) rows = nyl;
    const int ctas = (nyl + rows - 1) / rows;
    const size_t smem = smem_for(rows);
    int occ_r = 0;
    if (smem + 1024 <= (size_t)smem_optin) {
      ResidentFn rf = pick_resident(stencil);
      PLAN_CUDA(cudaFuncSetAttribute((const void*)rf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
      PLAN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_r, (const void*)rf, 512, smem));
    }
    // auto mode only where the neighbour handshakes do not dominate: at most
    // 4 CTA slabs (the 64^2 config: 2.9 vs 3.8 us per sweep; from 128^2 on
    // the streaming kernels win, profiles/r01_resident_vs_stream.jsonl)
    const bool wanted = opt.resident == 1 || ctas <= 4;
    if (occ_r >= 1 && ctas <= nsm * occ_r && wanted) {
      pl->resident = 1;
      pl->res_rows = rows;
      pl->res_ctas = ctas;
      pl->res_smem = smem;
      pl->res_halo_bytes = (size_t)ctas * 2 * 2 * R * ldS * sizeof(double);
    } else if (opt.resident == 1) {
      set_error("cjm_plan", "resident=1 but the grid does not fit in shared memory");
      return fail(CJM_ERR_INVALID_ARG);
    }
  }

  tt.mark("schedule+config");
  // ---- buffers: (ny_local + 2R) rows of pitch ld; interior column 0 at PADL
  cjm_buffer_layout(nx, &pl->ld, nullptr);
  pl->H = pl->world > 1 ? pl->K * R : R;
  const bool deep_external = pl->world > 1 && opt.external_halo && pl->K > 1;
  pl->Hu = deep_external ? pl->H : R;
  pl->Hr = deep_external ? pl->H : 0;
  pl->row_lo = std::max(-pl->H, -pl->y0);
  pl->row_hi = std::min(nyl + pl->H, ny - pl->y0);
  pl->buf_elems = (size_t)(nyl + 2 * pl->H) * pl->ld;
  pl->g_elems = (size_t)(nyl + 2 * pl->H) * pl->ld;
  PLAN_CUDA(cjm::pool_alloc(dev, pl->buf_elems * sizeof(double), (void**)&pl->buf[0]));
  PLAN_CUDA(cjm::pool_alloc(dev, pl->buf_elems * sizeof(double), (void**)&pl->buf[1]));
  PLAN_CUDA(cjm::pool_alloc(dev, pl->g_elems * sizeof(double), (void**)&pl->G));
  PLAN_CUDA(cudaMemset(pl->buf[0], 0, pl->buf_elems * sizeof(double)));
  PLAN_CUDA(cudaMemset(pl->buf[1], 0, pl->buf_elems * sizeof(double)));
  PLAN_CUDA(cudaMemset(pl->G, 0, pl->g_elems * sizeof(double)));
  if (mask) {
    pl->mask_r = mask_r;
    pl->nplanes = mask_r ? (2 * mask_r + 1) * (2 * mask_r + 1) : 5;
    pl->mask_qc = mask_r ? mask_r * (2 * mask_r + 1) + mask_r : 4;
    pl->a_elems = (size_t)pl->nplanes * ny * pl->ld;
    PLAN_CUDA(cjm::pool_alloc(dev, pl->a_elems * sizeof(double), (void**)&pl->A));
  }
  tt.mark("field buffers");
  PLAN_CUDA(cjm::pool_alloc(dev, (size_t)pl->P * sizeof(double), (void**)&pl->w_dev));
  PLAN_CUDA(cudaMemcpy(pl->w_dev, pl->sched.w.data(), (size_t)pl->P * sizeof(double),
                       cudaMemcpyHostToDevice));
  // one small block: partials (2 per CTA), result (2), state, real-error bits
  pl->small_bytes = ((size_t)pl->nctas * 2 + 2) * sizeof(double) + sizeof(cjm::SweepState) +
                    3 * sizeof(unsigned long long);
  PLAN_CUDA(cjm::pool_alloc(dev, pl->small_bytes, &pl->small_block));
  pl->partials = static_cast<double*>(pl->small_block);
  if (pl->resident) {
    PLAN_CUDA(cjm::pool_alloc(dev, pl->res_halo_bytes, (void**)&pl->res_halo));
    PLAN_CUDA(cjm::pool_alloc(dev, (size_t)pl->res_ctas * sizeof(unsigned int), (void**)&pl->res_flags));
  }
  pl->result = pl->partials + (size_t)pl->nctas * 2;
  pl->state = reinterpret_cast<cjm::SweepState*>(pl->result + 2);
  pl->err_bits = reinterpret_cast<unsigned long long*>(pl->state + 1);
  pl->dbg = pl->err_bits + 1;
  PLAN_CUDA(cudaMemset(pl->state, 0, sizeof(cjm::SweepState) + 3 * sizeof(unsigned long long)));
  PLAN_CUDA(cjm::pool_alloc_host(2 * sizeof(double), (void**)&pl->result_host));
  tt.mark("weights+small");
  PLAN_CUDA(cudaStreamCreateWithFlags(&pl->cap_stream, cudaStreamNonBlocking));
  PLAN_CUDA(cudaStreamCreateWithFlags(&pl->comm_stream, cudaStreamNonBlocking));
  PLAN_CUDA(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming));
  PLAN_CUDA(cudaEventCreateWithFlags(&pl->ev_join, cudaEventDisableTiming));
  for (auto& e : pl->ev) PLAN_CUDA(cudaEventCreate(&e));

  if (use_nccl) {
    ncclUniqueId id;
    std::memcpy(&id, opt.nccl_id, sizeof(id));
    CommKey key;
    std::memcpy(key.id, opt.nccl_id, sizeof(key.id));
    key.world = pl->world;
    key.rank = pl->rank;
    key.device = dev;
    // Cache decision: a cached, idle communicator for this id is reused (no
    // collective call); an unknown id is initialised (ncclCommInitRank, a
    // collective over the world).  Every rank makes the same plan calls in
    // the same order, so the decisions agree across ranks.  An id is
    // single-use for initialisation: a second LIVE plan with the same id
    // cannot get a communicator (re-initialising a consumed id would hang)
    // and is rejected -- pass a fresh cjm_get_nccl_id() for concurrent plans.
    bool init = false;
    {
      std::lock_guard<std::mutex> lk(g_comm_mu);
      auto it = g_comms.find(key);
      if (it == g_comms.end()) {
        init = true;
        g_comms[key] = {nullptr, 1};   // reserved while this plan initialises it
      } else if (it->second.second == 0 && it->second.first) {
        pl->comm = it->second.first;
        it->second.second = 1;
      }
    }
    if (!pl->comm && !init) {
      set_error("cjm_plan", "a live plan already uses this NCCL id (ids are single-use: pass a fresh "
                            "cjm_get_nccl_id for concurrent plans)");
      return fail(CJM_ERR_INVALID_ARG);
    }
    if (init) {
      ncclComm_t c = nullptr;
      ncclResult_t r = ncclCommInitRank(&c, pl->world, id, pl->rank);
      std::lock_guard<std::mutex> lk(g_comm_mu);
      if (r != ncclSuccess) {
        g_comms.erase(key);
        set_error("ncclCommInitRank", ncclGetErrorString(r));
        return fail(CJM_ERR_NCCL);
      }
      g_comms[key] = {c, 1};
      pl->comm = c;
    }
  }

  PLAN_CUDA(cudaDeviceSynchronize());
#undef PLAN_CUDA
  tt.mark("streams+nccl+sync");
  pl->plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = pl;
  return CJM_OK;
}

cjm_status cjm_plan(cjm_plan_t* out, int stencil, int nx, int ny, double h, int bc, double tol,
                    const cjm_options* opt) {
  if (stencil == CJM_STENCIL_MASK) {
    if (out) *out = nullptr;
    set_error("cjm_plan", "generic masks use cjm_plan_mask");
    return CJM_ERR_INVALID_ARG;
  }
  return plan_create(out, stencil, nx, ny, h, bc, tol, opt, nullptr);
}

cjm_status cjm_plan_mask(cjm_plan_t* out, int nx, int ny, double kappa_min, double kappa_max,
                         double tol, const cjm_options* opt) {
  if (!(kappa_min > 0.0 && kappa_max > kappa_min) || !std::isfinite(kappa_max)) {
    if (out) *out = nullptr;
    set_error("cjm_plan_mask", "need 0 < kappa_min < kappa_max < inf");
    return CJM_ERR_INVALID_ARG;
  }
  const double bounds[2] = {kappa_min, kappa_max};
  return plan_create(out, CJM_STENCIL_MASK, nx, ny, 1.0, CJM_BC_DIRICHLET, tol, opt, bounds);
}

cjm_status cjm_mask_set(cjm_plan_t p, const double* cW, const double* cE, const double* cS,
                        const double* cN, const double* cC, long long ld_c, void* cuda_stream) {
  if (!p || p->stencil != CJM_STENCIL_MASK || p->mask_r != 0 || !cW || !cE || !cS || !cN || !cC ||
      ld_c < p->nx) {
    set_error("cjm_mask_set", "invalid argument (not a 5-point mask plan, NULL array or ld_c < nx)");
    return CJM_ERR_INVALID_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long total = (long long)p->nx * p->ny;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  cjm::cjm_mask_prepare_kernel<<<blocks, 256, 0, st>>>(p->A, (long long)p->a_elems / p->nplanes,
                                                       p->ld, cW, cE, cS, cN, cC, ld_c, p->nx, p->ny);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  p->mask_ready = 1;
  return CJM_OK;
}

cjm_status cjm_plan_mask_n(cjm_plan_t* out, int nx, int ny, int radius, double kappa_min,
                           double kappa_max, double tol, const cjm_options* opt) {
  if (!(kappa_min > 0.0 && kappa_max > kappa_min) || !std::isfinite(kappa_max) ||
      (radius != 1 && radius != 2)) {
    if (out) *out = nullptr;
    set_error("cjm_plan_mask_n", "need radius 1 or 2 and 0 < kappa_min < kappa_max < inf");
    return CJM_ERR_INVALID_ARG;
  }
  const double bounds[2] = {kappa_min, kappa_max};
  return plan_create(out, CJM_STENCIL_MASK, nx, ny, 1.0, CJM_BC_DIRICHLET, tol, opt, bounds, radius);
}

cjm_status cjm_mask_set_n(cjm_plan_t p, const double* const* planes, long long ld_c,
                          void* cuda_stream) {
  if (!p || p->stencil != CJM_STENCIL_MASK || p->mask_r == 0 || !planes || ld_c < p->nx ||
      !planes[p->mask_qc]) {
    set_error("cjm_mask_set_n",
              "invalid argument (not a square-mask plan, NULL planes / centre plane, ld_c < nx)");
    return CJM_ERR_INVALID_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cjm::MaskPlanes mp{};
  unsigned int present = 0;
  for (int q = 0; q < p->nplanes; ++q) {
    mp.c[q] = planes[q];
    if (planes[q] && q != p->mask_qc) present |= 1u << q;
  }
  const long long total = (long long)p->nx * p->ny;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  cjm::cjm_maskn_prepare_kernel<<<blocks, 256, 0, st>>>(p->A, (long long)p->a_elems / p->nplanes,
                                                        p->ld, mp, p->nplanes, p->mask_qc, ld_c,
                                                        p->nx, p->ny);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  p->present = present;
  p->mask_ready = 1;
  return CJM_OK;
}

cjm_status cjm_mask_bounds(int nx, int ny, const double* cW, const double* cE, const double* cS,
                           const double* cN, const double* cC, long long ld_c, int iters,
                           double* kappa_min, double* kappa_max) {
  double kmin = 0, kmax = 0;
  if (!kappa_min || !kappa_max ||
      !cjm::mask_spectral_bounds(nx, ny, cW, cE, cS, cN, cC, ld_c, iters > 0 ? iters : 2000, &kmin,
                                 &kmax)) {
    set_error("cjm_mask_bounds", "invalid argument, zero / non-finite c_C or rho(N) >= 1");
    return CJM_ERR_INVALID_ARG;
  }
  *kappa_min = kmin;
  *kappa_max = kmax;
  return CJM_OK;
}

cjm_status cjm_mask_bounds_n(int nx, int ny, int radius, const double* const* planes, long long ld_c,
                             int iters, double* kappa_min, double* kappa_max) {
  double kmin = 0, kmax = 0;
  if (!kappa_min || !kappa_max ||
      !cjm::mask_spectral_bounds_n(radius, nx, ny, planes, ld_c, iters > 0 ? iters : 2000, &kmin,
                                   &kmax)) {
    set_error("cjm_mask_bounds_n",
              "invalid argument, zero / non-finite c_C or D^-1 A not positive definite");
    return CJM_ERR_INVALID_ARG;
  }
  *kappa_min = kmin;
  *kappa_max = kmax;
  return CJM_OK;
}

cjm_status cjm_plan_info(cjm_plan_t p, cjm_report* info, int* reach, int* y0, int* ny_local,
                         const double** host_weights) {
  if (!p) return CJM_ERR_INVALID_ARG;
  if (info) fill_static(p, info);
  if (reach) *reach = p->R;
  if (y0) *y0 = p->y0;
  if (ny_local) *ny_local = p->ny_local;
  if (host_weights) *host_weights = p->sched.w.data();
  return CJM_OK;
}

cjm_status cjm_solve(cjm_plan_t p, const double* rhs, long long ld_rhs, double* u, long long ld_u,
                     void* cuda_stream, cjm_report* rep) {
  return solve_impl(p, rhs, ld_rhs, u, ld_u, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice,
                    cuda_stream, rep);
}

cjm_status cjm_solve_ref(cjm_plan_t p, const double* rhs, long long ld_rhs, double* u, long long ld_u,
                         const double* u_ref, long long ld_ref, double real_tol, void* cuda_stream,
                         cjm_report* rep) {
  if (!u_ref) {
    set_error("cjm_solve_ref", "u_ref is NULL");
    return CJM_ERR_INVALID_ARG;
  }
  return solve_impl(p, rhs, ld_rhs, u, ld_u, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice,
                    cuda_stream, rep, u_ref, ld_ref, real_tol);
}

cjm_status cjm_solve_host(cjm_plan_t p, const double* rhs_host, long long ld_rhs, double* u_host,
                          long long ld_u, void* cuda_stream, cjm_report* rep) {
  return solve_impl(p, rhs_host, ld_rhs, u_host, ld_u, cudaMemcpyHostToDevice,
                    cudaMemcpyDeviceToHost, cuda_stream, rep);
}

cjm_status cjm_sweeps(cjm_plan_t p, const double* rhs, long long ld_rhs, double* u, long long ld_u,
                      long long first, long long count, void* cuda_stream, cjm_report* rep_out) {
  if (!check_layout(p, rhs, ld_rhs, u, ld_u) || !rhs || first < 0 || count < 0) {
    set_error("cjm_sweeps", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  if (p->world > 1 && !p->comm && count > p->K) {
    // external_halo: the caller refreshes the halos between calls; more than
    // one launch per call would read stale neighbour rows
    set_error("cjm_sweeps", "external_halo plans apply at most temporal_k sweeps per call");
    return CJM_ERR_INVALID_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cjm_report rep;
  fill_static(p, &rep);
  p->launches = 0;
  STATUS_TRY(stage_in(p, rhs, ld_rhs, u, ld_u, true, cudaMemcpyDeviceToDevice, st));
  STATUS_TRY(set_state(p, (unsigned long long)first, st));
  STATUS_TRY(halo_exchange(p, p->buf[0], st));
  CUDA_TRY(cudaEventRecord(p->ev[2], st));
  STATUS_TRY(run_hot(p, count, st, &rep.hot_launches));
  CUDA_TRY(cudaEventRecord(p->ev[3], st));
  STATUS_TRY(stage_out(p, p->host_cur, u, ld_u, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  rep.sweep_s = elapsed_s(p->ev[2], p->ev[3]);
  rep.sweeps_timed = count;
  rep.iterations = count;
  rep.kernel_launches = p->launches;
  if (rep_out) *rep_out = rep;
  return debug_verify(p);
}

cjm_status cjm_residual(cjm_plan_t p, const double* rhs, long long ld_rhs, const double* u,
                        long long ld_u, void* cuda_stream, double* l2, double* linf) {
  if (!check_layout(p, rhs, ld_rhs, u, ld_u) || !rhs) {
    set_error("cjm_residual", "invalid argument");
    return CJM_ERR_INVALID_ARG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  p->launches = 0;
  STATUS_TRY(stage_in(p, rhs, ld_rhs, u, ld_u, false, cudaMemcpyDeviceToDevice, st));
  STATUS_TRY(set_state(p, 0ull, st));
  STATUS_TRY(halo_exchange(p, p->buf[0], st));
  STATUS_TRY(launch_sweep(p, MODE_RESID, 1, st));
  double s, m;
  STATUS_TRY(fetch_result(p, st, &s, &m));
  const double sc = std::fabs(p->gscale);
  if (l2) *l2 = std::sqrt(s) / sc;
  if (linf) *linf = m / sc;
  return debug_verify(p);
}

const char* cjm_status_str(int s) {
  switch (s) {
    case CJM_OK: return "CJM_OK";
    case CJM_ERR_INVALID_ARG: return "CJM_ERR_INVALID_ARG";
    case CJM_ERR_UNSUPPORTED: return "CJM_ERR_UNSUPPORTED";
    case CJM_ERR_NOT_CONVERGED: return "CJM_ERR_NOT_CONVERGED";
    case CJM_ERR_DIVERGED: return "CJM_ERR_DIVERGED";
    case CJM_ERR_STAGNATED: return "CJM_ERR_STAGNATED";
    case CJM_ERR_CUDA: return "CJM_ERR_CUDA";
    case CJM_ERR_NCCL: return "CJM_ERR_NCCL";
    case CJM_ERR_OOM: return "CJM_ERR_OOM";
    default: return "CJM_ERR_UNKNOWN";
  }
}

const char* cjm_last_error(void) { return g_last_error.c_str(); }

#ifdef CJM_DIAG_TIMES
// diagnostic builds only: the per-CTA (start, end) %globaltimer stamps of the
// last hot launch, kept in the (otherwise unused) partials of hot launches
cjm_status cjm_diag_times(cjm_plan_t p, unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  cudaMemcpy(host, p->partials, sizeof(unsigned long long) * 2 * std::min(n, p->nctas),
             cudaMemcpyDeviceToHost);
  return (cjm_status)p->nctas;
}
#endif

cjm_status cjm_pool_trim(long long* cached_bytes_before) {
  if (cached_bytes_before) *cached_bytes_before = (long long)cjm::pool_cached_bytes();
  cjm::pool_trim();
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (auto it = g_comms.begin(); it != g_comms.end();) {
      if (it->second.second == 0) {
        ncclCommDestroy(it->second.first);
        it = g_comms.erase(it);
      } else {
        ++it;
      }
    }
  }
  return CJM_OK;
}

int cjm_version(void) { return 100 * CJM_VERSION_MAJOR + CJM_VERSION_MINOR; }

}  // extern "C"
