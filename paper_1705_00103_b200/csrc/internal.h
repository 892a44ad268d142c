// Internal declarations of libcjm (not part of the C ABI).
#pragma once

#include <cstddef>
#include <vector>

#include <cuda_runtime.h>

namespace cjm {

// Interior column 0 of every internal row sits at column PADL: 64-byte aligned
// rows, 16-byte aligned TMA row loads starting up to E + 2 columns to the left
// (E <= 6: temporal blocking depth K <= 4 for r = 1 and 2).
constexpr int PADL = 8;

struct Schedule {
  double kmin = 0, kmax = 0;
  long long m_min = 0, P = 0;
  std::vector<long long> t;  // Chebyshev zero index per sweep position
  std::vector<double> w;     // weight per sweep position
};

int stencil_reach(int stencil);
bool spectral_bounds(int stencil, int nx, int ny, double* kmin, double* kmax);
long long chebyshev_degree(double kmin, double kmax, double tol);
long long smooth_cycle_length(long long m, int* a_out, int* b_out);
std::vector<long long> lebedev23_order(int a, int b);
bool build_schedule(int stencil, int nx, int ny, double tol, int order, Schedule* s);
// the same from caller-given bounds (generic masks, NEXT-4)
bool build_schedule_bounds(double kmin, double kmax, double tol, int order, Schedule* s);
// host estimate of the spectral bounds of D^-1 A for a 5-point mask (mask_bounds.cpp)
bool mask_spectral_bounds(int nx, int ny, const double* cW, const double* cE, const double* cS,
                          const double* cN, const double* cC, long long ldc, int iters,
                          double* kmin, double* kmax);
// the same for a (2m+1)^2 mask (both ends by power iteration)
bool mask_spectral_bounds_n(int m, int nx, int ny, const double* const* c, long long ldc, int iters,
                            double* kmin, double* kmax);

// device-buffer cache (pool.cpp)
cudaError_t pool_alloc(int device, size_t bytes, void** out);
void pool_free(int device, size_t bytes, void* p);
void pool_trim();
cudaError_t pool_alloc_host(size_t bytes, void** out);
void pool_free_host(size_t bytes, void* p);
size_t pool_cached_bytes();

}  // namespace cjm
