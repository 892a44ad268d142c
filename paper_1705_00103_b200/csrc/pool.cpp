// Device-buffer cache of libcjm (the runtime's allocator).
//
// A plan owns ~3 field-sized buffers (two iterates and g: 3 x 134 MB at
// 4096^2, 3 x 8.6 GB at 32768^2).  cudaMalloc / cudaFree of buffers that size
// cost milliseconds to hundreds of milliseconds and cudaFree synchronises the
// device, so plans that are created and destroyed repeatedly (one plan per
// solve) would spend more time in the driver than in some solves.  Freed plan
// buffers are therefore kept here, keyed by (device, exact byte size), and
// handed to the next plan that asks for the same size.  cjm_pool_trim()
// returns everything to the driver.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"

namespace cjm {

namespace {
std::mutex g_mu;
std::multimap<std::pair<int, size_t>, void*> g_free;   // (device, bytes) -> block
size_t g_cached = 0;
constexpr size_t kMaxCached = size_t(96) << 30;         // never hold more than 96 GiB
}  // namespace

cudaError_t pool_alloc(int device, size_t bytes, void** out) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_free.find({device, bytes});
    if (it != g_free.end()) {
      *out = it->second;
      g_free.erase(it);
      g_cached -= bytes;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(out, bytes);
  if (e == cudaErrorMemoryAllocation) {   // give the cache back and retry once
    pool_trim();
    cudaGetLastError();
    e = cudaMalloc(out, bytes);
  }
  return e;
}

void pool_free(int device, size_t bytes, void* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_cached + bytes <= kMaxCached) {
      g_free.emplace(std::make_pair(device, bytes), p);
      g_cached += bytes;
      return;
    }
  }
  cudaFree(p);
}

void pool_trim() {
  std::multimap<std::pair<int, size_t>, void*> blocks;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    blocks.swap(g_free);
    g_cached = 0;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& kv : blocks) {
    cudaSetDevice(kv.first.first);
    cudaFree(kv.second);
  }
  cudaSetDevice(prev);
}

// pinned host blocks (the 16-byte D2H landing zones of the reductions)
namespace {
std::multimap<size_t, void*> g_host_free;
}

cudaError_t pool_alloc_host(size_t bytes, void** out) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_host_free.find(bytes);
    if (it != g_host_free.end()) {
      *out = it->second;
      g_host_free.erase(it);
      return cudaSuccess;
    }
  }
  return cudaMallocHost(out, bytes);
}

void pool_free_host(size_t bytes, void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  g_host_free.emplace(bytes, p);
}

size_t pool_cached_bytes() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_cached;
}

}  // namespace cjm
