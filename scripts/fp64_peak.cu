// fp64 pipe peak of the B200 (the denominator of bench.py's roofline.fp64_frac).
//
// Every thread runs NCH independent DFMA (or DADD) chains for ITER steps; the
// grid fills every SM with 32 warps.  Reported: lane-operations per second
// (one DFMA = one operation; FLOP/s = 2x that), the SM clock seen by the
// kernel (%clock64 against %globaltimer), and operations per SM per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak scripts/fp64_peak.cu
//   build/fp64_peak > profiles/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NCH = 8;
constexpr int ITER = 4096;

template <bool FMA>
__global__ void fp64_kernel(double* out, double b, double c, unsigned long long* clk) {
  double a[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) a[i] = threadIdx.x * 1e-9 + i;
  unsigned long long c0 = 0, t0 = 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  }
  for (int k = 0; k < ITER; ++k) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) a[i] = FMA ? __fma_rn(a[i], b, c) : __dadd_rn(a[i], c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains alive
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long c1, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    clk[0] = c1 - c0;
    clk[1] = t1 - t0;
  }
}

template <bool FMA>
double run(int nsm, double* out, unsigned long long* clk, double* mhz) {
  const int threads = 256, blocks = nsm * 8;   // 64 warps' worth of blocks per SM (2 waves of 32)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_kernel<FMA><<<blocks, threads>>>(out, 0.999999, 1e-7, clk);   // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    fp64_kernel<FMA><<<blocks, threads>>>(out, 0.999999, 1e-7, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  unsigned long long h[2];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  *mhz = h[1] ? 1e3 * (double)h[0] / (double)h[1] : 0.0;
  const double ops = (double)blocks * threads * NCH * ITER;
  return ops / (best * 1e-3);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  unsigned long long* clk;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&clk, 2 * sizeof(unsigned long long));
  double mhz_f = 0, mhz_a = 0;
  const double fma = run<true>(nsm, out, clk, &mhz_f);
  const double add = run<false>(nsm, out, clk, &mhz_a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  printf("{\"dfma_ops_per_s\": %.6e, \"dadd_ops_per_s\": %.6e, \"dfma_flops\": %.6e, "
         "\"sm_mhz_seen\": %.1f, \"dfma_per_sm_per_clk\": %.2f, \"sms\": %d, "
         "\"how\": \"scripts/fp64_peak.cu: %d independent DFMA / DADD chains per thread, %d steps, "
         "%d blocks x 256 threads, best of 10 (CUDA events); one DFMA = one fp64 pipe operation\"}\n",
         fma, add, 2 * fma, mhz_f, mhz_f > 0 ? fma / (nsm * mhz_f * 1e6) : 0.0, nsm, NCH, ITER,
         nsm * 8);
  return 0;
}
