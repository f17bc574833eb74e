// Integer-pipe microbenchmark: measures the B200's sustained throughput of
// 32-bit IMAD (d = a*b + c) and of IMAD.WIDE.U32 (64-bit d = a*b + c), the
// instruction the trailing-update kernel issues once per modular product.
// These measured rates are the roofline denominators reported by bench.py
// (BASELINE.md's 64 IMAD/clk/SM is the datasheet figure being checked).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 16;
constexpr int kIters = 4096;

__global__ void imad32_kernel(uint32_t* out, uint32_t seed,
                              unsigned long long* cycles) {
  uint32_t acc[kChains];
  const uint32_t b = seed | 1u;
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x + i;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = acc[i] * b + (uint32_t)it;
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicMax(cycles, (unsigned long long)(t1 - t0));
}

__global__ void imadwide_kernel(uint64_t* out, uint32_t seed,
                                unsigned long long* cycles) {
  uint64_t acc[kChains];
  uint32_t a[kChains];
  const uint32_t b = seed | 1u;
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = threadIdx.x + i;
    a[i] = threadIdx.x * 7 + i;
  }
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] += (uint64_t)a[i] * b;
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] ^= (uint32_t)acc[i];
  }
  const long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicMax(cycles, (unsigned long long)(t1 - t0));
}

}  // namespace

extern "C" {

// Returns ops/s for IMAD (kind 0) or IMAD.WIDE + one LOP (kind 1) over the
// whole device, and the SM clock implied by clock64 vs. event time (MHz).
int hgpu_probe_imad(int kind, double* ops_per_s, double* sm_mhz,
                    double* ops_per_clk_sm) {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // one wave: as many 512-thread CTAs per SM as are resident at once (the
  // register file limits it), so the kernel time is one CTA's cycle count
  const int threads = 512;
  int per_sm = 0;
  if (kind == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, imad32_kernel, threads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, imadwide_kernel, threads, 0);
  const int blocks = nsm * (per_sm > 0 ? per_sm : 1);
  void* out = nullptr;
  unsigned long long* cyc = nullptr;
  if (cudaMalloc(&out, (size_t)threads * blocks * 8) != cudaSuccess) return 2;
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_ms = 1e30f;
  unsigned long long best_cyc = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(cyc, 0, 8);
    cudaEventRecord(e0);
    if (kind == 0)
      imad32_kernel<<<blocks, threads>>>((uint32_t*)out, 12345u + rep, cyc);
    else
      imadwide_kernel<<<blocks, threads>>>((uint64_t*)out, 12345u + rep, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms) {
      best_ms = ms;
      cudaMemcpy(&best_cyc, cyc, 8, cudaMemcpyDeviceToHost);
    }
  }
  const double ops = (double)threads * blocks * kIters * kChains;
  *ops_per_s = ops / (best_ms * 1e-3);
  // every CTA is resident at once (one wave), so the kernel time is the
  // per-CTA cycle count at the SM clock
  *sm_mhz = (double)best_cyc / (best_ms * 1e-3) / 1e6;
  *ops_per_clk_sm = ops / ((double)best_cyc * nsm);
  cudaFree(out);
  cudaFree(cyc);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // extern "C"
