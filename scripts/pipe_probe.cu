// Probe: per-SM throughput of the candidate modular multiply-accumulate
// instructions for the trailing update: IMAD.WIDE.U32 with a
// 64-bit addend (what k_update_tiled issues) and DFMA (exact 48-bit products
// of 24-bit residues, sums < 2^53), each with 16 independent chains/thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp scripts/pipe_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_wide(uint64_t* out, uint32_t seed, int iters) {
  uint64_t acc[16];
  uint32_t a = seed + threadIdx.x, b = seed * 3 + blockIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] += (uint64_t)(a + j) * b;
    b += 0x9E3779B9u;
  }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s ^= acc[j];
  if (s == 42) out[0] = s;
}

__global__ void k_dfma(double* out, double seed, int iters) {
  double acc[16];
  double a = seed + threadIdx.x, b = seed * 3.0 + blockIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(a + j, b, acc[j]);
    b += 1.0;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 42.0) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  uint64_t* o;
  cudaMalloc(&o, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = nsm * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_wide<<<blocks, threads>>>(o, 7u, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 16;
    printf("IMAD.WIDE+64-bit add: %.3e ops/s\n", ops / (ms * 1e-3));
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>((double*)o, 1.5, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA: %.3e ops/s\n", ops / (ms * 1e-3));
  }
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d, max clock %d kHz\n", nsm, clk);
  return 0;
}
