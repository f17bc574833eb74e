// Latency of the reciprocal's building blocks on one 512-thread CTA
// (clock64 around each, thread 0's view, median of 8 trials).
#include "../../paper_0902_0852_b200/csrc/ldlt_kernels.cu"

#include <algorithm>
#include <cstdio>

using namespace hgpu;

__global__ void __launch_bounds__(512) prim(long long* out, int M, uint32_t* gout) {
  extern __shared__ uint32_t dsm[];
  __shared__ uint32_t red[64];
  uint32_t* A = dsm + 132;         // 132 guard words each side
  uint32_t* B = A + 512 + 264;
  uint32_t* O = B + 512 + 264;     // 1024
  unsigned long long* V = reinterpret_cast<unsigned long long*>(O + 1024);  // 1024
  uint32_t* pl = reinterpret_cast<uint32_t*>(V + 1024);                     // 3*6*1024
  for (int i = threadIdx.x; i < 2 * (512 + 264) + 132; i += blockDim.x) dsm[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += blockDim.x) A[i] = 0x9e3779b9u * (i + 1), B[i] = 0x85ebca6bu * (i + 7);
  __syncthreads();
  long long t0, t1;
  int slot = 0;
  auto rec = [&](long long a, long long b) { if (threadIdx.x == 0) out[slot] = b - a; ++slot; };
  for (int trial = 0; trial < 8; ++trial) {
    slot = trial * 16;
    t0 = clock64(); __syncthreads(); __syncthreads(); t1 = clock64(); rec(t0, t1);   // 0 two barriers
    t0 = clock64();
    rf::fast_resolve(M, false, [&](int k) -> int64_t { return (int64_t)A[k] + B[k]; },
                     [&](int k, uint32_t d) { O[k] = d; }, red);
    t1 = clock64(); rec(t0, t1);                                                    // 1 fast_resolve
    t0 = clock64();
    rf::fast_resolve(M, true, [&](int k) -> int64_t { return (int64_t)A[k] - B[k]; },
                     [&](int k, uint32_t d) { O[k] = d; }, red);
    t1 = clock64(); rec(t0, t1);                                                    // 2 fast_resolve biased
    t0 = clock64();
    cta_resolve(M, 32, [&](int k) -> int64_t { return (int64_t)A[k] - (int64_t)B[k]; },
                [&](int k, uint32_t d) { O[k] = d; }, red);
    t1 = clock64(); rec(t0, t1);                                                    // 3 cta_resolve
    t0 = clock64();
    const int len = cta_limb_len(O, M, red);
    t1 = clock64(); rec(t0, t1);                                                    // 4 limb_len
    if (threadIdx.x == 0) gout[0] = len;
    t0 = clock64();
    rf::cta_mul_fast(A, M, B, M, O, 2 * M, 0, pl, 3 * 6 * 1024, V, red);
    t1 = clock64(); rec(t0, t1);                                                    // 5 mul_fast MxM
    t0 = clock64();
    const int nseg = rf::wcols(A, M, B, M, 0, 2 * M, pl, 3 * 6 * 1024);
    __syncthreads();
    t1 = clock64(); rec(t0, t1);                                                    // 6 wcols + sync
    t0 = clock64();
    rf::col_reduce(pl, 2 * M, nseg, V);
    __syncthreads();
    t1 = clock64(); rec(t0, t1);                                                    // 7 reduce + sync
  }
  for (int i = threadIdx.x; i < 2 * M; i += blockDim.x) gout[1 + i] = O[i];
}

int main() {
  long long* d;
  uint32_t* g;
  cudaMalloc(&d, 8 * 16 * 8);
  cudaMalloc(&g, 4 * 2048);
  const size_t smem = (2 * (512 + 264) + 132 + 1024) * 4 + 1024 * 8 + 3 * 6 * 1024 * 4;
  cudaFuncSetAttribute(prim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[] = {"2 barriers", "fast_resolve", "fast_resolve(biased)", "cta_resolve", "limb_len",
                         "mul_fast", "wcols+sync", "reduce+sync"};
  for (int M : {4, 16, 64, 200, 400, 512}) {
    prim<<<1, 512, smem>>>(d, M, g);
    long long h[128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=%d:", M);
    for (int s = 0; s < 8; ++s) {
      long long v[8];
      for (int t = 0; t < 8; ++t) v[t] = h[t * 16 + s];
      std::sort(v, v + 8);
      printf("  %s %lld", names[s], v[4]);
    }
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
