// Microbenchmark of the CTA-wide limb product (cta_ops.cuh: cta_mul, G = 8)
// against a G-column variant (cta_mul2<G>) at the reciprocal's and the
// solve's sizes: clock64 cycles per call, one CTA alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_0902_0852_b200/csrc -o /tmp/mb scripts/mul_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "cta_ops.cuh"

using namespace hgpu;


template <int G>
__device__ inline void cta_mul2(const uint32_t* a, int na, const uint32_t* b,
                                int nb, uint32_t* out, int M_end, uint32_t* col,
                                uint32_t* red, int col_words = 0,
                                int k_begin = 0) {
  const int M = M_end - k_begin;
  const int ngroups = (M + G - 1) / G;
  const int minlen = min(na, nb);
  const int maxseg = max(1, ((col_words > 0 ? col_words : 3 * M) - 2 * M) / (3 * M));
  const int want = (2 * (int)blockDim.x + ngroups - 1) / max(ngroups, 1);
  const int bylen = max(1, (minlen + G - 1) / 32);
  const int nseg = max(1, min(min(min(maxseg, want), bylen), 16));
  const int seglen = (minlen + G - 1 + nseg - 1) / nseg;
  const int items = ngroups * nseg;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int g = nseg == 1 ? it : it / nseg, sgi = it - g * nseg;
    const int k0 = k_begin + g * G;
    uint64_t acc[G];
    uint32_t c2[G];
#pragma unroll
    for (int t = 0; t < G; ++t) acc[t] = 0ull, c2[t] = 0u;
    if (na > 0 && nb > 0) {
      const int glo = max(0, k0 - nb + 1);
      const int ghi = min(k0 + G - 1, na - 1);
      const int ilo = glo + sgi * seglen;
      const int ihi = min(ghi, ilo + seglen - 1);
      if (ilo <= ihi) col_block<G>(a, b, nb, k0, ilo, ihi, acc, c2);
    }
    uint32_t* pl = col + (size_t)sgi * 3 * M;
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int k = k0 + t - k_begin;
      if (k < M) {
        pl[k] = (uint32_t)acc[t];
        pl[M + k] = (uint32_t)(acc[t] >> 32);
        pl[2 * M + k] = c2[t];
      }
    }
  }
  __syncthreads();
  if (nseg > 1) {
    for (int k = threadIdx.x; k < M; k += blockDim.x) {
      uint64_t v = 0;
      for (int sg = 0; sg < nseg; ++sg) {
        const uint32_t* pl = col + (size_t)sg * 3 * M;
        v += pl[k];
        if (k >= 1) v += pl[M + k - 1];
        if (k >= 2) v += pl[2 * M + k - 2];
      }
      col[3 * (size_t)nseg * M + k] = (uint32_t)v;
      col[3 * (size_t)nseg * M + M + k] = (uint32_t)(v >> 32);
    }
    __syncthreads();
    const uint32_t* slo = col + 3 * (size_t)nseg * M;
    const uint32_t* shi = slo + M;
    cta_resolve(M, 32, [&](int k) -> int64_t { int64_t v = slo[k]; if (k >= 1) v += shi[k - 1]; return v; },
                [&](int k, uint32_t d) { out[k] = d; }, red);
    return;
  }
  const uint32_t* c0p = col;
  const uint32_t* c1p = col + M;
  const uint32_t* c2p = col + 2 * M;
  cta_resolve(M, 32, [&](int k) -> int64_t {
        int64_t v = c0p[k]; if (k >= 1) v += c1p[k - 1]; if (k >= 2) v += c2p[k - 2]; return v; },
      [&](int k, uint32_t d) { out[k] = d; }, red);
}

template <int VARIANT>
__global__ void __launch_bounds__(512) k_bench(int na, int nb, int reps, long long* cyc,
                                               uint32_t* out_g, int col_words_arg) {
  extern __shared__ uint32_t sm[];
  uint32_t* a = sm;
  uint32_t* b = a + na;
  const int M = na + nb;
  uint32_t* out = b + nb;
  uint32_t* col = out + M;
  const int col_words = col_words_arg;
  uint32_t* red = col + col_words;
  for (int i = threadIdx.x; i < na; i += blockDim.x) a[i] = 0x9E3779B9u * (i + 1);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) b[i] = 0x7F4A7C15u * (i + 3);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (VARIANT == 0) cta_mul(a, na, b, nb, out, M, col, red, col_words);
    else cta_mul2<16>(a, na, b, nb, out, M, col, red, col_words);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  for (int i = threadIdx.x; i < M; i += blockDim.x) out_g[i] = out[i];
}

int main() {
  const int sizes[][2] = {{650, 1038}, {650, 830}, {398, 340}, {676, 676}};
  long long* cyc;
  uint32_t* outg;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&outg, 4 * 4096);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(k_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (auto& s : sizes) {
    for (int threads : {256, 512}) for (int cw : {0, 3 * (s[0] + s[1]) * 2}) {
      long long c0 = 0, c1 = 0;
      std::vector<uint32_t> r0(4096), r1(4096);
      k_bench<0><<<1, threads, smem>>>(s[0], s[1], 5, cyc, outg, cw);
      cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(r0.data(), outg, 4 * 4096, cudaMemcpyDeviceToHost);
      k_bench<1><<<1, threads, smem>>>(s[0], s[1], 5, cyc, outg, cw);
      cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(r1.data(), outg, 4 * 4096, cudaMemcpyDeviceToHost);
      bool same = true;
      for (int i = 0; i < s[0] + s[1]; ++i) same &= r0[i] == r1[i];
      printf("cw %5d %4d x %4d, %3d threads: cta_mul %7lld cycles (%.2f prod/cyc), cta_mul2 %7lld cycles (%.2f prod/cyc) %s\n",
             cw, s[0], s[1], threads, c0, (double)s[0] * s[1] / c0, c1, (double)s[0] * s[1] / c1, same ? "same" : "DIFFERENT");
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
