// Determinant fold (ldlt.cpp:22-27 with FixedPoint::mul, fixed_point.cpp:40-53):
//   det_0 = 2^K,  det_{p+1} = tdiv_q_2exp(det_p * D_p, K)
// a strictly sequential chain of N big-by-medium products (the determinant
// reaches ~7.8 Mbit at BASELINE config 3).  Each step runs grid-wide:
//   F1 column sums of X*|D_p| (product scanning, 96-bit sums),
//   F2 per-chunk carry functions, F3 one-CTA scan of the chunk functions,
//   F4 digits with the resolved carry-in, emitted already shifted right by K.
// The sign is the product of the pivot signs, tracked on the host.
#include <cstdint>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"

namespace hgpu {

namespace {

constexpr int kFoldThreads = 256;
constexpr int kFoldG = 8;                            // columns per thread (F1)
constexpr int kChunk = kFoldThreads * 8;             // positions per chunk

// F1: column sums of X[0,nx) * D[0,nd) for columns [0, M).
__global__ void __launch_bounds__(kFoldThreads)
k_fold_colsum(const uint32_t* X, int nx, const uint32_t* D, int nd, int M,
              uint32_t* c0p, uint32_t* c1p, uint32_t* c2p) {
  extern __shared__ uint32_t Ds[];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) Ds[i] = D[i];
  __syncthreads();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = g * kFoldG;
  if (k0 >= M) return;
  uint32_t c0[kFoldG], c1[kFoldG], c2[kFoldG];
#pragma unroll
  for (int t = 0; t < kFoldG; ++t) c0[t] = c1[t] = c2[t] = 0u;
  // column k = sum_j D[j] X[k-j]
  const int jlo = max(0, k0 - nx + 1);
  const int jhi = min(nd - 1, k0 + kFoldG - 1);
  uint32_t w[kFoldG];  // w[t] = X[k0 + t - j]
#pragma unroll
  for (int t = 0; t < kFoldG; ++t) {
    const int i = k0 + t - jlo;
    w[t] = (i >= 0 && i < nx) ? __ldg(X + i) : 0u;
  }
  for (int j = jlo; j <= jhi; ++j) {
    const uint32_t dj = Ds[j];
#pragma unroll
    for (int t = 0; t < kFoldG; ++t)
      asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
          "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
          "addc.u32 %2, %2, 0;"
          : "+r"(c0[t]), "+r"(c1[t]), "+r"(c2[t])
          : "r"(dj), "r"(w[t]));
#pragma unroll
    for (int t = kFoldG - 1; t > 0; --t) w[t] = w[t - 1];
    const int i = k0 - j - 1;
    w[0] = (i >= 0 && i < nx) ? __ldg(X + i) : 0u;
  }
#pragma unroll
  for (int t = 0; t < kFoldG; ++t) {
    const int k = k0 + t;
    if (k < M) {
      c0p[k] = c0[t];
      c1p[k] = c1[t];
      c2p[k] = c2[t];
    }
  }
}

__device__ __forceinline__ int64_t fold_v(const uint32_t* c0p,
                                          const uint32_t* c1p,
                                          const uint32_t* c2p, int k, int M) {
  if (k >= M) return 0;
  int64_t v = c0p[k];
  if (k >= 1) v += c1p[k - 1];
  if (k >= 2) v += c2p[k - 2];
  return v;
}

__device__ __forceinline__ uint32_t carry_fn(int64_t v) { return cf_of(v, 32); }

// F2: carry function of each chunk of kChunk positions.
__global__ void __launch_bounds__(kFoldThreads)
k_fold_chunkfn(const uint32_t* c0p, const uint32_t* c1p, const uint32_t* c2p,
               int M, uint32_t* chunk_fn) {
  __shared__ uint32_t red[64];
  const int base = blockIdx.x * kChunk;
  const int per = kChunk / kFoldThreads;
  const int k0 = base + threadIdx.x * per;
  uint32_t F = kCfIdentity;
  for (int k = k0; k < k0 + per; ++k)
    F = cf_compose(carry_fn(fold_v(c0p, c1p, c2p, k, M)), F);
  // inclusive composition over the block = exclusive of a virtual next thread
  const uint32_t ex = cta_exclusive_compose(F, red);
  if (threadIdx.x == blockDim.x - 1) chunk_fn[blockIdx.x] = cf_compose(F, ex);
}

// F3: carry into every chunk (single CTA, sequential over warps of chunks).
__global__ void k_fold_scan(const uint32_t* chunk_fn, int nchunks,
                            int* chunk_carry) {
  __shared__ uint32_t red[64];
  __shared__ int carry_in;
  if (threadIdx.x == 0) carry_in = 0;
  __syncthreads();
  for (int b = 0; b < nchunks; b += blockDim.x) {
    const int i = b + threadIdx.x;
    const uint32_t f = i < nchunks ? chunk_fn[i] : kCfIdentity;
    const uint32_t ex = cta_exclusive_compose(f, red);
    const int cin = carry_in;
    if (i < nchunks) chunk_carry[i] = cf_apply(ex, cin);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_in = cf_apply(cf_compose(f, ex), cin);
    __syncthreads();
  }
}

// F4: digits of the product for this chunk (plus the next digit), emitted
// as X_new[i] = bits [32 i + K, 32 i + K + 32) of the product.
__global__ void __launch_bounds__(kFoldThreads)
k_fold_apply(const uint32_t* c0p, const uint32_t* c1p, const uint32_t* c2p,
             int M, const int* chunk_carry, int K, uint32_t* Xn, int nxn) {
  __shared__ uint32_t dig[kChunk + 1];
  __shared__ uint32_t red[64];
  const int base = blockIdx.x * kChunk;
  const int per = kChunk / kFoldThreads;
  const int k0 = threadIdx.x * per;  // local
  uint32_t F = kCfIdentity;
  for (int k = k0; k < k0 + per; ++k)
    F = cf_compose(carry_fn(fold_v(c0p, c1p, c2p, base + k, M)), F);
  const uint32_t ex = cta_exclusive_compose(F, red);
  const int cin_block = chunk_carry[blockIdx.x];
  int c = cf_apply(ex, cin_block);
  for (int k = k0; k < k0 + per; ++k) {
    const int64_t v = fold_v(c0p, c1p, c2p, base + k, M) + c;
    dig[k] = (uint32_t)v;
    c = (int)floor_shift(v, 32);
  }
  if (threadIdx.x == blockDim.x - 1) {
    // first digit of the next chunk
    const int64_t v = fold_v(c0p, c1p, c2p, base + kChunk, M) + c;
    dig[kChunk] = (uint32_t)v;
  }
  __syncthreads();
  const int a = K >> 5, b = K & 31;
  // output limbs i with source digit i + a inside [base, base + kChunk)
  const int ilo = max(0, base - a), ihi = min(nxn, base + kChunk - a);
  for (int i = ilo + threadIdx.x; i < ihi; i += blockDim.x) {
    const int s = i + a - base;  // in [0, kChunk)
    uint32_t v = dig[s] >> b;
    if (b) v |= dig[s + 1] << (32 - b);
    Xn[i] = v;
  }
}

}  // namespace

// Folds the n pivots (magnitudes in plimbs, lengths plen) into |det| at K
// bits.  X0/X1 ping-pong buffers of xcap limbs; col: 3*(xcap+pcap) words;
// chunk scratch: (xcap+pcap)/kChunk+2 words each.  Returns the final limb
// count (upper bound; the caller trims) or -1 if xcap is too small.
long long fold_pivots_device(const uint32_t* plimbs, const int* plen, int n,
                             int pcap, int K, uint32_t* X0, uint32_t* X1,
                             long long xcap, uint32_t* col, uint32_t* chunk_fn,
                             int* chunk_carry, cudaStream_t st,
                             long long* launches) {
  // X = 2^K
  long long nx = K / 32 + 1;
  if (nx > xcap) return -1;
  cudaMemsetAsync(X0, 0, nx * 4, st);
  const uint32_t one = 1u << (K % 32);
  cudaMemcpyAsync(X0 + K / 32, &one, 4, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);  // `one` lives on this stack frame
  uint32_t* X = X0;
  uint32_t* Y = X1;
  for (int p = 0; p < n; ++p) {
    const int nd = plen[p];
    const long long M = nx + nd;
    const long long nxn = M - K / 32;
    if (nxn > xcap || M > xcap + pcap) return -1;
    if (nxn <= 0) return 0;
    uint32_t* c0p = col;
    uint32_t* c1p = col + M;
    uint32_t* c2p = col + 2 * M;
    const int g1 = (int)((M + (long long)kFoldThreads * kFoldG - 1) /
                         ((long long)kFoldThreads * kFoldG));
    k_fold_colsum<<<g1, kFoldThreads, nd * 4, st>>>(
        X, (int)nx, plimbs + (long long)p * pcap, nd, (int)M, c0p, c1p, c2p);
    const int nchunks = (int)((M + kChunk - 1) / kChunk);
    k_fold_chunkfn<<<nchunks, kFoldThreads, 0, st>>>(c0p, c1p, c2p, (int)M,
                                                     chunk_fn);
    k_fold_scan<<<1, 1024, 0, st>>>(chunk_fn, nchunks, chunk_carry);
    k_fold_apply<<<nchunks, kFoldThreads, 0, st>>>(
        c0p, c1p, c2p, (int)M, chunk_carry, K, Y, (int)nxn);
    *launches += 4;
    uint32_t* t = X;
    X = Y;
    Y = t;
    nx = nxn;
  }
  if (X != X0) cudaMemcpyAsync(X0, X, nx * 4, cudaMemcpyDeviceToDevice, st);
  return nx;
}

}  // namespace hgpu
