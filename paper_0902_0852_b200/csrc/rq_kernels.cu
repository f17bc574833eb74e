// Rayleigh quotient of inverse iteration on the device (the
// north-star's "Rayleigh-quotient kernels" -- the reference finds lambda_1
// by the secant, secant.cpp:27-117, and has no such step, so
// oracle/pyoracle.py:inverse_iteration_py defines the arithmetic).
//
// After a solve the vectors u (the right-hand side) and y (the solution)
// sit in the solve's integer buffer, n signed limb integers each.  One step
// of the iteration needs
//   num = sum_i y_i u_i,  den = sum_i y_i y_i      (exact integers)
//   rho = s + tdiv(num 2^K, den)                   (one division, host)
//   u'  = y scaled by a power of two: tdiv_2exp(y_i, sh) or y_i 2^-sh
// Here the 2n multiprecision products, their exact sums and the rescaling
// run on the GPU; only num, den and the bit length of y leave the device.
//   k_rq_products  one CTA per entry: |y_i||u_i| and |y_i|^2 (cta_mul), as
//                  magnitude digits plus a sign
//   k_rq_reduce    one thread per limb column: signed sum over the entries
//   k_rq_carry     one carry pass over the column sums -> two's complement
//   k_rq_rescale   one CTA per entry: the shifted magnitude of y_i into u_i
#include <cstdint>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"

namespace hgpu {

namespace {
constexpr int kRqThreads = 256;

// words of one k_rq_products CTA for operands of at most `maxlen` limbs:
// Y | U | product 2 maxlen | column planes 3 * 2 maxlen | red 64
__host__ __device__ inline long long rq_words(int maxlen) {
  return 2LL * maxlen + 2LL * maxlen + 6LL * maxlen + 64;
}
}  // namespace

size_t rq_products_words(int maxlen) { return (size_t)rq_words(maxlen); }

// prod[(which * n + i) * M + k], which = 0: |y_i u_i|, 1: y_i^2, M = 2 maxlen
// columns (zero padded); psign[which * n + i] in {-1, 0, 1}.
__global__ void __launch_bounds__(kRqThreads)
k_rq_products(IntBuf v, int yi0, int ui0, int n, int Wv, int maxlen, uint32_t* prod,
              int* psign, uint32_t* gscratch, int* err) {
  extern __shared__ uint32_t sm_dyn[];
  uint32_t* sm = gscratch ? gscratch + (long long)blockIdx.x * rq_words(maxlen) : sm_dyn;
  uint32_t* Y = sm;
  uint32_t* U = Y + maxlen;
  uint32_t* P = U + maxlen;
  uint32_t* col = P + 2 * maxlen;
  uint32_t* red = col + 6 * maxlen;
  const int M = 2 * maxlen;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int hy = v.hdr[yi0 + i], hu = v.hdr[ui0 + i];
    const int ly = hy < 0 ? -hy : hy, lu = hu < 0 ? -hu : hu;
    if (ly > maxlen || lu > maxlen) {  // the host sized the layout too small
      if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
      return;
    }
    for (int k = threadIdx.x; k < ly; k += blockDim.x)
      Y[k] = v.limbs[(long long)(yi0 + i) * Wv + k];
    for (int k = threadIdx.x; k < lu; k += blockDim.x)
      U[k] = v.limbs[(long long)(ui0 + i) * Wv + k];
    __syncthreads();
    for (int which = 0; which < 2; ++which) {
      const uint32_t* B = which ? Y : U;
      const int lb = which ? ly : lu;
      const int nP = (ly == 0 || lb == 0) ? 0 : ly + lb;
      if (nP > 0) cta_mul(Y, ly, B, lb, P, nP, col, red);
      uint32_t* out = prod + ((long long)which * n + i) * M;
      for (int k = threadIdx.x; k < M; k += blockDim.x) out[k] = k < nP ? P[k] : 0u;
      if (threadIdx.x == 0)
        psign[which * n + i] = nP == 0 ? 0 : (which ? 1 : ((hy < 0) != (hu < 0) ? -1 : 1));
      __syncthreads();
    }
  }
}

// colsum[which * M + k] = sum_i psign * prod[..][k]  (|sum| < n 2^32)
__global__ void k_rq_reduce(const uint32_t* prod, const int* psign, int n, int M,
                            long long* colsum) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int which = blockIdx.y;
  if (k >= M) return;
  const uint32_t* p = prod + (long long)which * n * M + k;
  const int* sg = psign + which * n;
  long long s = 0;
  for (int i = 0; i < n; ++i) {
    const int g = sg[i];
    if (g == 0) continue;
    const long long d = (long long)p[(long long)i * M];
    s += g > 0 ? d : -d;
  }
  colsum[(long long)which * M + k] = s;
}

// out[which * (M + 2) + k]: the two's-complement limbs of sum_k colsum[k]
// 2^(32 k), M + 2 limbs (the last two hold the sign-extended final carry).
__global__ void k_rq_carry(const long long* colsum, int M, uint32_t* out) {
  constexpr int kChunk = 2048;
  __shared__ long long buf[kChunk];
  __shared__ uint32_t dig[kChunk];
  __shared__ long long carry_s;
  const int which = blockIdx.x;
  const long long* cs = colsum + (long long)which * M;
  uint32_t* o = out + (long long)which * (M + 2);
  if (threadIdx.x == 0) carry_s = 0;
  for (int k0 = 0; k0 < M; k0 += kChunk) {
    const int m = min(kChunk, M - k0);
    for (int k = threadIdx.x; k < m; k += blockDim.x) buf[k] = cs[k0 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
      long long c = carry_s;
      for (int k = 0; k < m; ++k) {
        const long long t = buf[k] + c;  // |buf| < 2^52, |c| < 2^31: no overflow
        dig[k] = (uint32_t)t;
        c = t >> 32;  // floor
      }
      carry_s = c;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) o[k0 + k] = dig[k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    o[M] = (uint32_t)carry_s;
    o[M + 1] = (uint32_t)(carry_s >> 32);
  }
}

// u_i = tdiv_2exp(y_i, sh) (sh > 0) or y_i 2^(-sh) (sh <= 0), every i < n
__global__ void __launch_bounds__(kRqThreads)
k_rq_rescale(IntBuf v, int yi0, int ui0, int n, int Wv, int sh, int* err) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int hy = v.hdr[yi0 + i];
    const int ly = hy < 0 ? -hy : hy;
    const uint32_t* Y = v.limbs + (long long)(yi0 + i) * Wv;
    uint32_t* U = v.limbs + (long long)(ui0 + i) * Wv;
    const int bits = limbs_bits(Y, ly) - sh;  // of the shifted magnitude
    const int len = bits <= 0 ? 0 : (bits + 31) / 32;
    if (len > Wv) {
      if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
      return;
    }
    for (int k = threadIdx.x; k < Wv; k += blockDim.x)
      U[k] = k < len ? field32(Y, ly, 32LL * k + sh) : 0u;
    if (threadIdx.x == 0) v.hdr[ui0 + i] = len == 0 ? 0 : (hy < 0 ? -len : len);
  }
}

cudaError_t configure_rq_kernels(int maxlen, bool* use_global) {
  int dev = 0, maxopt = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t need = rq_products_words(maxlen) * 4;
  *use_global = need > (size_t)maxopt;
  if (*use_global) return cudaSuccess;
  return cudaFuncSetAttribute(k_rq_products, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)need);
}

cudaError_t launch_rq_products(IntBuf v, int yi0, int ui0, int n, int Wv, int maxlen,
                               uint32_t* prod, int* psign, uint32_t* gscratch, int grid,
                               int* err, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = gscratch ? 0 : rq_products_words(maxlen) * 4;
  kernel_launch_count_add(1);
  k_rq_products<<<grid, kRqThreads, smem, st>>>(v, yi0, ui0, n, Wv, maxlen, prod, psign,
                                                gscratch, err);
  return cudaGetLastError();
}

cudaError_t launch_rq_reduce(const uint32_t* prod, const int* psign, int n, int M,
                             long long* colsum, uint32_t* out, cudaStream_t st) {
  dim3 grid((M + 127) / 128, 2);
  kernel_launch_count_add(1);
  k_rq_reduce<<<grid, 128, 0, st>>>(prod, psign, n, M, colsum);
  kernel_launch_count_add(1);
  k_rq_carry<<<2, 256, 0, st>>>(colsum, M, out);
  return cudaGetLastError();
}

cudaError_t launch_rq_rescale(IntBuf v, int yi0, int ui0, int n, int Wv, int sh, int* err,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  kernel_launch_count_add(1);
  k_rq_rescale<<<n, kRqThreads, 0, st>>>(v, yi0, ui0, n, Wv, sh, err);
  return cudaGetLastError();
}

}  // namespace hgpu
