// Transform-domain conversions shared by the LDL^T and the solve kernels:
// signed limb integer -> residues of its base-2^w digit polynomial -> NTT
// (transform_int), and back: inverse NTT, Garner CRT to signed coefficients,
// digit sums and one carry resolution to magnitude limbs (reconstruct_int).
// Both take the plan by reference, so one code path serves every
// (primes, length, digit width) plan.  All threads of the block must call.
#pragma once
#include <cstdint>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"

namespace hgpu {

// Loads a signed limb integer: returns sign, writes magnitude to dst (n limbs).
__device__ inline int load_int(const IntBuf& b, long long idx, int cap,
                               uint32_t* dst, int* len_out) {
  const int h = b.hdr[idx];
  const int len = h < 0 ? -h : h;
  const uint32_t* src = b.limbs + idx * (long long)cap;
  for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
  *len_out = len;
  __syncthreads();
  return h < 0 ? -1 : (h > 0 ? 1 : 0);
}

// Digit d_i (w bits) of |X| >> shift -> residues of the signed digit,
// forward NTT per prime, optional Montgomery scaling (x 2^32), store NW words
// to out.  sm: NW words of scratch, must not alias mag.
template <int RM = 16>
__device__ inline void transform_int(const DevPlan& P, const uint32_t* mag, int len,
                              long long shift, int sign, uint32_t* sm,
                              uint32_t* out, bool mont, const uint32_t* twm,
                              int* err) {
  const long long bits = (long long)limbs_bits(mag, len) - shift;
  if (bits > (long long)P.w * P.L) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapDigits);
  }
  const uint64_t dmask = (1ull << P.w) - 1ull;
  const bool word_digits = P.w == 32 && (shift & 31) == 0;  // digit i = limb i
  for (int gi = threadIdx.x; gi < P.NW; gi += blockDim.x) {
    const int j = gi >> P.logL, i = gi & (P.L - 1);
    const PrimeConsts& c = P.pc[j];
    const long long off = (long long)P.w * i + shift;
    uint64_t d;
    if (word_digits) {
      const long long li = i + (shift >> 5);
      d = li < len ? mag[li] : 0u;
    } else {
      d = ((uint64_t)field32(mag, len, off) | ((uint64_t)field32(mag, len, off + 32) << 32)) &
          dmask;
    }
    // d mod q: d = dh 2^32 + dl, dh 2^32 = dh r32 (Shoup), dl = dl * 1 (Shoup)
    uint32_t rr;
    if (P.w <= 27) {
      rr = (uint32_t)d;  // < 2^27 < q
    } else {
      const uint32_t dl = (uint32_t)d, dh = (uint32_t)(d >> 32);
      rr = reduce_2q(mul_shoup(dl, 1u, c.one_s, c.q), c.q);
      if (dh) {
        rr += reduce_2q(mul_shoup(dh, c.r32, c.r32s, c.q), c.q);
        rr = reduce_2q(rr, c.q);
      }
    }
    sm[gi] = (sign < 0 && rr) ? c.q - rr : rr;
  }
  __syncthreads();
  cta_ntt_fwd16<RM>(sm, P.np, P.logL, twm, P.pc);
  for (int gi = threadIdx.x; gi < P.NW; gi += blockDim.x) {
    uint32_t v = sm[gi];
    if (mont) {
      const PrimeConsts& c = P.pc[gi >> P.logL];
      v = reduce_2q(mont_mul(v, c.r64, c.q, c.qneg), c.q);
    }
    out[gi] = v;
  }
  __syncthreads();
}

// Inverse transform of A (np*L residues, bit-reversed, shared memory) back
// to the exact signed integer it represents: |value| in Lb[0, lcap) (zero
// padded), *len_out its limb length; returns the sign (+1 / -1), or 0 after
// flagging kCapCrt (coefficients out of the CRT range).  from = 1: A already
// holds the inverse transforms; from = 2: S already holds the digit sums
// (both computed elsewhere, e.g. split over a cluster).  Scratch: S and Dg
// hold L + T digit sums / digits; red is the scan scratch.  A is clobbered.
// Garner CRT of coefficient i's np residues (planes `stride` words apart),
// scaled by 1/L: the signed coefficient as a 128-bit two's complement value.
__device__ __forceinline__ unsigned __int128 garner_coef(const DevPlan& P, const uint32_t* A,
                                                         int stride, int i) {
  const int np = P.np;
  uint32_t a[kMaxPrimes];
  for (int j = 0; j < np; ++j) {
    const uint32_t q = P.pc[j].q;
    uint32_t v = reduce_2q(A[j * stride + i], q);
    a[j] = reduce_2q(mul_shoup(v, P.invL[j], P.invLp[j], q), q);
  }
  const uint32_t q0 = P.pc[0].q, q1 = P.pc[1].q;
  const uint32_t x0 = a[0];
  const uint32_t x0m1 = x0 >= q1 ? x0 - q1 : x0;
  const uint32_t x1 =
      reduce_2q(mul_shoup(a[1] + q1 - x0m1, P.g1, P.g1p, q1), q1);
  unsigned __int128 v = (unsigned __int128)x0 + (unsigned long long)x1 * q0;
  if (np >= 3) {
    const uint32_t q2 = P.pc[2].q;
    const uint32_t x0m2 = x0 >= q2 ? x0 - q2 : x0;
    uint32_t u = x0m2 + reduce_2q(mul_shoup(x1, P.q0m2, P.q0m2p, q2), q2);
    u = reduce_2q(u, q2);
    const uint32_t x2 =
        reduce_2q(mul_shoup(a[2] + q2 - u, P.g2, P.g2p, q2), q2);
    v += (unsigned __int128)x2 * P.q01;
    if (np == 4) {
      // x3 = (a3 - (x0 + x1 q0 + x2 q0 q1)) (q0 q1 q2)^-1  mod q3
      const uint32_t q3 = P.pc[3].q;
      const uint32_t x0m3 = x0 >= q3 ? x0 - q3 : x0;
      const uint32_t x2m3 = x2 >= q3 ? x2 - q3 : x2;
      uint32_t u3 = x0m3 + reduce_2q(mul_shoup(x1, P.q0m3, P.q0m3p, q3), q3);
      u3 = reduce_2q(u3, q3);
      u3 += reduce_2q(mul_shoup(x2m3, P.q01m3, P.q01m3p, q3), q3);
      u3 = reduce_2q(u3, q3);
      const uint32_t x3 =
          reduce_2q(mul_shoup(a[3] + q3 - u3, P.g3, P.g3p, q3), q3);
      const unsigned __int128 q012 =
          ((unsigned __int128)P.q012hi << 64) | P.q012lo;
      v += (unsigned __int128)x3 * q012;
    }
  }
  const unsigned __int128 Q = ((unsigned __int128)P.Qhi << 64) | P.Qlo;
  const unsigned __int128 H = ((unsigned __int128)P.Hhi << 64) | P.Hlo;
  if (v >= H) v -= Q;  // wraps to the two's complement of a negative value

  return v;
}

template <int RM = 16>
__device__ inline int reconstruct_int(const DevPlan& P, uint32_t* A, int64_t* S,
                                      uint64_t* Dg, uint32_t* Lb, int lcap,
                                      uint32_t* red, const uint32_t* itwm,
                                      int* err, int* len_out,
                                      long long* stamps = nullptr, int from = 0) {
  const int L = P.L, np = P.np, T = P.T, w = P.w;
  const int M = L + T;
  const uint64_t dmask = (1ull << w) - 1ull;
  // CRT (Garner), scaled by 1/L; signed result in np words, two's complement.
  if (from == 0) {
    cta_ntt_inv16<RM>(A, np, P.logL, itwm, P.pc);
  }
  if (stamps && threadIdx.x == 0) stamps[0] = clock64();
  if (from <= 1)
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const unsigned __int128 v = garner_coef(P, A, L, i);
    for (int t = 0; t < np; ++t) A[t * L + i] = (uint32_t)(v >> (32 * t));
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[1] = clock64();

  // Digit sums: s_k = sum_t piece_t(c_{k-t}); pieces are w-bit fields of the
  // two's complement coefficient, the top piece carries the sign.  With
  // w = 32 the pieces are the coefficient's words (sign words above the
  // np-th).
  if (from == 2) {
    // digit sums supplied by the caller
  } else if (w == 32) {
    for (int k = threadIdx.x; k < M; k += blockDim.x) {
      int64_t sk = 0;
      for (int t = 0; t < T; ++t) {
        const int i = k - t;
        if (i < 0 || i >= L) continue;
        const uint32_t top = A[(np - 1) * L + i];
        const uint32_t wt = t < np ? A[t * L + i] : ((top >> 31) ? 0xFFFFFFFFu : 0u);
        sk += t == T - 1 ? (int64_t)(int32_t)wt : (int64_t)wt;
      }
      S[k] = sk;
    }
  } else
  // one position per thread: piece t of coefficient k - t for t < T (T
  // decodes per position, every thread busy; the old 8-positions-per-thread
  // loop spent most of its time on out-of-range piece tests)
  for (int k = threadIdx.x; k < M; k += blockDim.x) {
    int64_t sk = 0;
    for (int t = 0; t < T; ++t) {
      const int i = k - t;
      if (i < 0 || i >= L) continue;
      unsigned __int128 cu = 0;
      for (int u = np - 1; u >= 0; --u) cu = (cu << 32) | A[u * L + i];
      cu <<= (128 - 32 * np);
      const __int128 c = ((__int128)cu) >> (128 - 32 * np);  // sign-extend
      const __int128 sh = c >> (w * t);
      sk += (t == T - 1) ? (int64_t)sh : (int64_t)((uint64_t)sh & dmask);
    }
    S[k] = sk;
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[2] = clock64();

  // One resolution of V = sum_k S_k 2^(wk) in two's complement: final carry
  // 0 -> V = D >= 0; -1 -> V = D - 2^(wM) < 0 and |V| = 2^(wM) - D, formed
  // digit-wise from the lowest nonzero digit k0 (zeros below it, 2^w - D_k0
  // at it, complemented digits above) instead of a second resolution.
  const int carry = cta_resolve(
      M, w,
      [&](int k) -> int64_t {
        int64_t vv = S[k] & (int64_t)dmask;
        if (k > 0) vv += S[k - 1] >> w;
        return vv;
      },
      [&](int k, uint64_t d) { Dg[k] = d; }, red);
  int sg = 1;
  bool bad = carry != 0 && carry != -1;
  if (carry == -1) {
    sg = -1;
    if (threadIdx.x == 0) red[0] = (uint32_t)M;
    __syncthreads();
    for (int k = threadIdx.x; k < M; k += blockDim.x)
      if (Dg[k]) {
        atomicMin(red, (uint32_t)k);
        break;
      }
    __syncthreads();
    const int k0 = (int)red[0];
    bad = k0 >= M;  // V = -2^(wM): magnitude does not fit M digits
    for (int k = threadIdx.x; k < M; k += blockDim.x)
      Dg[k] = k < k0 ? 0ull : (k == k0 ? ((dmask - Dg[k]) + 1ull) : (dmask - Dg[k]));
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapCrt);
    return 0;
  }
  // Pack base-2^w digits into 32-bit limbs of |W| (only the low 32 bits of
  // each shifted digit matter, so u64 wrap-around is harmless).
  const int nl = min(lcap, (int)(((long long)w * M + 31) / 32));
  if (w == 32) {
    for (int m = threadIdx.x; m < lcap; m += blockDim.x) Lb[m] = m < nl ? (uint32_t)Dg[m] : 0u;
  } else
  for (int m = threadIdx.x; m < lcap; m += blockDim.x) {
    uint64_t acc = 0;
    if (m < nl) {
      const int first = (32 * m) / w;
      for (int k = first; k < M && (long long)w * k < 32LL * m + 32; ++k) {
        const int shl = w * k - 32 * m;
        acc |= shl >= 0 ? (Dg[k] << shl) : (Dg[k] >> -shl);
      }
    }
    Lb[m] = (uint32_t)acc;
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[3] = clock64();
  const int len = cta_limb_len(Lb, lcap, red);
  if (threadIdx.x == 0 && (long long)w * M > 32LL * lcap) {
    for (int k = (32 * lcap) / w; k < M; ++k)
      if (Dg[k] && (long long)w * (k + 1) > 32LL * lcap)
        atomicOr(&err[kErrCapacity], kCapLimbs);
  }
  *len_out = len;
  return sg;
}

}  // namespace hgpu
