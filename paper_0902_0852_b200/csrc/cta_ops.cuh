// CTA-cooperative building blocks on shared-memory arrays:
//   * length-L number-theoretic transforms (Harvey lazy butterflies, Shoup
//     twiddles) in bit-reversed-output (forward) / bit-reversed-input
//     (inverse) order, so a length-L/2^k transform is a prefix of the
//     length-L one and one twiddle table serves every length;
//   * carry resolution of redundant digit sums by a block-wide scan over
//     carry *functions* (carry-in in {-1,0,1,2} -> carry-out), which makes
//     every multi-limb add/sub/normalise a constant-depth parallel step;
//   * schoolbook limb multiplication (product scanning, 96-bit column sums
//     on PTX carry chains), shifts and bit-field reads.
// All routines must be called by every thread of the block.
#pragma once
#include <cstdint>

#include "modarith.cuh"

namespace hgpu {

// ---------------------------------------------------------------- NTT ------

// Forward transforms of np residue planes x[j*L ...] (natural order in,
// values < 4q; bit-reversed order out, values < q), all primes in the same
// level loop so each radix-2 level costs one barrier.  tw/twp: per-prime
// tables T[m+i] = w^{(Lmax/2m) bitrev_m(i)} with Shoup companions, stride
// `ts` (shared by every L <= Lmax, which is what makes length-L/2^k
// transforms prefixes of length-L ones).
__device__ inline void cta_ntt_fwd_multi(uint32_t* x, int np, int logL,
                                         const uint32_t* tw,
                                         const uint32_t* twp, int ts,
                                         const PrimeConsts* pc) {
  const int L = 1 << logL, half = L >> 1;
  const int total = np * half;
  for (int lm = 0; lm < logL; ++lm) {
    const int m = 1 << lm;
    const int lt = logL - 1 - lm;  // t = L / (2m)
    for (int gb = threadIdx.x; gb < total; gb += blockDim.x) {
      const int j = gb >> (logL - 1);
      const int b = gb & (half - 1);
      const uint32_t q = pc[j].q, q2 = 2 * q;
      uint32_t* xj = x + j * L;
      const int i = b >> lt;
      const int j1 = (i << (lt + 1)) + (b & ((1 << lt) - 1));
      const int j2 = j1 + (1 << lt);
      uint32_t X = xj[j1];
      X = X >= q2 ? X - q2 : X;
      const uint32_t T = mul_shoup(xj[j2], tw[j * ts + m + i], twp[j * ts + m + i], q);
      xj[j1] = X + T;
      xj[j2] = X - T + q2;
    }
    __syncthreads();
  }
  for (int gi = threadIdx.x; gi < np * L; gi += blockDim.x) {
    const uint32_t q = pc[gi >> logL].q, q2 = 2 * q;
    uint32_t X = x[gi];
    X = X >= q2 ? X - q2 : X;
    x[gi] = X >= q ? X - q : X;
  }
  __syncthreads();
}

// Inverse transforms without the 1/L scale: bit-reversed in (values < 2q),
// natural order out (values < 2q).
__device__ inline void cta_ntt_inv_multi(uint32_t* x, int np, int logL,
                                         const uint32_t* itw,
                                         const uint32_t* itwp, int ts,
                                         const PrimeConsts* pc) {
  const int L = 1 << logL, half = L >> 1;
  const int total = np * half;
  for (int lt = 0; lt < logL; ++lt) {
    const int m = L >> (lt + 1);
    for (int gb = threadIdx.x; gb < total; gb += blockDim.x) {
      const int j = gb >> (logL - 1);
      const int b = gb & (half - 1);
      const uint32_t q = pc[j].q, q2 = 2 * q;
      uint32_t* xj = x + j * L;
      const int i = b >> lt;
      const int j1 = (i << (lt + 1)) + (b & ((1 << lt) - 1));
      const int j2 = j1 + (1 << lt);
      const uint32_t U = xj[j1], V = xj[j2];
      const uint32_t S = U + V;
      xj[j1] = S >= q2 ? S - q2 : S;
      xj[j2] = mul_shoup(U - V + q2, itw[j * ts + m + i], itwp[j * ts + m + i], q);
    }
    __syncthreads();
  }
}

// ------------------------------------------------ radix-16 NTT (SMEM) ------
// The same transforms as above, restructured for B200 SMEM: every pass does
// up to four butterfly levels on 16 registers per unit, so a length-2048
// transform is 3 passes (3 barriers) instead of 11, and the pass whose
// elements are contiguous (the last forward / first inverse pass) moves them
// with 16-byte vector loads.  Twiddles are in Montgomery form (one word):
//   mont_mul(a, w 2^32 mod q) = a w mod q  in [0, 2q)  for a < 2^32.
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t wm,
                                             uint32_t q, uint32_t qneg) {
  const uint64_t t = (uint64_t)a * wm;
  const uint32_t m = (uint32_t)t * qneg;
  return (uint32_t)((t + (uint64_t)m * q) >> 32);
}

template <int R>
__device__ __forceinline__ void load_unit(const uint32_t* xj, int base, int s,
                                          uint32_t* a) {
  if (s == 1 && R >= 4) {
#pragma unroll
    for (int u = 0; u < R; u += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(xj + base + u);
      a[u] = v.x; a[u + 1] = v.y; a[u + 2] = v.z; a[u + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < R; ++u) a[u] = xj[base + u * s];
  }
}
template <int R>
__device__ __forceinline__ void store_unit(uint32_t* xj, int base, int s,
                                           const uint32_t* a) {
  if (s == 1 && R >= 4) {
#pragma unroll
    for (int u = 0; u < R; u += 4)
      *reinterpret_cast<uint4*>(xj + base + u) = make_uint4(a[u], a[u + 1], a[u + 2], a[u + 3]);
  } else {
#pragma unroll
    for (int u = 0; u < R; ++u) xj[base + u * s] = a[u];
  }
}

// forward pass over levels [lm0, lm0 + log2 R)
template <int R>
__device__ inline void fwd_pass(uint32_t* x, int np, int logL, int lm0,
                                const uint32_t* twm, const PrimeConsts* pc) {
  constexpr int r = R == 2 ? 1 : (R == 4 ? 2 : (R == 8 ? 3 : 4));
  const int L = 1 << logL;
  const int ls = logL - lm0 - r;  // log2 s
  const int s = 1 << ls;
  const int lupp = logL - r;      // log2 units per prime
  const int total = np << lupp;
  for (int gu = threadIdx.x; gu < total; gu += blockDim.x) {
    const int j = gu >> lupp, v = gu & ((1 << lupp) - 1);
    const int i0 = v >> ls, jj = v & (s - 1);
    const int base = (i0 << (ls + r)) + jj;
    uint32_t* xj = x + j * L;
    const uint32_t* tw = twm + j * L;
    const uint32_t q = pc[j].q, q2 = 2 * q, qneg = pc[j].qneg;
    const int mi = (1 << lm0) + i0;
    uint32_t a[R];
    load_unit<R>(xj, base, s, a);
#pragma unroll
    for (int l = 0; l < r; ++l) {
      const int half = R >> (l + 1);
#pragma unroll
      for (int u = 0; u < R; ++u) {
        if (u & half) continue;
        const uint32_t w = tw[(mi << l) + (u >> (r - l))];
        uint32_t X = a[u];
        X = X >= q2 ? X - q2 : X;
        const uint32_t T = mont_mul(a[u + half], w, q, qneg);
        a[u] = X + T;
        a[u + half] = X - T + q2;
      }
    }
    store_unit<R>(xj, base, s, a);
  }
  __syncthreads();
}

// inverse (GS) pass over levels with half-sizes 2^lt0 .. 2^(lt0+log2R-1)
template <int R>
__device__ inline void inv_pass(uint32_t* x, int np, int logL, int lt0,
                                const uint32_t* itwm, const PrimeConsts* pc) {
  constexpr int r = R == 2 ? 1 : (R == 4 ? 2 : (R == 8 ? 3 : 4));
  const int L = 1 << logL;
  const int S = 1 << lt0;
  const int lupp = logL - r;
  const int total = np << lupp;
  for (int gu = threadIdx.x; gu < total; gu += blockDim.x) {
    const int j = gu >> lupp, v = gu & ((1 << lupp) - 1);
    const int bb = v >> lt0, jj = v & (S - 1);
    const int base = (bb << (lt0 + r)) + jj;
    uint32_t* xj = x + j * L;
    const uint32_t* tw = itwm + j * L;
    const uint32_t q = pc[j].q, q2 = 2 * q, qneg = pc[j].qneg;
    uint32_t a[R];
    load_unit<R>(xj, base, S, a);
#pragma unroll
    for (int l = 0; l < r; ++l) {
      const int half = 1 << l;
      const int ml = L >> (lt0 + l + 1);
#pragma unroll
      for (int u = 0; u < R; ++u) {
        if (u & half) continue;
        const uint32_t w = tw[ml + (bb << (r - l - 1)) + (u >> (l + 1))];
        const uint32_t U = a[u], V = a[u + half];
        const uint32_t Sm = U + V;
        a[u] = Sm >= q2 ? Sm - q2 : Sm;
        a[u + half] = mont_mul(U - V + q2, w, q, qneg);
      }
    }
    store_unit<R>(xj, base, S, a);
  }
  __syncthreads();
}

// Forward: natural in (< 4q), bit-reversed out (< q).  twm: [np][L] table
// T[m+i] in Montgomery form (any memory; shared memory when it fits).
// RM (16, 8 or 4): the widest pass; narrower passes use more threads per
// transform (the single-transform chains of the solve prefer them).
template <int RM = 16>
__device__ inline void cta_ntt_fwd16(uint32_t* x, int np, int logL,
                                     const uint32_t* twm, const PrimeConsts* pc) {
  // first pass takes logL mod 4 levels (large stride), then passes of 4;
  // the last pass (s = 1) moves contiguous 16-word units
  constexpr int rb = RM == 16 ? 4 : (RM == 8 ? 3 : 2);
  int lm = 0;
  while (lm < logL) {
    const int r = (lm == 0 && logL % rb) ? logL % rb : rb;
    switch (r) {
      case 1: fwd_pass<2>(x, np, logL, lm, twm, pc); break;
      case 2: fwd_pass<4>(x, np, logL, lm, twm, pc); break;
      case 3: fwd_pass<8>(x, np, logL, lm, twm, pc); break;
      default: fwd_pass<16>(x, np, logL, lm, twm, pc); break;
    }
    lm += r;
  }
  const int L = 1 << logL;
  for (int gi = threadIdx.x; gi < np * L; gi += blockDim.x) {
    const uint32_t q = pc[gi >> logL].q, q2 = 2 * q;
    uint32_t X = x[gi];
    X = X >= q2 ? X - q2 : X;
    x[gi] = X >= q ? X - q : X;
  }
  __syncthreads();
}

// Inverse without 1/L: bit-reversed in (< 2q), natural out (< 2q).
template <int RM = 16>
__device__ inline void cta_ntt_inv16(uint32_t* x, int np, int logL,
                                     const uint32_t* itwm, const PrimeConsts* pc) {
  // passes of 4 from the contiguous end (S = 1); the last takes the rest
  constexpr int rb = RM == 16 ? 4 : (RM == 8 ? 3 : 2);
  int lt = 0;
  while (lt < logL) {
    const int r = logL - lt >= rb ? rb : logL - lt;
    switch (r) {
      case 1: inv_pass<2>(x, np, logL, lt, itwm, pc); break;
      case 2: inv_pass<4>(x, np, logL, lt, itwm, pc); break;
      case 3: inv_pass<8>(x, np, logL, lt, itwm, pc); break;
      default: inv_pass<16>(x, np, logL, lt, itwm, pc); break;
    }
    lt += r;
  }
}

// ----------------------------------------------------- carry functions -----
// A carry function maps carry-in c in {-1,0,1,2} to carry-out in the same
// set.  It is stored as four bytes, byte (c+1) = out+1 in [0,3], so that
// composition is one byte permute: (later o earlier) byte i =
// later.byte[earlier.byte[i]].
constexpr uint32_t kCfIdentity = 0x03020100u;

__device__ __forceinline__ int cf_apply(uint32_t f, int c) {
  return (int)((f >> (8 * (c + 1))) & 0xFFu) - 1;
}
// later o earlier
__device__ __forceinline__ uint32_t cf_compose(uint32_t later,
                                               uint32_t earlier) {
  // selector nibble i = earlier byte i (each in [0,3])
  const uint32_t t = earlier | (earlier >> 4);
  const uint32_t sel = (t & 0xFFu) | ((t >> 8) & 0xFF00u);
  return __byte_perm(later, 0u, sel);
}

// Exclusive block-wide scan under composition: returns f_{t-1} o ... o f_0
// and, in *total, the composition of all threads' functions.
// `red` needs blockDim.x/32 words of shared memory.
__device__ inline uint32_t cta_exclusive_compose(uint32_t f, uint32_t* red,
                                                 uint32_t* total = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t x = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = cf_compose(x, y);
  }
  if (lane == 31) red[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < nw ? red[lane] : kCfIdentity;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = cf_compose(w, y);
    }
    if (lane < nw) red[lane] = w;
  }
  __syncthreads();
  const uint32_t before_warp = wid > 0 ? red[wid - 1] : kCfIdentity;
  if (total) *total = red[nw - 1];
  uint32_t excl = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl = kCfIdentity;
  __syncthreads();
  return cf_compose(excl, before_warp);
}

__device__ __forceinline__ int64_t floor_shift(int64_t v, int bits) {
  return v >> bits;  // arithmetic shift = floor division by 2^bits
}

// carry function of one position holding v (carry-out = floor((v+c)/2^bits))
__device__ __forceinline__ uint32_t cf_of(int64_t v, int bits) {
  uint32_t f = 0;
#pragma unroll
  for (int c = -1; c <= 2; ++c)
    f |= (uint32_t)(floor_shift(v + c, bits) + 1) << (8 * (c + 1));
  return f;
}

// Resolves sum_{k<M} v_k 2^{bits k} into digits d_k in [0, 2^bits), where
// getv(k) returns v_k in [-2^bits + 1, 3*2^bits - 2] (int64), bits <= 48.
// putd(k, d) receives every digit (uint64_t; callers with bits <= 32 may
// take it as uint32_t).  Returns the final carry (in {-1,0,1,2}) to all
// threads: the exact value is sum d_k 2^{bits k} + carry 2^{bits M}.
// `red` needs blockDim.x/32 words.  getv must not read what putd writes.
template <class GetV, class PutD>
__device__ int cta_resolve(int M, int bits, GetV getv, PutD putd,
                           uint32_t* red) {
  const int nt = blockDim.x;
  const int chunk = (M + nt - 1) / nt;
  const int k0 = min(M, (int)threadIdx.x * chunk);
  const int k1 = min(M, k0 + chunk);
  uint32_t F = kCfIdentity;
  for (int k = k0; k < k1; ++k) F = cf_compose(cf_of(getv(k), bits), F);
  uint32_t total;
  const uint32_t P = cta_exclusive_compose(F, red, &total);
  int c = cf_apply(P, 0);
  const int64_t mask = (int64_t(1) << bits) - 1;
  for (int k = k0; k < k1; ++k) {
    const int64_t v = getv(k) + c;
    putd(k, (uint64_t)(v & mask));  // bits <= 48: digits may exceed 32 bits
    c = (int)floor_shift(v, bits);
  }
  __syncthreads();  // digits visible to every thread on return
  return cf_apply(total, 0);
}

// ------------------------------------------- warp-level variants ---------
// The same carry-function resolution and products for one warp (all 32
// lanes), with __syncwarp only: the reciprocal's small Newton levels run on
// a single warp, where block-wide barriers would cost more than the work.

__device__ __forceinline__ uint32_t warp_exclusive_compose(uint32_t f,
                                                           uint32_t* total) {
  const int lane = threadIdx.x & 31;
  uint32_t x = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = cf_compose(x, y);
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  uint32_t excl = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl = kCfIdentity;
  return excl;
}

template <class GetV, class PutD>
__device__ int warp_resolve(int M, int bits, GetV getv, PutD putd) {
  const int lane = threadIdx.x & 31;
  const int chunk = (M + 31) / 32;
  const int k0 = min(M, lane * chunk);
  const int k1 = min(M, k0 + chunk);
  uint32_t F = kCfIdentity;
  for (int k = k0; k < k1; ++k) F = cf_compose(cf_of(getv(k), bits), F);
  uint32_t total;
  const uint32_t Pf = warp_exclusive_compose(F, &total);
  int c = cf_apply(Pf, 0);
  const int64_t mask = (int64_t(1) << bits) - 1;
  for (int k = k0; k < k1; ++k) {
    const int64_t v = getv(k) + c;
    putd(k, (uint64_t)(v & mask));
    c = (int)floor_shift(v, bits);
  }
  __syncwarp();
  return cf_apply(total, 0);
}

// ------------------------------------------------------- limb helpers -----

// Bits [off, off+32) of the non-negative integer a[0..n) (off may be < 0).
__device__ __forceinline__ uint32_t field32(const uint32_t* a, int n,
                                            long long off) {
  const long long li = off >> 5;
  const int sh = (int)(off & 31);
  const uint32_t lo = (li >= 0 && li < n) ? a[li] : 0u;
  if (sh == 0) return lo;
  const uint32_t hi = (li + 1 >= 0 && li + 1 < n) ? a[li + 1] : 0u;
  return (lo >> sh) | (hi << (32 - sh));
}

// Number of significant limbs (block-wide).  `red` needs 1 word.
__device__ inline int cta_limb_len(const uint32_t* a, int n, uint32_t* red) {
  if (threadIdx.x == 0) red[0] = 0;
  __syncthreads();
  int best = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (a[i]) best = i + 1;
  if (best) atomicMax(red, (uint32_t)best);
  __syncthreads();
  const int len = (int)red[0];
  __syncthreads();
  return len;
}

__device__ inline int warp_limb_len(const uint32_t* a, int n) {
  int best = 0;
  for (int i = threadIdx.x & 31; i < n; i += 32)
    if (a[i]) best = i + 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  return best;
}

__device__ __forceinline__ int limbs_bits(const uint32_t* a, int len) {
  return len == 0 ? 0 : 32 * (len - 1) + (32 - __clz(a[len - 1]));
}

// Column sums of a*b for the G columns k0..k0+G-1 over i in [ilo, ihi]:
// acc[t] + cc[t] 2^64 += sum_i a[i] b[k0+t-i].  The i-loop is unrolled by G,
// so the b-window sits in static registers (2G-1 values per block) and every
// product is one IMAD.WIDE.U32 with carry-out plus one IMAD.X, with G
// independent accumulator chains (measured 2x the throughput of the rolled
// loop, whose window shifts and CC chains cost register moves).
template <int G>
__device__ __forceinline__ void col_block(const uint32_t* a, const uint32_t* b,
                                          int nb, int k0, int ilo, int ihi,
                                          uint64_t* acc, uint32_t* cc) {
  for (int i = ilo; i <= ihi; i += G) {
    uint32_t av[G];
#pragma unroll
    for (int u = 0; u < G; ++u) av[u] = (i + u <= ihi) ? a[i + u] : 0u;
    uint32_t bw[2 * G - 1];  // bw[m] = b[k0 - i - (G-1) + m]
#pragma unroll
    for (int m = 0; m < 2 * G - 1; ++m) {
      const int j = k0 - i - (G - 1) + m;
      bw[m] = (j >= 0 && j < nb) ? b[j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int t = 0; t < G; ++t)
        asm("{\n\t.reg .u64 pr;\n\t"
            "mul.wide.u32 pr, %2, %3;\n\t"
            "add.cc.u64 %0, %0, pr;\n\t"
            "addc.u32 %1, %1, 0;\n\t}"
            : "+l"(acc[t]), "+r"(cc[t])
            : "r"(av[u]), "r"(bw[G - 1 + t - u]));
  }
}

// out[0..M) = low M limbs of a*b (M <= na+nb gives the exact product when
// M == na+nb).  Product scanning: a work item is a group of 8 consecutive
// output columns times one segment of its i-range, so long middle columns
// are split across threads (load balance); each item keeps 96-bit column
// sums (col_block) and writes them to its segment's planes.
// col: scratch of `col_words` >= 3*M words (more words allow more segments);
// out must not alias a, b or col.  red: blockDim/32+1 words.
// With k_begin > 0 only columns [k_begin, M) are formed (a "short product"):
// out[k - k_begin] holds the digits of sum_{k >= k_begin} col_k 2^{32 k},
// i.e. the top of the product without the carry from the dropped columns
// (below the true value by < min(na,nb) 2^{32 k_begin + 33}).
__device__ inline void cta_mul(const uint32_t* a, int na, const uint32_t* b,
                               int nb, uint32_t* out, int M_end, uint32_t* col,
                               uint32_t* red, int col_words = 0,
                               int k_begin = 0) {
  constexpr int G = 8;
  const int M = M_end - k_begin;  // columns formed
  const int ngroups = (M + G - 1) / G;
  const int minlen = min(na, nb);
  // split a group's i-range only when segments stay >= 32 iterations and
  // there are idle threads to take them
  // nseg > 1 needs 3*nseg*M words of planes plus 2*M for the reduced sums
  const int maxseg = max(1, ((col_words > 0 ? col_words : 3 * M) - 2 * M) / (3 * M));
  const int want = (2 * (int)blockDim.x + ngroups - 1) / max(ngroups, 1);
  const int bylen = max(1, (minlen + G - 1) / 32);
  const int nseg = max(1, min(min(min(maxseg, want), bylen), 16));
  const int seglen = (minlen + G - 1 + nseg - 1) / nseg;  // group i-range <= minlen+G-1
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
  // S_k = sum over segments of the column value at weight 2^(32k) (< 2^64),
  // reduced once into (lo, hi) planes 0 and 1 of segment 0's storage;
  // v_k = lo_k + hi_{k-1} then stays in the resolve domain.
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
    cta_resolve(
        M, 32,
        [&](int k) -> int64_t {
          int64_t v = slo[k];
          if (k >= 1) v += shi[k - 1];
          return v;
        },
        [&](int k, uint32_t d) { out[k] = d; }, red);
    return;
  }
  const uint32_t* c0p = col;
  const uint32_t* c1p = col + M;
  const uint32_t* c2p = col + 2 * M;
  cta_resolve(
      M, 32,
      [&](int k) -> int64_t {
        int64_t v = c0p[k];
        if (k >= 1) v += c1p[k - 1];
        if (k >= 2) v += c2p[k - 2];
        return v;
      },
      [&](int k, uint32_t d) { out[k] = d; }, red);
}

// Warp version of cta_mul (full product columns [0, M)): each lane forms
// groups of 4 consecutive columns (col_block), then a warp carry resolution.
// col: 3*M words; out must not alias a, b or col.
__device__ inline void warp_mul(const uint32_t* a, int na, const uint32_t* b,
                                int nb, uint32_t* out, int M, uint32_t* col) {
  constexpr int G = 4;
  for (int k0 = (threadIdx.x & 31) * G; k0 < M; k0 += 32 * G) {
    uint64_t acc[G];
    uint32_t c2[G];
#pragma unroll
    for (int t = 0; t < G; ++t) acc[t] = 0ull, c2[t] = 0u;
    const int ilo = max(0, k0 - nb + 1), ihi = min(k0 + G - 1, na - 1);
    if (ilo <= ihi) col_block<G>(a, b, nb, k0, ilo, ihi, acc, c2);
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int k = k0 + t;
      if (k < M) {
        col[k] = (uint32_t)acc[t];
        col[M + k] = (uint32_t)(acc[t] >> 32);
        col[2 * M + k] = c2[t];
      }
    }
  }
  __syncwarp();
  warp_resolve(
      M, 32,
      [&](int k) -> int64_t {
        int64_t v = col[k];
        if (k >= 1) v += col[M + k - 1];
        if (k >= 2) v += col[2 * M + k - 2];
        return v;
      },
      [&](int k, uint32_t d) { out[k] = d; });
}


}  // namespace hgpu
