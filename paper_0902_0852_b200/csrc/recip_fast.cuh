// Latency-lean pivot reciprocal (the chain's k_recip step).
//
// Same numbers as recip_body (ldlt_kernels.cu): the same Newton ladder
// (recip_levels), the same truncated divisor D' per level, the same low and
// high short products and the same resolves, so Y is bit-identical and the
// error contract |Y - 2^S/D| <= 4 that k_divide relies on carries over.  What
// changes is how each level is executed on the CTA:
//
//  * every level runs on the whole CTA (no single-warp phase): a product is
//    split into items of 4 output columns x 32 terms, so even a 7 x 5 limb
//    product finishes in one short pass and a 398 x 340 one spreads over
//    ~1200 items instead of a few hundred long serial chains;
//  * an item's column sums go to per-column shared-memory accumulators with
//    64-bit shared atomics (the low and high 32-bit halves separately, so no
//    sum can overflow), instead of per-segment planes and a reduction pass;
//  * the two tiny first levels (divisor <= 4 limbs) run on thread 0 alone in
//    128-bit registers, with no barrier inside.
//
// The ldlt.cpp arithmetic this serves: R_p[r] = tdiv_q(V_p[r] 2^{K/2}, V_p[p])
// (ldlt.cpp:15-20) for every row of stage p, all from one reciprocal of
// V_p[p].
#pragma once
#include "cta_ops.cuh"

namespace hgpu {
namespace rf {

constexpr int kSegMax = 6;  // i-range segments per column block (planes)

// 32-bit words of the launch's dynamic shared memory
__device__ __forceinline__ long long dyn_smem_words() {
  uint32_t b;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(b));
  return b / 4;
}

// Block-wide resolution of sum_{k<M} v_k 2^{32k} into 32-bit digits mod
// 2^{32M}, for v_k + bias in [0, 3 2^32) with bias = 0 or 2^32 - 1 (biased:
// v_k in [-2^32 + 1, 2^33]; the biases sum to 2^{32M} - 1, so a carry of 1
// into position 0 restores the value mod 2^{32M}).  With d_k = v_k mod 2^32
// and c_k = floor(v_k / 2^32) in {0, 1, 2}, s_k = d_k + c_{k-1} <= 2^32 + 1,
// and the remaining carries are binary: position k generates one (s_k >=
// 2^32) or propagates one (s_k = 2^32 - 1).  The carries into the positions
// of a warp are ((G|P) + G + c_in) ^ (G|P) ^ G on the ballot masks, and the
// same identity over the warps' summaries gives each warp's c_in: 512
// positions per round, two barriers per round (cta_resolve's carry-function
// scan costs several times that).  red: 3 * (blockDim / 32) + 2 words.
template <class GetV, class PutD>
__device__ inline void fast_resolve(int M, bool biased, GetV getv, PutD putd,
                                        uint32_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cw = red;           // [nw] top lane's c of each warp
  uint32_t* gp = red + nw;      // [nw] warp summary: bit0 out with c_in 0, bit1 with c_in 1
  uint32_t* lastc = red + 2 * nw;
  uint32_t cin_round = biased ? 1u : 0u;  // carry into the round's first position
  uint32_t c_before = 0;                  // c_{base-1}: previous round's last c
  for (int base = 0; base < M; base += blockDim.x) {
    const int k = base + (int)threadIdx.x;
    const int64_t vv = k < M ? getv(k) + (biased ? (int64_t)0xFFFFFFFFLL : 0) : 0;
    const uint32_t d = (uint32_t)vv, c = (uint32_t)((uint64_t)vv >> 32);  // c in {0, 1, 2}
    uint32_t cprev = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane == 31) cw[wid] = c;
    __syncthreads();
    if (lane == 0) cprev = wid > 0 ? cw[wid - 1] : c_before;
    const uint64_t sv = (uint64_t)d + cprev;
    const bool g = (sv >> 32) != 0;
    const bool pr = !g && (uint32_t)sv == 0xFFFFFFFFu;
    const uint32_t G = __ballot_sync(0xffffffffu, g), P = __ballot_sync(0xffffffffu, pr);
    const uint64_t x = (uint64_t)(G | P), y = G;
    if (lane == 0)
      gp[wid] = (uint32_t)((x + y) >> 32) | ((uint32_t)((x + y + 1) >> 32) << 1);
    if (threadIdx.x == blockDim.x - 1) lastc[0] = c;
    __syncthreads();
    // carries into the warps: generate = out with c_in 0, propagate = only with c_in 1
    const uint32_t f = lane < nw ? gp[lane] : 0u;
    const uint32_t Gw = __ballot_sync(0xffffffffu, f & 1u);
    const uint32_t Pw = __ballot_sync(0xffffffffu, (f >> 1) & ~f & 1u);
    const uint64_t xw = (uint64_t)(Gw | Pw), yw = Gw;
    const uint64_t tw = xw + yw + cin_round;
    const uint32_t cin_w = (uint32_t)(((tw ^ xw ^ yw) >> wid) & 1u);
    const uint64_t t = x + y + cin_w;
    const uint32_t cbit = (uint32_t)(((t ^ x ^ y) >> lane) & 1u);
    if (k < M) putd(k, (uint32_t)sv + cbit);
    cin_round = (uint32_t)((tw >> nw) & 1u);
    c_before = lastc[0];
    __syncthreads();  // red reuse, digits visible
  }
}

// 96-bit column accumulation: (lo, hi, cc) += a * b
__device__ __forceinline__ void mac96(uint32_t& lo, uint32_t& hi, uint32_t& cc, uint32_t a,
                                      uint32_t b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+r"(lo), "+r"(hi), "+r"(cc)
      : "r"(a), "r"(b));
}

// Column sums of a*b for columns [k_begin, k_end) (M = k_end - k_begin):
// warp tasks of 128 consecutive columns (lane: 4 adjacent columns) times one
// of nseg segments of the block's term range; task (block, s) writes its
// 3-word column sums to planes pl[(3 s + w) M + k].  Per 4 terms a lane
// loads a[i..i+3] (broadcast), splits them in 16-bit halves and a window of
// 7 values of b, and issues 32 carry-free IMAD.WIDE accumulations (each
// half product < 2^48): 16 limb products, no carry-flag chains, no bounds
// checks -- b needs kGuard zero words below b[0] and above b[nb-1].
constexpr int kGuard = 132;
__device__ inline int wcols(const uint32_t* a, int na, const uint32_t* b, int nb, int k_begin,
                            int k_end, uint32_t* pl, int pl_words) {
  const int M = k_end - k_begin;
  const int nblk = (M + 127) / 128;
  const int span = min(na, nb) + 127;  // terms of one block, at most
  const int nseg = max(1, min(min(kSegMax, pl_words / (3 * M)), (span + 63) / 64));
  const int seg = ((span + nseg - 1) / nseg + 3) & ~3;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int task = threadIdx.x >> 5; task < nblk * nseg; task += nw) {
    const int blk = task / nseg, sgi = task - blk * nseg;
    const int c0 = k_begin + blk * 128, k0 = c0 + 4 * lane;
    const int glo = max(0, c0 - nb + 1), ghi = min(c0 + 127, na - 1);
    const int ilo = glo + sgi * seg, ihi = min(ghi, ilo + seg - 1);
    uint64_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    int i = ilo;
    for (; i + 3 <= ihi; i += 4) {
      uint32_t al[4], ah[4], bw[7];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t av = a[i + u];
        al[u] = av & 0xFFFFu;
        ah[u] = av >> 16;
      }
      const uint32_t* bp = b + (k0 - i - 3);
#pragma unroll
      for (int m = 0; m < 7; ++m) bw[m] = bp[m];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          // a[i+u] * b[k0 + t - i - u] = bw[t - u + 3]
          lo[t] += (uint64_t)al[u] * bw[t - u + 3];
          hi[t] += (uint64_t)ah[u] * bw[t - u + 3];
        }
    }
    for (; i <= ihi; ++i) {
      const uint32_t av = a[i];
      const uint32_t* bp = b + (k0 - i);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        lo[t] += (uint64_t)(av & 0xFFFFu) * bp[t];
        hi[t] += (uint64_t)(av >> 16) * bp[t];
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int k = k0 + t;
      if (k < k_end) {
        const unsigned __int128 tot = (unsigned __int128)lo[t] + ((unsigned __int128)hi[t] << 16);
        const int kk = k - k_begin;
        pl[(3 * sgi + 0) * M + kk] = (uint32_t)tot;
        pl[(3 * sgi + 1) * M + kk] = (uint32_t)(tot >> 32);
        pl[(3 * sgi + 2) * M + kk] = (uint32_t)(tot >> 64);
      }
    }
  }
  return nseg;
}

// V[k] = column k's sum over the planes at weight 2^(32k): word 0 of column
// k, word 1 of k-1, word 2 of k-2 (< 3 nseg 2^32)
__device__ __forceinline__ void col_reduce(const uint32_t* pl, int M, int nseg,
                                           unsigned long long* V) {
  for (int k = threadIdx.x; k < M; k += blockDim.x) {
    unsigned long long v = 0;
    for (int s = 0; s < nseg; ++s) {
      v += pl[(3 * s) * M + k];
      if (k >= 1) v += pl[(3 * s + 1) * M + k - 1];
      if (k >= 2) v += pl[(3 * s + 2) * M + k - 2];
    }
    V[k] = v;
  }
}

// Limb value of position k from the reduced sums: [0, 2^32 + 3 kSegMax)
__device__ __forceinline__ int64_t vlimb(const unsigned long long* V, int k) {
  int64_t v = (int64_t)(V[k] & 0xFFFFFFFFull);
  if (k >= 1) v += (int64_t)(V[k - 1] >> 32);
  return v;
}

// out[0, M) = limbs of sum_{k_begin <= k < k_end} col_k 2^{32(k-k_begin)}
// minus sub (at limb subk), mod 2^(32 M) (the cta_mul short-product
// semantics; sub = 0 for a plain product).
__device__ __noinline__ void cta_mul_fast(const uint32_t* a, int na, const uint32_t* b, int nb,
                                    uint32_t* out, int M_end, int k_begin, uint32_t* pl,
                                    int pl_words, unsigned long long* V, uint32_t* red,
                                    int subk = -1, uint32_t sub = 0) {
  const int M = M_end - k_begin;
  const int nseg = wcols(a, na, b, nb, k_begin, M_end, pl, pl_words);
  __syncthreads();
  col_reduce(pl, M, nseg, V);
  __syncthreads();
  fast_resolve(
      M, subk >= 0,
      [&](int k) -> int64_t { return vlimb(V, k) - (k == subk ? (int64_t)sub : 0); },
      [&](int k, uint32_t d) { out[k] = d; }, red);
}

// Thread-serial low product for tiny operands: out[0, M) = low M limbs of a*b
// (exact, M <= na + nb).
__device__ inline void serial_mul(const uint32_t* a, int na, const uint32_t* b, int nb,
                                  uint32_t* out, int M) {
  unsigned __int128 carry = 0;
  for (int k = 0; k < M; ++k) {
    unsigned __int128 s = carry;
    const int ilo = max(0, k - nb + 1), ihi = min(k, na - 1);
    for (int i = ilo; i <= ihi; ++i) s += (unsigned long long)a[i] * b[k - i];
    out[k] = (uint32_t)s;
    carry = s >> 32;
  }
}


// ---- register ladder -------------------------------------------------------
// The first Newton levels (precision <= kRegBits) on warp 0 in registers: a
// 512-bit fixed-point reciprocal of the divisor's top 512 bits, one 32-bit
// limb per lane, operands exchanged by shuffles, so no level of it touches
// shared memory or a barrier (the shared-memory levels cost 12-19k cycles
// each for a few limbs of work).
constexpr int kRegBits = 400;

// Digits of sum_k v_k 2^(32 k) + cin mod 2^1024, lane k holding v_k < 3 2^32:
// after the carries c_k = v_k >> 32 move one lane up the remaining carries
// are binary, and the ballot identity of fast_resolve gives every lane's.
__device__ __forceinline__ uint32_t warp_digits(unsigned long long v, uint32_t cin) {
  const int lane = threadIdx.x & 31;
  const uint32_t d = (uint32_t)v, c = (uint32_t)(v >> 32);
  uint32_t cprev = __shfl_up_sync(0xffffffffu, c, 1);
  if (lane == 0) cprev = cin;
  const unsigned long long sv = (unsigned long long)d + cprev;
  const bool g = (sv >> 32) != 0;
  const bool pr = !g && (uint32_t)sv == 0xFFFFFFFFu;
  const uint32_t G = __ballot_sync(0xffffffffu, g), P = __ballot_sync(0xffffffffu, pr);
  const unsigned long long x = (unsigned long long)(G | P), y = G;
  const unsigned long long t = x + y;
  return (uint32_t)sv + (uint32_t)(((t ^ x ^ y) >> lane) & 1u);
}

// limb `lane` of a * b (a, b: 16 limbs, lane l < 16 holds limb l, 0 above)
__device__ __forceinline__ uint32_t warp_mul16(uint32_t a, uint32_t b) {
  const int lane = threadIdx.x & 31;
  unsigned long long lo = 0;
  uint32_t hi = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t ai = __shfl_sync(0xffffffffu, a, i);
    const int j = lane - i;
    uint32_t bj = __shfl_sync(0xffffffffu, b, j & 31);
    if (j < 0 || j > 15) bj = 0u;
    const unsigned long long p = (unsigned long long)ai * bj;
    lo += p;
    hi += lo < p ? 1u : 0u;
  }
  unsigned long long v = (uint32_t)lo;
  const uint32_t w1 = __shfl_up_sync(0xffffffffu, (uint32_t)(lo >> 32), 1);
  const uint32_t w2 = __shfl_up_sync(0xffffffffu, hi, 2);
  if (lane >= 1) v += w1;
  if (lane >= 2) v += w2;
  return warp_digits(v, 0u);
}

// Warp 0: lane l < 16 holds limb l of d in [2^511, 2^512); returns limb l of
// y = floor(2^(pa + 512) / d) within one unit (pa <= kRegBits).  x ~ 2^1022 / d
// (x / 2^510 ~ 1 / (d / 2^512) in (1, 2]) by four full-width Newton steps
// x <- x (2 - d x) from the FP64 seed (relative error 2^-51 -> 2^-102 ->
// 2^-204 -> 2^-408 -> the truncation floor of a few 2^-510), then
// y = x >> (510 - pa): the error of x is far below one unit of y.
__device__ inline uint32_t reg_reciprocal(uint32_t d, int pa) {
  const int lane = threadIdx.x & 31;
  const uint32_t d15 = __shfl_sync(0xffffffffu, d, 15), d14 = __shfl_sync(0xffffffffu, d, 14);
  const double dd = ldexp((double)d15, 32) + (double)d14;                      // [2^63, 2^64]
  const unsigned long long x63 = (unsigned long long)(ldexp(1.0, 126) / dd);   // x / 2^448
  uint32_t x = lane == 14 ? (uint32_t)x63 : lane == 15 ? (uint32_t)(x63 >> 32) : 0u;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {
    // T = floor(d x / 2^512) ~ 2^510;  E2 = 2^511 - T (2 - d x in units of 2^-510)
    const uint32_t pr = warp_mul16(d, x);
    const uint32_t t = __shfl_down_sync(0xffffffffu, pr, 16);  // lanes < 16: limb 16 + lane
    const unsigned long long m = lane == 15 ? 0x80000000ull : 0ull;
    // lanes >= 16 hold the bias alone: their digits resolve to zero
    const unsigned long long v = lane < 16 ? m + 0xFFFFFFFFull - t : 0xFFFFFFFFull;
    uint32_t e2 = warp_digits(v, 1u);
    if (lane >= 16) e2 = 0u;
    // x' = floor(x E2 / 2^510): bit 510 = limb 15, bit 30
    const uint32_t q = warp_mul16(x, e2);
    const uint32_t q15 = __shfl_down_sync(0xffffffffu, q, 15);
    const uint32_t q16 = __shfl_down_sync(0xffffffffu, q, 16);
    x = lane < 16 ? (q15 >> 30) | (q16 << 2) : 0u;
  }
  const int sh = 510 - pa;  // >= 110
  const int ws = sh >> 5, bs = sh & 31;
  const int src = lane + ws;
  uint32_t lo = __shfl_sync(0xffffffffu, x, src & 31);
  uint32_t hi = __shfl_sync(0xffffffffu, x, (src + 1) & 31);
  if (src > 15) lo = 0u;
  if (src + 1 > 15) hi = 0u;
  return bs ? (lo >> bs) | (hi << (32 - bs)) : lo;
}

}  // namespace rf

// The reciprocal of stage p's pivot value V_p[p] = vint[prow]; arguments and
// outputs as recip_body.  sm: shared scratch of rf_scratch_words(Lm) words.
__host__ __device__ inline long long rf_scratch_words(int Lm) {
  // Ds, Dt, Y | Pr, E (2 Lm + 4 each) | Tm (3 Lm + 4) | V (u64, 3 Lm + 4) |
  // planes (3 kSegMax (Lm + 4): every product of the ladder has <= Lm + 4
  // columns except small full products, which then take fewer segments)
  return (long long)(Lm + 4) * 3 + 2LL * (2 * Lm + 4) + 6 * rf::kGuard + (3 * Lm + 4) +
         2LL * (3 * Lm + 4) + 3LL * rf::kSegMax * (Lm + 4) + 64;
}

// Returns false (having done nothing) when the stage's precision needs more
// than avail_words of scratch; the caller then runs recip_body.
__device__ bool recip_fast_body(const DevPlan& P, IntBuf vint, long long prow,
                                const int* maxbitsV, int p, IntBuf piv, int dmax_bits,
                                uint32_t* Ybuf, int* ys, uint32_t* sm, long long avail_words,
                                int* err) {
  __shared__ uint32_t red[64];
  const long long t_entry = (P.debug & 256) ? clock64() : 0;
  const int h = vint.hdr[prow];
  const int nD = h < 0 ? -h : h;
  if (nD == 0) return true;  // flagged as ZeroPivot by k_extract
  const uint32_t* Dg = vint.limbs + prow * (long long)P.cap;
  const int n = limbs_bits(Dg, nD);
  int amax;
  if (dmax_bits > 0) {
    const int hp = piv.hdr[p];
    const int npl = hp < 0 ? -hp : hp;
    const int wpp = limbs_bits(piv.limbs + (long long)p * P.cap, npl);
    amax = (dmax_bits + 1 + wpp + 1) / 2 + 2;
  } else {
    amax = maxbitsV[p] + P.k2;
  }
  const int e = max(amax - n + 2, 1);
  const int G = 32;
  const int Pt = e + G;
  const int S = n + Pt;
  const int Lm = (Pt + G + 31) / 32 + 2;
  const int nYf = (Pt + 2 + 31) / 32 + 1;
  if (nYf > P.ycap) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return true;
  }
  if (rf_scratch_words(Lm) > avail_words) {
    if ((P.debug & 4096) && p % 100 == 50 && threadIdx.x == 0)
      printf("recip_fast p=%d falls back: Lm %d needs %lld words, %lld available (n %d amax %d)\n", p,
             Lm, rf_scratch_words(Lm), avail_words, n, amax);
    return false;
  }
  const int dbase = max(0, nD - (Lm + 2));
  const int nDs = nD - dbase;
  // Y, Pr and E are product operands b: kGuard zero words on either side
  // (wcols reads past their lengths).  Zeroed once: every buffer only grows
  // from level to level, so what lies past a length is zero.
  constexpr int GW = rf::kGuard;
  uint32_t* Ds = sm;                    // Lm + 4
  uint32_t* Dt = Ds + (Lm + 4);         // Lm + 4
  uint32_t* Y = Dt + (Lm + 4) + GW;     // Lm + 4 + 2 GW
  uint32_t* Pr = Y + (Lm + 4) + 2 * GW; // 2 Lm + 4 + 2 GW
  uint32_t* E = Pr + (2 * Lm + 4) + 2 * GW;
  uint32_t* Tm = E + (2 * Lm + 4) + GW;  // 3 Lm + 4
  const int zero_words = (int)(Tm - sm);
  // 10 Lm + 24 + 6 GW words from sm: even, so the 64-bit sums are aligned
  unsigned long long* V = reinterpret_cast<unsigned long long*>(Tm + (3 * Lm + 4));
  uint32_t* pl = reinterpret_cast<uint32_t*>(V + (3 * Lm + 4));
  const int pl_words = 3 * rf::kSegMax * (Lm + 4);
  for (int k = threadIdx.x; k < zero_words; k += blockDim.x) sm[k] = 0u;
  __syncthreads();
  for (int k = threadIdx.x; k < nDs; k += blockDim.x) Ds[k] = Dg[dbase + k];
  int lv[40];
  const int nl = recip_levels(Pt, lv);
  const int p0 = lv[0];
  // register ladder: levels [0, i0) replaced by one 512-bit reciprocal on
  // warp 0: Y_{i0} = floor(2^(n + lv[i0]) / D) within a unit (the ladder's
  // own levels keep a few units; every later level tolerates < 16)
  int i0 = 0;
  if (P.recip_fast & 2)
    while (i0 + 1 < nl && lv[i0 + 1] <= rf::kRegBits) ++i0;
  if (i0 == 0 && threadIdx.x == 0) {
    // seed as recip_body: floor(2^126 / top64(D)) >> (62 - p0), via FP64
    const uint32_t hi = field32(Dg + dbase, nDs, (long long)n - 32 - 32LL * dbase);
    const uint32_t lo = field32(Dg + dbase, nDs, (long long)n - 64 - 32LL * dbase);
    const double d = ldexp((double)hi, 32) + (double)lo;
    const unsigned long long y63 = (unsigned long long)(ldexp(1.0, 126) / d);
    const unsigned long long y0 = y63 >> (62 - p0);
    Y[0] = (uint32_t)y0;
    Y[1] = (uint32_t)(y0 >> 32);
  }
  __syncthreads();
  int nY = 2;
  // recip_body's warp-class levels (K0 = 0: full second product) are those
  // before the first with nDt > 128 or nY > 128
  bool warp_class = true;
  const bool prof = (P.debug & 256) && p == 50 && threadIdx.x == 0;
  if (i0 > 0) {
    const long long t_reg = prof ? clock64() : 0;
    const int pa = lv[i0];
    const int nYr = min(Lm, (pa + 2 + 31) / 32 + 1);
    if (threadIdx.x < 32) {
      const int l = (int)threadIdx.x;
      uint32_t dl = 0u;
      if (l < 16) dl = field32(Ds, nDs, (long long)n - 512 + 32LL * l - 32LL * dbase);
      const uint32_t yl = rf::reg_reciprocal(dl, pa);
      if (l < nYr && l < 16) Y[l] = yl;
    }
    __syncthreads();
    nY = nYr;
    if (prof) printf("recip_fast register ladder to level %d (pa=%d): %lld cycles (entry + %lld)\n", i0, pa,
                     clock64() - t_reg, t_reg - t_entry);
  }
  for (int i = i0; i + 1 < nl; ++i) {
    long long tph[6];
    if (prof) tph[0] = clock64();
    const int pa = lv[i], pb = lv[i + 1], dlt = pb - pa;
    const int mb = min(n, pb + G);
    const int t = n - mb;
    const int nDt = (mb + 31) / 32;
    if (warp_class && (nDt > 128 || nY > 128)) warp_class = false;
    const int nL = nDt + 1;
    const int Sb = mb + pa;
    const int nYn = min(Lm, (pb + 2 + 31) / 32 + 1);
    const int sh = Sb - dlt;
    const int K0 = warp_class ? 0 : max(0, (sh - 64) / 32);
    if (nDt <= 8 && nY <= 8) {
      // tiny level on thread 0: 128-bit serial arithmetic, no barriers
      if (threadIdx.x == 0) {
        for (int k = 0; k < nDt; ++k) Dt[k] = field32(Ds, nDs, 32LL * k + t - 32LL * dbase);
        rf::serial_mul(Dt, nDt, Y, nY, Pr, nL);
        // E = 2^Sb - Pr mod 2^(32 nL)
        int64_t c = 0;
        for (int k = 0; k < nL; ++k) {
          const int64_t av = (k == Sb / 32) ? (int64_t)(1u << (Sb % 32)) : 0;
          const int64_t v = av - (int64_t)Pr[k] + c;
          E[k] = (uint32_t)v;
          c = v >> 32;
        }
        const int sgn = (E[nL - 1] & 0x80000000u) ? -1 : 1;
        uint32_t* Ev = E;
        if (sgn < 0) {
          c = 0;
          for (int k = 0; k < nL; ++k) {
            const int64_t v = -(int64_t)E[k] + c;
            Pr[k] = (uint32_t)v;
            c = v >> 32;
          }
          Ev = Pr;
        }
        int nE = nL;
        while (nE > 0 && Ev[nE - 1] == 0) --nE;
        const int nT = nY + nE;
        if (nE > 0) rf::serial_mul(Y, nY, Ev, nE, Tm, nT);  // K0 == 0 here
        c = 0;
        for (int k = 0; k < nYn; ++k) {
          const int64_t yv = field32(Y, nY, 32LL * k - dlt);
          const int64_t tv = nE > 0 ? (int64_t)field32(Tm, nT, 32LL * k + sh) : 0;
          const int64_t v = (sgn > 0 ? yv + tv : yv - tv) + c;
          Dt[k] = (uint32_t)v;  // Dt is dead: staging for Y'
          c = v >> 32;
        }
        for (int k = 0; k < nYn; ++k) Y[k] = Dt[k];
      }
      __syncthreads();
      if (prof)
        printf("recip_fast lvl %d (thread 0) pa=%d pb=%d nDt=%d nY=%d: %lld cycles (entry + %lld)\n", i,
               pa, pb, nDt, nY, clock64() - tph[0], tph[0] - t_entry);
      nY = nYn;
      continue;
    }
    for (int k = threadIdx.x; k < nDt; k += blockDim.x)
      Dt[k] = field32(Ds, nDs, 32LL * k + t - 32LL * dbase);
    __syncthreads();
    if (prof) tph[1] = clock64();
    // F = D' Y - 2^Sb = -E mod 2^(32 nL) in one resolve with the product
    rf::cta_mul_fast(Dt, nDt, Y, nY, Pr, nL, 0, pl, pl_words, V, red, Sb / 32 < nL ? Sb / 32 : -1,
                     1u << (Sb % 32));
    if (prof) tph[2] = clock64();
    const int nF = cta_limb_len(Pr, nL, red);
    // E < 0 (F small positive): |E| = F; E > 0: |E| = -F; E = 0: nE = 0
    const int sgn = (nF == 0 || (Pr[nL - 1] & 0x80000000u)) ? 1 : -1;
    uint32_t* Ev = Pr;
    int nE = nF;
    if (nF > 0 && sgn > 0) {
      rf::fast_resolve(
          nL, true, [&](int k) -> int64_t { return -(int64_t)Pr[k]; },
          [&](int k, uint32_t dd) { E[k] = dd; }, red);
      Ev = E;
      nE = cta_limb_len(Ev, nL, red);
    }
    if (prof) tph[3] = clock64();
    const int nT = nY + nE;
    if (nE > 0) rf::cta_mul_fast(Y, nY, Ev, nE, Tm, nT, K0, pl, pl_words, V, red);
    if (prof) tph[4] = clock64();
    rf::fast_resolve(
        nYn, sgn < 0,
        [&](int k) -> int64_t {
          const int64_t yv = field32(Y, nY, 32LL * k - dlt);
          const int64_t tv =
              nE > 0 ? (int64_t)field32(Tm, nT - K0, 32LL * k + sh - 32LL * K0) : 0;
          return sgn > 0 ? yv + tv : yv - tv;
        },
        [&](int k, uint32_t dd) { Dt[k] = dd; }, red);
    for (int k = threadIdx.x; k < nYn; k += blockDim.x) Y[k] = Dt[k];
    __syncthreads();
    if (prof) {
      tph[5] = clock64();
      printf("recip_fast lvl %d pa=%d pb=%d nDt=%d nY=%d nE=%d: Dt %lld mul1 %lld E %lld mul2 %lld Yupd %lld\n",
             i, pa, pb, nDt, nY, nE, tph[1] - tph[0], tph[2] - tph[1], tph[3] - tph[2],
             tph[4] - tph[3], tph[5] - tph[4]);
    }
    nY = nYn;
  }
  const long long t_lv = prof ? clock64() : 0;
  for (int k = threadIdx.x; k < P.ycap; k += blockDim.x) Ybuf[k] = k < nY ? Y[k] : 0u;
  if (prof) printf("recip_fast store %lld cycles, total %lld\n", clock64() - t_lv, clock64() - t_entry);
  if (threadIdx.x == 0) {
    ys[0] = S;
    ys[1] = nY;
    ys[2] = amax;
  }
  return true;
}

}  // namespace hgpu
