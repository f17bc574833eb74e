// Triangular solves with the LDL^T factors for inverse iteration (SURVEY
// §8 a11; the north-star's step after the factorisation -- the reference
// itself finds lambda_1 by the secant and has no solve).  With A = M - sI =
// L D L^T, L[r][p] = R_p[r] 2^-k2 (the ratio columns of ldlt.cpp:57-58) and
// D_p = piv_p 2^-K, a right-hand side u at F fractional bits is solved in
// exact fixed point, truncating toward zero once per entry:
//   forward   z_r = u_r - tdiv_2exp( sum_{p<r} R_p[r] z_p , k2 )
//   diagonal  w_p = tdiv( z_p 2^K , piv_p )              (k_divide)
//   back      y_p = w_p - tdiv_2exp( sum_{r>p} R_p[r] y_r , k2 )
// The sums are accumulated column by column (one CTA per target row, exact
// two's-complement accumulators), so each sequential step is one parallel
// AXPY over the remaining rows.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"
#include "transform_ops.cuh"

#include <cooperative_groups.h>

namespace hgpu {

namespace {

// words of one k_solve_axpy CTA sized for operands of at most capX (x) and
// capC (R) limbs: X | C | max(Pr (capX + capC) + col 3 (capX + capC), the
// finish's scratch) | red 64
__host__ __device__ inline long long solve_finish_words(int Wv, int Wa) {
  return (long long)(Wa + 1) + (Wv + 1) + (Wv + 2) + 64;
}
__host__ __device__ inline long long solve_axpy_words(int capX, int capC,
                                                      int Wv, int Wa) {
  const long long prod = 4LL * (capX + capC);
  const long long fin = solve_finish_words(Wv, Wa);
  return (long long)capX + capC + (prod > fin ? prod : fin) + 64;
}

// index of R_p[r] (p < r < n) in the packed strictly-lower store
__device__ __forceinline__ long long lidx(int n, int p, int r) {
  return (long long)p * (n - 1) - (long long)p * (p - 1) / 2 + (r - p - 1);
}

}  // namespace

// out_i = base_i - tdiv_2exp(acc_i, k2)   (single CTA; acc two's complement)
// base/out are signed limb vectors of Wv limbs; `shift_out` > 0 additionally
// stores out_i << shift_out into out2 (the diagonal step's numerator).
// The same from |acc| (M1, Wa limbs, zero padded; Wa + 1 words of storage,
// reused as scratch) and its sign; T: Wv + 1, X: Wv + 2 words.
__device__ void solve_finish_mag(int Wv, int Wa, int k2, uint32_t* M1, bool neg,
                                 const Finish& f, uint32_t* T, uint32_t* X,
                                 uint32_t* red, int* err, int mlen = -1) {
  const IntBuf& base = f.base;
  const int bi = f.bi;
  const IntBuf& out = f.out;
  const int oi = f.oi;
  const IntBuf& out2 = f.out2;
  const int o2i = f.o2i, shift_out = f.shift_out;
  // t = sign * (|acc| >> k2)
  const int st = neg ? -1 : 1;
  // limbs of |acc| >> k2 (all Wv + 1 unless the caller knows |acc|'s length)
  const int tlen = mlen < 0 ? Wv + 1 : min(Wv + 1, max(0, mlen - (k2 >> 5)) + 1);
  for (int k = threadIdx.x; k < tlen; k += blockDim.x)
    T[k] = field32(M1, Wa, 32LL * k + k2);
  // X = |base - t|: with base = sb |B| and t = st |T|, base - t =
  // sb (|B| - sb st |T|), whose limb-wise digit sums stay in (-2^32, 2^33):
  // one resolve, and a second (negated) one only when |B| < |T| under the
  // subtraction.
  const int hb = base.hdr[bi];
  const int nb = hb < 0 ? -hb : hb;
  const int sb = hb < 0 ? -1 : 1;
  const int sbt = sb * st;
  const uint32_t* B = base.limbs + (long long)bi * Wv;
  __syncthreads();
  // |base - t| < 2^(32 max(nb, tlen) + 1): two spare limbs keep the
  // capacity check below exact
  const int W2 = min(Wv + 2, max(nb, tlen) + 2);
  auto inner = [&](int k) -> int64_t {
    const int64_t bv = k < nb ? (int64_t)B[k] : 0;
    const int64_t tv = k < tlen ? (int64_t)T[k] : 0;
    return sbt > 0 ? bv - tv : bv + tv;
  };
  const bool ineg =
      cta_resolve(W2, 32, inner, [&](int k, uint32_t d) { X[k] = d; }, red) < 0;
  if (ineg)
    cta_resolve(
        W2, 32, [&](int k) -> int64_t { return -inner(k); },
        [&](int k, uint32_t d) { X[k] = d; }, red);
  const bool rneg = (sb < 0) != ineg;
  const int len = cta_limb_len(X, W2, red);
  if (len > Wv) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return;
  }
  uint32_t* O = out.limbs + (long long)oi * Wv;
  for (int k = threadIdx.x; k < Wv; k += blockDim.x) O[k] = k < len ? X[k] : 0u;
  if (threadIdx.x == 0) out.hdr[oi] = len == 0 ? 0 : (rneg ? -len : len);
  if (shift_out > 0) {
    // numerator z << shift for the diagonal division (k_divide shifts by k2
    // itself, so the caller passes K - k2 = k2)
    const int bits = limbs_bits(X, len) + shift_out;
    const int n2 = len == 0 ? 0 : (bits + 31) / 32;
    uint32_t* O2 = out2.limbs + (long long)o2i * Wv;
    if (n2 > Wv) {
      if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
      return;
    }
    for (int k = threadIdx.x; k < Wv; k += blockDim.x)
      O2[k] = k < n2 ? field32(X, len, 32LL * k - shift_out) : 0u;
    if (threadIdx.x == 0) out2.hdr[o2i] = n2 == 0 ? 0 : (rneg ? -n2 : n2);
  }
}

__device__ void solve_finish(int Wv, int Wa, int k2, const uint32_t* acc_i,
                             const Finish& f, uint32_t* sm, int* err) {
  uint32_t* M1 = sm;           // Wa + 1
  uint32_t* T = M1 + Wa + 1;   // Wv + 1
  uint32_t* X = T + Wv + 1;    // Wv + 2
  uint32_t* red = X + Wv + 2;
  // |acc| and its sign
  const bool neg = (acc_i[Wa - 1] & 0x80000000u) != 0;
  cta_resolve(
      Wa, 32,
      [&](int k) -> int64_t {
        return neg ? -(int64_t)acc_i[k] : (int64_t)acc_i[k];
      },
      [&](int k, uint32_t d) { M1[k] = d; }, red);
  solve_finish_mag(Wv, Wa, k2, M1, neg, f, T, X, red, err);
}

__global__ void k_solve_finish(int Wv, int Wa, int k2, const uint32_t* acc_i,
                               Finish f, int* err) {
  extern __shared__ uint32_t sm[];
  solve_finish(Wv, Wa, k2, acc_i, f, sm, err);
}

// acc_t += R(a, b) * x_j  for the targets of step j:
//   forward (dir = 0): j = p, targets t = r in (p, n),  coefficient R_p[r]
//   back    (dir = 1): j = r, targets t = q in [0, r),  coefficient R_q[r]
// The first target (p+1, resp. r-1) is complete after this step: CTA 0
// takes it first and finishes it (solve_finish with `fin`), so the next
// step's operand is ready without a separate launch.
__global__ void __launch_bounds__(256) k_solve_axpy(int n, int cap, int Wv, int Wa, int k2, IntBuf L,
                             IntBuf xv, int xi, int j, int dir, uint32_t* acc,
                             Finish fin, int capX, int capC, uint32_t* gscratch,
                             int seg, int* err) {
  extern __shared__ uint32_t sm_dyn[];
  // operands and product scratch in shared memory, or (large plans) in this
  // CTA's slice of a global scratch (L1/L2-resident)
  uint32_t* sm =
      gscratch ? gscratch + (long long)blockIdx.x * solve_axpy_words(capX, capC, Wv, Wa)
               : sm_dyn;
  const int hx = xv.hdr[xi];
  const int nx = hx < 0 ? -hx : hx;
  const int sx = hx < 0 ? -1 : 1;
  uint32_t* X = sm;                   // capX
  uint32_t* C = X + capX;             // capC
  uint32_t* Pr = C + capC;            // capX + capC (also the finish scratch)
  uint32_t* col = Pr + capX + capC;   // 3 (capX + capC)
  uint32_t* red = Pr + max(4LL * (capX + capC), solve_finish_words(Wv, Wa));
  const int seg_words = seg ? 3 * (capX + capC) : 0;
  if (nx > capX) {  // the host sized the layout too small: it reruns
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return;
  }
  for (int i = threadIdx.x; i < nx; i += blockDim.x)
    X[i] = xv.limbs[(long long)xi * Wv + i];
  // targets in critical-first order: k = 0 is the row finished here
  const int ntg = dir == 0 ? n - j - 1 : j;
  for (int kk = blockIdx.x; kk < ntg; kk += gridDim.x) {
    const int t = dir == 0 ? j + 1 + kk : j - 1 - kk;
    const long long li = dir == 0 ? lidx(n, j, t) : lidx(n, t, j);
    const int hc = L.hdr[li];
    const int nc = hc < 0 ? -hc : hc;
    if (nc == 0 || nx == 0) {
      if (kk == 0) solve_finish(Wv, Wa, k2, acc + (long long)t * Wa, fin, Pr, err);
      continue;
    }
    if (nc > capC) {
      if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
      return;
    }
    const int sgn = (hc < 0 ? -1 : 1) * sx;
    for (int i = threadIdx.x; i < nc; i += blockDim.x)
      C[i] = L.limbs[li * cap + i];
    __syncthreads();
    const int nP = nc + nx;
    // one segment per group (measured fastest here; HGPU_SOLVE_SEG=1: as
    // many as the column scratch allows)
    cta_mul(C, nc, X, nx, Pr, nP, col, red, seg_words);
    uint32_t* a = acc + (long long)t * Wa;
    if (nP > Wa && threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    cta_resolve(
        Wa, 32,
        [&](int k) -> int64_t {
          const int64_t pv = k < nP ? (int64_t)Pr[k] : 0;
          return (int64_t)a[k] + (sgn > 0 ? pv : -pv);
        },
        [&](int k, uint32_t d) { col[k] = d; }, red);
    for (int k = threadIdx.x; k < Wa; k += blockDim.x) a[k] = col[k];
    __syncthreads();
    if (kk == 0) solve_finish(Wv, Wa, k2, a, fin, Pr, err);
  }
}

// bits of the signed limb integers idx0 + b*step, b < count (the
// reciprocal's precision bound for each batched division)
__global__ void k_int_bits(IntBuf v, int idx0, int step, int stride, int count,
                           int* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  const long long idx = idx0 + (long long)b * step;
  const int h = v.hdr[idx];
  const int n = h < 0 ? -h : h;
  out[b] = n == 0 ? 0 : limbs_bits(v.limbs + idx * stride, n);
}

// ------------------------------------ transform-domain AXPY (opt-in) ---
// The step's products R(t, j) x_j are pointwise in the residue-number NTT
// domain of a solve plan S (its own primes / length / digit width, chosen
// so that a whole column of products sums exactly: n * (L/2) * 2^(2w) <
// Q/4 and deg R + deg x < L).  Once per factorisation every L entry is
// transformed (Montgomery form, k_solve_rhat); per step the accumulators of
// all targets take one pointwise multiply-add (HBM-streaming), and the
// critical target alone is brought back to an exact integer (inverse NTT,
// Garner, carry resolution: reconstruct_int), finished (solve_finish_mag)
// and its new vector entry transformed for the next step.  The integer
// result of every accumulator equals k_solve_axpy's, so the solve is bit
// identical.

// shared-memory words of the critical CTA: A NW | forward, inverse twiddles
// NW each (staged while the pointwise update runs: from L2 they stall every
// butterfly) | S, Dg (L+T) x 2 words each | M1 Wa + 1 | T Wv + 1 | X Wv + 2 |
// red 64
__host__ __device__ inline long long solve_ntt_words(const DevPlan& S, int Wv, int Wa) {
  const long long M = S.L + S.T;
  return (S.tw_global ? 1LL : 3LL) * S.NW + 4 * M + (Wa + 1) + (Wv + 1) + (Wv + 2) + 64;
}
constexpr int kSolveNttThreads = 1024;

// every L entry (packed like L) -> its transform in Montgomery form
__global__ void __launch_bounds__(256) k_solve_rhat(const __grid_constant__ DevPlan S, int cap, IntBuf L,
                                                    long long e_begin, long long count,
                                                    EntryStore rhat, int* err) {
  extern __shared__ uint32_t sm[];
  uint32_t* buf = sm;           // NW
  uint32_t* mag = buf + S.NW;   // cap
  for (long long e = e_begin + blockIdx.x; e < e_begin + count; e += gridDim.x) {
    int len;
    const int sign = load_int(L, e, cap, mag, &len);
    transform_int(S, mag, len, 0, sign, buf, rhat.at(e), true, S.twm, err);
  }
}

// transform of the signed limb integer xv[xi] (stride Wv) -> xhat
__global__ void __launch_bounds__(512) k_solve_xhat(const __grid_constant__ DevPlan S, IntBuf xv, int xi, int Wv,
                                                    uint32_t* xhat, int xbmax, int* err) {
  extern __shared__ uint32_t sm[];
  uint32_t* buf = sm;
  uint32_t* mag = buf + S.NW;
  int len;
  const int sign = load_int(xv, xi, Wv, mag, &len);
  if (threadIdx.x == 0 && limbs_bits(mag, len) > xbmax)
    atomicOr(&err[kErrCapacity], kCapDegree);
  transform_int(S, mag, len, 0, sign, buf, xhat, false, S.twm, err);
}

// a + mont(x, r) mod q for 4 words of one prime
__device__ __forceinline__ uint4 pw_madd(uint4 a, uint4 x, uint4 r, const PrimeConsts& c) {
  auto f = [&](uint32_t av, uint32_t xv, uint32_t rv) {
    const uint32_t v = av + reduce_2q(mont_mul(xv, rv, c.q, c.qneg), c.q);
    return v >= c.q ? v - c.q : v;
  };
  return make_uint4(f(a.x, x.x, r.x), f(a.y, x.y, r.y), f(a.z, x.z, r.z), f(a.w, x.w, r.w));
}

// One step j (dir 0: forward, targets t > j, coefficient R_j[t]; dir 1:
// back, targets t < j, coefficient R_t[j]).  Block 0 finishes the critical
// target (t = j+1 resp. j-1) and writes xhat_out; blocks >= 1 stream the
// pointwise updates of the other targets.
template <int RM>
__global__ void __launch_bounds__(kSolveNttThreads) k_solve_ntt(const __grid_constant__ DevPlan S, int n, int Wv, int Wa, int k2,
                                                   EntryStore rhat,
                                                   const uint32_t* __restrict__ xhat_in,
                                                   uint32_t* xhat_out, uint32_t* acch,
                                                   int j, int dir, Finish fin, int xbmax,
                                                   int* err) {
  extern __shared__ uint32_t sm[];
  const int NW = S.NW;
  const int ntg = dir == 0 ? n - j - 1 : j;
  auto target = [&](int kk) { return dir == 0 ? j + 1 + kk : j - 1 - kk; };
  auto ridx = [&](int t) { return dir == 0 ? lidx(n, j, t) : lidx(n, t, j); };
  if (blockIdx.x > 0) {
    if (S.debug & 16384) return;  // timing aid: skip the pointwise updates
    // pointwise: items (kk >= 1, 4-word group), grid-stride over blocks >= 1
    const int g4 = NW / 4;
    const long long items = (long long)(ntg - 1) * g4;
    const long long stride = (long long)(gridDim.x - 1) * blockDim.x;
    for (long long it = (long long)(blockIdx.x - 1) * blockDim.x + threadIdx.x; it < items;
         it += stride) {
      const int kk = 1 + (int)(it / g4);
      const int q4 = (int)(it - (long long)(kk - 1) * g4);
      const int t = target(kk);
      const PrimeConsts& c = S.pc[(4 * q4) >> S.logL];
      uint4* a = reinterpret_cast<uint4*>(acch + (long long)t * NW) + q4;
      const uint4 r = __ldcs(reinterpret_cast<const uint4*>(rhat.at(ridx(t))) + q4);
      const uint4 x = reinterpret_cast<const uint4*>(xhat_in)[q4];
      *a = pw_madd(*a, x, r, c);
    }
    return;
  }
  if (ntg <= 0 || (S.debug & 32768)) return;  // (timing aid: skip the critical row)
  const int t = target(0);
  const int M = S.L + S.T;
  uint32_t* A = sm;
  // twiddles staged in shared memory, or (tw_global: plans whose 3 NW words
  // do not fit) read from global memory through L1
  uint32_t* twf_s = A + NW;
  uint32_t* twi_s = twf_s + NW;
  const uint32_t* twf = S.tw_global ? S.twm : twf_s;
  const uint32_t* twi = S.tw_global ? S.itwm : twi_s;
  int64_t* Ssum = reinterpret_cast<int64_t*>(S.tw_global ? A + NW : twi_s + NW);
  uint64_t* Dg = reinterpret_cast<uint64_t*>(Ssum + M);
  uint32_t* M1 = reinterpret_cast<uint32_t*>(Dg + M);
  uint32_t* T = M1 + Wa + 1;
  uint32_t* X = T + Wv + 1;
  uint32_t* red = X + Wv + 2;
  if (!S.tw_global)
    for (int i = threadIdx.x; i < NW / 4; i += blockDim.x) {
      reinterpret_cast<uint4*>(twf_s)[i] = reinterpret_cast<const uint4*>(S.twm)[i];
      reinterpret_cast<uint4*>(twi_s)[i] = reinterpret_cast<const uint4*>(S.itwm)[i];
    }
  const bool stamp = (S.debug & 8192) && (j == 500 || j == 501) && threadIdx.x == 0;
  long long c0 = stamp ? clock64() : 0, c1 = 0, c2 = 0, c3 = 0;
  unsigned long long g0 = 0;
  if (stamp) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  {
    const uint4* a = reinterpret_cast<const uint4*>(acch + (long long)t * NW);
    const uint4* r = reinterpret_cast<const uint4*>(rhat.at(ridx(t)));
    const uint4* x = reinterpret_cast<const uint4*>(xhat_in);
    for (int q4 = threadIdx.x; q4 < NW / 4; q4 += blockDim.x)
      reinterpret_cast<uint4*>(A)[q4] = pw_madd(a[q4], x[q4], __ldcs(r + q4), S.pc[(4 * q4) >> S.logL]);
  }
  __syncthreads();
  if (stamp) c1 = clock64();
  int len = 0;
  long long rs[4] = {0, 0, 0, 0};
  const int sg = reconstruct_int<RM>(S, A, Ssum, Dg, M1, Wa, red, twi, err, &len,
                                 stamp ? rs : nullptr);
  if (sg == 0) return;
  if (threadIdx.x == 0) M1[Wa] = 0u;
  __syncthreads();
  if (stamp) c2 = clock64();
  solve_finish_mag(Wv, Wa, k2, M1, sg < 0 && len > 0, fin, T, X, red, err, len);
  __syncthreads();
  if (stamp) c3 = clock64();
  // the finished entry, transformed for the next step
  int xl;
  const int xs = load_int(fin.out, fin.oi, Wv, X, &xl);
  if (threadIdx.x == 0 && limbs_bits(X, xl) > xbmax) atomicOr(&err[kErrCapacity], kCapDegree);
  transform_int<RM>(S, X, xl, 0, xs, A, xhat_out, false, twf, err);
  unsigned long long g1 = 0;
  if (stamp) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (stamp)
    printf("solve_ntt j=%d dir=%d ns %llu..%llu (%llu) clk %lld: pointwise %lld reconstruct %lld (intt %lld garner %lld "
           "digits %lld resolve+pack %lld) finish %lld transform %lld\n",
           j, dir, g0, g1, g1 - g0, clock64() - c0, c1 - c0, c2 - c1, rs[0] - c1, rs[1] - rs[0], rs[2] - rs[1], c2 - rs[2],
           c3 - c2, clock64() - c3);
}

// The same step with the critical row spread over a cluster of np CTAs (one
// prime each): every CTA updates and inverse-transforms its prime's slice
// of the critical accumulator and stores it into CTA 0's shared memory
// (DSMEM); CTA 0 runs Garner, the carry resolution and the finish; then
// every CTA transforms the new entry for its prime.  Both transforms of the
// chain run np-wide in parallel instead of np in a row.  Needs w = 32 (the
// solve plan's digits).
template <int RM>
__global__ void __launch_bounds__(kSolveNttThreads) k_solve_ntt_cl(
    const __grid_constant__ DevPlan S, int n, int Wv, int Wa, int k2, EntryStore rhat,
    const uint32_t* __restrict__ xhat_in, uint32_t* xhat_out, uint32_t* acch, int j, int dir,
    Finish fin, int xbmax, int* err) {
  namespace cg = cooperative_groups;
  extern __shared__ uint32_t sm[];
  const int NW = S.NW, L = S.L, np = S.np;
  const int ntg = dir == 0 ? n - j - 1 : j;
  auto target = [&](int kk) { return dir == 0 ? j + 1 + kk : j - 1 - kk; };
  auto ridx = [&](int t) { return dir == 0 ? lidx(n, j, t) : lidx(n, t, j); };
  const int nc = np;  // CTAs of the critical cluster (cluster 0)
  if ((int)blockIdx.x >= nc) {
    // launched early (programmatic dependent launch): wait for the previous
    // step's grid before reading x-hat and the accumulators
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (S.debug & 16384) return;
    const int g4 = NW / 4;
    const long long items = (long long)(ntg - 1) * g4;
    const long long stride = (long long)(gridDim.x - nc) * blockDim.x;
    for (long long it = (long long)(blockIdx.x - nc) * blockDim.x + threadIdx.x; it < items;
         it += stride) {
      const int kk = 1 + (int)(it / g4);
      const int q4 = (int)(it - (long long)(kk - 1) * g4);
      const int t = target(kk);
      const PrimeConsts& c = S.pc[(4 * q4) >> S.logL];
      uint4* a = reinterpret_cast<uint4*>(acch + (long long)t * NW) + q4;
      const uint4 r = __ldcs(reinterpret_cast<const uint4*>(rhat.at(ridx(t))) + q4);
      const uint4 x = reinterpret_cast<const uint4*>(xhat_in)[q4];
      *a = pw_madd(*a, x, r, c);
    }
    return;
  }
  // every CTA of cluster 0 reaches every cluster barrier (no early return)
  cg::cluster_group cl = cg::this_cluster();
  // arrive now, wait just before the first store into another CTA's shared
  // memory: a CTA's distributed shared memory may only be accessed once
  // every CTA of the cluster has started
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
  const int rk = (int)blockIdx.x;  // prime handled by this CTA
  const bool live = ntg > 0 && !(S.debug & 32768);
  const int t = live ? target(0) : 0;
  const int M = L + S.T;
  uint32_t* A = sm;
  uint32_t* twf_s = A + NW;
  uint32_t* twi_s = twf_s + NW;
  const uint32_t* twf = S.tw_global ? S.twm : twf_s;
  const uint32_t* twi = S.tw_global ? S.itwm : twi_s;
  int64_t* Ssum = reinterpret_cast<int64_t*>(S.tw_global ? A + NW : twi_s + NW);
  uint64_t* Dg = reinterpret_cast<uint64_t*>(Ssum + M);
  uint32_t* M1 = reinterpret_cast<uint32_t*>(Dg + M);
  uint32_t* T = M1 + Wa + 1;
  uint32_t* X = T + Wv + 1;
  uint32_t* red = X + Wv + 2;
  const PrimeConsts& c = S.pc[rk];
  uint32_t* Ar = A + rk * L;
  const int qs = (L + nc - 1) / nc;  // coefficients per CTA after the exchange
  if (live && !S.tw_global) {
    for (int i = threadIdx.x; i < L / 4; i += blockDim.x) {
      reinterpret_cast<uint4*>(twf_s + rk * L)[i] = reinterpret_cast<const uint4*>(S.twm + rk * L)[i];
      reinterpret_cast<uint4*>(twi_s + rk * L)[i] = reinterpret_cast<const uint4*>(S.itwm + rk * L)[i];
    }
  }
  // the twiddle staging above overlaps the previous step's tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (live) {
    const uint4* a = reinterpret_cast<const uint4*>(acch + (long long)t * NW + rk * L);
    const uint4* r = reinterpret_cast<const uint4*>(rhat.at(ridx(t)) + rk * L);
    const uint4* x = reinterpret_cast<const uint4*>(xhat_in + rk * L);
    for (int q4 = threadIdx.x; q4 < L / 4; q4 += blockDim.x)
      reinterpret_cast<uint4*>(Ar)[q4] = pw_madd(a[q4], x[q4], __ldcs(r + q4), c);
    __syncthreads();
    cta_ntt_inv16<RM>(Ar, 1, S.logL, twi + rk * L, &c);
  }
  asm volatile("barrier.cluster.wait;" ::: "memory");
  if (live) {
    // CTA q gets every prime of its coefficient slice [lo_q - (T-1), hi_q)
    for (int q = 0; q < nc; ++q) {
      if (q == rk) continue;
      const int lo = max(0, q * qs - (S.T - 1)), hi = min(L, (q + 1) * qs);
      uint32_t* Aq = cl.map_shared_rank(A, q) + rk * L;
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) Aq[i] = Ar[i];
    }
  }
  cl.sync();
  if (live) {
    // Garner for the slice (plus the T-1 coefficients below it), then the
    // digit sums of positions [lo, hi) (the last CTA also [L, L+T)) into
    // CTA 0's S
    const int lo = rk * qs, hi = min(L, lo + qs), glo = max(0, lo - (S.T - 1));
    const int gn = hi - glo;
    uint32_t* Cw = reinterpret_cast<uint32_t*>(Dg);  // np planes of gn words
    for (int i = glo + threadIdx.x; i < hi; i += blockDim.x) {
      const unsigned __int128 v = garner_coef(S, A, L, i);
      for (int u = 0; u < np; ++u) Cw[u * gn + (i - glo)] = (uint32_t)(v >> (32 * u));
    }
    __syncthreads();
    int64_t* S0 = cl.map_shared_rank(Ssum, 0);
    const int kend = rk == nc - 1 ? M : hi;
    for (int k = lo + threadIdx.x; k < kend; k += blockDim.x) {
      int64_t sk = 0;
      for (int u = 0; u < S.T; ++u) {
        const int i = k - u;
        if (i < glo || i >= hi) continue;
        const uint32_t top = Cw[(np - 1) * gn + (i - glo)];
        const uint32_t wt = u < np ? Cw[u * gn + (i - glo)] : ((top >> 31) ? 0xFFFFFFFFu : 0u);
        sk += u == S.T - 1 ? (int64_t)(int32_t)wt : (int64_t)wt;
      }
      S0[k] = sk;
    }
  }
  cl.sync();
  if (live && rk == 0) {
    int len = 0;
    const int sg = reconstruct_int<RM>(S, A, Ssum, Dg, M1, Wa, red, twi, err, &len, nullptr, 2);
    if (sg != 0) {
      if (threadIdx.x == 0) M1[Wa] = 0u;
      __syncthreads();
      solve_finish_mag(Wv, Wa, k2, M1, sg < 0 && len > 0, fin, T, X, red, err, len);
    }
    __threadfence();
  }
  cl.sync();
  if (live) {
    // the finished entry (global, written by CTA 0), transformed for prime rk
    int xl;
    const int xs = load_int(fin.out, fin.oi, Wv, X, &xl);
    if (threadIdx.x == 0 && rk == 0) {
      if (limbs_bits(X, xl) > xbmax) atomicOr(&err[kErrCapacity], kCapDegree);
      if (xl > L) atomicOr(&err[kErrCapacity], kCapDigits);
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const uint32_t d = i < xl ? X[i] : 0u;
      const uint32_t rr = reduce_2q(mul_shoup(d, 1u, c.one_s, c.q), c.q);
      Ar[i] = (xs < 0 && rr) ? c.q - rr : rr;
    }
    __syncthreads();
    cta_ntt_fwd16<RM>(Ar, 1, S.logL, twf + rk * L, &c);
    for (int i = threadIdx.x; i < L / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(xhat_out + rk * L)[i] = reinterpret_cast<const uint4*>(Ar)[i];
  }
}

// ------------------------------------------ tensor-core AXPY (opt-in) ---
// Every step's products R(t, j) x_j (x_j the vector entry just finished)
// share x_j, so they form one int8 GEMM on 7-bit digits (as the ratio GEMM,
// DESIGN.md §4): C[t][k'] = sum_i rdig(t)[i] xdig[k' - i], column k' of
// |R| |x| (digit products < 2^14, sums over <= 2^13 digits < 2^27: exact in
// int32).  The accumulators stay in those 7-bit columns as signed 64-bit
// sums (|.| < n 2^27), and a row's finish converts them to two's
// complement limbs and applies solve_finish.  Results equal k_solve_axpy's.

// packed lower triangle by rows: (r, q), q < r
__device__ __forceinline__ long long lidx_row(int r, int q) {
  return (long long)r * (r - 1) / 2 + q;
}

// 7-bit digits of |R_p[r]| of every stored entry, in column order (forward
// sweep: entry lidx(n,p,r)) and row order (back sweep: entry lidx_row(r,p)).
__global__ void k_solve_rdig(int n, int cap, IntBuf L, int kr, uint8_t* dcol,
                             uint8_t* drow, int* err) {
  const long long ne = (long long)n * (n - 1) / 2;
  for (long long li = blockIdx.x; li < ne; li += gridDim.x) {
    // column p of entry li: largest p with lidx(n, p, p+1) <= li
    int p = (int)((2.0 * n - 1 - sqrt((2.0 * n - 1) * (2.0 * n - 1) - 8.0 * li)) / 2);
    p = max(0, min(p, n - 2));
    while (p > 0 && lidx(n, p, p + 1) > li) --p;
    while (p + 1 < n - 1 && lidx(n, p + 1, p + 2) <= li) ++p;
    const int r = (int)(li - lidx(n, p, p + 1)) + p + 1;
    const int h = L.hdr[li];
    const int len = h < 0 ? -h : h;
    const uint32_t* src = L.limbs + li * (long long)cap;
    if (threadIdx.x == 0 && len > 0 && (limbs_bits(src, len) + 6) / 7 > kr)
      atomicOr(&err[kErrCapacity], kCapLimbs);
    uint32_t* c = reinterpret_cast<uint32_t*>(dcol + li * kr);
    uint32_t* rw = reinterpret_cast<uint32_t*>(drow + lidx_row(r, p) * kr);
    for (int i = threadIdx.x; i < kr / 4; i += blockDim.x) {
      uint32_t w = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        w |= (field32(src, len, 7LL * (4 * i + u)) & 127u) << (8 * u);
      c[i] = w;
      rw[i] = w;
    }
  }
}

// T[k'][i] = 7-bit digit k' - i of |x| (entry xi of xv), k' < mc, i < kr
__global__ void k_solve_toeplitz(IntBuf xv, int xi, int Wv, int kr, int mc,
                                 uint8_t* T, int* err) {
  extern __shared__ uint32_t xs[];
  const int h = xv.hdr[xi];
  const int nx = h < 0 ? -h : h;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) xs[i] = xv.limbs[(long long)xi * Wv + i];
  __syncthreads();
  const long long nxd = nx == 0 ? 0 : (limbs_bits(xs, nx) + 6) / 7;
  if (blockIdx.x == 0 && threadIdx.x == 0 && nxd + kr > mc)
    atomicOr(&err[kErrCapacity], kCapLimbs);  // product columns beyond mc
  const int per_row = kr / 16;
  const long long total = (long long)mc * per_row;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int kc = (int)(idx / per_row);
    const int i0 = (int)(idx - (long long)kc * per_row) * 16;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const long long jd = (long long)kc - (i0 + u);
      if (jd >= 0 && jd < nxd)
        w[u >> 2] |= (field32(xs, nx, 7 * jd) & 127u) << (8 * (u & 3));
    }
    reinterpret_cast<uint4*>(T + (long long)kc * kr)[i0 / 16] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// acc7[t] += s_t C[row(t)] for the targets of step j; the first target is
// complete afterwards and finished here (solve_finish), as in k_solve_axpy.
__global__ void __launch_bounds__(256)
k_solve_acc_tc(int n, int Wv, int Wa, int k2, IntBuf L, IntBuf xv, int xi, int j,
               int dir, const int32_t* C, int mc, long long* acc7, Finish fin,
               int* err) {
  extern __shared__ uint32_t sm_dyn[];
  const int hx = xv.hdr[xi];
  const int sx = hx < 0 ? -1 : 1;
  const int ntg = dir == 0 ? n - j - 1 : j;
  const int J = mc / 4;        // 28-bit super-digits
  const int Mres = J + 2;
  long long* Dsd = reinterpret_cast<long long*>(sm_dyn);          // J
  uint32_t* dig = reinterpret_cast<uint32_t*>(Dsd + J);           // Mres
  uint32_t* limbs = dig + Mres;                                   // Wa
  uint32_t* fscr = limbs + Wa;                                    // finish
  for (int kk = blockIdx.x; kk < ntg; kk += gridDim.x) {
    const int t = dir == 0 ? j + 1 + kk : j - 1 - kk;
    const long long li = dir == 0 ? lidx(n, j, t) : lidx(n, t, j);
    const int hc = L.hdr[li];
    long long* a = acc7 + (long long)t * mc;
    if (hc != 0 && hx != 0) {
      const long long crow = dir == 0 ? kk : t;
      const int32_t* c = C + crow * mc;
      const bool neg = (hc < 0) != (sx < 0);
      for (int k = threadIdx.x; k < mc; k += blockDim.x)
        a[k] += neg ? -(long long)c[k] : (long long)c[k];
    }
    if (kk != 0) continue;
    __syncthreads();
    // columns -> base-2^28 super-digit sums D_j (|D_j| < 2^58)
    for (int q = threadIdx.x; q < J; q += blockDim.x)
      Dsd[q] = a[4 * q] + a[4 * q + 1] * 128 + a[4 * q + 2] * 16384 + a[4 * q + 3] * 2097152;
    __syncthreads();
    const long long m28 = (1ll << 28) - 1;
    const int carry = cta_resolve(
        Mres, 28,
        [&](int q) -> int64_t {
          int64_t v = q < J ? (Dsd[q] & m28) : 0;
          if (q >= 1 && q - 1 < J) v += (Dsd[q - 1] >> 28) & m28;
          if (q >= 2 && q - 2 < J) v += Dsd[q - 2] >> 56;
          return v;
        },
        [&](int q, uint64_t d) { dig[q] = (uint32_t)d; }, fscr);
    if (carry > 0 || carry < -1) {
      if (threadIdx.x == 0) atomicOr(&err[kErrInternal], kIntDivision);
      return;
    }
    // two's complement limbs over Wa (sign-filled above the digits)
    const long long top = 28LL * Mres;
    for (int m = threadIdx.x; m < Wa; m += blockDim.x) {
      uint64_t accw = 0;
      for (int k = (32 * m) / 28; k < Mres && 28 * k < 32 * m + 32; ++k) {
        const int shl = 28 * k - 32 * m;
        accw |= shl >= 0 ? ((uint64_t)dig[k] << shl) : ((uint64_t)dig[k] >> -shl);
      }
      uint32_t v = (uint32_t)accw;
      if (carry < 0) {
        const long long lo = 32LL * m;
        if (lo >= top) v = 0xFFFFFFFFu;
        else if (lo + 32 > top) v |= 0xFFFFFFFFu << (int)(top - lo);
      }
      limbs[m] = v;
    }
    __syncthreads();
    solve_finish(Wv, Wa, k2, limbs, fin, fscr, err);
  }
}

size_t solve_acc_tc_smem_words(int Wv, int Wa, int mc) {
  const long long J = mc / 4;
  return (size_t)(2 * J + (J + 2) + Wa + solve_finish_words(Wv, Wa) + 64);
}

cudaError_t launch_solve_rdig(int n, int cap, IntBuf L, int kr, uint8_t* dcol,
                              uint8_t* drow, int* err, cudaStream_t st) {
  if (n < 2) return cudaSuccess;
  const long long ne = (long long)n * (n - 1) / 2;
  k_solve_rdig<<<(unsigned)std::min<long long>(ne, 8192), 128, 0, st>>>(n, cap, L, kr, dcol,
                                                                    drow, err);
  return cudaGetLastError();
}

cudaError_t launch_solve_toeplitz(IntBuf xv, int xi, int Wv, int kr, int mc,
                                  uint8_t* T, int* err, cudaStream_t st) {
  const long long words = (long long)mc * (kr / 16);
  const int blocks = (int)std::min<long long>((words + 255) / 256, 2048);
  k_solve_toeplitz<<<blocks, 256, (size_t)Wv * 4, st>>>(xv, xi, Wv, kr, mc, T, err);
  return cudaGetLastError();
}

cudaError_t launch_solve_acc_tc(int n, int Wv, int Wa, int k2, IntBuf L, IntBuf xv,
                                int xi, int j, int dir, const int32_t* C, int mc,
                                long long* acc7, const Finish& fin, int grid_cap,
                                int* err, cudaStream_t st) {
  const int rows = dir == 0 ? n - j - 1 : j;
  if (rows <= 0) return cudaSuccess;
  const size_t smem = solve_acc_tc_smem_words(Wv, Wa, mc) * 4;
  k_solve_acc_tc<<<std::min(rows, grid_cap), 256, smem, st>>>(
      n, Wv, Wa, k2, L, xv, xi, j, dir, C, mc, acc7, fin, err);
  return cudaGetLastError();
}

size_t solve_axpy_smem_words(int capX, int capC, int Wv, int Wa) {
  return (size_t)solve_axpy_words(capX, capC, Wv, Wa);
}
size_t solve_finish_smem_words(int Wv, int Wa) {
  return (size_t)solve_finish_words(Wv, Wa);
}

cudaError_t launch_solve_axpy(int n, int cap, int Wv, int Wa, int k2, IntBuf L,
                              IntBuf xv, int xi, int j, int dir, uint32_t* acc,
                              const Finish& fin, int capX, int capC,
                              uint32_t* gscratch, int grid_cap, int* err,
                              cudaStream_t st) {
  const int rows = dir == 0 ? n - j - 1 : j;
  if (rows <= 0) return cudaSuccess;
  const size_t smem =
      gscratch ? 0 : solve_axpy_smem_words(capX, capC, Wv, Wa) * 4;
  static const int seg = [] {
    const char* e = getenv("HGPU_SOLVE_SEG");
    return e ? atoi(e) : 0;
  }();
  k_solve_axpy<<<min(rows, grid_cap), 256, smem, st>>>(
      n, cap, Wv, Wa, k2, L, xv, xi, j, dir, acc, fin, capX, capC, gscratch,
      seg, err);
  return cudaGetLastError();
}

cudaError_t launch_solve_finish(int Wv, int Wa, int k2, const uint32_t* acc_i,
                                const Finish& fin, int* err, cudaStream_t st) {
  const size_t smem = solve_finish_smem_words(Wv, Wa) * 4;
  k_solve_finish<<<1, 256, smem, st>>>(Wv, Wa, k2, acc_i, fin, err);
  return cudaGetLastError();
}

cudaError_t launch_int_bits_batch(IntBuf v, int idx0, int step, int stride,
                                  int count, int* out, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  k_int_bits<<<(count + 127) / 128, 128, 0, st>>>(v, idx0, step, stride, count,
                                                  out);
  return cudaGetLastError();
}

size_t solve_ntt_smem_words(const DevPlan& S, int Wv, int Wa) {
  return (size_t)solve_ntt_words(S, Wv, Wa);
}

cudaError_t configure_solve_ntt(DevPlan& S, int cap, int Wv, int Wa, int* ok) {
  int dev = 0, maxopt = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // twiddles from global memory when staging them would not fit (or when
  // HGPU_SOLVE_TW_GLOBAL=1 asks for it)
  const char* twg = getenv("HGPU_SOLVE_TW_GLOBAL");
  S.tw_global = twg && atoi(twg) ? 1 : 0;
  if (!S.tw_global && solve_ntt_words(S, Wv, Wa) * 4 > (size_t)maxopt) S.tw_global = 1;
  const size_t step = solve_ntt_words(S, Wv, Wa) * 4;
  const size_t rh = ((size_t)S.NW + cap) * 4, xh = ((size_t)S.NW + Wv) * 4;
  *ok = step <= (size_t)maxopt && rh <= (size_t)maxopt && xh <= (size_t)maxopt;
  if (!*ok) return cudaSuccess;
  cudaError_t e;
  for (auto k : {k_solve_ntt<16>, k_solve_ntt<8>, k_solve_ntt<4>, k_solve_ntt_cl<16>,
                 k_solve_ntt_cl<8>, k_solve_ntt_cl<4>})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step)) !=
        cudaSuccess)
      return e;
  if ((e = cudaFuncSetAttribute(k_solve_rhat, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)rh)) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(k_solve_xhat, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)xh);
}

cudaError_t launch_solve_rhat(const DevPlan& S, int cap, IntBuf L, long long count,
                              EntryStore rhat, int grid_cap, int* err, cudaStream_t st,
                              long long e_begin) {
  if (count <= 0) return cudaSuccess;
  // every resident CTA slot (each transform is a latency-bound chain)
  const size_t smem = ((size_t)S.NW + cap) * 4;
  int dev = 0, nsm = 1, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_rhat, 256, smem);
  const long long grid = std::max<long long>(grid_cap, (long long)nsm * std::max(1, per_sm));
  k_solve_rhat<<<(int)std::min<long long>(count, grid), 256, smem, st>>>(S, cap, L, e_begin,
                                                                        count, rhat, err);
  return cudaGetLastError();
}

cudaError_t launch_solve_xhat(const DevPlan& S, IntBuf xv, int xi, int Wv, uint32_t* xhat,
                              int xbmax, int* err, cudaStream_t st) {
  k_solve_xhat<<<1, 512, ((size_t)S.NW + Wv) * 4, st>>>(S, xv, xi, Wv, xhat, xbmax, err);
  return cudaGetLastError();
}

cudaError_t launch_solve_ntt(const DevPlan& S, int n, int Wv, int Wa, int k2,
                             EntryStore rhat, const uint32_t* xhat_in,
                             uint32_t* xhat_out, uint32_t* acch, int j, int dir,
                             const Finish& fin, int grid, int xbmax, int* err,
                             cudaStream_t st) {
  const int ntg = dir == 0 ? n - j - 1 : j;
  if (ntg <= 0) return cudaSuccess;
  const long long items = (long long)(ntg - 1) * (S.NW / 4);
  const int pw = (int)std::min<long long>((items + kSolveNttThreads - 1) / kSolveNttThreads,
                                          grid);
  // widest NTT pass of the critical row's transforms (HGPU_SOLVE_RADIX)
  static const int radix = [] {
    const char* e = getenv("HGPU_SOLVE_RADIX");
    return e ? atoi(e) : 16;
  }();
  // the critical row on a cluster of np CTAs (HGPU_SOLVE_CLUSTER, 32-bit
  // digits only)
  static const int use_cl = [] {
    const char* e = getenv("HGPU_SOLVE_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  const size_t smem = solve_ntt_words(S, Wv, Wa) * 4;
  if (use_cl && S.w == 32 && S.np > 1) {
    auto kc = radix == 8 ? k_solve_ntt_cl<8> : (radix == 4 ? k_solve_ntt_cl<4> : k_solve_ntt_cl<16>);
    const int nc = S.np;
    const int grid_pw = ((pw + nc - 1) / nc) * nc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc + grid_pw);
    cfg.blockDim = dim3(kSolveNttThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch (HGPU_SOLVE_PDL): the next step's CTAs
    // are placed while this one drains and wait in griddepcontrol.wait
    static const int pdl = [] {
      const char* e = getenv("HGPU_SOLVE_PDL");
      return e ? atoi(e) : 1;
    }();
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kc, S, n, Wv, Wa, k2, rhat, xhat_in, xhat_out, acch, j, dir,
                              fin, xbmax, err);
  }
  auto kern = radix == 8 ? k_solve_ntt<8> : (radix == 4 ? k_solve_ntt<4> : k_solve_ntt<16>);
  kern<<<1 + pw, kSolveNttThreads, smem, st>>>(
      S, n, Wv, Wa, k2, rhat, xhat_in, xhat_out, acch, j, dir, fin, xbmax, err);
  return cudaGetLastError();
}

cudaError_t configure_solve_tc(int Wv, int Wa, int mc, int* ok) {
  int dev = 0, maxopt = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t smem = solve_acc_tc_smem_words(Wv, Wa, mc) * 4;
  *ok = smem <= (size_t)maxopt && (size_t)Wv * 4 <= (size_t)maxopt;
  if (!*ok) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_solve_acc_tc,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_solve_toeplitz, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Wv * 4);
}

cudaError_t configure_solve_kernels(int cap, int Wv, int Wa, bool* axpy_global) {
  cudaError_t e;
  int dev = 0, maxopt = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // the attribute admits the worst-case layout; launches use the layout of
  // the operand sizes actually met (more CTAs per SM)
  *axpy_global = solve_axpy_smem_words(Wv, cap, Wv, Wa) * 4 > (size_t)maxopt;
  if (!*axpy_global &&
      (e = cudaFuncSetAttribute(
           k_solve_axpy, cudaFuncAttributeMaxDynamicSharedMemorySize,
           (int)(solve_axpy_smem_words(Wv, cap, Wv, Wa) * 4))) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(k_solve_finish,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(solve_finish_smem_words(Wv, Wa) * 4));
}

}  // namespace hgpu
