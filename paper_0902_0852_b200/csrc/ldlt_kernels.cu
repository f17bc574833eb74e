// sm_100a kernels of the LDL^T engine.  Each kernel cites the reference step
// it reproduces (/root/reference/proj/src/ldlt.cpp).  Arithmetic is exact:
// the only roundings are the reference's own truncations (tdiv_q_2exp for the
// column values, tdiv_q for the ratios), so results are bit-identical.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"
#include "transform_ops.cuh"

namespace hgpu {

// ------------------------------------------------------------ helpers -----

__device__ __forceinline__ bool stage_aborted(const int* err) {
  return *(volatile const int*)&err[kErrZeroPivot] != INT_MAX ||
         *(volatile const int*)&err[kErrCapacity] != 0;
}

// Stages the Montgomery twiddle tables in shared memory (when the plan says
// they fit) and returns the pointers the transforms should use.
// A CTA that transforms a single integer reads the tables from global
// memory (L1) instead: staging them costs more than it saves (`stage`).
__device__ inline void stage_tables(const DevPlan& P, uint32_t* sm_fwd,
                                    uint32_t* sm_inv, const uint32_t** fwd,
                                    const uint32_t** inv, bool stage = true) {
  if (P.tw_smem && stage) {
    for (int i = threadIdx.x; i < P.NW; i += blockDim.x) {
      if (sm_fwd) sm_fwd[i] = P.twm[i];
      if (sm_inv) sm_inv[i] = P.itwm[i];
    }
    __syncthreads();
    if (fwd) *fwd = sm_fwd;
    if (inv) *inv = sm_inv;
  } else {
    if (fwd) *fwd = P.twm;
    if (inv) *inv = P.itwm;
  }
}

// ------------------------------------------------------ forward transform --
// For items i in [0,count): integer (in_base + i) of `src` -> transform at
// out + (out_base + i)*NW.  Records deg = floor((bits-1)/w) via atomicMax.
// Used for the strip moments and the shift at setup, and by ranks that
// receive a panel over NCCL.  Grid-stride over items.
__global__ void k_fwd_ints(const __grid_constant__ DevPlan P, IntBuf src, long long in_base,
                           uint32_t* out, long long out_base, int count,
                           int mont, int* maxdeg, int* err) {
  extern __shared__ uint32_t sm[];
  if (err && stage_aborted(err)) return;
  uint32_t* tab = sm;
  uint32_t* buf = sm + (P.tw_smem ? P.NW : 0);
  uint32_t* mag = buf + P.NW;
  const uint32_t* twm;
  stage_tables(P, tab, nullptr, &twm, nullptr);
  for (int item = blockIdx.x; item < count; item += gridDim.x) {
    int len;
    const int sign = load_int(src, in_base + item, P.cap, mag, &len);
    if (maxdeg && len > 0 && threadIdx.x == 0)
      atomicMax(maxdeg, (limbs_bits(mag, len) - 1) / P.w);
    transform_int(P, mag, len, 0, sign, buf,
                  out + (out_base + item) * (long long)P.NW, mont != 0, twm, err);
  }
}

// ------------------------------------------------------- workspace init ----
// ldlt.cpp:38-44: cols[c][r-c] = strip[r+c], cols[c][0] -= x.  By linearity
// the transform of strip[2c]-x is that[2c] - xhat.  grid.x: word blocks,
// grid.y: column c (all rows r >= c of an owned column).
__global__ void k_init_w(const __grid_constant__ DevPlan P, const uint32_t* that, const uint32_t* xhat,
                         const long long* colbase, uint32_t* W) {
  const int c = blockIdx.y;
  const long long base = colbase[c];
  if (base < 0) return;
  const int wd = blockIdx.x * blockDim.x + threadIdx.x;
  if (wd >= P.NW) return;
  const uint32_t q = P.pc[wd / P.L].q;
  for (int r = c; r < P.n; ++r) {
    uint32_t v = that[(long long)(r + c) * P.NW + wd];
    if (r == c) {
      const uint32_t xv = xhat[wd];
      v = v >= xv ? v - xv : v + q - xv;
    }
    W[(base + (r - c)) * P.NW + wd] = v;
  }
}

// The same with four words per thread (NW and L multiples of 4, so a group
// lies within one prime) and the rows of a column split over grid.z: a pure
// HBM write stream (config 3: 8.2 GB per factorisation).
__global__ void k_init_w4(const __grid_constant__ DevPlan P, const uint32_t* that, const uint32_t* xhat,
                          const long long* colbase, uint32_t* W) {
  const int c = blockIdx.y;
  const long long base = colbase[c];
  if (base < 0) return;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;  // group of 4 words
  if (4 * g >= P.NW) return;
  const long long NW4 = P.NW / 4;
  const uint4* src = reinterpret_cast<const uint4*>(that);
  uint4* dst = reinterpret_cast<uint4*>(W);
  for (int r = c + blockIdx.z; r < P.n; r += gridDim.z) {
    uint4 v = __ldg(src + (long long)(r + c) * NW4 + g);
    if (r == c) {
      const uint32_t q = P.pc[(4 * g) / P.L].q;
      const uint4 xv = reinterpret_cast<const uint4*>(xhat)[g];
      v.x = v.x >= xv.x ? v.x - xv.x : v.x + q - xv.x;
      v.y = v.y >= xv.y ? v.y - xv.y : v.y + q - xv.y;
      v.z = v.z >= xv.z ? v.z - xv.z : v.z + q - xv.z;
      v.w = v.w >= xv.w ? v.w - xv.w : v.w + q - xv.w;
    }
    __stcs(dst + (base + (r - c)) * NW4 + g, v);
  }
}

// ------------------------------------------------------------ extraction ---
// Stage p, rows r in [p, n): W[r][p] back to an exact integer (inverse NTT,
// CRT, carry resolution).  Then
//   pivot = W[p][p], ZeroPivot if 0                    (ldlt.cpp:48-50)
//   V_p[r] = tdiv_q_2exp(W[r][p], K/2)                 (ldlt.cpp:54-55)
//   ZeroPivot if V_p[p] == 0 and p < n-1               (ldlt.cpp:56)
// V goes to vint[slot][r]; the full pivot to piv[p].
__device__ void extract_body(const DevPlan& P, const uint32_t* W, const long long* colbase,
                             int p, int r_begin, int r_end, IntBuf vint,
                             long long vrow0, IntBuf piv, int* maxbitsV,
                             uint32_t* vhat, int* maxdegV, int* err, int round,
                             uint8_t* vdig, int kd, int bx, int gx) {
  extern __shared__ uint32_t sm[];
  __shared__ int s_bump;
  if (stage_aborted(err)) return;
  const int L = P.L, np = P.np, T = P.T, w = P.w;
  const int M = L + T;
  // rows this CTA extracts: with one, the tables are read from global memory
  // (and take no shared memory: the launch may size it without them)
  const bool multi = r_begin + bx + gx < r_end;
  const int tw_words = (P.tw_smem && multi) ? P.NW : 0;
  uint32_t* tabf = sm;
  uint32_t* tabi = sm + tw_words;
  uint32_t* A = tabi + tw_words;  // np*L residues -> CRT words
  int64_t* S = reinterpret_cast<int64_t*>(A + P.NW);  // M digit sums
  uint64_t* Dg = reinterpret_cast<uint64_t*>(S + M);  // M digits
  uint32_t* Lb = reinterpret_cast<uint32_t*>(Dg + M); // cap limbs of |W|
  uint32_t* red = Lb + P.cap;                         // scan scratch
  // HGPU_DEBUG & 1024: phase clocks of sampled pivot-row extractions
  long long xs[12];
  const bool xph = (P.debug & 1024) && p % 100 == 50 && r_begin == p && threadIdx.x == 0;
  if (xph) xs[0] = clock64();
  const uint32_t* twm;
  const uint32_t* itwm;
  stage_tables(P, tabf, tabi, &twm, &itwm, multi);
  const uint64_t dmask = (1ull << w) - 1ull;

  for (int r = r_begin + bx; r < r_end; r += gx) {
    if (xph) xs[1] = clock64();
    const uint32_t* src = W + (colbase[p] + (r - p)) * (long long)P.NW;
    for (int i = threadIdx.x; i < P.NW / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(A)[i] = reinterpret_cast<const uint4*>(src)[i];
    __syncthreads();
    if (xph) xs[2] = clock64();
    int len = 0;
    const int sg = reconstruct_int(P, A, S, Dg, Lb, P.cap, red, itwm, err, &len,
                                   xph ? xs + 3 : nullptr);
    if (xph) xs[7] = clock64();
    if (sg == 0) return;
    const int wsign = len == 0 ? 0 : sg;

    if (r == p) {  // pivot
      if (threadIdx.x == 0) {
        piv.hdr[p] = wsign * len;
        // the interval elimination checks only V_p (ldlt.cpp:110-111)
        if (len == 0 && round == 0) atomicMin(&err[kErrZeroPivot], p);
      }
      uint32_t* dst = piv.limbs + (long long)p * P.cap;
      for (int m = threadIdx.x; m < P.cap; m += blockDim.x) dst[m] = Lb[m];
    }
    // V = W >> k2: truncated toward zero (round 0, tdiv_q_2exp), or toward
    // -inf / +inf (round 1 / 2: the interval bounds, ldlt.cpp:105-108).  The
    // magnitude is |W| >> k2, plus one when the rounding moves away from zero
    // and a bit below k2 is set.  Built in Vb (the digit buffer is dead now).
    uint32_t* Vb = reinterpret_cast<uint32_t*>(Dg);
    if (threadIdx.x == 0) s_bump = 0;
    __syncthreads();
    if ((round == 1 && wsign < 0) || (round == 2 && wsign > 0)) {
      const int full = P.k2 / 32, rb = P.k2 % 32;
      bool any = false;
      for (int m = threadIdx.x; m < min(full, len); m += blockDim.x)
        any |= Lb[m] != 0u;
      if (threadIdx.x == 0 && rb && full < len && (Lb[full] & ((1u << rb) - 1u)))
        any = true;
      if (any) s_bump = 1;
    }
    __syncthreads();
    if (s_bump) {
      cta_resolve(
          P.cap, 32,
          [&](int k) -> int64_t {
            return (int64_t)field32(Lb, len, 32LL * k + P.k2) + (k == 0 ? 1 : 0);
          },
          [&](int k, uint32_t d) { Vb[k] = d; }, red);
    } else {
      for (int m = threadIdx.x; m < P.cap; m += blockDim.x)
        Vb[m] = field32(Lb, len, 32LL * m + P.k2);
      __syncthreads();
    }
    const long long vidx = vrow0 + r;
    uint32_t* vdst = vint.limbs + vidx * P.cap;
    for (int m = threadIdx.x; m < P.cap; m += blockDim.x) vdst[m] = Vb[m];
    const int vlen = cta_limb_len(Vb, P.cap, red);
    const int vbits = limbs_bits(Vb, vlen);
    if (vdig && r > p) {  // 7-bit digits of |V| for the ratio GEMM
      uint32_t* drow = reinterpret_cast<uint32_t*>(vdig + (long long)r * kd);
      for (int i = threadIdx.x; i < kd / 4; i += blockDim.x) {
        uint32_t wv = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          wv |= (field32(Vb, vlen, 7LL * (4 * i + u)) & 127u) << (8 * u);
        drow[i] = wv;
      }
    }
    const int vsign = vlen == 0 ? 0 : wsign;
    if (threadIdx.x == 0) {
      vint.hdr[vidx] = vsign * vlen;
      if (r == p && vlen == 0 && p < P.n - 1) atomicMin(&err[kErrZeroPivot], p);
      if (r > p) {
        atomicMax(&maxbitsV[p], vbits);
        if (vbits > 0) atomicMax(&maxdegV[p], (vbits - 1) / w);
      }
    }
    if (xph) xs[8] = clock64();
    // transform of V_p[r] for the trailing update (rows r > p)
    if (r > p)
      transform_int(P, Vb, vlen, 0, vsign, A, vhat + vidx * (long long)P.NW,
                    false, twm, err);
    __syncthreads();
    if (xph) {
      xs[9] = clock64();
      printf("extract p=%d tables %lld load %lld iNTT %lld garner %lld digitsums %lld "
             "resolve+pack %lld V+len %lld fwdNTT %lld cycles\n", p, xs[1] - xs[0],
             xs[2] - xs[1], xs[3] - xs[2], xs[4] - xs[3], xs[5] - xs[4], xs[7] - xs[5],
             xs[8] - xs[7], xs[9] - xs[8]);
    }
  }
}

// Near / far rows of stage p in one launch: each CTA takes a row, applies the
// panel's pending stages to its entry W[r][p] (k_update_col's arithmetic, as
// k_pivot does for the pivot entry) and extracts it (extract_body).  One
// launch instead of two per stage on the panel's latency path, and no wait
// for the column update's grid to drain.
__global__ void __launch_bounds__(256)
k_col_extract(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase, const uint32_t* Vhat,
              const uint32_t* Rhat, long long row_stride_slot, int nslots, int p, int r_begin,
              int r_end, IntBuf vint, long long vrow0, IntBuf piv, int* maxbitsV, uint32_t* vhat,
              int* maxdegV, int* err, uint8_t* vdig, int kd) {
  if (stage_aborted(err)) return;
  const long long NW = P.NW;
  for (int r = r_begin + blockIdx.x; r < r_end; r += gridDim.x) {
    if (nslots > 0) {
      uint32_t* dst = W + (colbase[p] + (r - p)) * NW;
      const uint32_t* vp = Vhat + (long long)p * NW;
      const uint32_t* rp = Rhat + (long long)r * NW;
      for (int wd = threadIdx.x; wd < P.NW; wd += blockDim.x) {
        uint64_t acc = 0;
        int s = 0;
        for (; s + 1 < nslots; s += 2) {
          const long long o0 = s * row_stride_slot + wd, o1 = o0 + row_stride_slot;
          const uint32_t v0 = __ldg(vp + o0), r0 = __ldg(rp + o0);
          const uint32_t v1 = __ldg(vp + o1), r1 = __ldg(rp + o1);
          acc += (uint64_t)v0 * r0;
          acc += (uint64_t)v1 * r1;
        }
        if (s < nslots) {
          const long long o0 = s * row_stride_slot + wd;
          acc += (uint64_t)__ldg(vp + o0) * __ldg(rp + o0);
        }
        const PrimeConsts& pc = P.pc[wd / P.L];
        const uint32_t t32 = reduce_sum64(acc, pc);
        const uint32_t old = dst[wd];
        dst[wd] = old >= t32 ? old - t32 : old + pc.q - t32;
      }
      __syncthreads();
    }
    extract_body(P, W, colbase, p, r, r + 1, vint, vrow0, piv, maxbitsV, vhat, maxdegV, err, 0,
                 vdig, kd, 0, 1);
    __syncthreads();
  }
}

#ifdef HGPU_EXTRACT_MINB  // experiment: cap k_extract's registers (512 threads x MINB CTAs per SM)
__global__ void __launch_bounds__(512, HGPU_EXTRACT_MINB)
#else
__global__ void
#endif
k_extract(const __grid_constant__ DevPlan P, const uint32_t* W, const long long* colbase,
                          int p, int r_begin, int r_end, IntBuf vint,
                          long long vrow0, IntBuf piv, int* maxbitsV,
                          uint32_t* vhat, int* maxdegV, int* err, int round,
                          uint8_t* vdig, int kd) {
  extract_body(P, W, colbase, p, r_begin, r_end, vint, vrow0, piv, maxbitsV,
               vhat, maxdegV, err, round, vdig, kd, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------- reciprocal --
// Per stage, one CTA: Y ~ 2^S / |V_p| within a few units, S = n + Pt with
// n = bits(V_p) and Pt = e + 32, where e bounds the bits of every ratio of the
// stage.  Newton with precision doubling: level i holds Y_i ~ 2^(n_i+p_i)/D_i
// for D_i = D truncated to its top n_i = min(n, p_{i+1}+G) bits, and
//   Y_{i+1} = Y_i 2^d + (Y_i (2^(n'+p_i) - D' Y_i)) / 2^(n'+p_i-d),
// d = p_{i+1} - p_i.  Only the last level touches Pt-sized operands, so the
// whole reciprocal costs ~3 Pt x Pt limb products.  ys[0] = S, ys[1] = nY.
__device__ inline int recip_levels(int Pt, int* lv) {
  // lv[0] <= 48 < ... < lv[k] = Pt, lv[i] = ceil(lv[i+1]/2) + 8
  int tmp[40], k = 0;
  tmp[k++] = Pt;
  while (tmp[k - 1] > 48) tmp[k] = (tmp[k - 1] + 1) / 2 + 8, ++k;
  for (int i = 0; i < k; ++i) lv[i] = tmp[k - 1 - i];
  return k;
}

__device__ void recip_body(const DevPlan& P, IntBuf vint, long long prow,
                           const int* maxbitsV, int p, IntBuf piv, int dmax_bits,
                           uint32_t* Ybuf, int* ys, uint32_t* gscratch,
                           int use_gscratch, int* err, int b,
                           long long scratch_words = 0) {
  extern __shared__ uint32_t sm_dyn[];
  __shared__ uint32_t red[64];
  if (stage_aborted(err)) return;
  {
    // b: batched instance (0 in the LDL^T)
    prow += (long long)b * P.bat_vrow;
    maxbitsV += b * P.bat_mb;
    Ybuf += b * P.bat_ybuf;
    ys += b * P.bat_ys;
    gscratch += b * P.bat_scr;
  }
  const int h = vint.hdr[prow];
  const int nD = h < 0 ? -h : h;
  if (nD == 0) return;  // flagged as ZeroPivot by k_extract
  const uint32_t* Dg = vint.limbs + prow * (long long)P.cap;  // global
  const int n = limbs_bits(Dg, nD);
  // max over rows of bits(V_r 2^k2): exact (after the bulk extraction) or,
  // when dmax_bits > 0, the PD bound |W_rp|^2 <= W_rr W_pp with
  // bits(W_rr) <= dmax_bits, so the reciprocal can run concurrently with the
  // extraction of the other rows; k_divide verifies the bound per row.
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
  const int Lm = (Pt + G + 31) / 32 + 2;  // limbs of any D' or Y
  const int nYf = (Pt + 2 + 31) / 32 + 1;
  if (nYf > P.ycap) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return;
  }
  uint32_t* sm = use_gscratch ? gscratch : sm_dyn;
  // the top Lm + 2 limbs of D: every level reads D' (its top <= 32 Lm - 64
  // bits) from here instead of global memory
  const int dbase = max(0, nD - (Lm + 2));
  const int nDs = nD - dbase;
  uint32_t* Ds = sm;                 // Lm + 2
  for (int k = threadIdx.x; k < nDs; k += blockDim.x) Ds[k] = Dg[dbase + k];
  __syncthreads();
  sm += Lm + 2;
  uint32_t* Dt = sm;                 // Lm
  uint32_t* Y = Dt + Lm;             // Lm
  uint32_t* Pr = Y + Lm;             // 2 Lm + 1
  uint32_t* E = Pr + 2 * Lm + 1;     // 2 Lm + 2
  uint32_t* Tm = E + 2 * Lm + 2;     // 3 Lm + 2
  uint32_t* col = Tm + 3 * Lm + 2;   // 2 * 3 (3 Lm + 2)
  // product planes: up to 6 segments' worth, fewer when the caller's scratch
  // (scratch_words > 0) is sized to the stage's bound
  int segs = 6;
  if (scratch_words > 0)
    segs = (int)min(6LL, (scratch_words - 10LL * Lm - 71) / (3LL * Lm + 2));
  if (segs < 1) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return;
  }
  const int col_words = segs * (3 * Lm + 2);
  int lv[40];
  const int nl = recip_levels(Pt, lv);
  // seed: Y_0 = floor(2^(n+p0)/D) ~ (2^126/top64(D)) >> (62 - p0)
  const int p0 = lv[0];
  if (threadIdx.x == 0) {
    const uint32_t hi = field32(Ds, nDs, (long long)n - 32 - 32LL * dbase);
    const uint32_t lo = field32(Ds, nDs, (long long)n - 64 - 32LL * dbase);
    const double d = ldexp((double)hi, 32) + (double)lo;  // [2^63, 2^64)
    const unsigned long long y63 =
        (unsigned long long)(ldexp(1.0, 126) / d);        // (2^62, 2^63]
    const unsigned long long y0 = y63 >> (62 - p0);
    Y[0] = (uint32_t)y0;
    Y[1] = (uint32_t)(y0 >> 32);
  }
  __syncthreads();
  int nY = 2;
  const bool prof = (P.debug & 256) && p == 50 && threadIdx.x == 0;
  // one Newton level; kWarp: run by warp 0 alone (small levels)
  auto level = [&](auto warp_tag, int i) {
    constexpr bool kWarp = decltype(warp_tag)::value;
    const int t0 = kWarp ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    const int ts = kWarp ? 32 : (int)blockDim.x;
    auto sync = [] {
      if (kWarp) __syncwarp(); else __syncthreads();
    };
    auto resolve = [&](int M, auto getv, auto putd) {
      if constexpr (kWarp) return warp_resolve(M, 32, getv, putd);
      else return cta_resolve(M, 32, getv, putd, red);
    };
    // out = columns [k_begin, M) of a*b (the warp path forms all of [0, M))
    auto mul = [&](const uint32_t* a, int na, const uint32_t* b, int nb,
                   uint32_t* out, int M, int k_begin) {
      if constexpr (kWarp) warp_mul(a, na, b, nb, out, M, col);
      else cta_mul(a, na, b, nb, out, M, col, red, col_words, k_begin);
    };
    long long tph[6];
    if (prof) tph[0] = clock64();
    const int pa = lv[i], pb = lv[i + 1], dlt = pb - pa;
    const int mb = min(n, pb + G);   // bits of D'
    const int t = n - mb;
    const int nDt = (mb + 31) / 32;
    for (int k = t0; k < nDt; k += ts) Dt[k] = field32(Ds, nDs, 32LL * k + t - 32LL * dbase);
    sync();
    // E = 2^Sb - D' Y, Sb = mb + pa.  Y is within a few units at precision
    // pa, so |E| < 2^(mb+3) <= 2^(32 nDt + 3): the low nL = nDt + 1 limbs of
    // the product (a low short product) determine E, read as a two's
    // complement number mod 2^(32 nL).
    const int nL = nDt + 1;
    if (prof) tph[1] = clock64();
    mul(Dt, nDt, Y, nY, Pr, nL, 0);
    if (prof) tph[2] = clock64();
    const int Sb = mb + pa;
    resolve(
        nL,
        [&](int k) -> int64_t {
          const int64_t av = (k == Sb / 32) ? (int64_t)(1u << (Sb % 32)) : 0;
          return av - (int64_t)Pr[k];
        },
        [&](int k, uint32_t dd) { E[k] = dd; });
    const int sgn = (E[nL - 1] & 0x80000000u) ? -1 : 1;
    uint32_t* Ev = E;
    if (sgn < 0) {  // |E| = 2^(32 nL) - E
      resolve(
          nL, [&](int k) -> int64_t { return -(int64_t)E[k]; },
          [&](int k, uint32_t dd) { Pr[k] = dd; });
      Ev = Pr;
    }
    const int nE = kWarp ? warp_limb_len(Ev, nL) : cta_limb_len(Ev, nL, red);
    if (prof) tph[3] = clock64();
    // Tm = Y |E|, only from column K0 on: Y' below uses Tm >> sh, and the
    // dropped columns sum to < min(nY,nE) 2^(32 K0 + 33) <= 2^(sh - 21), so
    // Y' moves by at most one unit (|Y - 2^S/D| <= 4 at the last level)
    const int nYn = min(Lm, (pb + 2 + 31) / 32 + 1);
    const int sh = Sb - dlt;
    const int K0 = kWarp ? 0 : max(0, (sh - 64) / 32);
    const int nT = nY + nE;
    if (nE > 0) mul(Y, nY, Ev, nE, Tm, nT, K0);
    if (prof) tph[4] = clock64();
    // Y' = Y 2^dlt +- Tm >> (Sb - dlt)
    resolve(
        nYn,
        [&](int k) -> int64_t {
          const int64_t yv = field32(Y, nY, 32LL * k - dlt);
          const int64_t tv =
              nE > 0 ? (int64_t)field32(Tm, nT - K0, 32LL * k + sh - 32LL * K0) : 0;
          return sgn > 0 ? yv + tv : yv - tv;
        },
        [&](int k, uint32_t dd) { Pr[k] = dd; });
    for (int k = t0; k < nYn; k += ts) Y[k] = Pr[k];
    sync();
    if (prof) {
      tph[5] = clock64();
      printf("recip lvl %d%s pa=%d pb=%d nDt=%d nY=%d nE=%d: Dt %lld mul1 %lld E %lld mul2 %lld Yupd %lld\n",
             i, kWarp ? "w" : "", pa, pb, nDt, nY, nE, tph[1] - tph[0],
             tph[2] - tph[1], tph[3] - tph[2], tph[4] - tph[3], tph[5] - tph[4]);
    }
    nY = nYn;
  };
  // levels whose operands stay within kWarpLimbs run on warp 0 alone
  constexpr int kWarpLimbs = 128;
  __shared__ int s_next[2];
  int i = 0;
  if (threadIdx.x < 32) {
    for (; i + 1 < nl; ++i) {
      const int nDt = (min(n, lv[i + 1] + G) + 31) / 32;
      if (nDt > kWarpLimbs || nY > kWarpLimbs) break;
      level(std::true_type{}, i);
    }
    if (threadIdx.x == 0) {
      s_next[0] = i;
      s_next[1] = nY;
    }
  }
  __syncthreads();
  i = s_next[0];
  nY = s_next[1];
  for (; i + 1 < nl; ++i) level(std::false_type{}, i);
  for (int k = threadIdx.x; k < P.ycap; k += blockDim.x)
    Ybuf[k] = k < nY ? Y[k] : 0u;
  if (threadIdx.x == 0) {
    ys[0] = S;
    ys[1] = nY;
    ys[2] = amax;
  }
}

}  // namespace hgpu
#include "recip_fast.cuh"
namespace hgpu {

__global__ void __launch_bounds__(512) k_recip(const __grid_constant__ DevPlan P, IntBuf vint, long long prow,
                        const int* maxbitsV, int p, IntBuf piv, int dmax_bits,
                        uint32_t* Ybuf, int* ys, uint32_t* gscratch,
                        int use_gscratch, int* err) {
  extern __shared__ uint32_t sm_dyn[];
  if (P.recip_fast && !use_gscratch && gridDim.y == 1) {
    if (stage_aborted(err)) return;
    if (recip_fast_body(P, vint, prow, maxbitsV, p, piv, dmax_bits, Ybuf, ys, sm_dyn,
                        rf::dyn_smem_words(), err))
      return;
  }
  recip_body(P, vint, prow, maxbitsV, p, piv, dmax_bits, Ybuf, ys, gscratch,
             use_gscratch, err, blockIdx.y);
}


// Quotient from the top of the product.  Pr[0, nPs) holds the product
// columns from limb K0 on, i.e. F 2^shs with F = |V| Y / 2^sh lowered by
// < 2^-32 (dropped columns) and within 2^-32 of |V| 2^k2 / |D| (k_recip's
// |Y - 2^S/D| <= 4), shs = sh - 32 K0 >= 32.  When the 32 fraction bits of F
// lie in [4, 2^32-5], q = floor(F) exactly; otherwise floor(F) is within one
// of q and the remainder window |V| 2^k2 - q~ D over nD+2 limbs decides the
// correction exactly.  `away`: interval rounding bumps a non-integer
// quotient away from zero.  Writes |q| to Qt (Qt may alias neither Pr nor
// col); Pr is reused as the window scratch.  Returns the limb count of |q|,
// or -1 after raising kCapLimbs.
__device__ int ratio_quotient(const DevPlan& P, uint32_t* Pr, int nPs, int shs,
                              uint32_t* Qt, uint32_t* col, uint32_t* red, int CY,
                              const uint32_t* Vg, int na, const uint32_t* Dg,
                              int nD, bool away, int* err) {
  int nq;
  const int nQ = max(0, (int)((32LL * nPs - shs + 31) / 32));
  for (int i = threadIdx.x; i < nQ; i += blockDim.x)
    Qt[i] = field32(Pr, nPs, 32LL * i + shs);
  const uint32_t frac = field32(Pr, nPs, (long long)shs - 32);
  __syncthreads();
  nq = cta_limb_len(Qt, nQ, red);
  const bool exact_needed = shs < 32 || frac < 4u || frac > 0xFFFFFFFAu;
  int bump = (away && !exact_needed) ? 1 : 0;  // fast path: never exact
  if (exact_needed) {
    // remainder window: |V| 2^k2 - q~ D  (mod 2^(32 nw)), nw = nD + 2
    const int nw = nD + 2;
    uint32_t* Wa = Pr;
    uint32_t* Wb = Pr + nw;
    cta_mul(Qt, nq, Dg, nD, Wb, nw, col, red, 3 * CY);
    cta_resolve(
        nw, 32,
        [&](int k) -> int64_t {
          return (int64_t)field32(Vg, na, 32LL * k - P.k2) - (int64_t)Wb[k];
        },
        [&](int k, uint32_t d) { Wa[k] = d; }, red);
    int adj = 0;
    if (Wa[nw - 1] & 0x80000000u) {
      adj = -1;  // remainder negative: q~ was one too large
    } else {
      cta_resolve(
          nw, 32,
          [&](int k) -> int64_t {
            return (int64_t)Wa[k] - (int64_t)(k < nD ? Dg[k] : 0u);
          },
          [&](int k, uint32_t d) { Wb[k] = d; }, red);
      if (!(Wb[nw - 1] & 0x80000000u)) {
        adj = 1;
        cta_resolve(
            nw, 32,
            [&](int k) -> int64_t {
              return (int64_t)Wb[k] - (int64_t)(k < nD ? Dg[k] : 0u);
            },
            [&](int k, uint32_t d) { Wa[k] = d; }, red);
        if (!(Wa[nw - 1] & 0x80000000u) && threadIdx.x == 0)
          atomicOr(&err[kErrInternal], kIntDivision);
      }
    }
    if (away) {
      // remainder: Wa (adj 0), Wb (adj +1), Wa + D (adj -1)
      const uint32_t* rem = adj == 1 ? Wb : Wa;
      if (adj == -1) {
        __syncthreads();
        cta_resolve(
            nw, 32,
            [&](int k) -> int64_t {
              return (int64_t)Wa[k] + (int64_t)(k < nD ? Dg[k] : 0u);
            },
            [&](int k, uint32_t d) { Wb[k] = d; }, red);
        rem = Wb;
      }
      bump = cta_limb_len(rem, nw, red) != 0 ? 1 : 0;
    }
    adj += bump;
    bump = 0;
    if (adj != 0) {
      const int nn = nq + 1;
      cta_resolve(
          nn, 32,
          [&](int k) -> int64_t {
            return (int64_t)(k < nq ? Qt[k] : 0u) + (k == 0 ? adj : 0);
          },
          [&](int k, uint32_t d) { col[k] = d; }, red);
      for (int i = threadIdx.x; i < nn; i += blockDim.x) Qt[i] = col[i];
      __syncthreads();
      nq = cta_limb_len(Qt, nn, red);
    }
    // every thread has read the window signs before Pr is reused below
    __syncthreads();
  }
  if (bump) {
    const int nn = nq + 1;
    cta_resolve(
        nn, 32,
        [&](int k) -> int64_t {
          return (int64_t)(k < nq ? Qt[k] : 0u) + (k == 0 ? 1 : 0);
        },
        [&](int k, uint32_t d) { col[k] = d; }, red);
    for (int i = threadIdx.x; i < nn; i += blockDim.x) Qt[i] = col[i];
    __syncthreads();
    nq = cta_limb_len(Qt, nn, red);
  }
  if (nq > P.cap) {
    if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
    return -1;
  }
  return nq;
}

// ---------------------------------------------------------------- ratios ---
// Stage p, rows r in (p, n):  R_p[r] = tdiv_q(V_p[r] << K/2, V_p[p])
// (ldlt.cpp:15-20, 57-58).  With A = |V_r| 2^{K/2}, D = |V_p|, n = bits(D):
//   F = (|V_r| >> t) * Y / 2^{S-K/2-t},   t = max(0, n - K/2 - 40),
// differs from A/D by <= 2^-32 (|Y - 2^S/D| <= 4 from k_recip, and
// S = n + e + 32 with 2^e >= 4 A/D; the dropped low bits of V cost < 2^-39),
// and the product is formed only from column K0 = (sh-75)/32 up, which
// lowers F by < 2^-32 more.  So when the 32 fraction bits of F lie in
// [4, 2^32-5], q = floor(F) exactly and no remainder is needed.  Otherwise
// (e.g. exact quotients) floor(F) is within one of q and the remainder
// window A - q~ D over nD+2 limbs decides the correction exactly.
__device__ void divide_body(const DevPlan& P, IntBuf vint, long long vrow0, int p,
                            int r_begin, int r_end,
                            const uint32_t* Ybuf, const int* ys, IntBuf rint,
                            long long rrow0, uint32_t* rhat, int* maxdegR,
                            uint32_t* gscratch, int use_gscratch, int* err,
                            IvDiv iv, int bx, int gx, int b) {
  extern __shared__ uint32_t sm_dyn[];
  if (stage_aborted(err)) return;
  const int cap = P.cap, ycap = P.ycap;
  const long long span = div_span_words(cap, ycap);
  const long long cta_words = span + div_extra_words(P);
  {
    // b: batched instance (0 in the LDL^T)
    vrow0 += (long long)b * P.bat_vrow;
    rrow0 += (long long)b * P.bat_rrow;
    Ybuf += b * P.bat_ybuf;
    ys += b * P.bat_ys;
    gscratch += (long long)b * gx * cta_words;
  }
  // one row per CTA: twiddles from global memory, no table region
  const bool multi = r_begin + bx + gx < r_end;
  uint32_t* tab = sm_dyn;
  uint32_t* sm = use_gscratch ? gscratch + (long long)bx * cta_words
                              : sm_dyn + ((P.tw_smem && multi) ? P.NW : 0);
  const uint32_t* twm;
  stage_tables(P, tab, nullptr, &twm, nullptr, multi);
  const int CY = (cap + ycap + 2 + 3) & ~3;  // 16-byte aligned regions
  uint32_t* Vt = sm;                 // cap      } later: Qt (cap + ycap)
  uint32_t* Y = Vt + cap;            // ycap     }
  uint32_t* Pr = Vt + CY;            // CY       later: windows Wa | Wb, NTT
  uint32_t* col = Pr + CY;           // 3 CY
  uint32_t* red = col + 3 * CY;      // 64
  uint32_t* Qt = Vt;
  const long long pidx = vrow0 + p;
  // interval mode: the pivot interval [D.lo, D.hi] is sign-definite (else
  // ZeroPivot aborted the stage); sd is its sign
  const int sd = iv.mode == 0 ? 0 : (vint.hdr[pidx] > 0 ? 1 : -1);

  for (int r = r_begin + bx; r < r_end; r += gx) {
    const long long vidx = vrow0 + r;
    // numerator bound and divisor (ldlt.cpp:113-131 restated per corner):
    //   R.lo = floor(min corner): N = sd > 0 ? V.lo : V.hi, D = N > 0 ? D.hi : D.lo
    //   R.hi = ceil(max corner):  N = sd > 0 ? V.hi : V.lo, D = N > 0 ? D.lo : D.hi
    IntBuf nb = vint;
    bool use_hi_div = false;
    if (iv.mode != 0) {
      const bool n_lo = (iv.mode == 1) == (sd > 0);
      nb = n_lo ? vint : iv.vhi;
      const int hn = nb.hdr[vidx];
      use_hi_div = (iv.mode == 1) == (hn > 0);
    }
    const IntBuf db = use_hi_div ? iv.vhi : vint;
    const uint32_t* Yb = use_hi_div ? iv.yhi : Ybuf;
    const int* yb = use_hi_div ? iv.yshi : ys;
    const int S = yb[0], nY = yb[1], amax_used = yb[2];
    const int hd = db.hdr[pidx];
    const int nD = hd < 0 ? -hd : hd;
    const int sD = hd < 0 ? -1 : (hd > 0);
    const uint32_t* Dg = db.limbs + pidx * cap;
    const int n = nD ? limbs_bits(Dg, nD) : 0;
    const int hv = nb.hdr[vidx];
    const int na = hv < 0 ? -hv : hv;
    const int sV = hv < 0 ? -1 : (hv > 0);
    const uint32_t* Vg = nb.limbs + vidx * cap;   // global, read-only
    const long long ridx = rrow0 + r;
    uint32_t* dst = rint.limbs + ridx * cap;
    int nq = 0;
    if (na > 0 && nD > 0) {
      const int vbits = limbs_bits(Vg, na);
      if (vbits + P.k2 > amax_used) {  // reciprocal too short for this row
        if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapAmax);
        return;
      }
      const int tv = max(0, n - P.k2 - 40);
      const int nt = max(0, (vbits - tv + 31) / 32);
      for (int i = threadIdx.x; i < nt; i += blockDim.x)
        Vt[i] = field32(Vg, na, 32LL * i + tv);
      for (int i = threadIdx.x; i < nY; i += blockDim.x) Y[i] = Yb[i];
      __syncthreads();
      const int nP = nt + nY;
      const int sh = S - P.k2 - tv;
      // short product: columns below K0 move F by < 2^-32 (see the header)
      const int K0 = max(0, (sh - 75) / 32);
      const int nPs = nP - K0;
      const int shs = sh - 32 * K0;
      cta_mul(Vt, nt, Y, nY, Pr, nP, col, red, 3 * CY, K0);
      // interval rounding: one more unit of magnitude when the exact quotient
      // is not an integer and the rounding points away from zero
      const bool away = (iv.mode == 1 && sV * sD < 0) || (iv.mode == 2 && sV * sD > 0);
      nq = ratio_quotient(P, Pr, nPs, shs, Qt, col, red, CY, Vg, na, Dg, nD, away, err);
      if (nq < 0) return;
    }
    const int rsign = nq == 0 ? 0 : sV * sD;
    for (int i = threadIdx.x; i < cap; i += blockDim.x)
      dst[i] = i < nq ? Qt[i] : 0u;
    if (threadIdx.x == 0) {
      rint.hdr[ridx] = rsign * nq;
      if (nq > 0 && maxdegR) atomicMax(maxdegR, (limbs_bits(Qt, nq) - 1) / P.w);
    }
    // transform of R_p[r] (Montgomery form) for the trailing update; the
    // NTT buffer reuses the Barrett scratch when it is large enough
    if (rhat) {
      uint32_t* X = P.NW <= 4 * CY ? Pr : sm + span;
      transform_int(P, Qt, nq, 0, rsign, X, rhat + ridx * (long long)P.NW,
                    true, twm, err);
    } else {
      __syncthreads();
    }
  }
}

#ifndef HGPU_DIVIDE_MINB
#define HGPU_DIVIDE_MINB 3  // 80 registers; 4: 64 registers (experiment)
#endif
__global__ void __launch_bounds__(256, HGPU_DIVIDE_MINB) k_divide(const __grid_constant__ DevPlan P, IntBuf vint, long long vrow0, int p,
                         int r_begin, int r_end,
                         const uint32_t* Ybuf, const int* ys, IntBuf rint,
                         long long rrow0, uint32_t* rhat, int* maxdegR,
                         uint32_t* gscratch, int use_gscratch, int* err,
                         IvDiv iv) {
  divide_body(P, vint, vrow0, p, r_begin, r_end, Ybuf, ys, rint, rrow0, rhat,
              maxdegR, gscratch, use_gscratch, err, iv, blockIdx.x, gridDim.x,
              blockIdx.y);
}

// A single row (the pivot chain's next row) with 512 threads; the multi-row
// kernel above is held to 80 registers so that a CTA fits beside two
// trailing-update CTAs on an SM instead of waiting for one to leave.
__global__ void __launch_bounds__(512) k_divide1(const __grid_constant__ DevPlan P, IntBuf vint, long long vrow0, int p,
                         int r_begin, int r_end,
                         const uint32_t* Ybuf, const int* ys, IntBuf rint,
                         long long rrow0, uint32_t* rhat, int* maxdegR,
                         uint32_t* gscratch, int use_gscratch, int* err,
                         IvDiv iv) {
  divide_body(P, vint, vrow0, p, r_begin, r_end, Ybuf, ys, rint, rrow0, rhat,
              maxdegR, gscratch, use_gscratch, err, iv, blockIdx.x, gridDim.x,
              blockIdx.y);
}

// Pivot chain of stage p in one CTA (the three steps of the helper stream,
// fused to save two launches per stage): column p's pivot entry receives the
// panel's stages [0, s) (as k_update_col), is extracted (k_extract, row p:
// pivot, V_p[p], ZeroPivot) and the stage's reciprocal is formed (k_recip).
__device__ __forceinline__ void pivot_body(
    const DevPlan& P, uint32_t* W, const long long* colbase, const uint32_t* Vhat,
    const uint32_t* Rhat, long long row_stride_slot, int nslots, int p, IntBuf vint,
    long long vrow0, IntBuf piv, int* maxbitsV, uint32_t* vhat, int* maxdegV, int dmax_bits,
    uint32_t* Ybuf, int* ys, uint32_t* gscratch, int use_gscratch, int* err, PivotDiv pd) {
  if (stage_aborted(err)) return;
  // HGPU_DEBUG & 4096: phase clocks of sampled stages (timing aid)
  const bool ph = (P.debug & 4096) && p % 100 == 50 && threadIdx.x == 0;
  long long t[5];
  if (ph) t[0] = clock64();
  if (pd.on) {
    // R_{p-1}[p] of the previous stage of the panel (k_divide, one row)
    divide_body(P, vint, pd.vrow0, p - 1, p, p + 1, pd.Ybuf, pd.ys, pd.rint,
                pd.vrow0, pd.rhat, pd.maxdegR, pd.dscr, pd.use_dscr, err, IvDiv{},
                0, 1, 0);
    __syncthreads();
    if (stage_aborted(err)) return;
  }
  if (ph) t[1] = clock64();
  if (nslots > 0) {
    const long long NW = P.NW;
    uint32_t* dst = W + colbase[p] * NW;
    const uint32_t* vp = Vhat + (long long)p * NW;
    const uint32_t* rp = Rhat + (long long)p * NW;
    for (int wd = threadIdx.x; wd < P.NW; wd += blockDim.x) {
      uint64_t acc = 0;
      for (int s = 0; s < nslots; ++s) {
        const long long off = s * row_stride_slot + wd;
        acc += (uint64_t)__ldg(vp + off) * __ldg(rp + off);
      }
      const PrimeConsts& pc = P.pc[wd / P.L];
      const uint32_t t32 = reduce_sum64(acc, pc);
      const uint32_t old = dst[wd];
      dst[wd] = old >= t32 ? old - t32 : old + pc.q - t32;
    }
    __syncthreads();
  }
  if (ph) t[2] = clock64();
  extract_body(P, W, colbase, p, p, p + 1, vint, vrow0, piv, maxbitsV, vhat,
               maxdegV, err, 0, nullptr, 0, 0, 1);
  __syncthreads();
  if (ph) t[3] = clock64();
  if (p < P.n - 1) {
    extern __shared__ uint32_t sm_dyn[];
    if (!(P.recip_fast && !use_gscratch &&
          recip_fast_body(P, vint, vrow0 + p, maxbitsV, p, piv, dmax_bits, Ybuf, ys, sm_dyn,
                          rf::dyn_smem_words(), err))) {
      recip_body(P, vint, vrow0 + p, maxbitsV, p, piv, dmax_bits, Ybuf, ys,
                 gscratch, use_gscratch, err, 0, pd.recip_words);
    }
  }
  if (ph) {
    t[4] = clock64();
    printf("k_pivot p=%d div %lld col %lld extract %lld recip %lld cycles\n", p,
           t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3]);
  }
}

__global__ void __launch_bounds__(512)
k_pivot(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase, const uint32_t* Vhat,
        const uint32_t* Rhat, long long row_stride_slot, int nslots, int p,
        IntBuf vint, long long vrow0, IntBuf piv, int* maxbitsV, uint32_t* vhat,
        int* maxdegV, int dmax_bits, uint32_t* Ybuf, int* ys, uint32_t* gscratch,
        int use_gscratch, int* err, PivotDiv pd) {
  pivot_body(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, p, vint, vrow0, piv, maxbitsV,
             vhat, maxdegV, dmax_bits, Ybuf, ys, gscratch, use_gscratch, err, pd);
}

// The same chain step in a footprint that fits beside two k_update_tiled
// CTAs on one SM (256 threads, <= 80 registers: 20K of the 64K registers;
// the 512-thread kernel needs a whole SM's register file, so in the step it
// waits for an SM to drain completely).
__global__ void __launch_bounds__(256, 3)
k_pivot_lean(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase, const uint32_t* Vhat,
             const uint32_t* Rhat, long long row_stride_slot, int nslots, int p,
             IntBuf vint, long long vrow0, IntBuf piv, int* maxbitsV, uint32_t* vhat,
             int* maxdegV, int dmax_bits, uint32_t* Ybuf, int* ys, uint32_t* gscratch,
             int use_gscratch, int* err, PivotDiv pd) {
  pivot_body(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, p, vint, vrow0, piv, maxbitsV,
             vhat, maxdegV, dmax_bits, Ybuf, ys, gscratch, use_gscratch, err, pd);
}

// ------------------------------------------- ratios on the tensor cores ---
// The stage's bulk division R_p[r] = tdiv_q(V_p[r] 2^k2, V_p[p]) for many
// rows is one product of every |V_p[r]| with the stage's reciprocal Y, i.e. a
// limb convolution with a common operand: a GEMM.  In 7-bit digits
//   C[r][k'] = sum_i vdig[r][i] * T[k'][i],   T[k'][i] = ydig[K0d + k' - i],
// is column K0d + k' of |V_r| Y (products < 2^14, sums over <= 2^13 digits
// stay < 2^27: exact in int32), computed by an int8 x int8 -> int32 tensor
// core GEMM.  k_ratio_finish turns each row's columns back into limbs and
// applies ratio_quotient, so the results equal k_divide's bit for bit.
// K0d = ((sh - 59) / 7) rounded down to a multiple of 32 (7 K0d is a whole
// limb offset): the dropped columns sum to < 2^26.1 2^(7 K0d) <= 2^(sh-32),
// so F is lowered by < 2^-32 as in k_divide (there with V truncated; here V
// is whole, sh = S - k2).
__device__ __forceinline__ int ratio_k0d(int sh) {
  return sh < 59 ? 0 : ((sh - 59) / 7) & ~31;
}

// T[k'][i] (ncols x kd bytes, row k' contiguous) for the stage's Y.  One
// thread per 16 bytes.
__global__ void k_toeplitz(const uint32_t* Ybuf, const int* ys, int k2, int kd,
                           int ncols, uint8_t* T, const int* err) {
  extern __shared__ uint32_t ysm[];
  if (stage_aborted(err)) return;
  const int nY = ys[1];
  const int k0d = ratio_k0d(ys[0] - k2);
  for (int i = threadIdx.x; i < nY; i += blockDim.x) ysm[i] = Ybuf[i];
  __syncthreads();
  const int per_row = kd / 16;
  const long long total = (long long)ncols * per_row;
  const long long nyd = (32LL * nY + 6) / 7;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int kc = (int)(idx / per_row);
    const int i0 = (int)(idx - (long long)kc * per_row) * 16;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const long long j = (long long)k0d + kc - (i0 + u);
      if (j >= 0 && j < nyd) {
        const uint32_t d = field32(ysm, nY, 7 * j) & 127u;
        w[u >> 2] |= d << (8 * (u & 3));
      }
    }
    reinterpret_cast<uint4*>(T + (long long)kc * kd)[i0 / 16] =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Rows r in [r_begin, r_end) of stage p from the GEMM's columns
// C[(r - r_begin) * ncols + k'] (see above); same outputs as k_divide.
__global__ void k_ratio_finish(const __grid_constant__ DevPlan P, IntBuf vint, long long vrow0, int p,
                               int r_begin, int r_end, const uint32_t* Ybuf,
                               const int* ys, const int32_t* C, int ncols,
                               IntBuf rint, long long rrow0, uint32_t* rhat,
                               int* maxdegR, uint32_t* gscratch,
                               int use_gscratch, int* err) {
  extern __shared__ uint32_t sm_dyn[];
  if (stage_aborted(err)) return;
  const int cap = P.cap, ycap = P.ycap;
  const long long span = div_span_words(cap, ycap);
  const long long cta_words = span + div_extra_words(P);
  uint32_t* tab = sm_dyn;
  uint32_t* sm = use_gscratch ? gscratch + (long long)blockIdx.x * cta_words
                              : sm_dyn + (P.tw_smem ? P.NW : 0);
  const uint32_t* twm;
  stage_tables(P, tab, nullptr, &twm, nullptr);
  const int CY = (cap + ycap + 2 + 3) & ~3;
  uint32_t* Qt = sm;                 // cap + ycap: digits, then |q|
  uint32_t* Pr = sm + CY;            // CY: product top, windows, NTT
  uint32_t* col = Pr + CY;           // 3 CY: super-digits, then scratch
  uint32_t* red = col + 3 * CY;      // 64
  const long long pidx = vrow0 + p;
  const int S = ys[0], nY = ys[1], amax_used = ys[2];
  const int ybits = limbs_bits(Ybuf, nY);
  const int sh = S - P.k2;
  const int k0d = ratio_k0d(sh);
  const int shs = sh - 7 * k0d;
  const int J = ncols / 4;  // 28-bit super-digits
  const uint64_t m28 = (1ull << 28) - 1ull;
  for (int r = r_begin + blockIdx.x; r < r_end; r += gridDim.x) {
    const long long vidx = vrow0 + r;
    const int hd = vint.hdr[pidx];
    const int nD = hd < 0 ? -hd : hd;
    const int sD = hd < 0 ? -1 : (hd > 0);
    const uint32_t* Dg = vint.limbs + pidx * cap;
    const int hv = vint.hdr[vidx];
    const int na = hv < 0 ? -hv : hv;
    const int sV = hv < 0 ? -1 : (hv > 0);
    const uint32_t* Vg = vint.limbs + vidx * cap;
    const long long ridx = rrow0 + r;
    uint32_t* dst = rint.limbs + ridx * cap;
    int nq = 0;
    if (na > 0 && nD > 0) {
      const int vbits = limbs_bits(Vg, na);
      if (vbits + P.k2 > amax_used) {  // reciprocal too short for this row
        if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapAmax);
        return;
      }
      // every nonzero column of |V| Y lies below K0d + ncols
      if ((vbits + ybits + 6) / 7 + 1 > k0d + ncols) {
        if (threadIdx.x == 0) atomicOr(&err[kErrCapacity], kCapLimbs);
        return;
      }
      const int32_t* Cr = C + (long long)(r - r_begin) * ncols;
      uint64_t* Dsd = reinterpret_cast<uint64_t*>(col);
      for (int j = threadIdx.x; j < J; j += blockDim.x) {
        const int4 c4 = reinterpret_cast<const int4*>(Cr)[j];
        Dsd[j] = (uint64_t)(uint32_t)c4.x + ((uint64_t)(uint32_t)c4.y << 7) +
                 ((uint64_t)(uint32_t)c4.z << 14) + ((uint64_t)(uint32_t)c4.w << 21);
      }
      __syncthreads();
      const int carry = cta_resolve(
          J + 1, 28,
          [&](int j) -> int64_t {
            int64_t v = j < J ? (int64_t)(Dsd[j] & m28) : 0;
            if (j > 0) v += (int64_t)(Dsd[j - 1] >> 28);
            return v;
          },
          [&](int j, uint64_t d) { Qt[j] = (uint32_t)d; }, red);
      if (carry != 0) {
        if (threadIdx.x == 0) atomicOr(&err[kErrInternal], kIntDivision);
        return;
      }
      const int nPs = (28 * (J + 1) + 31) / 32;
      for (int m = threadIdx.x; m < nPs; m += blockDim.x) {
        uint64_t acc = 0;
        for (int k = (32 * m) / 28; k <= J && 28 * k < 32 * m + 32; ++k) {
          const int shl = 28 * k - 32 * m;
          acc |= shl >= 0 ? ((uint64_t)Qt[k] << shl) : ((uint64_t)Qt[k] >> -shl);
        }
        Pr[m] = (uint32_t)acc;
      }
      __syncthreads();
      nq = ratio_quotient(P, Pr, nPs, shs, Qt, col, red, CY, Vg, na, Dg, nD,
                          false, err);
      if (nq < 0) return;
    }
    const int rsign = nq == 0 ? 0 : sV * sD;
    for (int i = threadIdx.x; i < cap; i += blockDim.x)
      dst[i] = i < nq ? Qt[i] : 0u;
    if (threadIdx.x == 0) {
      rint.hdr[ridx] = rsign * nq;
      if (nq > 0 && maxdegR) atomicMax(maxdegR, (limbs_bits(Qt, nq) - 1) / P.w);
    }
    if (rhat) {
      uint32_t* X = P.NW <= 4 * CY ? Pr : sm + span;
      transform_int(P, Qt, nq, 0, rsign, X, rhat + ridx * (long long)P.NW,
                    true, twm, err);
    } else {
      __syncthreads();
    }
  }
}

// --------------------------------------------------------- trailing update -
// W[r][c] -= sum_{s} Vhat[s][c] * Rhat[s][r]   for c in [c_begin, c_end),
// r in [c, n), pointwise in the transform domain (ldlt.cpp:65-71, summed over
// the panel's stages: exact, so order-free).  One thread per transform word,
// a TILE x TILE (r,c) register tile, one 64-bit accumulator per pair for the
// whole panel (products < 2^56, <= 256 stages), one Montgomery reduction.
template <int TILE>
__global__ void __launch_bounds__(128)
k_update(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase,
         const uint32_t* Vhat, const uint32_t* Rhat, long long row_stride_slot,
         int nslots, int c_begin, int c_end, int nct, int nrt, const int* err) {
  if (stage_aborted(err)) return;
  // grid.x walks the (r,c) tiles, grid.y the word blocks: all tiles of one
  // word block run together, so the panel's operand slice for those words
  // (2 x kb x n x 128 words) stays L2-resident while every tile reuses it.
  const int wd = blockIdx.y * blockDim.x + threadIdx.x;
  if (wd >= P.NW) return;
  int t = blockIdx.x, ct = 0;
  while (t >= nrt - ct) {
    t -= nrt - ct;
    ++ct;
  }
  const int rt = ct + t;
  const int c0 = c_begin + ct * TILE;
  const int r0 = c_begin + rt * TILE;
  const PrimeConsts pc = P.pc[wd / P.L];
  const long long NW = P.NW;

  // out-of-range rows/columns are clamped to a valid one and never stored
  const uint32_t* rp[TILE];
  const uint32_t* vp[TILE];
#pragma unroll
  for (int i = 0; i < TILE; ++i) rp[i] = Rhat + (long long)min(r0 + i, P.n - 1) * NW + wd;
#pragma unroll
  for (int j = 0; j < TILE; ++j) vp[j] = Vhat + (long long)min(c0 + j, c_end - 1) * NW + wd;

  uint64_t acc[TILE][TILE];
#pragma unroll
  for (int i = 0; i < TILE; ++i)
#pragma unroll
    for (int j = 0; j < TILE; ++j) acc[i][j] = 0;

  uint32_t a[TILE], b[TILE];
#pragma unroll
  for (int i = 0; i < TILE; ++i) a[i] = __ldg(rp[i]);
#pragma unroll
  for (int j = 0; j < TILE; ++j) b[j] = __ldg(vp[j]);
  for (int s = 1; s <= nslots; ++s) {
    // prefetch the next stage while this one multiplies
    uint32_t an[TILE], bn[TILE];
    const long long off = (s < nslots ? s : s - 1) * row_stride_slot;
#pragma unroll
    for (int i = 0; i < TILE; ++i) an[i] = __ldg(rp[i] + off);
#pragma unroll
    for (int j = 0; j < TILE; ++j) bn[j] = __ldg(vp[j] + off);
#pragma unroll
    for (int i = 0; i < TILE; ++i)
#pragma unroll
      for (int j = 0; j < TILE; ++j) acc[i][j] += (uint64_t)a[i] * b[j];
#pragma unroll
    for (int i = 0; i < TILE; ++i) a[i] = an[i];
#pragma unroll
    for (int j = 0; j < TILE; ++j) b[j] = bn[j];
  }
#pragma unroll
  for (int j = 0; j < TILE; ++j) {
    const int c = c0 + j;
    if (c >= c_end) continue;
    const long long base = colbase[c];
#pragma unroll
    for (int i = 0; i < TILE; ++i) {
      const int r = r0 + i;
      if (r < c || r >= P.n) continue;
      uint32_t* ptr = W + (base + (r - c)) * NW + wd;
      const uint32_t t32 = reduce_sum64(acc[i][j], pc);
      const uint32_t old = *ptr;
      *ptr = old >= t32 ? old - t32 : old + pc.q - t32;
    }
  }
}

// ------------------------------------------------ trailing update (SMEM) --
// Same contract as k_update.  A CTA (4 warps) owns a 16 x 16 (r,c) tile and
// 32 consecutive transform words; warp w computes the 8 x 8 sub-tile
// (w>>1, w&1), lane = word.  Each stage's operands -- 16 rows of Rhat and 16
// columns of Vhat, 32 words each (4 KB) -- are staged into shared memory by
// cp.async through a kStages-deep pipeline, so the L2 latency hides behind
// the 64 IMAD.WIDE of the stages in flight and every operand word fetched
// from L2 feeds 16 products (0.5 B/product).
namespace {
constexpr int kUT = 16;        // CTA tile edge
#ifndef HGPU_USTAGES
#define HGPU_USTAGES 4
#endif
constexpr int kUStages = HGPU_USTAGES;    // cp.async pipeline depth
constexpr int kUWords = 32;    // words per CTA

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
}  // namespace

#ifdef HGPU_UPD_MAXREG  // experiment: leave register headroom beside three update CTAs
__global__ void __maxnreg__(HGPU_UPD_MAXREG)
#else
__global__ void __launch_bounds__(128, 2)
#endif
k_update_tiled(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase,
               const uint32_t* Vhat, const uint32_t* Rhat,
               long long row_stride_slot, int nslots, int c_begin, int c_end,
               int nct, int nrt, const int* err, int r_lo, int r_hi, int rect) {
  __shared__ __align__(16) uint32_t sm[kUStages][2 * kUT][kUWords];
  // the tile's own workspace words, prefetched at entry so the epilogue's
  // read-modify-write never waits on HBM
  extern __shared__ __align__(16) uint32_t sW[];  // [kUT*kUT][kUWords]
  if (stage_aborted(err)) return;
  const int w0 = blockIdx.y * kUWords;
  // tiles: the lower triangle r >= c of columns [c_begin, c_end) (rows from
  // r_lo = c_begin), or (rect) the rectangle [r_lo, r_hi) x [c_begin, c_end)
  int t = blockIdx.x, ct = 0, rt;
  if (rect) {
    ct = t / nrt;
    rt = t - ct * nrt;
  } else {
    while (t >= nrt - ct) {
      t -= nrt - ct;
      ++ct;
    }
    rt = ct + t;
  }
  const int c0 = c_begin + ct * kUT;
  const int r0 = r_lo + rt * kUT;
  const long long NW = P.NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // loader: 32 operand rows x 8 chunks of 16 B = 256 chunks, 2 per thread
  const uint32_t* src[2];
  int dst_k[2], dst_w[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int chunk = tid + 128 * h;
    const int k = chunk >> 3, part = chunk & 7;
    const uint32_t* base;
    if (k < kUT) base = Rhat + (long long)min(r0 + k, r_hi - 1) * NW;
    else base = Vhat + (long long)min(c0 + k - kUT, c_end - 1) * NW;
    src[h] = base + w0 + part * 4;
    dst_k[h] = k;
    dst_w[h] = part * 4;
  }
  auto issue = [&](int s) {
    const int buf = s % kUStages;
    const long long off = s * row_stride_slot;
#pragma unroll
    for (int h = 0; h < 2; ++h) cp_async16(&sm[buf][dst_k[h]][dst_w[h]], src[h] + off);
  };
  // W tile prefetch: 256 pairs x 8 chunks of 16 B, 16 per thread, committed
  // with the first operand stage
#ifndef HGPU_UPD_NOPREFETCH
#pragma unroll 4
  for (int h = 0; h < (kUT * kUT * 8) / 128; ++h) {
    const int chunk = tid + 128 * h;
    const int pair = chunk >> 3, part = chunk & 7;
    const int r = r0 + (pair >> 4), c = c0 + (pair & 15);
    if (c < c_end && r >= c && r < r_hi)
      cp_async16(&sW[pair * kUWords + part * 4],
                 W + (colbase[c] + (r - c)) * NW + w0 + part * 4);
  }
#endif
#pragma unroll
  for (int s = 0; s < kUStages - 1; ++s) {
    if (s < nslots) issue(s);
    cp_async_commit();
  }

  const int rm = (warp >> 1) * 8, cm = (warp & 1) * 8;
  uint64_t acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0;

  for (int s = 0; s < nslots; ++s) {
    if (s + kUStages - 1 < nslots) issue(s + kUStages - 1);
    cp_async_commit();
    cp_async_wait<kUStages - 1>();
    __syncthreads();
    const int buf = s % kUStages;
    uint32_t a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = sm[buf][rm + i][lane];
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = sm[buf][kUT + cm + j][lane];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] += (uint64_t)a[i] * b[j];
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();

  const int wd = w0 + lane;
  if (wd >= P.NW) return;
  const PrimeConsts pc = P.pc[wd / P.L];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + cm + j;
    if (c >= c_end) continue;
    const long long base = colbase[c];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + rm + i;
      if (r < c || r >= r_hi) continue;
      const uint32_t t32 = reduce_sum64(acc[i][j], pc);
#ifndef HGPU_UPD_NOPREFETCH
      const uint32_t old = sW[((rm + i) * kUT + cm + j) * kUWords + lane];
#else
      const uint32_t old = W[(base + (r - c)) * NW + wd];
#endif
      W[(base + (r - c)) * NW + wd] = old >= t32 ? old - t32 : old + pc.q - t32;
    }
  }
}

// -------------------------------------------------------- column update ---
// In-panel, left-looking: right before column c is extracted it receives
// every earlier stage of its panel at once,
//   W[r][c] -= sum_{s < ns} Vhat[s][c] * Rhat[s][r],   r in [c, n),
// so each entry of the panel is read-modify-written once per column instead
// of once per stage.  Thread: one word x TR rows.
template <int TR>
__global__ void __launch_bounds__(128)
k_update_col(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase,
             const uint32_t* Vhat, const uint32_t* Rhat,
             long long row_stride_slot, int nslots, int c, int r_begin,
             int r_end, const int* err) {
  if (stage_aborted(err)) return;
  const int wd = blockIdx.y * blockDim.x + threadIdx.x;
  if (wd >= P.NW) return;
  const int r0 = r_begin + blockIdx.x * TR;
  const PrimeConsts pc = P.pc[wd / P.L];
  const long long NW = P.NW;
  // rows r0 .. r0 + TR - 1 (consecutive: one base pointer; rows past r_end
  // read the last valid row and are not written)
  const int nv = min(TR, r_end - r0);
  const uint32_t* rp = Rhat + (long long)r0 * NW + wd;
  const uint32_t* vp = Vhat + (long long)c * NW + wd;
  uint64_t acc[TR];
#pragma unroll
  for (int i = 0; i < TR; ++i) acc[i] = 0;
  // the stage loop is unrolled so that the loads of several stages are in
  // flight together: the kernel is bound by L2 latency (one dependent round
  // trip per stage otherwise), and in the step that latency is several times
  // what it is alone
#ifndef HGPU_COL_UNROLL
#define HGPU_COL_UNROLL 4
#endif
  constexpr int kColUnroll = HGPU_COL_UNROLL;
#pragma unroll kColUnroll
  for (int s = 0; s < nslots; ++s) {
    const long long off = s * row_stride_slot;
    const uint32_t b = __ldg(vp + off);
    uint32_t a[TR];
#pragma unroll
    for (int i = 0; i < TR; ++i) a[i] = __ldg(rp + off + (long long)min(i, nv - 1) * NW);
#pragma unroll
    for (int i = 0; i < TR; ++i) acc[i] += (uint64_t)a[i] * b;
  }
  uint32_t* wp = W + (colbase[c] + (r0 - c)) * NW + wd;
  uint32_t old[TR];
#pragma unroll
  for (int i = 0; i < TR; ++i) old[i] = i < nv ? wp[(long long)i * NW] : 0u;
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    if (i >= nv) continue;
    const uint32_t t32 = reduce_sum64(acc[i], pc);
    wp[(long long)i * NW] = old[i] >= t32 ? old[i] - t32 : old[i] + pc.q - t32;
  }
}

// -------------------------------------------------------------- validate ---
// Checks the transform capacity after the factorisation: for every stage
// deg V + deg R < L (no cyclic wrap) and the accumulated coefficient bound
// sum_p (min(degV,degR)+1)(2^w-1)^2 + 2^(w+1) < Q/2 (exact CRT).
__global__ void k_validate(const __grid_constant__ DevPlan P, const int* maxdegV, const int* maxdegR,
                           int nstages, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long double dig = (long double)((1ull << P.w) - 1ull);
  long double bound = 2.0L * (dig + 1.0L);
  const long double dig2 = dig * dig;
  for (int p = 0; p < nstages; ++p) {
    const int dv = maxdegV[p], dr = maxdegR[p];
    if (dv < 0 || dr < 0) continue;
    if (dv + dr >= P.L) atomicOr(&err[kErrCapacity], kCapDegree);
    bound += (long double)(min(dv, dr) + 1) * dig2;
  }
  const long double half =
      (long double)P.Hhi * 18446744073709551616.0L + (long double)P.Hlo;
  if (bound >= half * 0.5L) atomicOr(&err[kErrCapacity], kCapCoeff);
}

// ------------------------------------------------------ launch wrappers --

static thread_local long long g_launches = 0;
long long kernel_launch_count() { return g_launches; }
long long kernel_launch_count_add(long long k) { return g_launches += k; }

// HGPU_SYNC_DEBUG=1: synchronise after every launch so a fault is reported
// by the launch that caused it (debug aid; off by default).
static cudaError_t post_launch(cudaStream_t st) {
  static const bool sync_debug = [] {
    const char* e = getenv("HGPU_SYNC_DEBUG");
    return e && *e == '1';
  }();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_debug) e = cudaStreamSynchronize(st);
  return e;
}

cudaError_t launch_fwd_ints(const DevPlan& P, IntBuf src, long long in_base,
                            uint32_t* out, long long out_base, int count,
                            int mont, int* maxdeg, int* err,
                            cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = (size_t)((P.tw_smem ? P.NW : 0) + P.NW + P.cap) * 4;
  ++g_launches;
  k_fwd_ints<<<min(count, P.grid_cap), 256, smem, st>>>(
      P, src, in_base, out, out_base, count, mont, maxdeg, err);
  return post_launch(st);
}

cudaError_t launch_init_w(const DevPlan& P, const uint32_t* that,
                          const uint32_t* xhat, const long long* colbase,
                          uint32_t* W, cudaStream_t st) {
  ++g_launches;
  if (P.NW % 4 == 0 && P.L % 4 == 0) {
    dim3 grid((P.NW / 4 + 255) / 256, P.n, 4);
    k_init_w4<<<grid, 256, 0, st>>>(P, that, xhat, colbase, W);
    return post_launch(st);
  }
  dim3 grid((P.NW + 255) / 256, P.n);
  k_init_w<<<grid, 256, 0, st>>>(P, that, xhat, colbase, W);
  return post_launch(st);
}

// threads of a multi-row extraction / division CTA (HGPU_ROW_THREADS: 128 or
// 256; experiment)
static int row_threads() {
  static const int v = [] {
    const char* e = getenv("HGPU_ROW_THREADS");
    const int t = e ? atoi(e) : 256;
    return t == 128 ? 128 : 256;
  }();
  return v;
}

size_t extract_smem_bytes(const DevPlan& P, bool staged) {
  const int M = P.L + P.T;
  return (size_t)((P.tw_smem && staged ? 2 * P.NW : 0) + P.NW + 4 * M + P.cap + 64) * 4;
}

cudaError_t launch_extract(const DevPlan& P, const uint32_t* W,
                           const long long* colbase, int p, int r_begin,
                           int r_end, IntBuf vint, long long vrow0, IntBuf piv,
                           int* maxbitsV, uint32_t* vhat, int* maxdegV,
                           int* err, cudaStream_t st, int round,
                           uint8_t* vdig, int kd) {
  const int rows = r_end - r_begin;
  if (rows <= 0) return cudaSuccess;
  ++g_launches;
  // a single row is on the pivot chain: give it more threads; one row per
  // CTA needs no twiddle tables in shared memory
  k_extract<<<min(rows, P.grid_cap), rows == 1 ? 512 : row_threads(),
              extract_smem_bytes(P, rows > P.grid_cap), st>>>(
      P, W, colbase, p, r_begin, r_end, vint, vrow0, piv, maxbitsV, vhat,
      maxdegV, err, round, vdig, kd);
  return post_launch(st);
}

static int recip_threads() {
  static const int t = [] {
    const char* e = getenv("HGPU_RECIP_THREADS");
    const int v = e ? atoi(e) : 512;
    return (v >= 32 && v <= 512 && v % 32 == 0) ? v : 512;
  }();
  return t;
}

long long recip_words_bound(const DevPlan& P, int dmax_bits, int segs) {
  // e <= (dmax - k2)/2 + k2 + 6 (the pivot has more than k2 bits), Pt = e + 32
  const long long e = (long long)(dmax_bits - P.k2) / 2 + P.k2 + 6;
  const long long Lm = (e + 32 + 32 + 31) / 32 + 2;
  return 10 * Lm + 71 + (long long)segs * (3 * Lm + 2) + 8;
}

long long recip_fast_words_bound(const DevPlan& P, int dmax_bits) {
  const long long e = (long long)(dmax_bits - P.k2) / 2 + P.k2 + 6;
  const long long Lm = (e + 32 + 32 + 31) / 32 + 2;
  return rf_scratch_words((int)Lm);
}

// recip_body's scratch at the reciprocal capacity ycap (+ guard limbs)
static size_t recip_body_words(const DevPlan& P) {
  const size_t Lm = (size_t)P.ycap + 4;
  return (Lm + 2) + Lm + Lm + (2 * Lm + 1) + (2 * Lm + 2) + (3 * Lm + 2) + 6 * (3 * Lm + 2) + 64;
}

// Global scratch for either body at ycap.  The fast body needs ~35 words per
// limb of the stage's actual precision (Lm, usually far below ycap): in
// shared memory it runs whenever the launch's dynamic shared memory holds
// that, and otherwise the stage uses recip_body (recip_fast_body checks).
size_t recip_scratch_words(const DevPlan& P) {
  return std::max(recip_body_words(P), (size_t)rf_scratch_words(P.ycap + 4));
}

// the dynamic shared memory k_pivot / k_recip may take: the opt-in limit per
// block less their static shared memory (set by configure_kernels)
static size_t g_pivot_dyn = 0, g_recip_dyn = 0;

cudaError_t launch_recip(const DevPlan& P, IntBuf vint, long long prow,
                         const int* maxbitsV, int p, IntBuf piv, int dmax_bits,
                         uint32_t* Ybuf, int* ys, uint32_t* scratch,
                         int use_gscratch, int* err, cudaStream_t st) {
  ++g_launches;
  const size_t smem =
      use_gscratch ? 0 : std::min(recip_scratch_words(P) * 4, std::max(g_recip_dyn, recip_body_words(P) * 4));
  k_recip<<<1, recip_threads(), smem, st>>>(P, vint, prow, maxbitsV, p, piv,
                                            dmax_bits, Ybuf, ys, scratch,
                                            use_gscratch, err);
  return post_launch(st);
}

cudaError_t launch_pivot(const DevPlan& P, uint32_t* W, const long long* colbase,
                         const uint32_t* Vhat, const uint32_t* Rhat,
                         long long row_stride_slot, int nslots, int p,
                         IntBuf vint, long long vrow0, IntBuf piv, int* maxbitsV,
                         uint32_t* vhat, int* maxdegV, int dmax_bits,
                         uint32_t* Ybuf, int* ys, uint32_t* scratch,
                         int use_gscratch, int* err, cudaStream_t st,
                         const PivotDiv& pd) {
  ++g_launches;
  size_t smem = std::max(extract_smem_bytes(P, true),
                         use_gscratch ? (size_t)0 : (size_t)pd.recip_words * 4);
  if (pd.on)
    smem = std::max(smem, pd.use_dscr ? (size_t)(P.tw_smem ? P.NW : 0) * 4
                                      : divide_smem_words(P) * 4);
  static const int threads = [] {
    const char* e = getenv("HGPU_PIVOT_THREADS");
    const int v = e ? atoi(e) : 512;
    return (v >= 128 && v <= 512 && v % 32 == 0) ? v : 512;
  }();
  // k_pivot fills a whole SM's register file, so it always runs alone on its
  // SM: give it all the shared memory the SM has, so the fast reciprocal
  // runs at any precision that fits (the bound from dmax is far too loose
  // for the small pivots of these matrices).
  PivotDiv q = pd;
  if (threads != 256 && !use_gscratch && g_pivot_dyn > smem) {
    smem = g_pivot_dyn;
    q.recip_words = std::min<long long>((long long)recip_scratch_words(P), (long long)(smem / 4));
  }
  if (threads == 256)
    k_pivot_lean<<<1, 256, smem, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots,
                                       p, vint, vrow0, piv, maxbitsV, vhat, maxdegV,
                                       dmax_bits, Ybuf, ys, scratch, use_gscratch, err, q);
  else
    k_pivot<<<1, threads, smem, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots,
                                  p, vint, vrow0, piv, maxbitsV, vhat, maxdegV,
                                  dmax_bits, Ybuf, ys, scratch, use_gscratch, err, q);
  return post_launch(st);
}

cudaError_t launch_recip_batch(const DevPlan& P, IntBuf vint, long long prow,
                               const int* maxbitsV, uint32_t* Ybuf, int* ys,
                               uint32_t* scratch, int batch, int* err,
                               cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  ++g_launches;
  k_recip<<<dim3(1, batch), recip_threads(), 0, st>>>(
      P, vint, prow, maxbitsV, 0, IntBuf{nullptr, nullptr}, 0, Ybuf, ys,
      scratch, 1, err);
  return post_launch(st);
}

cudaError_t launch_divide_batch(const DevPlan& P, IntBuf vint,
                                long long vrow0, const uint32_t* Ybuf,
                                const int* ys, IntBuf rint, long long rrow0,
                                uint32_t* gscratch, int batch, int* err,
                                cudaStream_t st) {
  if (batch <= 0 || P.n - 1 <= 0) return cudaSuccess;
  ++g_launches;
  k_divide<<<dim3(min(P.n - 1, P.grid_cap), batch), 256,
             (size_t)(P.tw_smem ? P.NW : 0) * 4, st>>>(
      P, vint, vrow0, 0, 1, 2, Ybuf, ys, rint, rrow0, nullptr, nullptr,
      gscratch, 1, err, IvDiv{});
  return post_launch(st);
}

size_t divide_smem_words(const DevPlan& P) {
  return (size_t)(P.tw_smem ? P.NW : 0) + div_span_words(P.cap, P.ycap) +
         div_extra_words(P);
}

cudaError_t launch_divide(const DevPlan& P, IntBuf vint, long long vrow0,
                          int p, int r_begin, int r_end, const uint32_t* Ybuf,
                          const int* ys, IntBuf rint, long long rrow0,
                          uint32_t* rhat, int* maxdegR, uint32_t* gscratch,
                          int use_gscratch, int* err, cudaStream_t st,
                          const IvDiv* iv) {
  r_begin = max(r_begin, p + 1);
  r_end = min(r_end, P.n);
  const int rows = r_end - r_begin;
  if (rows <= 0) return cudaSuccess;
  // one row per CTA: no twiddle table in shared memory
  const size_t tw = rows <= P.grid_cap && P.tw_smem ? (size_t)P.NW * 4 : 0;
  const size_t smem = (use_gscratch ? (size_t)(P.tw_smem ? P.NW : 0) * 4
                                    : divide_smem_words(P) * 4) - tw;
  ++g_launches;
  if (rows == 1)
    k_divide1<<<1, 512, smem, st>>>(P, vint, vrow0, p, r_begin, r_end, Ybuf, ys, rint, rrow0,
                                    rhat, maxdegR, gscratch, use_gscratch, err,
                                    iv ? *iv : IvDiv{});
  else
    k_divide<<<min(rows, P.grid_cap), row_threads(), smem, st>>>(
        P, vint, vrow0, p, r_begin, r_end, Ybuf, ys, rint, rrow0, rhat, maxdegR,
        gscratch, use_gscratch, err, iv ? *iv : IvDiv{});
  return post_launch(st);
}

cudaError_t launch_toeplitz(const DevPlan& P, const uint32_t* Ybuf,
                            const int* ys, int kd, int ncols, uint8_t* T,
                            const int* err, cudaStream_t st) {
  ++g_launches;
  const long long words = (long long)ncols * (kd / 16);
  const int blocks = (int)std::min<long long>((words + 255) / 256, 4096);
  k_toeplitz<<<blocks, 256, (size_t)P.ycap * 4, st>>>(Ybuf, ys, P.k2, kd, ncols,
                                                      T, err);
  return post_launch(st);
}

cudaError_t launch_ratio_finish(const DevPlan& P, IntBuf vint, long long vrow0,
                                int p, int r_begin, int r_end,
                                const uint32_t* Ybuf, const int* ys,
                                const int32_t* C, int ncols, IntBuf rint,
                                long long rrow0, uint32_t* rhat, int* maxdegR,
                                uint32_t* gscratch, int use_gscratch, int* err,
                                cudaStream_t st) {
  const int rows = r_end - r_begin;
  if (rows <= 0) return cudaSuccess;
  const size_t smem = use_gscratch ? (size_t)(P.tw_smem ? P.NW : 0) * 4
                                   : divide_smem_words(P) * 4;
  ++g_launches;
  k_ratio_finish<<<min(rows, P.grid_cap), 256, smem, st>>>(
      P, vint, vrow0, p, r_begin, r_end, Ybuf, ys, C, ncols, rint, rrow0, rhat,
      maxdegR, gscratch, use_gscratch, err);
  return post_launch(st);
}

// HGPU_UPD_PAD (bytes): dynamic shared memory requested per k_update_tiled
// CTA (at least its 32 KB tile); ~76 KB holds the update to two CTAs per SM,
// leaving every SM a slot for the panel's single-row kernels (experiment)
static size_t upd_smem() {
  static const size_t v = [] {
    const char* e = getenv("HGPU_UPD_PAD");
#ifndef HGPU_UPD_NOPREFETCH
    const size_t base = (size_t)kUT * kUT * kUWords * 4;
#else
    const size_t base = 0;
#endif
    return e ? std::max(base, (size_t)atol(e)) : base;
  }();
  return v;
}

cudaError_t launch_update(const DevPlan& P, int tile, uint32_t* W,
                          const long long* colbase, const uint32_t* Vhat,
                          const uint32_t* Rhat, long long row_stride_slot,
                          int nslots, int c_begin, int c_end, const int* err,
                          cudaStream_t st, int r_hi) {
  if (c_begin >= c_end || nslots <= 0) return cudaSuccess;
  if (r_hi >= 0 && !(tile == 16 && P.NW % kUWords == 0)) return cudaErrorInvalidValue;
  if (tile == 16 && P.NW % kUWords == 0) {
    const int rows_end = r_hi >= 0 ? min(r_hi, P.n) : P.n;
    if (rows_end <= c_begin) return cudaSuccess;
    const int nct = (c_end - c_begin + kUT - 1) / kUT;
    const int nrt = (rows_end - c_begin + kUT - 1) / kUT;
    long long tiles = 0;
    if (nrt < nct) return cudaErrorInvalidValue;  // (the kernel's tile walk)
    for (int ct = 0; ct < nct; ++ct) tiles += nrt - ct;
    dim3 grid((unsigned)tiles, P.NW / kUWords);
    ++g_launches;
    k_update_tiled<<<grid, 128, upd_smem(), st>>>(P, W, colbase, Vhat, Rhat,
                                         row_stride_slot, nslots, c_begin,
                                         c_end, nct, nrt, err, c_begin, rows_end, 0);
    return cudaGetLastError();
  }
  if (tile == 16) tile = 8;
  const int nct = (c_end - c_begin + tile - 1) / tile;
  const int nrt = (P.n - c_begin + tile - 1) / tile;
  long long tiles = 0;
  for (int ct = 0; ct < nct; ++ct) tiles += nrt - ct;
  dim3 grid((unsigned)tiles, (P.NW + 127) / 128);
  ++g_launches;
  if (tile == 8)
    k_update<8><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat,
                                      row_stride_slot, nslots, c_begin, c_end,
                                      nct, nrt, err);
  else
    k_update<4><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat,
                                      row_stride_slot, nslots, c_begin, c_end,
                                      nct, nrt, err);
  return post_launch(st);
}

cudaError_t launch_update_rect(const DevPlan& P, uint32_t* W,
                               const long long* colbase, const uint32_t* Vhat,
                               const uint32_t* Rhat, long long row_stride_slot,
                               int nslots, int c_begin, int c_end, int r_lo,
                               int r_hi, const int* err, cudaStream_t st) {
  if (c_begin >= c_end || r_lo >= r_hi || nslots <= 0) return cudaSuccess;
  if (P.NW % kUWords != 0 || r_lo < c_end) return cudaErrorInvalidValue;
  const int nct = (c_end - c_begin + kUT - 1) / kUT;
  const int nrt = (r_hi - r_lo + kUT - 1) / kUT;
  dim3 grid((unsigned)(nct * nrt), P.NW / kUWords);
  ++g_launches;
  k_update_tiled<<<grid, 128, upd_smem(), st>>>(
      P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c_begin, c_end, nct, nrt,
      err, r_lo, r_hi, 1);
  return post_launch(st);
}

cudaError_t launch_col_extract(const DevPlan& P, uint32_t* W, const long long* colbase,
                               const uint32_t* Vhat, const uint32_t* Rhat,
                               long long row_stride_slot, int nslots, int p, int r_begin,
                               int r_end, IntBuf vint, long long vrow0, IntBuf piv,
                               int* maxbitsV, uint32_t* vhat, int* maxdegV, int* err,
                               cudaStream_t st, uint8_t* vdig, int kd) {
  const int rows = r_end - r_begin;
  if (rows <= 0) return cudaSuccess;
  ++g_launches;
  k_col_extract<<<min(rows, P.grid_cap), 256, extract_smem_bytes(P, false), st>>>(
      P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, p, r_begin, r_end, vint, vrow0, piv,
      maxbitsV, vhat, maxdegV, err, vdig, kd);
  return post_launch(st);
}

cudaError_t launch_update_col(const DevPlan& P, uint32_t* W,
                              const long long* colbase, const uint32_t* Vhat,
                              const uint32_t* Rhat, long long row_stride_slot,
                              int nslots, int c, int r_begin, int r_end,
                              const int* err, cudaStream_t st) {
  if (nslots <= 0 || r_begin >= r_end) return cudaSuccess;
  // rows per thread (HGPU_COL_TR: 2, 4, 8 or 16).  4 (40 registers: many
  // small CTAs that fit beside the trailing update's) measured best in the
  // step: 241.7 ms against 249.4 / 246.8 for 8 / 16 at config 3
  static const int tr = [] {
    const char* e = getenv("HGPU_COL_TR");
    const int v = e ? atoi(e) : 4;
    return (v == 2 || v == 8 || v == 16) ? v : 4;
  }();
  // threads per CTA (HGPU_COL_THREADS: 64 or 128)
  static const int ct = [] {
    const char* e = getenv("HGPU_COL_THREADS");
    return (e && atoi(e) == 64) ? 64 : 128;
  }();
  dim3 grid((r_end - r_begin + tr - 1) / tr, (P.NW + ct - 1) / ct);
  ++g_launches;
  if (ct == 64 && tr == 4) {
    k_update_col<4><<<grid, 64, 0, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c,
                                         r_begin, r_end, err);
    return post_launch(st);
  }
  if (tr == 2)
    k_update_col<2><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c,
                                          r_begin, r_end, err);
  else if (tr == 4)
    k_update_col<4><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c,
                                          r_begin, r_end, err);
  else if (tr == 8)
    k_update_col<8><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c,
                                          r_begin, r_end, err);
  else
    k_update_col<16><<<grid, 128, 0, st>>>(P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c,
                                           r_begin, r_end, err);
  return post_launch(st);
}

cudaError_t launch_validate(const DevPlan& P, const int* maxdegV,
                            const int* maxdegR, int nstages, int* err,
                            cudaStream_t st) {
  ++g_launches;
  k_validate<<<1, 32, 0, st>>>(P, maxdegV, maxdegR, nstages, err);
  return post_launch(st);
}

cudaError_t configure_kernels(const DevPlan& P, size_t* div_smem,
                              bool* div_global, bool* recip_global) {
  int dev;
  cudaGetDevice(&dev);
  int maxopt = 0;
  cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t ext = extract_smem_bytes(P, true);
  const size_t fwd = (size_t)((P.tw_smem ? P.NW : 0) + P.NW + P.cap) * 4;
  if ((int)ext > maxopt || (int)fwd > maxopt) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_extract,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ext)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_fwd_ints,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fwd)) != cudaSuccess)
    return e;
    if ((e = cudaFuncSetAttribute(k_col_extract,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ext)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_fwd_ints,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fwd)) != cudaSuccess)
    return e;
  auto dyn_cap = [&](const void* f) -> size_t {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 0;
    return (size_t)maxopt > fa.sharedSizeBytes ? (size_t)maxopt - fa.sharedSizeBytes : 0;
  };
  if ((e = cudaFuncSetAttribute(k_update_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::min(upd_smem(), dyn_cap((const void*)k_update_tiled)))) !=
      cudaSuccess)
    return e;
  g_pivot_dyn = std::min(dyn_cap((const void*)k_pivot), dyn_cap((const void*)k_pivot_lean));
  g_recip_dyn = dyn_cap((const void*)k_recip);
  const size_t rec = recip_body_words(P) * 4;
  {
    if ((e = cudaFuncSetAttribute(k_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)g_pivot_dyn)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(k_pivot_lean, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)g_pivot_dyn)) != cudaSuccess)
      return e;
  }
  // the reciprocal CTA runs beside the bulk kernels; shared-memory scratch
  // is faster even at ~190 KB (measured at config 3: 421 -> 405 ms per
  // factorisation), so it is used whenever it fits.  HGPU_RECIP_SMEM=0
  // keeps the scratch in global memory (L1/L2-resident) instead.
  const char* rg = getenv("HGPU_RECIP_SMEM");
  const bool want_smem = rg ? *rg == '1' : true;
  *recip_global = rec > std::min(g_recip_dyn, g_pivot_dyn) || !want_smem;
  if (!*recip_global) {
    if ((e = cudaFuncSetAttribute(k_recip,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)g_recip_dyn)) != cudaSuccess)
      return e;
  }
  const size_t div = divide_smem_words(P) * 4;
  *div_smem = div;
  *div_global = (int)div > maxopt;
  if (*div_global) {
    const int tab = (P.tw_smem ? P.NW : 0) * 4;
    if ((e = cudaFuncSetAttribute(k_divide,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  tab)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(k_divide1,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  tab)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(k_ratio_finish,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  tab)) != cudaSuccess)
      return e;
  } else {
    if ((e = cudaFuncSetAttribute(k_divide,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)div)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(k_divide1,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)div)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(k_ratio_finish,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)div)) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

}  // namespace hgpu
