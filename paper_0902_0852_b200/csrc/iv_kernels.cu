// Interval LDL^T kernels (ldlt_det_interval, ldlt.cpp:79-152).
// Each workspace entry is an interval [lo, hi] kept as two transforms; the
// column values and ratios are interval bounds with directed rounding
// (k_extract round 1/2, k_divide IvDiv).  The update subtracts the interval
// product: W.lo -= max corner, W.hi -= min corner (ldlt.cpp:136-148).  In the
// transform domain a corner cannot be compared, but which corner is extreme
// follows from the signs of the two intervals alone, unless both straddle
// zero: that case is flagged (kCapStraddle) instead of guessed.
#include <cstdint>

#include "cta_ops.cuh"
#include "ldlt_kernels.cuh"

namespace hgpu {

namespace {

// class of an interval bound pair: +1 lo > 0, -1 hi < 0, 0 contains zero
__device__ __forceinline__ int iv_class(int hlo, int hhi) {
  return hlo > 0 ? 1 : (hhi < 0 ? -1 : 0);
}

// Corner selection for the max and min of [v.lo,v.hi] x [r.lo,r.hi] given
// the classes cv, cr (not both 0).  Bit 0: use v.hi; bit 1: use r.hi.
//   max: v.hi iff cr > 0 or (cr == 0 and cv > 0); r.hi iff cv > 0 or (cv == 0 and cr > 0)
//   min: v.hi iff cr < 0 or (cr == 0 and cv > 0); r.hi iff cv < 0 or (cv == 0 and cr > 0)
__device__ __forceinline__ int sel_max(int cv, int cr) {
  const int vh = (cr > 0 || (cr == 0 && cv > 0)) ? 1 : 0;
  const int rh = (cv > 0 || (cv == 0 && cr > 0)) ? 2 : 0;
  return vh | rh;
}
__device__ __forceinline__ int sel_min(int cv, int cr) {
  const int vh = (cr < 0 || (cr == 0 && cv > 0)) ? 1 : 0;
  const int rh = (cv < 0 || (cv == 0 && cr > 0)) ? 2 : 0;
  return vh | rh;
}

}  // namespace

// Classes of rows [r_begin, r_end) of one slot row block (V or R bounds);
// the pivot row p (when check_pivot) must be sign-definite for p < n-1
// (ldlt.cpp:110-111: ZeroPivot).
__global__ void k_iv_classify(IntBuf lo, IntBuf hi, long long row0, int r_begin,
                              int r_end, int8_t* cls, int p, int check_pivot,
                              int n, int* err, int* nonpos) {
  for (int r = r_begin + blockIdx.x * blockDim.x + threadIdx.x; r < r_end;
       r += gridDim.x * blockDim.x) {
    const int c = iv_class(lo.hdr[row0 + r], hi.hdr[row0 + r]);
    cls[row0 + r] = (int8_t)c;
    if (c <= 0 && nonpos) atomicOr(nonpos, 1);
    if (check_pivot && r == p && c == 0 && p < n - 1)
      atomicMin(&err[kErrZeroPivot], p);
  }
}

// W.lo[r][c] -= sum_s max corner, W.hi[r][c] -= sum_s min corner, for the
// stages s in [s_begin, s_end) of a slot set, columns c in [c_begin, c_end),
// rows r in [max(c, r_min), n).  Vlo/Vhi/Rlo/Rhi: slot-set transforms (R in
// Montgomery form), entry (s, r) at ((s*n) + r)*NW; clsV/clsR likewise per
// (s, r).  grid.x: (column tile, row tile) pairs, grid.y: blocks of 128
// transform words; each thread one word of a 4x4 (r, c) tile.
constexpr int kIvT = 4;
__global__ void __launch_bounds__(128)
k_update_iv(const __grid_constant__ DevPlan P, uint32_t* Wlo, uint32_t* Whi, const long long* colbase,
            const uint32_t* Vlo, const uint32_t* Vhi, const uint32_t* Rlo,
            const uint32_t* Rhi, const int8_t* clsV, const int8_t* clsR,
            int s_begin, int s_end, int c_begin, int c_end, int r_min,
            int nrt, const int* gate, int* err) {
  if (*(volatile const int*)&err[kErrZeroPivot] != INT_MAX ||
      *(volatile const int*)&err[kErrCapacity] != 0)
    return;
  // all-positive panels take the tiled point kernels instead (iv_engine.cpp)
  if (gate && *(volatile const int*)gate == 0) return;
  const int wd = blockIdx.y * blockDim.x + threadIdx.x;
  if (wd >= P.NW) return;
  const int n = P.n;
  const int ct = blockIdx.x / nrt, rt = blockIdx.x % nrt;
  const int c0 = c_begin + ct * kIvT;
  const int rbase = max(c_begin, r_min);
  const int r0 = rbase + rt * kIvT;
  if (c0 >= c_end || r0 >= n || r0 + kIvT - 1 < c0) return;  // above diagonal
  const long long NW = P.NW;
  const PrimeConsts pc = P.pc[wd / P.L];
  uint64_t alo[kIvT][kIvT], ahi[kIvT][kIvT];
#pragma unroll
  for (int i = 0; i < kIvT; ++i)
#pragma unroll
    for (int j = 0; j < kIvT; ++j) alo[i][j] = ahi[i][j] = 0;
  bool straddle = false;
  for (int s = s_begin; s < s_end; ++s) {
    const long long sb = (long long)s * n;
    uint32_t vl[kIvT], vh[kIvT], rl[kIvT], rh[kIvT];
    int cv[kIvT], cr[kIvT];
#pragma unroll
    for (int j = 0; j < kIvT; ++j) {
      const int c = min(c0 + j, n - 1);
      vl[j] = Vlo[(sb + c) * NW + wd];
      vh[j] = Vhi[(sb + c) * NW + wd];
      cv[j] = clsV[sb + c];
    }
#pragma unroll
    for (int i = 0; i < kIvT; ++i) {
      const int r = min(r0 + i, n - 1);
      rl[i] = Rlo[(sb + r) * NW + wd];
      rh[i] = Rhi[(sb + r) * NW + wd];
      cr[i] = clsR[sb + r];
    }
#pragma unroll
    for (int i = 0; i < kIvT; ++i)
#pragma unroll
      for (int j = 0; j < kIvT; ++j) {
        straddle |= (cv[j] == 0 && cr[i] == 0 && r0 + i >= c0 + j &&
                     r0 + i < n && c0 + j < c_end);
        const int a = sel_max(cv[j], cr[i]), b = sel_min(cv[j], cr[i]);
        alo[i][j] += (uint64_t)((a & 1) ? vh[j] : vl[j]) * ((a & 2) ? rh[i] : rl[i]);
        ahi[i][j] += (uint64_t)((b & 1) ? vh[j] : vl[j]) * ((b & 2) ? rh[i] : rl[i]);
      }
  }
  if (straddle) atomicOr(&err[kErrCapacity], kCapStraddle);
#pragma unroll
  for (int j = 0; j < kIvT; ++j) {
    const int c = c0 + j;
    if (c >= c_end) continue;
#pragma unroll
    for (int i = 0; i < kIvT; ++i) {
      const int r = r0 + i;
      if (r < c || r >= n) continue;
      const long long e = (colbase[c] + (r - c)) * NW + wd;
      const uint32_t tl = reduce_sum64(alo[i][j], pc);
      const uint32_t th = reduce_sum64(ahi[i][j], pc);
      const uint32_t wl = Wlo[e], wh = Whi[e];
      Wlo[e] = wl >= tl ? wl - tl : wl + pc.q - tl;
      Whi[e] = wh >= th ? wh - th : wh + pc.q - th;
    }
  }
}

cudaError_t launch_iv_classify(IntBuf lo, IntBuf hi, long long row0,
                               int r_begin, int r_end, int8_t* cls, int p,
                               int check_pivot, int n, int* err, int* nonpos,
                               cudaStream_t st) {
  const int rows = r_end - r_begin;
  if (rows <= 0) return cudaSuccess;
  k_iv_classify<<<(rows + 255) / 256, 256, 0, st>>>(
      lo, hi, row0, r_begin, r_end, cls, p, check_pivot, n, err, nonpos);
  return cudaGetLastError();
}

cudaError_t launch_update_iv(const DevPlan& P, uint32_t* Wlo, uint32_t* Whi,
                             const long long* colbase, const uint32_t* Vlo,
                             const uint32_t* Vhi, const uint32_t* Rlo,
                             const uint32_t* Rhi, const int8_t* clsV,
                             const int8_t* clsR, int s_begin, int s_end,
                             int c_begin, int c_end, int r_min,
                             const int* gate, int* err, cudaStream_t st) {
  if (c_begin >= c_end || s_begin >= s_end) return cudaSuccess;
  const int rbase = std::max(c_begin, r_min);
  if (rbase >= P.n) return cudaSuccess;
  const int nct = (c_end - c_begin + kIvT - 1) / kIvT;
  const int nrt = (P.n - rbase + kIvT - 1) / kIvT;
  const dim3 grid((unsigned)(nct * nrt), (unsigned)((P.NW + 127) / 128));
  k_update_iv<<<grid, 128, 0, st>>>(P, Wlo, Whi, colbase, Vlo, Vhi, Rlo, Rhi,
                                    clsV, clsR, s_begin, s_end, c_begin, c_end,
                                    r_min, nrt, gate, err);
  return cudaGetLastError();
}

}  // namespace hgpu
