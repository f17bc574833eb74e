// Device-side data layout and kernel declarations of the B200 LDL^T engine.
//
// HBM layout:
//   W       workspace, lower triangle of the owned columns, column-major
//           packed: entry (r,c) at colbase[c] + (r-c); every entry is NW =
//           np*L residues (np primes x L NTT points, bit-reversed order),
//           i.e. the number-theoretic transform of the entry's base-2^w digit
//           polynomial.  The rank-kb trailing update is pointwise there.
//   Vint/Rint  per panel slot s and row r: the truncated column value
//           V_p[r] and ratio R_p[r] as signed limb integers (hdr = sign*len,
//           cap 32-bit limbs).  This is what a panel owner broadcasts.
//   Vhat/Rhat  their transforms (Rhat in Montgomery form), per slot and row.
//   piv     the full pivots W_pp (for the determinant fold).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "modarith.cuh"

namespace hgpu {

// Error words (device int32[kErrWords]).
enum : int {
  kErrZeroPivot = 0,  // first stage with a zero pivot (atomicMin), INT_MAX if none
  kErrCapacity = 1,   // bitmask: transform / limb capacity exceeded
  kErrInternal = 2,   // bitmask: arithmetic self-check failed
  kErrWords = 4
};
enum : int {
  kCapDigits = 1,     // an integer needs more than L digits
  kCapLimbs = 2,      // an integer needs more than cap limbs
  kCapCrt = 4,        // residue reconstruction out of range
  kCapDegree = 8,     // deg V + deg R >= L somewhere
  kCapCoeff = 16,     // accumulated coefficient bound reaches Q/2
  kCapAmax = 32,      // PD bound on the ratio sizes violated (non-PD shift)
  kCapStraddle = 64,  // interval update: both bounds straddle zero
  kIntDivision = 1,   // quotient correction out of range
  kIntRecip = 2,      // reciprocal did not converge
};

struct DevPlan {
  int n;        // matrix order
  int K;        // fractional bits
  int k2;       // K/2
  int np;       // primes in use (2 or 3)
  int logL, L;  // transform length
  int w;        // digit width in bits (<= 48)
  int T;        // w-bit pieces per reconstructed coefficient
  int cap;      // limbs per stored integer
  int ycap;     // limbs of the per-stage reciprocal
  int NW;       // np*L words per transformed number
  int Lmax;     // twiddle table stride
  PrimeConsts pc[kMaxPrimes];
  uint32_t invL[kMaxPrimes], invLp[kMaxPrimes];
  // Garner constants (q0 > q1 > q2)
  uint32_t g1, g1p;          // q0^-1 mod q1
  uint32_t g2, g2p;          // (q0 q1)^-1 mod q2
  uint32_t q0m2, q0m2p;      // q0 mod q2
  unsigned long long q01;    // q0*q1
  // fourth prime (np == 4)
  uint32_t g3, g3p;          // (q0 q1 q2)^-1 mod q3
  uint32_t q0m3, q0m3p;      // q0 mod q3
  uint32_t q01m3, q01m3p;    // q0 q1 mod q3
  unsigned long long q012lo, q012hi;  // q0 q1 q2 (128-bit)
  unsigned long long Qlo, Qhi, Hlo, Hhi;  // Q and Q/2 (128-bit)
  const uint32_t* tw;   // [np][Lmax]
  const uint32_t* twp;
  const uint32_t* itw;
  const uint32_t* itwp;
  const uint32_t* twm;  // [np][L] forward twiddles, Montgomery form
  const uint32_t* itwm; // [np][L] inverse twiddles, Montgomery form
  int tw_smem;          // 1: kernels stage the Montgomery tables in SMEM
  int grid_cap;         // CTAs for grid-stride row kernels
  int debug;            // HGPU_DEBUG bits (bisection aid), 0 in production
  int recip_fast;       // 1: recip_fast_body (recip_fast.cuh) on shared scratch
  int tw_global;        // solve plans: 1 = NTT twiddles read from global (L1/L2)
                        // instead of staged in shared memory (large NW)
  // batched division (the triangular solve's diagonal): instance b =
  // blockIdx.y offsets its rows, reciprocal and scratch by b * these strides
  // (all 0 in the LDL^T, where gridDim.y == 1)
  int bat_vrow, bat_rrow, bat_ys, bat_mb;
  long long bat_ybuf, bat_scr;
};

// Fixed-size records (nw words each) kept in chunks of 2^shift records, so
// a multi-GB store is assembled from pool blocks of a few hundred MB.
struct EntryStore {
  uint32_t* const* chunk;
  int shift;
  long long nw;
  __device__ __forceinline__ uint32_t* at(long long e) const {
    return chunk[e >> shift] + (e & ((1LL << shift) - 1)) * nw;
  }
};

struct IntBuf {  // count integers, each hdr (sign*len) + cap limbs
  int* hdr;
  uint32_t* limbs;
};

// Interval division (ldlt_det_interval, ldlt.cpp:113-131): mode 1 gives the
// lower ratio bound floor(min corner), mode 2 the upper bound ceil(max
// corner).  The launch's vint/Ybuf/ys hold the lower bounds V.lo and the
// reciprocal of |D.lo|; vhi/yhi/yshi the upper bounds and that of |D.hi|.
struct IvDiv {
  int mode;  // 0: point LDL^T (tdiv_q)
  IntBuf vhi;
  const uint32_t* yhi;
  const int* yshi;
};

// Shared-memory words of one k_divide CTA (layout in ldlt_kernels.cu).
__host__ __device__ inline long long div_span_words(int cap, int ycap) {
  const long long CY = ((long long)cap + ycap + 2 + 3) & ~3LL;
  return 5 * CY + 64;
}

// Extra words when the NTT buffer (NW) does not fit the Barrett scratch.
__host__ __device__ inline long long div_extra_words(const DevPlan& P) {
  const long long CY = ((long long)P.cap + P.ycap + 2 + 3) & ~3LL;
  return (long long)P.NW <= 4 * CY ? 0 : (long long)P.NW;
}

// Host launch wrappers (ldlt_kernels.cu).
cudaError_t launch_fwd_ints(const DevPlan& P, IntBuf src, long long in_base,
                            uint32_t* out, long long out_base, int count,
                            int mont, int* maxdeg, int* err, cudaStream_t st);
cudaError_t launch_init_w(const DevPlan& P, const uint32_t* that,
                          const uint32_t* xhat, const long long* colbase,
                          uint32_t* W, cudaStream_t st);
cudaError_t launch_extract(const DevPlan& P, const uint32_t* W,
                           const long long* colbase, int p, int r_begin,
                           int r_end, IntBuf vint, long long vrow0, IntBuf piv,
                           int* maxbitsV, uint32_t* vhat, int* maxdegV,
                           int* err, cudaStream_t st, int round = 0,
                           uint8_t* vdig = nullptr, int kd = 0);
size_t recip_scratch_words(const DevPlan& P);
cudaError_t launch_recip(const DevPlan& P, IntBuf vint, long long prow,
                         const int* maxbitsV, int p, IntBuf piv, int dmax_bits,
                         uint32_t* Ybuf, int* ys, uint32_t* scratch,
                         int use_gscratch, int* err, cudaStream_t st);
size_t divide_smem_words(const DevPlan& P);
// Optional first step of k_pivot: R_{p-1}[p] by the previous stage's
// reciprocal (k_divide for one row), vint/rint rows at vrow0 (stage p-1)
struct PivotDiv {
  int on;
  long long vrow0;
  const uint32_t* Ybuf;
  const int* ys;
  IntBuf rint;
  uint32_t* rhat;
  int* maxdegR;
  uint32_t* dscr;
  int use_dscr;
  // shared-memory words for the reciprocal (recip_words_bound), which
  // also sizes the launch's dynamic shared memory
  long long recip_words;
};
// reciprocal scratch words for diagonal entries of at most dmax_bits bits
// (PD bound on the stage's precision, as k_recip computes it) and `segs`
// product segments
// shared-memory words of recip_fast_body at that bound
long long recip_fast_words_bound(const DevPlan& P, int dmax_bits);
long long recip_words_bound(const DevPlan& P, int dmax_bits, int segs);
// stage p's pivot chain in one CTA: (pd) the previous stage's ratio of row p,
// the pivot-entry update with the panel's first nslots stages, its
// extraction, and (p < n-1) the reciprocal
cudaError_t launch_pivot(const DevPlan& P, uint32_t* W, const long long* colbase,
                         const uint32_t* Vhat, const uint32_t* Rhat,
                         long long row_stride_slot, int nslots, int p,
                         IntBuf vint, long long vrow0, IntBuf piv, int* maxbitsV,
                         uint32_t* vhat, int* maxdegV, int dmax_bits,
                         uint32_t* Ybuf, int* ys, uint32_t* scratch,
                         int use_gscratch, int* err, cudaStream_t st,
                         const PivotDiv& pd);
// gridDim.y = batch independent reciprocal / division instances (P.bat_*)
cudaError_t launch_recip_batch(const DevPlan& P, IntBuf vint, long long prow,
                               const int* maxbitsV, uint32_t* Ybuf, int* ys,
                               uint32_t* scratch, int batch, int* err,
                               cudaStream_t st);
cudaError_t launch_divide_batch(const DevPlan& P, IntBuf vint,
                                long long vrow0, const uint32_t* Ybuf,
                                const int* ys, IntBuf rint, long long rrow0,
                                uint32_t* gscratch, int batch, int* err,
                                cudaStream_t st);
// rows r in [max(r_begin, p+1), min(r_end, n)) of stage p
cudaError_t launch_divide(const DevPlan& P, IntBuf vint, long long vrow0,
                          int p, int r_begin, int r_end, const uint32_t* Ybuf,
                          const int* ys, IntBuf rint, long long rrow0,
                          uint32_t* rhat, int* maxdegR, uint32_t* gscratch,
                          int use_gscratch, int* err, cudaStream_t st,
                          const IvDiv* iv = nullptr);
// Ratio GEMM: T[k'][i] = 7-bit digit K0d + k' - i of the
// stage's reciprocal; C = T^T vdig on the tensor cores (cuBLAS int8); the
// finish kernel gives the same R_p[r] (and R^) as launch_divide.
cudaError_t launch_toeplitz(const DevPlan& P, const uint32_t* Ybuf,
                            const int* ys, int kd, int ncols, uint8_t* T,
                            const int* err, cudaStream_t st);
cudaError_t launch_ratio_finish(const DevPlan& P, IntBuf vint, long long vrow0,
                                int p, int r_begin, int r_end,
                                const uint32_t* Ybuf, const int* ys,
                                const int32_t* C, int ncols, IntBuf rint,
                                long long rrow0, uint32_t* rhat, int* maxdegR,
                                uint32_t* gscratch, int use_gscratch, int* err,
                                cudaStream_t st);
cudaError_t launch_update(const DevPlan& P, int tile, uint32_t* W,
                          const long long* colbase, const uint32_t* Vhat,
                          const uint32_t* Rhat, long long row_stride_slot,
                          int nslots, int c_begin, int c_end, const int* err,
                          cudaStream_t st, int r_hi = -1);  // rows below r_hi only (tiled kernel)
// rectangle rows [r_lo, r_hi) x columns [c_begin, c_end), r_lo >= c_end
cudaError_t launch_update_rect(const DevPlan& P, uint32_t* W,
                               const long long* colbase, const uint32_t* Vhat,
                               const uint32_t* Rhat, long long row_stride_slot,
                               int nslots, int c_begin, int c_end, int r_lo,
                               int r_hi, const int* err, cudaStream_t st);
cudaError_t launch_update_col(const DevPlan& P, uint32_t* W,
                              const long long* colbase, const uint32_t* Vhat,
                              const uint32_t* Rhat, long long row_stride_slot,
                              int nslots, int c, int r_begin, int r_end,
                              const int* err, cudaStream_t st);
cudaError_t launch_validate(const DevPlan& P, const int* maxdegV,
                            const int* maxdegR, int nstages, int* err,
                            cudaStream_t st);
// tensor-core trailing update of one band (tc_update.cu)
// column update of rows [r_begin, r_end) with the panel's nslots pending
// stages fused with their extraction (one CTA per row)
cudaError_t launch_col_extract(const DevPlan& P, uint32_t* W, const long long* colbase,
                               const uint32_t* Vhat, const uint32_t* Rhat,
                               long long row_stride_slot, int nslots, int p, int r_begin,
                               int r_end, IntBuf vint, long long vrow0, IntBuf piv,
                               int* maxbitsV, uint32_t* vhat, int* maxdegV, int* err,
                               cudaStream_t st, uint8_t* vdig, int kd);
cudaError_t launch_update_tc(const DevPlan& P, uint32_t* W, const long long* colbase,
                             const uint32_t* Vhat, const uint32_t* Rhat,
                             long long row_stride_slot, int nslots, int c_begin, int c_end,
                             const int* err, cudaStream_t st);
cudaError_t configure_update_tc();
long long kernel_launch_count_add(long long k);
long long kernel_launch_count();
// iv_kernels.cu (interval LDL^T)
// nonpos (optional): set to 1 when some class is not +1
cudaError_t launch_iv_classify(IntBuf lo, IntBuf hi, long long row0,
                               int r_begin, int r_end, int8_t* cls, int p,
                               int check_pivot, int n, int* err, int* nonpos,
                               cudaStream_t st);
cudaError_t launch_update_iv(const DevPlan& P, uint32_t* Wlo, uint32_t* Whi,
                             const long long* colbase, const uint32_t* Vlo,
                             const uint32_t* Vhi, const uint32_t* Rlo,
                             const uint32_t* Rhi, const int8_t* clsV,
                             const int8_t* clsR, int s_begin, int s_end,
                             int c_begin, int c_end, int r_min,
                             const int* gate, int* err, cudaStream_t st);
// solve_kernels.cu (inverse iteration)
size_t solve_axpy_smem_words(int capX, int capC, int Wv, int Wa);
size_t solve_finish_smem_words(int Wv, int Wa);
// One row's finish: out[oi] = base[bi] - tdiv_2exp(acc_row, k2) and, with
// shift_out > 0, out2[o2i] = out[oi] << shift_out (the diagonal numerator).
struct Finish {
  IntBuf base;
  int bi;
  IntBuf out;
  int oi;
  IntBuf out2;
  int o2i, shift_out;
};
// One solve step: every target row accumulates R * x_j; the first target's
// finish (`fin`) runs in the same launch.  gscratch: null (shared-memory
// operands) or solve_axpy_smem_words(cap, Wv) words per CTA of global
// scratch (plans too large for shared memory).
// capX / capC: the smem layout's operand capacities (x, R limbs); a larger
// operand raises kCapLimbs and the host reruns with the full capacities
cudaError_t launch_solve_axpy(int n, int cap, int Wv, int Wa, int k2, IntBuf L,
                              IntBuf xv, int xi, int j, int dir, uint32_t* acc,
                              const Finish& fin, int capX, int capC,
                              uint32_t* gscratch, int grid_cap, int* err,
                              cudaStream_t st);
cudaError_t launch_solve_finish(int Wv, int Wa, int k2, const uint32_t* acc_i,
                                const Finish& fin, int* err, cudaStream_t st);
// tensor-core AXPY of the triangular solves (solve_kernels.cu, opt-in)
cudaError_t launch_solve_rdig(int n, int cap, IntBuf L, int kr, uint8_t* dcol,
                              uint8_t* drow, int* err, cudaStream_t st);
cudaError_t launch_solve_toeplitz(IntBuf xv, int xi, int Wv, int kr, int mc,
                                  uint8_t* T, int* err, cudaStream_t st);
cudaError_t launch_solve_acc_tc(int n, int Wv, int Wa, int k2, IntBuf L, IntBuf xv,
                                int xi, int j, int dir, const int32_t* C, int mc,
                                long long* acc7, const Finish& fin, int grid_cap,
                                int* err, cudaStream_t st);
// transform-domain AXPY of the triangular solves (solve_kernels.cu, opt-in):
// plan S, per-factorisation transforms of L, per-step launch
size_t solve_ntt_smem_words(const DevPlan& S, int Wv, int Wa);
cudaError_t configure_solve_ntt(DevPlan& S, int cap, int Wv, int Wa, int* ok);
cudaError_t launch_solve_rhat(const DevPlan& S, int cap, IntBuf L, long long count,
                              EntryStore rhat, int grid_cap, int* err, cudaStream_t st,
                              long long e_begin = 0);  // entries [e_begin, e_begin + count)
cudaError_t launch_solve_xhat(const DevPlan& S, IntBuf xv, int xi, int Wv, uint32_t* xhat,
                              int xbmax, int* err, cudaStream_t st);
cudaError_t launch_solve_ntt(const DevPlan& S, int n, int Wv, int Wa, int k2,
                             EntryStore rhat, const uint32_t* xhat_in,
                             uint32_t* xhat_out, uint32_t* acch, int j, int dir,
                             const Finish& fin, int grid, int xbmax, int* err,
                             cudaStream_t st);
cudaError_t configure_solve_tc(int Wv, int Wa, int mc, int* ok);
cudaError_t launch_int_bits_batch(IntBuf v, int idx0, int step, int stride,
                                  int count, int* out, cudaStream_t st);
cudaError_t configure_solve_kernels(int cap, int Wv, int Wa, bool* axpy_global);
// rq_kernels.cu (the Rayleigh quotient of inverse iteration on the device):
// products |y_i u_i|, y_i^2 of the solve buffer's rows yi0 + i, ui0 + i
// (M = 2 maxlen columns each, sign apart), their exact signed sums as M + 2
// two's-complement limbs (out[0..M+2): num, out[M+2..2M+4): den), and the
// next start vector u_i = y_i scaled by 2^-sh (truncated toward zero).
size_t rq_products_words(int maxlen);
cudaError_t configure_rq_kernels(int maxlen, bool* use_global);
cudaError_t launch_rq_products(IntBuf v, int yi0, int ui0, int n, int Wv, int maxlen,
                               uint32_t* prod, int* psign, uint32_t* gscratch, int grid,
                               int* err, cudaStream_t st);
cudaError_t launch_rq_reduce(const uint32_t* prod, const int* psign, int n, int M,
                             long long* colsum, uint32_t* out, cudaStream_t st);
cudaError_t launch_rq_rescale(IntBuf v, int yi0, int ui0, int n, int Wv, int sh, int* err,
                              cudaStream_t st);
// fold_kernels.cu
long long fold_pivots_device(const uint32_t* plimbs, const int* plen, int n,
                             int pcap, int K, uint32_t* X0, uint32_t* X1,
                             long long xcap, uint32_t* col, uint32_t* chunk_fn,
                             int* chunk_carry, cudaStream_t st,
                             long long* launches);  // kernels launched by this thread
cudaError_t configure_kernels(const DevPlan& P, size_t* div_smem,
                              bool* div_global, bool* recip_global);

}  // namespace hgpu
