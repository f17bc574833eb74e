// Host side of the B200 LDL^T engine: transform plan, HBM buffers, the
// stage/panel schedule, and the column-block-cyclic multi-GPU protocol.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hgpu.h"
#include "ldlt_kernels.cuh"

namespace hgpu {

struct Error : std::runtime_error {
  hgpu_status status;
  long pivot = -1;
  int cap_flags = 0;
  Error(hgpu_status s, const std::string& what)
      : std::runtime_error(what), status(s) {}
};

// Device memory from the device's stream-ordered pool, which keeps freed
// blocks for reuse: building a matrix (GBs of workspace) after another one
// costs no cudaMalloc.  On exhaustion the pool is trimmed and the
// allocation retried.  dev_free waits for the device first.
void* dev_alloc(size_t bytes);
void dev_free(void* p);

// Signed limb integer (GMP-style size) on the host.
struct HostInt {
  int32_t size = 0;
  std::vector<uint32_t> limbs;
};

struct Plan {
  int n = 0, K = 0, np = 0, L = 0, logL = 0, w = 0, T = 0, cap = 0, ycap = 0;
  int kb = 32;         // panel width (columns per block)
  int tile = 16;       // update CTA tile (16: SMEM-staged kernel)
  long long entries = 0;  // workspace entries on this rank
  double workspace_bytes() const { return double(entries) * np * L * 4.0; }
};

// Picks (primes, length, digit width) minimising np*L such that every
// product V_p[c] R_p[r] fits the cyclic length and the accumulated digit
// coefficients stay below Q/4.  `bits` bounds the
// magnitude of any workspace entry and product (PD bound + margin).
Plan choose_plan(int n, int K, int bits, int min_logL = 0);

struct FactorResult {
  int n = 0, K = 0;
  std::vector<HostInt> pivots;
  std::vector<std::vector<HostInt>> ratios;  // [p][r-p-1], if captured
  HostInt det;
  bool have_det = false, have_ratios = false;
  int capture_rows = 0;  // ratios captured for stages and rows < capture_rows
  double device_ms = 0;
  long update_launches = 0;
  double update_ms = 0, update_products = 0;
  long long launches = 0;  // our kernels launched by the factorisation
  double fold_ms = 0;
  // interval factorisation (ldlt_det_interval): pivots = lower bounds,
  // pivots_hi = upper bounds; det = [det, det_hi] when folded; det_sign
  // (+1 / -1 / 0 indeterminate) as FixedInterval::sign (fixed_interval.cpp)
  bool interval = false;
  std::vector<HostInt> pivots_hi;
  HostInt det_hi;
  int det_sign = 0;
  bool det_exact_zero = false;  // folded det interval is exactly [0, 0]
  double net_ms = 0;  // receivers' wait + pull of panels (device time, {net})
};

// In-process rank group (hgpu_matrix_new_group, engine.cpp): W ranks of
// one column-block-cyclic factorisation in this process, on one or more
// devices, driven by host threads and ordered by CUDA events.
struct PeerGroup;

class Matrix {
 public:
  Matrix(int n, int K, const int32_t* sizes, const uint32_t* limbs, int device);
  ~Matrix();
  void set_comm(int rank, int world, const unsigned char* id);
  // Makes this matrix rank 0 of an in-process group over `devices` (one
  // rank per entry; a device may repeat, e.g. to run the multi-rank schedule
  // on one GPU).  The other ranks are owned by this one; factor() drives
  // them all.  A panel's owner publishes its slot set and every other rank
  // pulls the panel's integers from the owner's memory (peer reads over
  // NVLink across GPUs) straight into its own transforms (ldlt.cpp:255-307's
  // owner / receiver roles; no NCCL, no device-side waiting).
  void make_group(const std::vector<int>& devices);
  int world() const { return world_; }
  FactorResult factor(const HostInt& x, unsigned flags);
  // PrecisionMismatch as in ldlt.cpp:36 when x carries other frac bits.
  FactorResult factor_checked(const HostInt& x, long x_frac_bits,
                              unsigned flags) {
    if (x_frac_bits != K_)
      throw Error(HGPU_ERR_PRECISION_MISMATCH,
                  "fractional precision mismatch: " +
                      std::to_string(x_frac_bits) + " vs " +
                      std::to_string(K_));
    return factor(x, flags);
  }
  const Plan& plan_or_build() {
    if (!W_ && !ws_released_) build(0);
    return plan_;
  }
  int frac_bits() const { return K_; }
  // HGPU_CAPTURE keeps only the leading rows x rows block (0: all)
  void set_capture_rows(int rows) { capture_rows_ = rows; }
  // new moments of the same order and precision (hgpu_matrix_set_strip)
  void set_strip(const int32_t* sizes, const uint32_t* limbs);
  int chain_sms() const { return chain_sms_; }
  // Solves (M - sI) y = u with the factors of the last HGPU_KEEP_L
  // factorisation (solve_kernels.cu); u, y at F fractional bits.
  std::vector<HostInt> solve(const std::vector<HostInt>& u, long long* launches);
  // Device-resident inverse iteration (host/rqi.cpp): the start vector stays
  // in the solve buffer, y.u and y.y are formed by rq_kernels.cu, and the next
  // start vector is y rescaled in place; only num, den and bits(y) come back.
  void set_start(const std::vector<HostInt>& u);
  std::vector<HostInt> solve_resident(long long* launches, bool download);
  void rayleigh(HostInt& num, HostInt& den, long& ybits, long long* launches);
  void rescale_start(long sh, long long* launches);
  // mode 0: integer AXPY, 1: tensor-core AXPY, 2: transform-domain AXPY
  std::vector<HostInt> solve_impl(long long* launches, int mode, bool download);
  void ensure_solve_buffers();
  int order() const { return n_; }
  const HostInt& strip_entry(int s) const { return strip_[s]; }
  // Interval mode (iv_engine.cpp): the constructor's strip holds the lower
  // bounds; this supplies the upper bounds (HankelIntervalMatrix).
  void set_interval_hi(const int32_t* sizes, const uint32_t* limbs);
  bool is_interval() const { return interval_; }
  // ldlt_det_interval (ldlt.cpp:79-152) at the shift [xlo, xhi].
  FactorResult factor_interval(const HostInt& xlo, const HostInt& xhi,
                               unsigned flags);

 private:
  FactorResult factor_group(const HostInt& x, unsigned flags);
  long long slot_row0(int b) const { return (long long)(b % nsets_) * plan_.kb * n_; }
  // group transport (engine.cpp): owner publishes panel b, receivers wait for
  // it and pull, owner waits for the pulls before reusing a slot set
  void group_publish(int b, cudaStream_t st);
  Matrix* group_await(int b, int owner, cudaStream_t st);
  void group_pulled(int b, cudaStream_t st);
  void group_wait_pulled(int b, cudaStream_t st);
  void group_merge_err(int* herr);
  void parse_strip(const int32_t* sizes, const uint32_t* limbs);
  void build(int min_logL);
  void alloc_slots();
  void release_workspace();   // W and slot sets back to the pool (solves)
  void reclaim_workspace();   // ... and taken again by the next factorisation
  void release_solve_transforms();
  void release();
  void run(const HostInt& x, unsigned flags, FactorResult& res);
  void panel_broadcast(int owner, int p0, int ns, long long row0,
                       cudaStream_t st);
  void fold(FactorResult& res);
  int ratio_gemm_kd(int db) const;
  int ratio_gemm_ncols(int db) const;
  // R_p[r] for rows [max(r_begin, p+1), r_end) by the int8 ratio GEMM on
  // stream s with operand set `which` (0 near, 1 far)
  void ratio_gemm(int which, int p, int r_begin, int r_end, IntBuf vint,
                  long long row0, const uint32_t* yb, const int* yss,
                  IntBuf rint, int* maxdegR, uint32_t* dscr, cudaStream_t s);
  void keep_panel_L(int p0, int ns, long long row0set, cudaStream_t st,
                    IntBuf src);
  void build_interval();
  void release_interval();
  void run_interval(const HostInt& xlo, const HostInt& xhi, unsigned flags,
                    FactorResult& res);

  int n_, K_, device_;
  int capture_rows_ = 0;
  std::vector<HostInt> strip_;
  int strip_bits_ = 0;
  Plan plan_;
  DevPlan dp_{};
  int rank_ = 0, world_ = 1;
  void* comm_ = nullptr;  // ncclComm_t
  std::shared_ptr<PeerGroup> group_;                // in-process group, or null
  std::vector<std::unique_ptr<Matrix>> peers_;      // ranks 1.. (rank 0 only)
  std::vector<cudaEvent_t> grp_ready_ev_, grp_pulled_ev_;
  std::vector<cudaEvent_t> net_ev_;  // receivers: [2b] before, [2b+1] after a panel's arrival
  long long grp_run_ = 0;
  std::vector<long long> colbase_h_;
  std::vector<int> owned_blocks_;
  // device buffers
  uint32_t *tw_ = nullptr, *W_ = nullptr, *that_ = nullptr, *xhat_ = nullptr;
  long long* colbase_ = nullptr;
  int* strip_hdr_ = nullptr;
  uint32_t* strip_limbs_ = nullptr;
  int* x_hdr_ = nullptr;
  uint32_t* x_limbs_ = nullptr;
  int* vhdr_ = nullptr;
  uint32_t* vlimbs_ = nullptr;
  int* rhdr_ = nullptr;
  uint32_t* rlimbs_ = nullptr;
  uint32_t *vhat_ = nullptr, *rhat_ = nullptr;
  int* phdr_ = nullptr;
  uint32_t* plimbs_ = nullptr;
  uint32_t *ybuf_ = nullptr, *rscratch_ = nullptr, *dscratch_ = nullptr,
           *dscratch2_ = nullptr, *dscratch3_ = nullptr;
  static constexpr int kYRing = 128;
  // rows [p0, p0 + near_rows_) of a panel run in step with the pivot chain,
  // the rest on the far stream (HGPU_NEAR, default two panels)
  int near_rows_ = 34;
  // ratio GEMM (HGPU_RATIO_GEMM bits: 1 far rows, 2 near rows; 0 = k_divide,
  // the default: the int8 path is exact but measured slower end to end)
  int ratio_gemm_ = 0;
  int rg_kd_ = 0, rg_ncols_ = 0;
  uint8_t* vdig_ = nullptr;             // n x kd digits of |V_p[r]|
  uint8_t* rg_t_[2] = {nullptr, nullptr};  // per stream (near, far): T
  int32_t* rg_c_[2] = {nullptr, nullptr};  // per stream: GEMM output
  uint8_t* rg_ws_[2] = {nullptr, nullptr};
  void* blas_[2] = {nullptr, nullptr};     // cublasHandle_t per stream
  static constexpr size_t kBlasWorkspace = 32u << 20;
  int* ys_ = nullptr;
  int* stats_ = nullptr;  // maxbitsV | maxdegV | maxdegR, n each
  int* err_ = nullptr;
  size_t div_smem_ = 0;
  bool div_global_ = false;
  bool recip_global_ = false;
  cudaStream_t stream_ = nullptr;        // bulk (trailing updates)
  cudaStream_t stream_panel_ = nullptr;  // panel factorisation, high priority
  cudaStream_t stream_helper_ = nullptr; // pivot -> reciprocal chain
  cudaStream_t stream_far_ = nullptr;    // far rows of the panel (may lag)
  static constexpr int kMaxFarLanes = 4;
  int far_prio_ = 0;  // stream priority of the far lanes (HGPU_FAR_PRIO levels below the chain)
  int far_lanes_ = 3;  // far-row streams (HGPU_FAR_LANES; 3: 255 ms, 2: 265 ms at config 3)
  cudaStream_t far_streams_[kMaxFarLanes] = {};  // [0] = stream_far_
  cudaEvent_t far_ev_[kMaxFarLanes] = {};
  cudaStream_t stream_upd1_ = nullptr;   // trailing update: next band, catch-up
  cudaStream_t stream_upd2_ = nullptr;   // trailing update: deferred bands
  int defer_ = 4;   // panels the deferred trailing update may lag (HGPU_DEFER)
  bool fused_pivot_ = true;  // k_pivot: one launch per chain stage (HGPU_FUSED_PIVOT)
  int pivot_segs_ = 6;       // k_pivot's reciprocal product segments (HGPU_PIVOT_SEGS)
  int nsets_ = 2;   // V/R slot sets (2 + deferral, memory permitting)
  int chain_sms_ = 0;  // SMs reserved for the pivot chain (green context), 0 = none
  // HGPU_SM_SPLIT partition (CUgreenCtx of the chain's and the other SMs)
  void* split_ga_ = nullptr;
  void* split_gb_ = nullptr;
  std::vector<cudaEvent_t> pev_, sev_;
  bool recip_bound_ = true;  // reciprocal precision from the PD bound
  // whole L factor (HGPU_KEEP_L): R_p[r], p < r, packed strictly lower
  int* lhdr_ = nullptr;
  uint32_t* llimbs_ = nullptr;
  bool have_L_ = false;
  // solve buffers
  int sWv_ = 0, sWa_ = 0;
  int* svhdr_ = nullptr;        // vectors u | z | w | y (4n rows)
  uint32_t* svlimbs_ = nullptr;
  uint32_t* sacc_ = nullptr;    // n x Wa two's complement
  uint32_t* sgscr_ = nullptr;   // k_solve_axpy scratch when SMEM is too small
  int* spair_hdr_ = nullptr;    // (piv_p, z_p 2^k2) pairs, 2n rows
  uint32_t* spair_limbs_ = nullptr;
  int* sbits_ = nullptr;
  // Rayleigh quotient on the device (rq_kernels.cu)
  bool start_resident_ = false, have_y_ = false;
  std::vector<HostInt> saved_start_;  // the start vector across a re-plan
  int last_ulimbs_ = 0, last_ylimbs_ = 0;  // widest u / y entry of the last solve
  int rq_maxlen_ = 0, rq_grid_ = 0;
  uint32_t *rq_prod_ = nullptr, *rq_out_ = nullptr, *rq_scr_ = nullptr;
  long long* rq_colsum_ = nullptr;
  int* rq_sign_ = nullptr;
  uint32_t *sybuf_ = nullptr, *srscr_ = nullptr, *sdscr_ = nullptr;
  int* sys_ = nullptr;
  int dmax_bits_ = 0;
  // tensor-core solve AXPY (HGPU_SOLVE_TC): L digits (column and row order),
  // Toeplitz operand, GEMM output, 7-bit-column accumulators
  bool solve_tc_ = false;
  // transform-domain solve AXPY (HGPU_SOLVE_NTT): solve plan, transforms of
  // the L entries (per factorisation), accumulators, double-buffered x-hat
  int solve_ntt_ = 1;  // 0: off, 1: with fallback to the integer AXPY, 2: strict
  DevPlan sdp_{};
  int sdp_bits_ = 0, sdp_xbits_ = 0;
  uint32_t *stw_ = nullptr, *acch_ = nullptr, *sxhat_ = nullptr;
  std::vector<uint32_t*> lhat_chunks_;  // L-entry transforms, 2^lhat_shift_ per chunk
  uint32_t** lhat_tab_ = nullptr;       // device copy of the chunk pointers
  int lhat_shift_ = 0;
  EntryStore lhat_store() const { return EntryStore{lhat_tab_, lhat_shift_, (long long)sdp_.NW}; }
  long long lhat_for_ = -1;
  // L-entry transforms during the factorisation (HGPU_PRE_LHAT): once a solve
  // plan exists, every panel's ratio columns are transformed right after they
  // are copied to the L store, on a lowest-priority stream; the next solve
  // keeps them if the plan still fits and no entry was flagged
  bool pre_lhat_ = true;
  cudaStream_t stream_lhat_ = nullptr;
  cudaEvent_t lhat_ev_ = nullptr;
  int* lhat_err_ = nullptr;
  long long lhat_pre_for_ = -1;
  int far_sub_ = 16;  // far rows' in-panel sub-panel width (HGPU_FAR_SUB, 0 = off; 16 with the 4-row column update: 241.7 ms, 8: 246.3 ms)
  int edf_h_ = 1;    // EDF trailing-update horizon in panels (HGPU_EDF, 0 = off)
  // slot sets are reused when memory is short (configs 4, 5): the panels whose
  // sets come up for reuse are flushed (all their remaining bands) this many
  // panels ahead of the reuse, in batches of up to flush_batch_ panels per
  // launch (HGPU_FLUSH_AHEAD / HGPU_FLUSH_BATCH; 0 / 1: at the reuse, one by one)
  int flush_ahead_ = 2, flush_batch_ = 4;
  int edf_run_ = 8;  // panels accumulated by one EDF update launch (HGPU_EDF_RUN, 1-8)
  // pivot entry's earlier stages ahead of k_pivot (HGPU_PRE_ENTRY)
  bool pre_entry_ = true;
  // trailing update on the tensor cores (tc_update.cu, HGPU_UPDATE_TC=1);
  // bit-identical, measured slower than k_update_tiled: off by default
  bool update_tc_ = false;
  // near (bit 1) / far (bit 2) rows' column update fused with the extraction
  // (k_col_extract, HGPU_COL_EXTRACT)
  int col_extract_ = 0;
  // band b+1 receives panel b's stages sub-panel by sub-panel during the
  // panel instead of all at its end (HGPU_LOOKAHEAD)
  int lookahead_ = 0;  // 1: on su1, 2: on su2 (lowest priority)
  bool ws_released_ = false;
  bool strip_dirty_ = false;          // set_strip: re-send and re-transform
  uint32_t* strip_stage_ = nullptr;    // pinned host staging of the strip
  size_t strip_stage_words_ = 0;  // W / slot sets handed to the solves' transforms
  // the chain's next row on its own stream (HGPU_NEXT_ROW)
  bool next_row_ = false;
  cudaStream_t stream_next_ = nullptr;
  std::vector<cudaEvent_t> sn_ev_;
  cudaStream_t stream_pre_ = nullptr;
  std::vector<cudaEvent_t> pre_ev_;
  // near rows' column update ahead of the panel stream (HGPU_PRE_NEAR): column
  // c receives the panel's stages up to c-2 on its own stream as soon as the
  // ratios of stage c-2 exist, so the panel stream applies only stage c-1
  // far rows beyond the next panel's near window lag the chain by up to one
  // panel (HGPU_LAG_FAR): the panel ends when the chain, the near rows and
  // lane 0 (the next panel's near rows) are done; band b+1 is updated for
  // those rows at once and for the rest when the other lanes finish
  bool lag_far_ = false;  // bit-exact; 254.0 ms with four lanes against 254.6: off
  cudaStream_t stream_join_ = nullptr;
  std::vector<cudaEvent_t> lag_ev_;  // [2b]: panel b early, [2b+1]: band b far rows updated
  bool pre_near_ = false;  // bit-exact, measured equal (255.0 vs 254.7 ms): off
  cudaStream_t stream_pre2_ = nullptr;
  std::vector<cudaEvent_t> pre2_ev_;
  std::vector<cudaEvent_t> edf_ev_;
  int solve_xlimbs_ = 0;          // widest z / y entry of the solves so far
  long long factor_serial_ = 0;   // KEEP_L factorisations so far
  long long rdig_for_ = -1;       // factor_serial_ the digits belong to
  int tc_kr_ = 0, tc_mc_ = 0;
  uint8_t *rdig_col_ = nullptr, *rdig_row_ = nullptr, *tc_t_ = nullptr,
          *tc_ws_ = nullptr;
  int32_t* tc_c_ = nullptr;
  long long* tc_acc_ = nullptr;
  void* tc_blas_ = nullptr;
  // interval mode: upper-bound copies of the per-entry buffers (the point
  // buffers hold the lower bounds) and the sign classes of V, R bounds
  bool interval_ = false;
  std::vector<HostInt> strip_hi_;
  uint32_t *W2_ = nullptr, *that2_ = nullptr, *xhat2_ = nullptr;
  int* strip2_hdr_ = nullptr;
  uint32_t* strip2_limbs_ = nullptr;
  int* x2_hdr_ = nullptr;
  uint32_t* x2_limbs_ = nullptr;
  int *vhdr2_ = nullptr, *rhdr2_ = nullptr, *phdr2_ = nullptr;
  uint32_t *vlimbs2_ = nullptr, *rlimbs2_ = nullptr, *plimbs2_ = nullptr;
  uint32_t *vhat2_ = nullptr, *rhat2_ = nullptr, *ybuf2_ = nullptr;
  int* ys2_ = nullptr;
  int8_t *clsv_ = nullptr, *clsr_ = nullptr;
  int* ivgate_ = nullptr;  // {INT_MAX, nonpositive bound seen, 0, 0}
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  // HGPU_TIMELINE=<file>: per-launch start/end events (scheduling analysis)
  struct TlRec {
    int kind, p;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> tl_pool_;
  std::vector<TlRec> tl_;
  size_t tl_used_ = 0;
  std::vector<cudaEvent_t> uev_;
};

int block_owner(long block, int world);

}  // namespace hgpu
