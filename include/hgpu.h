/* hgpu — B200 (sm_100a) engine for the reference's O(N^3) hot path: the
 * square-root-free LDL^T determinant of the Hankel moment matrix M - xI.
 *
 * This is the thin C ABI the host C++ (the DetEvaluator seam) calls.  It
 * replaces, bit for bit:
 *   ldlt_det_serial    /root/reference/proj/src/ldlt.hpp:30-31  (ldlt.cpp:31-77)
 *   ldlt_det_parallel  /root/reference/proj/src/ldlt.hpp:56-57  (ldlt.cpp:315-341)
 *   LdltCapture        /root/reference/proj/src/ldlt.hpp:16-19
 *   ZeroPivot          /root/reference/proj/src/errors.hpp:49-58
 *
 * Numbers cross the boundary as GMP-style signed limb vectors: a signed
 * int32 size (sign of the value times the number of little-endian 32-bit
 * limbs, 0 for zero) and the limbs.  A strip of 2n-1 mantissas is passed as
 * `sizes[2n-1]` plus all limbs concatenated in order.  Every mantissa carries
 * frac_bits fractional bits (FixedPoint, fixed_point.hpp:12-22).
 *
 * Ownership: inputs are copied; results are owned by the returned handle.
 * Threading: one call at a time per matrix handle.  Status-returning
 * functions never throw; the message of the last failure in the calling
 * thread is available from hgpu_last_error().
 */
#ifndef HGPU_H
#define HGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hgpu_status {
  HGPU_OK = 0,
  HGPU_ERR_INVALID_ARGUMENT = 1,
  HGPU_ERR_ZERO_PIVOT = 2,         /* heig::ZeroPivot; see hgpu_last_zero_pivot */
  HGPU_ERR_PRECISION_MISMATCH = 3, /* heig::PrecisionMismatch (ldlt.cpp:36) */
  HGPU_ERR_CUDA = 4,               /* device unavailable or a CUDA failure */
  HGPU_ERR_CAPACITY = 5,           /* a value outgrew every plan that fits */
  HGPU_ERR_INTERNAL = 6,           /* an exactness self-check failed */
  HGPU_ERR_COMM = 7,               /* heig::ChannelFailure (errors.hpp:107-111) */
  HGPU_ERR_PRECISION_EXHAUSTED = 8, /* NoProgress / SignViolation /
                                       RootHitAtPrecision (errors.hpp:60-80):
                                       raise frac_bits and retry */
  HGPU_ERR_INTERVAL_STRADDLE = 9    /* interval LDL^T: a column-value bound
                                       and a ratio bound both contain zero,
                                       so the extreme corner of their product
                                       depends on magnitudes (not supported
                                       in the transform domain) */
} hgpu_status;

/* factor flags */
#define HGPU_CAPTURE 1u /* keep the ratio columns (LdltCapture) */
#define HGPU_FOLD 2u    /* fold the pivots into det (ldlt.cpp:22-27) */
#define HGPU_PROFILE 4u /* time every trailing-update launch with events */
#define HGPU_KEEP_L 8u  /* keep the whole L factor on the device (solves) */

typedef struct hgpu_matrix hgpu_matrix;
typedef struct hgpu_factor hgpu_factor;

/* Uploads the anti-diagonal strip of an order-n Hankel matrix (the
 * HankelMatrix of hankel_matrix.hpp:17-42) to `device` and sizes the
 * transform plan.  Replaces the per-call workspace init of ldlt.cpp:38-44. */
hgpu_status hgpu_matrix_new(long n, long frac_bits, const int32_t* strip_sizes,
                            const uint32_t* strip_limbs, int device,
                            hgpu_matrix** out);
void hgpu_matrix_free(hgpu_matrix* m);

/* The reference's on-disk interchange of a matrix (hankel_matrix.cpp:52-87):
 * one line per anti-diagonal, "s=<index> hex=<mantissa, base 16> fracbits=<K>".
 * hgpu_matrix_new_from_dump reads such a file the way load_matrix_dump does
 * (lines in order of s, empty lines skipped, 2n-1 anti-diagonals; anything
 * else is the reference's MalformedInput -> HGPU_ERR_INVALID_ARGUMENT with
 * its message) and uploads the strip; n and frac_bits (the last line's, as in
 * the reference) are reported.  hgpu_matrix_dump writes the matrix's strip in
 * the same format (dump_matrix, :52-57), so a strip can go from either side
 * to the other unchanged. */
hgpu_status hgpu_matrix_new_from_dump(const char* path, int device, hgpu_matrix** out,
                                      long* n, long* frac_bits);
hgpu_status hgpu_matrix_dump(const hgpu_matrix* m, const char* path);

/* Multi-GPU: join a column-block-cyclic factorisation as `rank` of `world`
 * (one process per GPU).  `nccl_id` is the 128-byte ncclUniqueId produced by
 * hgpu_nccl_unique_id on rank 0 and shared by the caller.  Must be called
 * before the first factorisation; world == 1 is the default. */
hgpu_status hgpu_nccl_unique_id(unsigned char out[128]);
hgpu_status hgpu_matrix_set_comm(hgpu_matrix* m, int rank, int world,
                                 const unsigned char nccl_id[128]);

/* Multi-GPU in one process (the reference's worker threads, ldlt.cpp:315-341,
 * with workers -> ranks): `world` column-block-cyclic ranks on
 * devices[0..world-1], driven by host threads of the calling process.  A
 * device may repeat (several ranks on one GPU: the multi-rank schedule on a
 * single device).  The panel owner publishes each finished panel with a CUDA
 * event; every other rank reads the panel's integers directly from the
 * owner's memory (NVLink peer loads between GPUs) into its own transforms.
 * The handle is rank 0: hgpu_ldlt_factor, the eigenvalue drivers and the
 * accessors use it as a single matrix (bit-identical to world 1). */
hgpu_status hgpu_matrix_new_group(long n, long frac_bits,
                                  const int32_t* strip_sizes,
                                  const uint32_t* strip_limbs, const int* devices,
                                  int world, hgpu_matrix** out);
/* Ranks behind the handle (1 unless grouped or joined by set_comm). */
int hgpu_matrix_world(const hgpu_matrix* m);

/* New moments for the same order and frac_bits (the strip of another beta,
 * or the same one re-sent): the next hgpu_ldlt_factor copies and transforms
 * them; the transform plan, workspace and streams are kept when the new
 * strip fits the plan (otherwise they are rebuilt there).  Inputs copied. */
hgpu_status hgpu_matrix_set_strip(hgpu_matrix* m, const int32_t* strip_sizes,
                                  const uint32_t* strip_limbs);

/* HGPU_CAPTURE keeps only the leading rows x rows block of the ratio
 * columns (stages p < rows, rows r < rows; 0 = all, the default).  The
 * leading block of the submatrix-order LDL^T is the factorisation of the
 * leading block (ldlt.cpp:65-71 touches indices < rows only there), so a
 * full-size run can be checked against the reference on a leading block
 * without copying every ratio to the host. */
hgpu_status hgpu_matrix_set_capture_rows(hgpu_matrix* m, long rows);

/* det(M - xI) by square-root-free LDL^T (ldlt_det_serial / _parallel).
 * x must carry the matrix's frac_bits.  On HGPU_ERR_ZERO_PIVOT the pivot
 * index is available from hgpu_last_zero_pivot(). */
hgpu_status hgpu_ldlt_factor(hgpu_matrix* m, int32_t x_size,
                             const uint32_t* x_limbs, long x_frac_bits,
                             unsigned flags, hgpu_factor** out);

long hgpu_factor_order(const hgpu_factor* f);
long hgpu_factor_frac_bits(const hgpu_factor* f);
/* Pivot D_p at frac_bits (LdltCapture::pivots). */
hgpu_status hgpu_factor_pivot(const hgpu_factor* f, long p, int32_t* size,
                              const uint32_t** limbs);
/* Ratio R_p[r] at frac_bits/2, r > p (LdltCapture::ratio_columns);
 * requires HGPU_CAPTURE. */
hgpu_status hgpu_factor_ratio(const hgpu_factor* f, long p, long r,
                              int32_t* size, const uint32_t** limbs);
/* fold_pivots (ldlt.cpp:22-27) at frac_bits; requires HGPU_FOLD. */
hgpu_status hgpu_factor_det(const hgpu_factor* f, int32_t* size,
                            const uint32_t** limbs);
/* Device time of the factorisation (CUDA events), and with HGPU_PROFILE the
 * trailing-update kernel statistics: launches, summed ms, modular products. */
double hgpu_factor_device_ms(const hgpu_factor* f);
hgpu_status hgpu_factor_update_stats(const hgpu_factor* f, long* launches,
                                     double* ms, double* products);
/* Multi-rank runs: device time the receiving ranks spent waiting for and
 * pulling published panels, summed over ranks (the reference's {net},
 * timing.hpp:7-39).  0 on one rank. */
double hgpu_factor_net_ms(const hgpu_factor* f);
/* Number of device kernels the factorisation launched. */
long long hgpu_factor_launches(const hgpu_factor* f);
void hgpu_factor_free(hgpu_factor* f);

/* Smallest eigenvalue of the resident matrix at its frac_bits: the
 * reference's secant on P(x) = det(M - xI) (secant.cpp:27-117) with every
 * probe a GPU factorisation + fold, stopping when the top `digits`
 * significant decimals of successive iterates agree (the reference: 15).
 * Outputs (malloc'd, free with hgpu_string_free; each may be NULL):
 *   eigenvalue  `digits`-digit truncation, scientific notation
 *   trace       one line per recorded iterate: "<x hex> <det hex>"
 * On HGPU_ERR_PRECISION_EXHAUSTED the caller escalates frac_bits, as
 * driver.cpp:100-130 does. */
hgpu_status hgpu_smallest_eigenvalue(hgpu_matrix* m, int digits,
                                     char** eigenvalue, char** trace,
                                     long* iterations, double* det_seconds);
void hgpu_string_free(char* s);

/* ---- moments (build_matrix / build_interval_matrix, hankel_matrix.cpp) ----
 * The 2n-1 anti-diagonals (1/beta) Gamma((1+s)/beta), beta = beta_num /
 * beta_den, at frac_bits: interval == 0 gives build_matrix's round-to-nearest
 * strip in lo (hi = lo if requested), interval != 0 the certified
 * [floor, ceil] bounds of build_interval_matrix.  Host code (all threads),
 * bit-identical to the reference's Gamma enclosures (gamma.cpp:101-230).
 * Outputs are malloc'd; release each with hgpu_buffer_free.  hi_* may be
 * null when interval == 0. */
hgpu_status hgpu_build_moments(long n, unsigned long beta_num,
                               unsigned long beta_den, long frac_bits,
                               int interval, int32_t** lo_sizes,
                               uint32_t** lo_limbs, int32_t** hi_sizes,
                               uint32_t** hi_limbs);
void hgpu_buffer_free(void* p);

/* ---- interval LDL^T (ldlt_det_interval, ldlt.cpp:79-152) ----------------
 * An interval matrix holds the lower and upper bounds of every moment
 * (HankelIntervalMatrix; bounds in order, same frac_bits).  It runs on one
 * GPU.  Replaces the reference's serial interval elimination (ldlt.cpp:79). */
hgpu_status hgpu_interval_matrix_new(long n, long frac_bits,
                                     const int32_t* lo_sizes,
                                     const uint32_t* lo_limbs,
                                     const int32_t* hi_sizes,
                                     const uint32_t* hi_limbs, int device,
                                     hgpu_matrix** out);
/* ldlt_det_interval(m, [xlo, xhi]): pivot intervals (hgpu_factor_pivot = lower
 * bound, hgpu_factor_pivot_hi = upper bound) and, with HGPU_FOLD, the exact
 * determinant interval (hgpu_factor_det / hgpu_factor_det_hi, folded with
 * FixedInterval::mul semantics).  ZeroPivot(p) when [V.lo, V.hi][p] contains
 * zero (ldlt.cpp:110-111); HGPU_ERR_INTERVAL_STRADDLE when a column-value bound
 * and a ratio bound both contain zero. */
hgpu_status hgpu_ldlt_interval(hgpu_matrix* m, int32_t xlo_size,
                               const uint32_t* xlo_limbs, int32_t xhi_size,
                               const uint32_t* xhi_limbs, long x_frac_bits,
                               unsigned flags, hgpu_factor** out);
hgpu_status hgpu_factor_pivot_hi(const hgpu_factor* f, long p, int32_t* size,
                                 const uint32_t** limbs);
hgpu_status hgpu_factor_det_hi(const hgpu_factor* f, int32_t* size,
                               const uint32_t** limbs);
/* FixedInterval::sign of the determinant interval: 1, -1, 0 (indeterminate) */
int hgpu_factor_det_sign(const hgpu_factor* f);
/* verify_eigenvalue (verify.cpp:8-42) on an interval matrix at its own
 * frac_bits: a = x truncated to `digits` significant digits (the reference
 * uses 15), b = a + 1 ulp in the last digit; status 0 verified (det(M-aI) > 0,
 * det(M-bI) < 0), 1 refuted, 2 inconclusive; signs 1/-1/0; probes are
 * malloc'd strings (hgpu_string_free). */
hgpu_status hgpu_verify_eigenvalue(hgpu_matrix* m, const char* x_decimal,
                                   int digits, int* status, int* lower_sign,
                                   int* upper_sign, char** probe_low,
                                   char** probe_high);

/* The same, also reporting VerifyOutcome::lower_exact_zero (verify.cpp:26-27):
 * 1 when the folded det(M - aI) interval is exactly [0, 0], i.e. the probe a
 * is itself an eigenvalue and bracketing cannot decide at any precision
 * (driver.cpp:161-170 stops with a diagnosis instead of escalating). */
hgpu_status hgpu_verify_eigenvalue_ex(hgpu_matrix* m, const char* x_decimal,
                                      int digits, int* status, int* lower_sign,
                                      int* upper_sign, int* lower_exact_zero,
                                      char** probe_low, char** probe_high);

/* Smallest eigenvalue by inverse iteration with Rayleigh-quotient shifts
 * (the north-star's lambda_min step; no reference counterpart -- SURVEY §0
 * D1 -- and pinned against oracle/pyoracle.py:inverse_iteration_py).  Each
 * step solves (M - s I) y = u_k with the GPU L, D factors of M - s I
 * (HGPU_KEEP_L; forward and back triangular solves, exact with one
 * truncation per entry) and sets rho_k = s + (y.u_k)/(y.y); the iterate stays
 * on the device (dot products and rescaling by rq_kernels.cu).  Phase 1 keeps
 * s = sigma until rho's relative change is < 2^-32, phase 2 refactors at
 * s = rho_k each step until it is < 2^-max(64, frac_bits/16), phase 3 keeps
 * those factors; stop when the change is below 2^-(frac_bits/2) or stalls.  u: n signed
 * limb vectors at frac_bits (e.g. the seed-0 uniform[-1,1] start vector);
 * sigma: the first shift (0 is fine).  Outputs as for
 * hgpu_smallest_eigenvalue; `trace` lists every rho_k in hex. */
hgpu_status hgpu_inverse_iteration(hgpu_matrix* m, const int32_t* u_sizes,
                                   const uint32_t* u_limbs, int32_t sigma_size,
                                   const uint32_t* sigma_limbs, int max_iter,
                                   int digits, char** eigenvalue, char** trace,
                                   long* iterations, double* seconds);

/* Plan introspection: primes, transform length, digit width, limb capacity,
 * workspace bytes on this rank. */
hgpu_status hgpu_matrix_plan(const hgpu_matrix* m, int* nprimes, int* length,
                             int* digit_bits, int* cap_limbs,
                             double* workspace_bytes);

/* Column-block owner (reflected round-robin of assignment.hpp:15-23 applied
 * to blocks of `block` columns). */
int hgpu_block_owner(long block_index, int world);

/* Returns every idle block of the device's stream-ordered memory pool to the
 * driver (the engine keeps freed blocks for reuse, so repeated matrices skip
 * cudaMalloc): lets a caller measure a cold start in a warm process. */
hgpu_status hgpu_trim_pool(int device);

long hgpu_last_zero_pivot(void);
const char* hgpu_last_error(void);
const char* hgpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HGPU_H */
