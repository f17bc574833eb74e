// Smallest eigenvalue by inverse iteration with Rayleigh-quotient shifts
// (the north-star's lambda_min step; the reference itself has
// no such path -- SURVEY §0 D1 -- so tests/ pin this against the restatement
// oracle/pyoracle.py:inverse_iteration_py, bit for bit).
//
// Fixed point at K fractional bits throughout (K = the matrix precision).
// Phase 1 (shifted inverse iteration) keeps the factors of M - s_0 I and only
// re-solves; once the relative change of rho is below 2^-32 (or after 64
// plain steps) phase 2 (Rayleigh-quotient iteration) refactors at s = rho;
// once it is below 2^-max(64, K/16) phase 3 keeps those factors again (each
// solve then gains ~K/8 bits for the price of a solve, not a factorisation):
// Every O(n) multiprecision step runs on the GPU and the iterate never
// leaves it: the host keeps only sigma, rho and the stopping rule.
//   factor   M - s_k I = L D L^T          (GPU LDL^T, HGPU_KEEP_L)
//   solve    (M - s_k I) y = u_k          (GPU triangular solves, exact with
//                                          one truncation per entry)
//   rho_k  = s_k + tdiv((y.u_k) 2^K, y.y)  (= y^T M y / y^T y for the exact y,
//                                          since M y = s_k y + u_k)
//   stop   when |rho_k - rho_{k-1}| 2^(K/2) <= |rho_k| (relative change below
//          2^-(K/2), the north-star rule), rho_k == rho_{k-1}, or after two
//          changes that fail to go below the smallest change so far (the
//          arithmetic noise floor)
//   next   u_{k+1} = y scaled by a power of two so that max |u_i| lies in
//          [1/2, 1);  s_{k+1} = rho_k in phase 2
// A zero last pivot means s_k is an eigenvalue at this precision (as in
// secant.cpp:36-52); it is returned as is.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/hgpu.h"
#include "../engine.h"
#include "bigz.h"

namespace hgpu {
Matrix* matrix_impl(hgpu_matrix* m);
void set_last_error(const std::string& s, long pivot);

namespace {

char* dup_c(const std::string& s) {
  char* o = static_cast<char*>(std::malloc(s.size() + 1));
  if (o) std::memcpy(o, s.c_str(), s.size() + 1);
  return o;
}

Z from_host(const HostInt& h) { return Z::from_limbs(h.size, h.limbs.data()); }

// phase switch and stall rule (oracle/pyoracle.py RQI_* constants)
constexpr long kSwitchBits = 32;  // phase 1 -> 2: relative change < 2^-32
constexpr long kMaxPlain = 64;    // ... or this many phase-1 steps
constexpr int kStall = 2;         // changes not below the smallest so far
// phase 2 -> 3: relative change < 2^-final_bits(K)
long final_bits(long k) { return std::max(64L, k / 16); }

}  // namespace
}  // namespace hgpu

extern "C" hgpu_status hgpu_inverse_iteration(
    hgpu_matrix* m, const int32_t* u_sizes, const uint32_t* u_limbs,
    int32_t sigma_size, const uint32_t* sigma_limbs, int max_iter, int digits,
    char** eigenvalue, char** trace, long* iterations, double* seconds) {
  using namespace hgpu;
  try {
    Matrix* mm = matrix_impl(m);
    if (!mm || !u_sizes || max_iter < 1 || digits < 1)
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad argument");
    const long n = mm->order(), k = mm->frac_bits(), k2 = k / 2;
    const auto t0 = std::chrono::steady_clock::now();
    // the start vector goes to the device once; every later iterate stays
    // there (solve -> Rayleigh quotient -> rescale, engine.cpp / rq_kernels.cu)
    {
      std::vector<HostInt> uh(n);
      const uint32_t* src = u_limbs;
      for (long i = 0; i < n; ++i) {
        const int len = std::abs(u_sizes[i]);
        uh[i].size = u_sizes[i];
        uh[i].limbs.assign(src, src + len);
        src += len;
      }
      mm->set_start(uh);
    }
    Z sigma = Z::from_limbs(sigma_size, sigma_limbs);
    Z rho_prev, d_min, rho;
    bool have_prev = false, have_dmin = false, factored = false;
    int phase = 1;
    const long fbits = final_bits(k);
    int stall = 0;
    long plain = 0;
    std::string tr;
    long it = 0;
    const bool verbose = std::getenv("HGPU_RQI_TRACE") != nullptr;
    double t_factor = 0, t_solve = 0;
    for (; it < max_iter; ++it) {
      auto ta = std::chrono::steady_clock::now();
      if (!factored) {
        std::vector<uint32_t> sl;
        HostInt sx;
        sx.size = sigma.to_limbs(sl);
        sx.limbs = sl;
        try {
          mm->factor(sx, HGPU_KEEP_L);
        } catch (const Error& e) {
          if (e.status == HGPU_ERR_ZERO_PIVOT && e.pivot == n - 1) {
            rho = sigma;  // sigma is an eigenvalue at this precision
            tr += rho.hex() + "\n";
            ++it;
            break;
          }
          throw;
        }
        factored = true;
      }
      auto tb = std::chrono::steady_clock::now();
      long long nl = 0;
      mm->solve_resident(&nl, false);
      // y.u, y.y: 2n products of ~K-bit integers and their exact sums on the
      // device; the host receives the two sums and max bits(y_i)
      long ybits = 0;
      Z num, den;
      {
        HostInt hn, hd;
        mm->rayleigh(hn, hd, ybits, &nl);
        num = from_host(hn);
        den = from_host(hd);
      }
      if (den.sgn() == 0) throw Error(HGPU_ERR_INTERNAL, "solve returned zero");
      rho = sigma + tdiv(shl(num, (unsigned long)k), den);
      tr += rho.hex() + "\n";
      if (verbose) {
        auto tc = std::chrono::steady_clock::now();
        const double f = std::chrono::duration<double>(tb - ta).count();
        const double sv = std::chrono::duration<double>(tc - tb).count();
        t_factor += f;
        t_solve += sv;
        const Z d = rho - rho_prev;
        std::fprintf(stderr, "rqi it %ld %s factor %.3fs solve %.3fs log2|drho/rho| %ld\n",
                     it, phase == 1 ? "plain" : phase == 2 ? "rqi" : "final", f, sv,
                     have_prev ? (long)(d.bits() - rho.bits()) : 0L);
      }
      if (have_prev) {
        Z d = rho - rho_prev;
        if (d.sgn() < 0) d = Z(0) - d;
        const Z a = rho.sgn() < 0 ? Z(0) - rho : rho;
        if (d.sgn() == 0 || cmp(shl(d, (unsigned long)k2), a) <= 0) {
          ++it;
          break;
        }
        if (have_dmin && cmp(d, d_min) >= 0) {
          if (++stall >= kStall) {
            ++it;
            break;
          }
        } else {
          d_min = d;
          have_dmin = true;
        }
        if (phase == 1 && (cmp(shl(d, (unsigned long)kSwitchBits), a) <= 0 ||
                           plain >= kMaxPlain))
          phase = 2;
        else if (phase == 2 && cmp(shl(d, (unsigned long)fbits), a) <= 0)
          phase = 3;
      }
      rho_prev = rho;
      have_prev = true;
      if (phase == 1) ++plain;
      // next start vector: y scaled so that max |u_i| lies in [1/2, 1)
      // (tdiv_2exp(y_i, sh) for sh > 0, else y_i 2^-sh), in place on the device
      mm->rescale_start(ybits - k, &nl);
      if (phase == 2) {
        sigma = rho;
        factored = false;
      }
    }
    if (verbose)
      std::fprintf(stderr, "rqi total factor %.3fs solve %.3fs\n", t_factor, t_solve);
    if (eigenvalue) {
      if (rho.sgn() <= 0)
        throw Error(HGPU_ERR_PRECISION_EXHAUSTED, "non-positive Rayleigh quotient");
      *eigenvalue = dup_c(sig_digits(rho, k, digits, false));
    }
    if (trace) *trace = dup_c(tr);
    if (iterations) *iterations = it;
    if (seconds)
      *seconds = std::chrono::duration<double>(
                     std::chrono::steady_clock::now() - t0).count();
    return HGPU_OK;
  } catch (const Error& e) {
    set_last_error(e.what(), e.pivot);
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what(), -1);
    return HGPU_ERR_INTERNAL;
  }
}
