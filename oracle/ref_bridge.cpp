// extern "C" bridge over the reference sources compiled unchanged from
// /root/reference/proj/src (see oracle/Makefile).  TEST INFRASTRUCTURE ONLY:
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load this library as the checker or as the timed CPU
// baseline; the product never links it.
//
// Numbers cross the boundary as signed hexadecimal strings (GMP get_str(16)),
// so the Python side can parse them into exact ints.  Every function returns
// a malloc'd string that the caller releases with oref_free; failures are
// reported in-band as "error <kind> <detail>".
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "assignment.hpp"
#include "channel.hpp"
#include "decimal.hpp"
#include "driver.hpp"
#include "hankel_matrix.hpp"
#include "ldlt.hpp"
#include "verify.hpp"
#include "secant.hpp"
#include "timing.hpp"

using namespace heig;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

HankelMatrix load(const char* dump) {
  std::istringstream is(dump);
  return load_matrix_dump(is);
}

FixedPoint fixed_from_hex(const char* hex, long k) {
  return FixedPoint(mpz_class(std::string(hex), 16), k);
}

template <typename F>
char* guarded(F&& f) {
  try {
    return dup(f());
  } catch (const ZeroPivot& zp) {
    return dup("error ZeroPivot " + std::to_string(zp.pivot_index) + " " +
               std::to_string(zp.frac_bits));
  } catch (const std::exception& e) {
    return dup(std::string("error exception ") + e.what());
  }
}

}  // namespace

extern "C" {

void oref_free(char* p) { std::free(p); }

// build_matrix(n, p/q, k) -> dump text (hankel_matrix.cpp:13-31, :52-57).
char* oref_build_strip(long n, unsigned long bnum, unsigned long bden,
                       long k) {
  return guarded([&] {
    HankelMatrix m = build_matrix(n, Rational(bnum, bden), k);
    std::ostringstream os;
    dump_matrix(m, os);
    return os.str();
  });
}

// build_interval_matrix -> "s lo_hex hi_hex" lines (hankel_matrix.cpp:33-50).
char* oref_build_interval_strip(long n, unsigned long bnum, unsigned long bden,
                                long k) {
  return guarded([&] {
    HankelIntervalMatrix m = build_interval_matrix(n, Rational(bnum, bden), k);
    std::ostringstream os;
    for (long s = 0; s < 2 * n - 1; ++s)
      os << s << " " << m.anti_diagonal(s).lo().mantissa().get_str(16) << " "
         << m.anti_diagonal(s).hi().mantissa().get_str(16) << "\n";
    return os.str();
  });
}

// ldlt_det_serial with LdltCapture (ldlt.cpp:31-77).  Output lines:
//   det <hex>
//   pivot <p> <hex>            (workspace precision K)
//   ratio <p> <r> <hex>        (half precision K/2), only if capture != 0
char* oref_ldlt_serial(const char* dump, const char* x_hex, int capture) {
  return guarded([&] {
    HankelMatrix m = load(dump);
    FixedPoint x = fixed_from_hex(x_hex, m.frac_bits());
    LdltCapture cap;
    FixedPoint det = ldlt_det_serial(m, x, capture ? &cap : nullptr);
    std::ostringstream os;
    os << "det " << det.mantissa().get_str(16) << "\n";
    if (capture) {
      for (size_t p = 0; p < cap.pivots.size(); ++p)
        os << "pivot " << p << " " << cap.pivots[p].mantissa().get_str(16)
           << "\n";
      for (size_t p = 0; p < cap.ratio_columns.size(); ++p)
        for (size_t i = 0; i < cap.ratio_columns[p].size(); ++i)
          os << "ratio " << p << " " << (p + 1 + i) << " "
             << cap.ratio_columns[p][i].mantissa().get_str(16) << "\n";
    }
    return os.str();
  });
}

// ldlt_det_parallel with the unthrottled in-process channel
// (ldlt.cpp:315-341, channel.cpp:10-47).  Output: "det <hex>\nseconds <s>".
char* oref_ldlt_parallel(const char* dump, const char* x_hex, long workers) {
  return guarded([&] {
    HankelMatrix m = load(dump);
    FixedPoint x = fixed_from_hex(x_hex, m.frac_bits());
    SharedMemoryChannel ch;
    ParallelDetResult r = ldlt_det_parallel(m, x, workers, ch);
    std::ostringstream os;
    os << "det " << r.determinant.mantissa().get_str(16) << "\n"
       << "seconds " << r.timing.total_seconds << "\n";
    return os.str();
  });
}

// Sign of det(M - xI) for a decimal probe, via the plain LDL^T at the matrix
// precision (decimal.cpp decimal_to_fixed_floor, ldlt.cpp:31-77).
char* oref_det_sign_decimal(const char* dump, const char* decimal) {
  return guarded([&] {
    HankelMatrix m = load(dump);
    FixedPoint x = decimal_to_fixed_floor(decimal, m.frac_bits());
    FixedPoint det = ldlt_det_serial(m, x);
    return std::to_string(det.sign());
  });
}

// Same sign through the reference's multi-worker path (ldlt.cpp:315-341,
// SharedMemoryChannel): the only practical CPU route at configs 4/5.
// Output: "sign <s>\nbits <log2|det|>\nseconds <wall>".
char* oref_det_sign_parallel_decimal(const char* dump, const char* decimal,
                                     long workers) {
  return guarded([&] {
    HankelMatrix m = load(dump);
    FixedPoint x = decimal_to_fixed_floor(decimal, m.frac_bits());
    SharedMemoryChannel ch;
    ParallelDetResult r = ldlt_det_parallel(m, x, workers, ch);
    std::ostringstream os;
    os << "sign " << r.determinant.sign() << "\n"
       << "bits " << mpz_sizeinbase(r.determinant.mantissa().get_mpz_t(), 2) << "\n"
       << "seconds " << r.timing.total_seconds << "\n";
    return os.str();
  });
}

// Interval-certified sign of det(M - aI) for a decimal probe a at kv bits
// (hankel_matrix.cpp:33-50, decimal.cpp decimal_to_interval,
// ldlt.cpp:79-152).  "1", "-1", "0" (straddles) or a ZeroPivot error.
char* oref_interval_sign_decimal(long n, unsigned long bnum, unsigned long bden,
                                 long kv, const char* decimal) {
  return guarded([&] {
    HankelIntervalMatrix m = build_interval_matrix(n, Rational(bnum, bden), kv);
    FixedInterval a = decimal_to_interval(decimal, kv);
    FixedInterval det = ldlt_det_interval(m, a);
    Sign s = FixedInterval::sign(det);
    return std::string(s == Sign::Positive ? "1"
                                           : (s == Sign::Negative ? "-1" : "0"));
  });
}

// ldlt_det_interval (ldlt.cpp:79-152) on a given interval strip.  `strip`
// lines: "<lo_hex> <hi_hex>" per anti-diagonal at k fractional bits; the
// shift is [xlo, xhi].  Output: "det <lo_hex> <hi_hex>" (or the error line).
char* oref_ldlt_interval(const char* strip, long k, const char* xlo_hex,
                         const char* xhi_hex) {
  return guarded([&] {
    std::istringstream is(strip);
    std::vector<FixedInterval> ad;
    std::string lo, hi;
    while (is >> lo >> hi)
      ad.emplace_back(fixed_from_hex(lo.c_str(), k), fixed_from_hex(hi.c_str(), k));
    const long n = ((long)ad.size() + 1) / 2;
    HankelIntervalMatrix m(n, Rational(1, 1), k, std::move(ad));
    FixedInterval x(fixed_from_hex(xlo_hex, k), fixed_from_hex(xhi_hex, k));
    FixedInterval det = ldlt_det_interval(m, x);
    std::ostringstream os;
    os << "det " << det.lo().mantissa().get_str(16) << " "
       << det.hi().mantissa().get_str(16) << "\n";
    return os.str();
  });
}

// decimal_to_interval (decimal.cpp:166-180): "<lo_hex> <hi_hex>".
char* oref_decimal_to_interval(const char* s, long frac_bits) {
  return guarded([&] {
    FixedInterval v = decimal_to_interval(s, frac_bits);
    return v.lo().mantissa().get_str(16) + " " + v.hi().mantissa().get_str(16);
  });
}

// verify_eigenvalue (verify.cpp:8-42) on build_interval_matrix(n, beta, kv):
// "<status> <lower_sign> <upper_sign> <probe_low> <probe_high> <lower_exact_zero>" with status
// 0 verified, 1 refuted, 2 inconclusive and signs 1/-1/0 (0: indeterminate).
char* oref_verify(long n, unsigned long bnum, unsigned long bden, long kv,
                  const char* x_decimal) {
  return guarded([&] {
    HankelIntervalMatrix m = build_interval_matrix(n, Rational(bnum, bden), kv);
    FixedPoint x = decimal_to_fixed_floor(x_decimal, kv);
    VerifyOutcome o = verify_eigenvalue(m, x);
    auto sg = [](Sign s) {
      return s == Sign::Positive ? "1" : (s == Sign::Negative ? "-1" : "0");
    };
    std::ostringstream os;
    os << (o.status == VerifyStatus::Verified ? 0
           : o.status == VerifyStatus::Refuted ? 1 : 2)
       << " " << sg(o.lower_sign) << " " << sg(o.upper_sign) << " "
       << o.probe_low << " " << o.probe_high << " " << (o.lower_exact_zero ? 1 : 0);
    return os.str();
  });
}

// Secant iteration on the plain serial determinant (secant.cpp:27-117).
// Output lines: "iterate <x_hex> <det_hex>" per recorded iterate, then
// "eigenvalue <15 digits>", "iterations <n>", "exact_root_hit <0|1>".
char* oref_secant(const char* dump) {
  return guarded([&] {
    HankelMatrix m = load(dump);
    long k = m.frac_bits();
    DetEvaluator eval = [&](const FixedPoint& x) {
      return ldlt_det_serial(m, x);
    };
    SecantTrace tr = secant_smallest_eigenvalue(m, eval, k);
    std::ostringstream os;
    for (const SecantIterate& it : tr.iterates)
      os << "iterate " << it.x.mantissa().get_str(16) << " "
         << it.det.mantissa().get_str(16) << "\n";
    os << "eigenvalue " << truncate_sig_digits(tr.eigenvalue(), 15) << "\n"
       << "iterations " << tr.iterations << "\n"
       << "exact_root_hit " << (tr.exact_root_hit ? 1 : 0) << "\n";
    return os.str();
  });
}

// Decimal helpers (decimal.cpp:143-180) with a caller-chosen digit count, so
// the parity harness can compare more than the reference's 15 digits.
char* oref_truncate_sig_digits(const char* x_hex, long frac_bits, int digits) {
  return guarded([&] {
    return truncate_sig_digits(fixed_from_hex(x_hex, frac_bits), digits);
  });
}
char* oref_bump_last_digit(const char* s) {
  return guarded([&] { return bump_last_digit(s); });
}
char* oref_decimal_to_fixed_floor(const char* s, long frac_bits) {
  return guarded([&] {
    return decimal_to_fixed_floor(s, frac_bits).mantissa().get_str(16);
  });
}

// Reflected round-robin owner map (assignment.hpp:15-23): "o0 o1 ...".
char* oref_column_owners(long n, long workers) {
  return guarded([&] {
    ColumnAssignment a(n, workers);
    std::ostringstream os;
    for (long o : a.owners()) os << o << " ";
    return os.str();
  });
}

}  // extern "C"
