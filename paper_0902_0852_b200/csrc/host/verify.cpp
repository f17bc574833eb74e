// Certification of a computed lambda_min (verify_eigenvalue, verify.cpp:8-42)
// on the GPU interval LDL^T: with a = x (a decimal string) truncated to
// `digits` significant digits and b = a + one unit in the last digit, Verified means
// det(M - aI) > 0 and det(M - bI) < 0 as enclosed by ldlt_det_interval, i.e.
// lambda_1 lies in [a, b).  The decimal helpers mirror decimal.cpp
// (DecimalSci::parse :112-141, bump_last_digit :155-164,
// decimal_to_interval :166-180).
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../../include/hgpu.h"
#include "../engine.h"
#include "bigz.h"

namespace hgpu {
Matrix* matrix_impl(hgpu_matrix* m);
void set_last_error(const std::string& s, long pivot);

namespace {

struct Sci {
  Z digits;
  int num_digits = 0;
  long exponent = 0;
};

// "D[.D+]e[-]E" (decimal.cpp:112-141)
Sci parse_sci(const std::string& s) {
  auto fail = [&]() -> Sci {
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "malformed decimal: " + s);
  };
  size_t i = 0;
  if (s.empty() || !std::isdigit((unsigned char)s[0])) return fail();
  std::string digs(1, s[i++]);
  if (i < s.size() && s[i] == '.') {
    const size_t start = ++i;
    while (i < s.size() && std::isdigit((unsigned char)s[i])) digs += s[i++];
    if (i == start) return fail();
  }
  if (i >= s.size() || s[i] != 'e') return fail();
  const size_t exp_start = ++i;
  if (i < s.size() && s[i] == '-') ++i;
  const size_t dig_start = i;
  while (i < s.size() && std::isdigit((unsigned char)s[i])) ++i;
  if (i != s.size() || dig_start == i) return fail();
  Sci d;
  __gmpz_set_str(d.digits.p(), digs.c_str(), 10);
  d.num_digits = (int)digs.size();
  d.exponent = std::strtol(s.c_str() + exp_start, nullptr, 10);
  return d;
}

std::string sci_string(const Sci& d) {
  const std::string ds = d.digits.dec();
  std::string out(1, ds[0]);
  if (ds.size() > 1) out += "." + ds.substr(1);
  return out + "e" + std::to_string(d.exponent);
}

std::string bump_last_digit(const std::string& s) {
  Sci d = parse_sci(s);
  d.digits = d.digits + Z(1);
  if (cmp(d.digits, pow10((unsigned long)d.num_digits)) >= 0) {
    d.digits = tdiv(d.digits, Z(10));  // 9.99 -> 1.00, exponent + 1
    d.exponent += 1;
  }
  return sci_string(d);
}

// [floor, ceil] of the decimal at frac_bits
void decimal_to_interval(const std::string& s, long frac_bits, Z& lo, Z& hi) {
  const Sci d = parse_sci(s);
  const long p = d.exponent - d.num_digits + 1;  // value = digits 10^p
  if (p >= 0) {
    lo = shl(d.digits * pow10((unsigned long)p), (unsigned long)frac_bits);
    hi = lo;
    return;
  }
  const Z num = shl(d.digits, (unsigned long)frac_bits);
  const Z den = pow10((unsigned long)-p);
  lo = fdiv(num, den);
  Z c;
  __gmpz_cdiv_q(c.p(), num.p(), den.p());
  hi = c;
}

HostInt host_int(const Z& z) {
  HostInt h;
  h.size = z.to_limbs(h.limbs);
  return h;
}

char* dup_c(const std::string& s) {
  char* o = static_cast<char*>(std::malloc(s.size() + 1));
  if (o) std::memcpy(o, s.c_str(), s.size() + 1);
  return o;
}

}  // namespace
}  // namespace hgpu

extern "C" hgpu_status hgpu_verify_eigenvalue(hgpu_matrix* m,
                                              const char* x_decimal, int digits,
                                              int* status, int* lower_sign,
                                              int* upper_sign,
                                              char** probe_low,
                                              char** probe_high) {
  return hgpu_verify_eigenvalue_ex(m, x_decimal, digits, status, lower_sign,
                                   upper_sign, nullptr, probe_low, probe_high);
}

extern "C" hgpu_status hgpu_verify_eigenvalue_ex(hgpu_matrix* m,
                                                 const char* x_decimal, int digits,
                                                 int* status, int* lower_sign,
                                                 int* upper_sign,
                                                 int* lower_exact_zero,
                                                 char** probe_low,
                                                 char** probe_high) {
  using namespace hgpu;
  try {
    Matrix* mm = matrix_impl(m);
    if (!mm || !x_decimal || digits < 1)
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad argument");
    if (!mm->is_interval())
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "verify needs an interval matrix");
    const long kv = mm->frac_bits();
    // a = x truncated to `digits` significant digits (truncate_sig_digits of
    // the decimal's exact value: its digit string cut or zero-padded)
    Sci xs = parse_sci(x_decimal);
    if (xs.digits.sgn() <= 0)
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "verify needs x > 0");
    {
      std::string ds = xs.digits.dec();
      if ((int)ds.size() != xs.num_digits)
        throw Error(HGPU_ERR_INVALID_ARGUMENT, "verify needs d.ddd...e<exp> with d != 0");
      if ((int)ds.size() > digits) ds.resize(digits);
      while ((int)ds.size() < digits) ds += '0';
      __gmpz_set_str(xs.digits.p(), ds.c_str(), 10);
      xs.num_digits = digits;
    }
    const std::string a = sci_string(xs);
    const std::string b = bump_last_digit(a);
    int ls = 0, us = 0, st = 2;  // 0 verified, 1 refuted, 2 inconclusive
    bool lz = false;  // det(M - aI) == [0, 0] (verify.cpp:26-27)
    try {
      Z alo, ahi, blo, bhi;
      decimal_to_interval(a, kv, alo, ahi);
      decimal_to_interval(b, kv, blo, bhi);
      const FactorResult ra = mm->factor_interval(host_int(alo), host_int(ahi), 0);
      ls = ra.det_sign;
      lz = ra.det_exact_zero;
      us = mm->factor_interval(host_int(blo), host_int(bhi), 0).det_sign;
      if (ls > 0 && us < 0) st = 0;
      else if (ls < 0 || us > 0) st = 1;
    } catch (const Error& e) {
      // a pivot enclosure straddled zero: not enough precision
      if (e.status != HGPU_ERR_ZERO_PIVOT) throw;
      st = 2;
    }
    if (status) *status = st;
    if (lower_sign) *lower_sign = ls;
    if (upper_sign) *upper_sign = us;
    if (lower_exact_zero) *lower_exact_zero = lz ? 1 : 0;
    if (probe_low) *probe_low = dup_c(a);
    if (probe_high) *probe_high = dup_c(b);
    return HGPU_OK;
  } catch (const Error& e) {
    set_last_error(e.what(), e.pivot);
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what(), -1);
    return HGPU_ERR_INTERNAL;
  }
}
