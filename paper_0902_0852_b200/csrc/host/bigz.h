// Minimal RAII big integer over the GMP mpz ABI, plus the fixed-point and
// decimal semantics of the reference that the driver layer needs:
//   FixedPoint::mul / div truncate toward zero   (fixed_point.cpp:40-71)
//   truncate_sig_digits / round_sig_digits        (decimal.cpp:47-95,143-155)
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "gmp_decl.h"

namespace hgpu {

class Z {
 public:
  Z() { __gmpz_init(z_); }
  explicit Z(long v) { __gmpz_init_set_si(z_, v); }
  Z(const Z& o) { __gmpz_init_set(z_, o.z_); }
  Z(Z&& o) noexcept {
    __gmpz_init(z_);
    __gmpz_swap(z_, o.z_);
  }
  ~Z() { __gmpz_clear(z_); }
  Z& operator=(const Z& o) {
    if (this != &o) __gmpz_set(z_, o.z_);
    return *this;
  }
  Z& operator=(Z&& o) noexcept {
    __gmpz_swap(z_, o.z_);
    return *this;
  }
  hg_mpz_ptr p() { return z_; }
  hg_mpz_srcptr p() const { return z_; }
  int sgn() const { return z_->_mp_size < 0 ? -1 : (z_->_mp_size > 0); }
  long bits() const { return sgn() == 0 ? 0 : (long)__gmpz_sizeinbase(z_, 2); }

  static Z from_limbs(int32_t size, const uint32_t* limbs) {
    Z r;
    const int n = size < 0 ? -size : size;
    if (n) __gmpz_import(r.z_, (size_t)n, -1, 4, 0, 0, limbs);
    if (size < 0) __gmpz_neg(r.z_, r.z_);
    return r;
  }
  int32_t to_limbs(std::vector<uint32_t>& out) const {
    out.assign(((size_t)bits() + 31) / 32 + 1, 0u);
    size_t cnt = 0;
    if (sgn()) __gmpz_export(out.data(), &cnt, -1, 4, 0, 0, z_);
    out.resize(cnt);
    return sgn() < 0 ? -(int32_t)cnt : (int32_t)cnt;
  }
  std::string hex() const {
    char* s = __gmpz_get_str(nullptr, 16, z_);
    std::string r(s);
    std::free(s);
    return r;
  }
  std::string dec() const {
    char* s = __gmpz_get_str(nullptr, 10, z_);
    std::string r(s);
    std::free(s);
    return r;
  }

 private:
  hg_mpz_struct z_[1];
};

inline Z operator+(const Z& a, const Z& b) { Z r; __gmpz_add(r.p(), a.p(), b.p()); return r; }
inline Z operator-(const Z& a, const Z& b) { Z r; __gmpz_sub(r.p(), a.p(), b.p()); return r; }
inline Z operator*(const Z& a, const Z& b) { Z r; __gmpz_mul(r.p(), a.p(), b.p()); return r; }
inline int cmp(const Z& a, const Z& b) { const int c = __gmpz_cmp(a.p(), b.p()); return (c > 0) - (c < 0); }
inline bool operator==(const Z& a, const Z& b) { return cmp(a, b) == 0; }
inline Z shl(const Z& a, unsigned long k) { Z r; __gmpz_mul_2exp(r.p(), a.p(), k); return r; }
inline Z tdiv_2exp(const Z& a, unsigned long k) { Z r; __gmpz_tdiv_q_2exp(r.p(), a.p(), k); return r; }
inline Z tdiv(const Z& a, const Z& b) { Z r; __gmpz_tdiv_q(r.p(), a.p(), b.p()); return r; }
inline Z fdiv(const Z& a, const Z& b) { Z r; __gmpz_fdiv_q(r.p(), a.p(), b.p()); return r; }
inline Z pow10(unsigned long e) { Z r; __gmpz_ui_pow_ui(r.p(), 10, e); return r; }
inline Z pow2(unsigned long e) { Z r(1); return shl(r, e); }

// Fixed-point (mantissa, frac bits K) arithmetic at one shared K.
inline Z fx_mul(const Z& a, const Z& b, long k) { return tdiv_2exp(a * b, (unsigned long)k); }
inline Z fx_div(const Z& a, const Z& b, long k) { return tdiv(shl(a, (unsigned long)k), b); }

// floor(log10(m 2^-f)) for m > 0, exact.
inline long decimal_exponent(const Z& m, long f) {
  const long bits = m.bits();
  long e = (long)__builtin_floor((double)(bits - 1 - f) * 0.30102999566398119521);
  auto lt = [&](long p) {  // m 2^-f < 10^p
    if (p >= 0) return cmp(m, shl(pow10((unsigned long)p), (unsigned long)f)) < 0;
    return cmp(m * pow10((unsigned long)-p), pow2((unsigned long)f)) < 0;
  };
  while (lt(e)) --e;
  while (!lt(e + 1)) ++e;
  return e;
}

// `digits` significant decimal digits of m 2^-f (m > 0), "d.ddde<exp>".
inline std::string sig_digits(const Z& m, long f, int digits, bool nearest) {
  long e = decimal_exponent(m, f);
  auto compute = [&](long t) {
    Z num = m, den = pow2((unsigned long)f);
    if (t >= 0) num = num * pow10((unsigned long)t);
    else den = den * pow10((unsigned long)-t);
    if (!nearest) return tdiv(num, den);
    Z two(2);
    return tdiv_2exp(fdiv(num * two + den, den), 1);  // round half up
  };
  Z d = compute(digits - 1 - e);
  const Z high = pow10((unsigned long)digits), low = pow10((unsigned long)digits - 1);
  while (cmp(d, high) >= 0) d = compute(digits - 1 - (++e));
  while (cmp(d, low) < 0) d = compute(digits - 1 - (--e));
  const std::string ds = d.dec();
  std::string out(1, ds[0]);
  if (digits > 1) out += "." + ds.substr(1);
  return out + "e" + std::to_string(e);
}

}  // namespace hgpu
