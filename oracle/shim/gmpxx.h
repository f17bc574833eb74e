// Minimal C++ value class over the GMP mpz ABI, written for the oracle build
// only (test infrastructure, never the product path).  It provides the subset
// of the gmpxx `mpz_class` surface the reference sources use: construction
// from machine integers and strings, arithmetic/shift/bitwise operators,
// comparisons, get_str/get_mpz_t, and the free functions sgn/abs/cmp/swap.
// gmpxx semantics are kept where they matter for bit-exactness:
//   operator/ and operator% truncate toward zero (mpz_tdiv_q / mpz_tdiv_r),
//   operator>> floors (mpz_fdiv_q_2exp).
#ifndef ORACLE_SHIM_GMPXX_H
#define ORACLE_SHIM_GMPXX_H

#include <cstdlib>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

#include "gmp.h"

class mpz_class {
 public:
  mpz_class() { mpz_init(z_); }
  mpz_class(const mpz_class& o) { mpz_init_set(z_, o.z_); }
  mpz_class(mpz_class&& o) noexcept {
    mpz_init(z_);
    mpz_swap(z_, o.z_);
  }
  template <typename T,
            typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
  mpz_class(T v) {
    if (std::is_signed<T>::value)
      mpz_init_set_si(z_, static_cast<long>(v));
    else
      mpz_init_set_ui(z_, static_cast<unsigned long>(v));
  }
  explicit mpz_class(double d) {
    mpz_init(z_);
    mpz_set_d(z_, d);
  }
  explicit mpz_class(const char* s, int base = 0) {
    mpz_init(z_);
    if (mpz_set_str(z_, s, base) != 0) {
      mpz_clear(z_);
      throw std::invalid_argument("mpz_set_str");
    }
  }
  explicit mpz_class(const std::string& s, int base = 0)
      : mpz_class(s.c_str(), base) {}
  explicit mpz_class(mpz_srcptr p) { mpz_init_set(z_, p); }
  ~mpz_class() { mpz_clear(z_); }

  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) mpz_set(z_, o.z_);
    return *this;
  }
  mpz_class& operator=(mpz_class&& o) noexcept {
    mpz_swap(z_, o.z_);
    return *this;
  }
  template <typename T,
            typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
  mpz_class& operator=(T v) {
    if (std::is_signed<T>::value)
      mpz_set_si(z_, static_cast<long>(v));
    else
      mpz_set_ui(z_, static_cast<unsigned long>(v));
    return *this;
  }

  mpz_ptr get_mpz_t() { return z_; }
  mpz_srcptr get_mpz_t() const { return z_; }

  std::string get_str(int base = 10) const {
    char* p = mpz_get_str(nullptr, base, z_);
    std::string s(p);
    std::free(p);
    return s;
  }
  long get_si() const { return mpz_get_si(z_); }
  unsigned long get_ui() const { return mpz_get_ui(z_); }
  double get_d() const { return mpz_get_d(z_); }

  mpz_class& operator+=(const mpz_class& o) { mpz_add(z_, z_, o.z_); return *this; }
  mpz_class& operator-=(const mpz_class& o) { mpz_sub(z_, z_, o.z_); return *this; }
  mpz_class& operator*=(const mpz_class& o) { mpz_mul(z_, z_, o.z_); return *this; }
  mpz_class& operator/=(const mpz_class& o) { mpz_tdiv_q(z_, z_, o.z_); return *this; }
  mpz_class& operator%=(const mpz_class& o) { mpz_tdiv_r(z_, z_, o.z_); return *this; }
  mpz_class& operator&=(const mpz_class& o) { mpz_and(z_, z_, o.z_); return *this; }
  mpz_class& operator|=(const mpz_class& o) { mpz_ior(z_, z_, o.z_); return *this; }
  mpz_class& operator^=(const mpz_class& o) { mpz_xor(z_, z_, o.z_); return *this; }
  mpz_class& operator<<=(unsigned long b) { mpz_mul_2exp(z_, z_, b); return *this; }
  mpz_class& operator>>=(unsigned long b) { mpz_fdiv_q_2exp(z_, z_, b); return *this; }
  mpz_class& operator++() { mpz_add_ui(z_, z_, 1); return *this; }
  mpz_class& operator--() { mpz_sub_ui(z_, z_, 1); return *this; }
  mpz_class operator++(int) { mpz_class t(*this); ++*this; return t; }
  mpz_class operator--(int) { mpz_class t(*this); --*this; return t; }

  mpz_class operator-() const { mpz_class r; mpz_neg(r.z_, z_); return r; }
  mpz_class operator+() const { return *this; }

 private:
  mpz_t z_;
};

#define ORACLE_MPZ_BINOP(op, fn)                                           \
  inline mpz_class operator op(const mpz_class& a, const mpz_class& b) {   \
    mpz_class r;                                                           \
    fn(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t());                       \
    return r;                                                              \
  }
ORACLE_MPZ_BINOP(+, mpz_add)
ORACLE_MPZ_BINOP(-, mpz_sub)
ORACLE_MPZ_BINOP(*, mpz_mul)
ORACLE_MPZ_BINOP(/, mpz_tdiv_q)
ORACLE_MPZ_BINOP(%, mpz_tdiv_r)
ORACLE_MPZ_BINOP(&, mpz_and)
ORACLE_MPZ_BINOP(|, mpz_ior)
ORACLE_MPZ_BINOP(^, mpz_xor)
#undef ORACLE_MPZ_BINOP

// Mixed operands with machine integers go through a temporary mpz_class.
#define ORACLE_MPZ_MIXED(op)                                                  \
  template <typename T, typename std::enable_if<std::is_integral<T>::value,   \
                                                int>::type = 0>               \
  inline mpz_class operator op(const mpz_class& a, T b) {                     \
    return a op mpz_class(b);                                                 \
  }                                                                           \
  template <typename T, typename std::enable_if<std::is_integral<T>::value,   \
                                                int>::type = 0>               \
  inline mpz_class operator op(T a, const mpz_class& b) {                     \
    return mpz_class(a) op b;                                                 \
  }
ORACLE_MPZ_MIXED(+)
ORACLE_MPZ_MIXED(-)
ORACLE_MPZ_MIXED(*)
ORACLE_MPZ_MIXED(/)
ORACLE_MPZ_MIXED(%)
#undef ORACLE_MPZ_MIXED

inline mpz_class operator<<(const mpz_class& a, unsigned long b) {
  mpz_class r;
  mpz_mul_2exp(r.get_mpz_t(), a.get_mpz_t(), b);
  return r;
}
inline mpz_class operator>>(const mpz_class& a, unsigned long b) {
  mpz_class r;
  mpz_fdiv_q_2exp(r.get_mpz_t(), a.get_mpz_t(), b);
  return r;
}
template <typename T,
          typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
inline mpz_class operator<<(const mpz_class& a, T b) {
  return a << static_cast<unsigned long>(b);
}
template <typename T,
          typename std::enable_if<std::is_integral<T>::value, int>::type = 0>
inline mpz_class operator>>(const mpz_class& a, T b) {
  return a >> static_cast<unsigned long>(b);
}

inline int cmp(const mpz_class& a, const mpz_class& b) {
  int c = mpz_cmp(a.get_mpz_t(), b.get_mpz_t());
  return c < 0 ? -1 : (c > 0 ? 1 : 0);
}
#define ORACLE_MPZ_CMP(op)                                                    \
  inline bool operator op(const mpz_class& a, const mpz_class& b) {           \
    return mpz_cmp(a.get_mpz_t(), b.get_mpz_t()) op 0;                        \
  }                                                                           \
  template <typename T, typename std::enable_if<std::is_integral<T>::value,   \
                                                int>::type = 0>               \
  inline bool operator op(const mpz_class& a, T b) {                          \
    return mpz_cmp(a.get_mpz_t(), mpz_class(b).get_mpz_t()) op 0;             \
  }                                                                           \
  template <typename T, typename std::enable_if<std::is_integral<T>::value,   \
                                                int>::type = 0>               \
  inline bool operator op(T a, const mpz_class& b) {                          \
    return mpz_cmp(mpz_class(a).get_mpz_t(), b.get_mpz_t()) op 0;             \
  }
ORACLE_MPZ_CMP(==)
ORACLE_MPZ_CMP(!=)
ORACLE_MPZ_CMP(<)
ORACLE_MPZ_CMP(<=)
ORACLE_MPZ_CMP(>)
ORACLE_MPZ_CMP(>=)
#undef ORACLE_MPZ_CMP

inline int sgn(const mpz_class& a) { return mpz_sgn(a.get_mpz_t()); }
inline mpz_class abs(const mpz_class& a) {
  mpz_class r;
  mpz_abs(r.get_mpz_t(), a.get_mpz_t());
  return r;
}
inline mpz_class sqrt(const mpz_class& a) {
  mpz_class r;
  mpz_sqrt(r.get_mpz_t(), a.get_mpz_t());
  return r;
}
inline void swap(mpz_class& a, mpz_class& b) { mpz_swap(a.get_mpz_t(), b.get_mpz_t()); }

inline std::ostream& operator<<(std::ostream& os, const mpz_class& a) {
  return os << a.get_str(10);
}

#endif
