// Moment generation: the 2N-1 anti-diagonals
//   M_s = (1/beta) Gamma((1+s)/beta)
// at K fractional bits, as build_matrix / build_interval_matrix produce them
// (hankel_matrix.cpp:13-50), with the Gamma enclosures of gamma.cpp:101-230
// restated in directed integer arithmetic over GMP, bit for bit:
//   * Gamma(a/b) for a/b in (1, 2): r^z e^-r sum_k r^k / (z ... (z+k)) with
//     cutoff r ~ 0.693 (p + 160), e^-r from the factorial series of e and
//     binary powering, every step rounded outward (gamma_base);
//   * other arguments: the recurrence Gamma(z+1) = z Gamma(z) as an exact
//     rational lift onto the base value, at a 1024-bucketed precision that is
//     raised until the enclosure is at most 4 ulps wide (gamma_core);
//   * integer arguments: (m-1)! exactly.
// The distinct base values are computed once; the moments then run on all
// host threads (each is independent).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../../include/hgpu.h"
#include "bigz.h"

namespace hgpu {
void set_last_error(const std::string& s, long pivot);

namespace {

Z fdiv_2exp(const Z& a, long k) {
  Z r;
  __gmpz_fdiv_q_2exp(r.p(), a.p(), (unsigned long)k);
  return r;
}
Z cdiv_2exp(const Z& a, long k) {
  Z r;
  __gmpz_cdiv_q_2exp(r.p(), a.p(), (unsigned long)k);
  return r;
}
Z cdiv(const Z& a, const Z& b) {
  Z r;
  __gmpz_cdiv_q(r.p(), a.p(), b.p());
  return r;
}
Z zu(unsigned long v) {
  Z r;
  __gmpz_set_ui(r.p(), v);
  return r;
}
long nbits(const Z& a) { return (long)__gmpz_sizeinbase(a.p(), 2); }

// value in [lo, hi] 2^-exp2 (gamma.cpp ScaledInterval)
struct SI {
  Z lo, hi;
  long exp2 = 0;
  void normalize(long max_bits) {
    const long b = nbits(hi);
    if (b <= max_bits) return;
    const long s = b - max_bits;
    lo = fdiv_2exp(lo, s);
    hi = cdiv_2exp(hi, s);
    exp2 -= s;
  }
  static SI mul(const SI& a, const SI& b, long max_bits) {
    SI r{a.lo * b.lo, a.hi * b.hi, a.exp2 + b.exp2};
    r.normalize(max_bits);
    return r;
  }
  std::pair<Z, Z> at_scale(long target) const {
    const long s = target - exp2;
    if (s >= 0) return {shl(lo, (unsigned long)s), shl(hi, (unsigned long)s)};
    return {fdiv_2exp(lo, -s), cdiv_2exp(hi, -s)};
  }
};

SI euler_e(long prec) {
  long m = 2, bits = 1;
  while (bits < prec + 4) {
    ++m;
    bits += nbits(zu((unsigned long)m)) - 1;
  }
  const Z unit = pow2((unsigned long)prec);
  Z acc = unit;
  for (long k = m; k >= 1; --k) {
    Z t;
    __gmpz_fdiv_q_ui(t.p(), acc.p(), (unsigned long)k);
    acc = unit + t;
  }
  return {acc, acc + zu((unsigned long)(m + 2)), prec};
}

SI exp_neg(unsigned long r, long prec) {
  const long work = prec + 96;
  const SI e = euler_e(work);
  SI acc{zu(1), zu(1), 0};
  SI base = e;
  const long max_bits = work + 64;
  for (unsigned long k = r; k > 0; k >>= 1) {
    if (k & 1) acc = SI::mul(acc, base, max_bits);
    base = SI::mul(base, base, max_bits);
  }
  const long lo_bits = nbits(acc.lo);
  const long s = work + lo_bits - acc.exp2 + 2;
  const Z num = pow2((unsigned long)(acc.exp2 + s));
  SI inv{fdiv(num, acc.hi), cdiv(num, acc.lo), s};
  inv.normalize(max_bits);
  return inv;
}

std::pair<Z, Z> gamma_base(unsigned long a, unsigned long b, long prec) {
  const long pser = prec + 96;
  const unsigned long r =
      (unsigned long)(((long long)(pser + 64) * 693148LL) / 1000000LL) + 2;
  const Z num0 = pow2((unsigned long)pser) * zu(b);
  Z ulo = fdiv(num0, zu(a)), uhi = cdiv(num0, zu(a));
  Z slo = ulo, shi = uhi;
  const Z rb = zu(r) * zu(b);
  Z divisor = zu(a);
  const unsigned long max_terms = 64 * (pser + r) + 1024;
  const Z one = zu(1), bz = zu(b);
  for (unsigned long k = 1;; ++k) {
    if (k > max_terms) throw std::runtime_error("gamma series failed to converge");
    divisor = divisor + bz;
    ulo = fdiv(ulo * rb, divisor);
    uhi = cdiv(uhi * rb, divisor);
    slo = slo + ulo;
    shi = shi + uhi;
    if (k >= 2 * r && cmp(uhi, one) <= 0) {
      shi = shi + zu(2);
      break;
    }
  }
  const SI sum{slo, shi, pser};
  const unsigned long c = a - b;
  SI rpow{zu(r), zu(r), 0};
  if (c != 0) {
    Z arg;
    __gmpz_ui_pow_ui(arg.p(), r, c);
    arg = shl(arg, (unsigned long)(pser * (long)b));
    Z root;
    __gmpz_root(root.p(), arg.p(), b);
    const SI frac{root, root + one, pser};
    rpow = SI::mul(rpow, frac, pser + 64);
  }
  const SI er = exp_neg(r, pser);
  const long max_bits = pser + 64;
  const SI g = SI::mul(SI::mul(rpow, er, max_bits), sum, max_bits);
  auto lh = g.at_scale(prec);
  lh.second = lh.second + one;
  return lh;
}

struct Key {
  unsigned long num, den;
  long bits;
  bool operator<(const Key& o) const {
    if (num != o.num) return num < o.num;
    if (den != o.den) return den < o.den;
    return bits < o.bits;
  }
};

class GammaCache {
 public:
  std::pair<Z, Z> base(unsigned long a, unsigned long b, long prec) {
    const Key key{a, b, prec};
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = base_.find(key);
      if (it != base_.end()) return it->second;
    }
    auto v = gamma_base(a, b, prec);
    std::lock_guard<std::mutex> lk(mu_);
    return base_.emplace(key, std::move(v)).first->second;
  }

 private:
  std::mutex mu_;
  std::map<Key, std::pair<Z, Z>> base_;
};

struct Lift {
  unsigned long base_num = 0;
  Z num, den;
  long bits = 0;
};

Lift lift_of(unsigned long num, unsigned long den) {
  Lift l;
  l.num = zu(1);
  l.den = zu(1);
  const unsigned long q = num / den;
  if (q >= 1) {
    const unsigned long steps = q - 1;
    l.base_num = num - steps * den;
    for (unsigned long j = 1; j <= steps; ++j)
      __gmpz_mul_ui(l.num.p(), l.num.p(), num - j * den);
    __gmpz_ui_pow_ui(l.den.p(), den, steps);
  } else {
    if (num > ULONG_MAX - den) throw std::runtime_error("gamma argument overflow");
    l.base_num = num + den;
    l.num = zu(den);
    l.den = zu(num);
  }
  l.bits = nbits(l.num) - nbits(l.den);
  return l;
}

long base_prec(long frac_bits, long lift_bits, int attempt) {
  const long prec = frac_bits + 80 + std::max(0L, lift_bits + 8) + 64L * attempt;
  return ((prec + 1023) / 1024) * 1024;
}

// certified enclosure of Gamma(num/den) at 2^frac_bits (gamma_core)
std::pair<Z, Z> gamma_core(GammaCache& cache, unsigned long num,
                           unsigned long den, long frac_bits) {
  if (den == 1) {
    Z f;
    __gmpz_fac_ui(f.p(), num - 1);
    f = shl(f, (unsigned long)frac_bits);
    return {f, f};
  }
  const Lift l = lift_of(num, den);
  for (int attempt = 0;; ++attempt) {
    const long prec = base_prec(frac_bits, l.bits, attempt);
    const auto b = cache.base(l.base_num, den, prec);
    Z lo = fdiv(b.first * l.num, l.den);
    Z hi = cdiv(b.second * l.num, l.den);
    lo = fdiv_2exp(lo, prec - frac_bits);
    hi = cdiv_2exp(hi, prec - frac_bits);
    if (cmp(hi - lo, zu(4)) <= 0) return {lo, hi};
    if (attempt >= 3) throw std::runtime_error("gamma enclosure failed to tighten");
  }
}

unsigned long gcd_u(unsigned long a, unsigned long b) {
  while (b) {
    const unsigned long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

}  // namespace

// The strip of build_matrix (interval == false: round to nearest at K) or
// build_interval_matrix (interval == true: [floor, ceil] at K) for
// beta = bnum/bden.  Throws std::runtime_error on argument overflow.
void build_moments(long n, unsigned long bnum, unsigned long bden, long k,
                   bool interval, std::vector<Z>& lo, std::vector<Z>& hi) {
  if (n < 1 || bnum == 0 || bden == 0)
    throw std::runtime_error("bad moment configuration");
  const unsigned long g = gcd_u(bnum, bden);
  bnum /= g;
  bden /= g;
  const long ns = 2 * n - 1;
  lo.assign(ns, Z());
  hi.assign(ns, Z());
  const long guarded = k + 8;
  GammaCache cache;
  // reduced Gamma arguments (1+s) bden / bnum
  std::vector<std::pair<unsigned long, unsigned long>> args(ns);
  for (long s = 0; s < ns; ++s) {
    const unsigned long kk = (unsigned long)(1 + s);
    if (kk > ULONG_MAX / bden) throw std::runtime_error("gamma argument overflow");
    const unsigned long a = kk * bden, d = bnum, gg = gcd_u(a, d);
    args[s] = {a / gg, d / gg};
  }
  // distinct base values first (the expensive part), in parallel
  {
    std::map<Key, int> bases;
    for (const auto& ad : args)
      if (ad.second != 1) {
        const Lift l = lift_of(ad.first, ad.second);
        bases.emplace(Key{l.base_num, ad.second, base_prec(guarded, l.bits, 0)}, 0);
      }
    std::vector<Key> keys;
    for (const auto& kv : bases) keys.push_back(kv.first);
    std::vector<std::thread> th;
    for (const Key& key : keys)
      th.emplace_back([&cache, key] { cache.base(key.num, key.den, key.bits); });
    for (auto& t : th) t.join();
  }
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  std::vector<std::string> errs(nt);
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        for (long s = t; s < ns; s += nt) {
          const auto gi = gamma_core(cache, args[s].first, args[s].second, guarded);
          // fold in 1/beta = bden/bnum outward (hankel_matrix.cpp:22-25)
          const Z l = fdiv(gi.first * zu(bden), zu(bnum));
          const Z h = cdiv(gi.second * zu(bden), zu(bnum));
          if (interval) {
            lo[s] = fdiv_2exp(l, 8);
            hi[s] = cdiv_2exp(h, 8);
          } else {
            // midpoint, rounded to nearest at K (hankel_matrix.cpp:26-28)
            Z mid = fdiv_2exp(l + h, 1);
            mid = mid + pow2(7);
            lo[s] = fdiv_2exp(mid, 8);
            hi[s] = lo[s];
          }
        }
      } catch (const std::exception& e) {
        errs[t] = e.what();
      }
    });
  for (auto& x : th) x.join();
  for (const auto& e : errs)
    if (!e.empty()) throw std::runtime_error(e);
}

}  // namespace hgpu

namespace {
void pack(const std::vector<hgpu::Z>& v, int32_t** sizes, uint32_t** limbs,
          long* nlimbs) {
  std::vector<int32_t> sz;
  std::vector<uint32_t> lb, tmp;
  for (const hgpu::Z& z : v) {
    sz.push_back(z.to_limbs(tmp));
    lb.insert(lb.end(), tmp.begin(), tmp.end());
  }
  *sizes = static_cast<int32_t*>(std::malloc(sz.size() * sizeof(int32_t) + 1));
  *limbs = static_cast<uint32_t*>(std::malloc(lb.size() * sizeof(uint32_t) + 1));
  if (!*sizes || !*limbs) throw std::bad_alloc();
  std::copy(sz.begin(), sz.end(), *sizes);
  std::copy(lb.begin(), lb.end(), *limbs);
  if (nlimbs) *nlimbs = (long)lb.size();
}
}  // namespace

extern "C" hgpu_status hgpu_build_moments(long n, unsigned long beta_num,
                                          unsigned long beta_den, long frac_bits,
                                          int interval, int32_t** lo_sizes,
                                          uint32_t** lo_limbs,
                                          int32_t** hi_sizes,
                                          uint32_t** hi_limbs) {
  try {
    if (n < 1 || n > 100000 || frac_bits < 0 || !lo_sizes || !lo_limbs)
      throw std::invalid_argument("bad argument");
    std::vector<hgpu::Z> lo, hi;
    hgpu::build_moments(n, beta_num, beta_den, frac_bits, interval != 0, lo, hi);
    pack(lo, lo_sizes, lo_limbs, nullptr);
    if (hi_sizes && hi_limbs) pack(hi, hi_sizes, hi_limbs, nullptr);
    return HGPU_OK;
  } catch (const std::invalid_argument& e) {
    hgpu::set_last_error(e.what(), -1);
    return HGPU_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    hgpu::set_last_error(e.what(), -1);
    return HGPU_ERR_INVALID_ARGUMENT;
  }
}

extern "C" void hgpu_buffer_free(void* p) { std::free(p); }
