// Host driver on the B200 determinant: secant smallest eigenvalue with
// precision escalation (/root/reference/proj/src/driver.cpp:80-178) and the
// reference's whole-run C ABI (include/hankel_eig.h).  Every determinant
// probe is a GPU LDL^T factorisation plus the GPU determinant fold.
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <new>
#include <optional>
#include <sstream>
#include <string>

#include "../../../include/hankel_eig.h"
#include "../../../include/hgpu.h"
#include "../engine.h"
#include "secant.h"

namespace hgpu {

// host/moments.cpp
void build_moments(long n, unsigned long bnum, unsigned long bden, long k,
                   bool interval, std::vector<Z>& lo, std::vector<Z>& hi);

namespace {

struct Rational {
  unsigned long num = 1, den = 1;
  std::string str() const { return std::to_string(num) + "/" + std::to_string(den); }
};

unsigned long gcd_ul(unsigned long a, unsigned long b) {
  while (b) {
    const unsigned long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// "p/q" or "p" in lowest terms; anything else rejected (rational.hpp:33-49)
Rational parse_rational(const std::string& s) {
  auto digits = [](const std::string& t) {
    if (t.empty()) return false;
    for (char c : t)
      if (c < '0' || c > '9') return false;
    return true;
  };
  const size_t slash = s.find('/');
  const std::string p = slash == std::string::npos ? s : s.substr(0, slash);
  const std::string q = slash == std::string::npos ? "1" : s.substr(slash + 1);
  if (!digits(p) || !digits(q))
    throw std::invalid_argument("expected rational p/q, got '" + s + "'");
  const unsigned long pn = std::stoul(p), qn = std::stoul(q);
  if (pn == 0 || qn == 0) throw std::invalid_argument("rational must be positive");
  const unsigned long g = gcd_ul(pn, qn);
  return {pn / g, qn / g};
}

struct RunConfig {
  long n = 1;
  Rational beta;
  long k_bits = 0;
  long workers = 1;
  double net_bandwidth = std::numeric_limits<double>::infinity();
  double net_latency_ms = 0;
  bool verify = true;
  std::string dump_path;
};

struct RunResult {
  long n = 0, k_bits = 0, kv_bits = 0, workers = 1, iterations = 0;
  Rational beta;
  std::string eigenvalue, condition_lower_bound, diagnosis;
  bool verified = false;
  double total_s = 0, compute_s = 0, net_s = 0, div_s = 0;
};

struct InvalidConfig : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PrecisionCap : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Refuted : std::runtime_error {  // errors.hpp:102-105
  using std::runtime_error::runtime_error;
};

// choose_initial_precision (driver.cpp:15-21): max(512, 8n, 4n ceil(1/beta)),
// rounded up to a multiple of 64.
long initial_precision(long n, const Rational& b) {
  const long inv_ceil = (long)((b.den + b.num - 1) / b.num);
  const long k = std::max({512L, 8 * n, 4 * n * std::max(1L, inv_ceil)});
  return ((k + 63) / 64) * 64;
}

long precision_cap() {
  if (const char* env = std::getenv("HANKEL_EIG_PRECISION_CAP")) {
    char* end = nullptr;
    const long cap = std::strtol(env, &end, 10);
    if (end && *end == '\0' && cap >= 64) return cap;
    throw InvalidConfig("HANKEL_EIG_PRECISION_CAP must be an integer >= 64");
  }
  return 1L << 21;
}

long escalate(long k, long cap) {
  if (2 * k > cap)
    throw PrecisionCap("precision escalation to " + std::to_string(2 * k) +
                       " bits exceeds cap " + std::to_string(cap));
  return 2 * k;
}

// Moments (1/beta) Gamma((1+s)/beta) at K bits when the Gamma arguments are
// integers (1/beta = m integral): m * (m(1+s)-1)!, exact, which is what the
// reference's build_matrix yields there (hankel_matrix.cpp:13-31).
// build_matrix (hankel_matrix.cpp:13-31): every beta, through the Gamma
// enclosures restated in host/moments.cpp (exact factorials when 1/beta is
// integral).
std::vector<Z> exact_moments(long n, const Rational& b, long k) {
  std::vector<Z> lo, hi;
  build_moments(n, b.num, b.den, k, false, lo, hi);
  return lo;
}

// workers (driver.cpp:102-114: one thread per worker in ldlt_det_parallel)
// -> column-block-cyclic ranks, one per GPU from HGPU_DEVICE on, at most the
// devices present.  HGPU_RANK_DEVICES="d0,d1,..." names the rank devices
// explicitly (a device may repeat: the multi-rank schedule on one GPU).
std::vector<int> rank_devices(long workers, int base) {
  std::vector<int> devs;
  if (const char* e = std::getenv("HGPU_RANK_DEVICES")) {
    for (const char* c = e; *c;) {
      char* end = nullptr;
      const long d = std::strtol(c, &end, 10);
      if (end == c) break;
      devs.push_back((int)d);
      c = *end == ',' ? end + 1 : end;
    }
    if (!devs.empty()) return devs;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 1;
  const long w = std::max(1L, std::min<long>(workers, (long)ndev - base));
  for (long i = 0; i < w; ++i) devs.push_back(base + (int)i);
  return devs;
}

std::unique_ptr<Matrix> upload(const std::vector<Z>& strip, long k, int device) {
  std::vector<int32_t> sizes;
  std::vector<uint32_t> limbs, tmp;
  for (const Z& z : strip) {
    sizes.push_back(z.to_limbs(tmp));
    limbs.insert(limbs.end(), tmp.begin(), tmp.end());
  }
  auto m = std::make_unique<Matrix>((int)((strip.size() + 1) / 2), (int)k,
                                    sizes.data(), limbs.data(), device);
  return m;
}

// The DetEvaluator: GPU factorisation + GPU fold (ldlt_det_serial semantics).
DetFn gpu_det(Matrix& m, long k, double* seconds, double* net = nullptr) {
  return [&m, k, seconds, net](const Z& x) -> Z {
    std::vector<uint32_t> xl;
    HostInt xi;
    xi.size = x.to_limbs(xl);
    xi.limbs = xl;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      FactorResult r = m.factor(xi, HGPU_FOLD);
      // timing.hpp:7-39: {net} is the receivers' wait for and pull of the
      // published panels (per-rank average, CUDA events); receivers never
      // divide (every ratio comes from the owner), so {d} stays 0 as with
      // the reference's unthrottled channel; {c} is the rest
      const double nets = r.net_ms * 1e-3 / std::max(1, m.world());
      if (net) *net += nets;
      if (seconds)
        *seconds += std::chrono::duration<double>(
                        std::chrono::steady_clock::now() - t0).count() - nets;
      return Z::from_limbs(r.det.size, r.det.limbs.data());
    } catch (const Error& e) {
      if (seconds)
        *seconds += std::chrono::duration<double>(
                        std::chrono::steady_clock::now() - t0).count();
      if (e.status == HGPU_ERR_ZERO_PIVOT) {
        SecantError se(SecantError::ZeroPivot, e.what());
        se.pivot = e.pivot;
        throw se;
      }
      throw;
    }
  };
}

int device_from_env() {
  if (const char* d = std::getenv("HGPU_DEVICE")) return std::atoi(d);
  return 0;
}

RunResult run(const RunConfig& cfg) {
  if (cfg.n < 1) throw InvalidConfig("order must be >= 1");
  if (cfg.workers < 1) throw InvalidConfig("workers must be >= 1");
  if (cfg.k_bits != 0) {
    if (cfg.k_bits < 64) throw InvalidConfig("precision must be >= 64 bits");
    if (cfg.k_bits % 2 != 0)
      throw InvalidConfig("precision must be even (column buffers carry half)");
  }
  if (!(cfg.net_bandwidth > 0))
    throw InvalidConfig("net bandwidth must be positive or inf");
  if (cfg.net_latency_ms < 0) throw InvalidConfig("net latency must be >= 0");
  const long cap = precision_cap();
  long k = cfg.k_bits ? cfg.k_bits : initial_precision(cfg.n, cfg.beta);
  if (k > cap)
    throw PrecisionCap("precision " + std::to_string(k) + " exceeds cap " +
                       std::to_string(cap));
  RunResult res;
  res.n = cfg.n;
  res.beta = cfg.beta;
  res.workers = cfg.workers;
  const auto t0 = std::chrono::steady_clock::now();
  std::optional<Z> hint;
  long hint_k = 0;
  SecantTrace tr;
  std::vector<Z> strip;
  for (;;) {
    strip = exact_moments(cfg.n, cfg.beta, k);
    const std::vector<int> devs = rank_devices(cfg.workers, device_from_env());
    std::unique_ptr<Matrix> m = upload(strip, k, devs[0]);
    if (devs.size() > 1) m->make_group(devs);
    try {
      std::optional<Z> acc;
      if (hint) acc = shl(*hint, (unsigned long)(k - hint_k));
      tr = secant_smallest_eigenvalue(cfg.n, strip[0],
                                      gpu_det(*m, k, &res.compute_s, &res.net_s), k, 15,
                                      acc ? &*acc : nullptr);
      break;
    } catch (const SecantError& e) {
      if (e.kind == SecantError::RootHitAtPrecision) {
        hint = e.probe;
        hint_k = k;
      }
      k = escalate(k, cap);
    }
  }
  res.k_bits = k;
  res.iterations = tr.iterations;
  const Z& lam = tr.eigenvalue();
  res.eigenvalue = sig_digits(lam, k, 15, false);
  if (!cfg.dump_path.empty()) {
    std::ofstream os(cfg.dump_path);
    if (!os) throw std::runtime_error("cannot open dump file: " + cfg.dump_path);
    for (size_t s = 0; s < strip.size(); ++s)
      os << "s=" << s << " hex=" << strip[s].hex() << " fracbits=" << k << "\n";
  }
  if (cfg.verify) {
    // driver.cpp:140-175: certify on the interval matrix at Kv = 2K, doubling
    // Kv while inconclusive.  The exact moments make lo = hi.
    long kv = 2 * k;
    for (;;) {
      // build_interval_matrix (hankel_matrix.cpp:33-50)
      std::vector<Z> vlo, vhi;
      build_moments(cfg.n, cfg.beta.num, cfg.beta.den, kv, true, vlo, vhi);
      std::vector<int32_t> sizes, sizes_hi;
      std::vector<uint32_t> limbs, limbs_hi, tmp;
      for (size_t i = 0; i < vlo.size(); ++i) {
        sizes.push_back(vlo[i].to_limbs(tmp));
        limbs.insert(limbs.end(), tmp.begin(), tmp.end());
        sizes_hi.push_back(vhi[i].to_limbs(tmp));
        limbs_hi.insert(limbs_hi.end(), tmp.begin(), tmp.end());
      }
      const auto tv = std::chrono::steady_clock::now();
      hgpu_matrix* im = nullptr;
      hgpu_status hs = hgpu_interval_matrix_new(
          cfg.n, kv, sizes.data(), limbs.data(), sizes_hi.data(),
          limbs_hi.data(), device_from_env(), &im);
      int st = 2, ls = 0, us = 0, lz = 0;
      char *pa = nullptr, *pb = nullptr;
      if (hs == HGPU_OK)
        hs = hgpu_verify_eigenvalue_ex(im, res.eigenvalue.c_str(), 15, &st, &ls,
                                       &us, &lz, &pa, &pb);
      hgpu_matrix_free(im);
      const std::string probe_low = pa ? pa : "";
      hgpu_string_free(pa);
      hgpu_string_free(pb);
      if (hs != HGPU_OK) throw std::runtime_error(hgpu_last_error());
      res.compute_s += std::chrono::duration<double>(
                           std::chrono::steady_clock::now() - tv).count();
      res.kv_bits = kv;
      if (st == 0) {
        res.verified = true;
        break;
      }
      if (st == 1)
        throw Refuted(
            "refuted: interval verification contradicted the converged value at " +
            probe_low);
      if (lz) {
        // driver.cpp:161-170: det(M - aI) = [0, 0], the truncated probe is
        // itself an eigenvalue; bracketing cannot decide at any precision
        res.verified = false;
        res.diagnosis = "det(M - aI) is exactly zero: the 15-digit probe " + probe_low +
                        " is itself an eigenvalue; bracketing verification does not apply";
        break;
      }
      kv = escalate(kv, cap);
    }
  }
  // condition_lower_bound (driver.cpp:48-54): M[n-1][n-1] / lambda_1
  res.condition_lower_bound =
      sig_digits(fx_div(strip[2 * cfg.n - 2], lam, k), k, 3, true);
  res.total_s = std::chrono::duration<double>(
                    std::chrono::steady_clock::now() - t0).count();
  return res;
}

std::string fmt_double(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  double back = std::strtod(buf, nullptr);
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    back = std::strtod(buf, nullptr);
    if (back == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

// report.cpp:10-26 schema (keys in the sorted order nlohmann::json emits)
std::string to_json(const RunResult& r) {
  std::ostringstream os;
  os << "{\n"
     << "  \"beta\": \"" << r.beta.str() << "\",\n"
     << "  \"condition_lower_bound\": \"" << r.condition_lower_bound << "\",\n"
     << "  \"eigenvalue\": \"" << r.eigenvalue << "\",\n"
     << "  \"iterations\": " << r.iterations << ",\n"
     << "  \"k_bits\": " << r.k_bits << ",\n"
     << "  \"kv_bits\": " << r.kv_bits << ",\n"
     << "  \"n\": " << r.n << ",\n"
     << "  \"timing\": {\n"
     << "    \"compute_s\": " << fmt_double(r.compute_s) << ",\n"
     << "    \"div_s\": " << fmt_double(r.div_s) << ",\n"
     << "    \"net_s\": " << fmt_double(r.net_s) << ",\n"
     << "    \"total_s\": " << fmt_double(r.total_s) << "\n"
     << "  },\n"
     << "  \"verified\": " << (r.verified ? "true" : "false") << ",\n"
     << "  \"workers\": " << r.workers << "\n"
     << "}";
  return os.str();
}

// report.cpp:47-76 summary layout
std::string summary(const RunResult& r) {
  std::ostringstream os;
  os << "N=" << r.n << " beta=" << r.beta.str() << " workers=" << r.workers
     << " K=" << r.k_bits;
  if (r.kv_bits > 0) os << " Kv=" << r.kv_bits;
  os << "\n";
  os << "smallest eigenvalue : " << r.eigenvalue << "\n";
  os << "verified            : " << (r.verified ? "yes" : "no");
  if (!r.diagnosis.empty()) os << "  (" << json_escape(r.diagnosis) << ")";
  os << "\n";
  os << "iterations          : " << r.iterations << "\n";
  os << "cond(M) lower bound : " << r.condition_lower_bound << "\n";
  const double total = r.total_s;
  auto pct = [&](double s) { return total > 0 ? 100.0 * s / total : 0.0; };
  char buf[160];
  std::snprintf(buf, sizeof buf, "Total Time    %10.3f s\n", total);
  os << buf;
  std::snprintf(buf, sizeof buf, "Computation   %9.1f%%  (%.3f)\n",
                pct(r.compute_s), r.compute_s);
  os << buf;
  std::snprintf(buf, sizeof buf, "Net + Divs    %9.1f%%  (%.3f)\n",
                pct(r.net_s + r.div_s), r.net_s + r.div_s);
  os << buf;
  return os.str();
}

thread_local std::string t_heig_error;

heig_status heig_fail(heig_status s, const char* what) {
  t_heig_error = what ? what : "unknown error";
  return s;
}

char* dup_string(const std::string& s) {
  char* o = static_cast<char*>(std::malloc(s.size() + 1));
  if (o) std::memcpy(o, s.c_str(), s.size() + 1);
  return o;
}

}  // namespace
}  // namespace hgpu

struct heig_config {
  hgpu::RunConfig cfg;
};
struct heig_result {
  hgpu::RunResult res;
  std::string beta_str;
};

using hgpu::heig_fail;

namespace hgpu {
Matrix* matrix_impl(hgpu_matrix* m);
void set_last_error(const std::string& s, long pivot);
}  // namespace hgpu

extern "C" {

hgpu_status hgpu_smallest_eigenvalue(hgpu_matrix* m, int digits,
                                     char** eigenvalue, char** trace,
                                     long* iterations, double* det_seconds) {
  using namespace hgpu;
  try {
    Matrix* mm = matrix_impl(m);
    if (!mm || digits < 1) throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad argument");
    const long k = mm->frac_bits();
    const HostInt& m00 = mm->strip_entry(0);
    const Z z00 = Z::from_limbs(m00.size, m00.limbs.data());
    double secs = 0;
    SecantTrace tr = secant_smallest_eigenvalue(mm->order(), z00,
                                                gpu_det(*mm, k, &secs), k, digits);
    if (eigenvalue) *eigenvalue = dup_string(sig_digits(tr.eigenvalue(), k, digits, false));
    if (trace) {
      std::string s;
      for (const SecantIterate& it : tr.iterates) s += it.x.hex() + " " + it.det.hex() + "\n";
      *trace = dup_string(s);
    }
    if (iterations) *iterations = tr.iterations;
    if (det_seconds) *det_seconds = secs;
    return HGPU_OK;
  } catch (const SecantError& e) {
    set_last_error(e.what(), e.kind == SecantError::ZeroPivot ? e.pivot : -1);
    return e.kind == SecantError::ZeroPivot ? HGPU_ERR_ZERO_PIVOT
                                            : HGPU_ERR_PRECISION_EXHAUSTED;
  } catch (const Error& e) {
    set_last_error(e.what(), e.pivot);
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what(), -1);
    return HGPU_ERR_INTERNAL;
  }
}

void hgpu_string_free(char* s) { std::free(s); }

heig_config* heig_config_new(void) { return new (std::nothrow) heig_config{}; }
void heig_config_free(heig_config* cfg) { delete cfg; }

heig_status heig_config_set_n(heig_config* cfg, long n) {
  if (!cfg || n < 1) return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "n must be >= 1");
  cfg->cfg.n = n;
  return HEIG_OK;
}

heig_status heig_config_set_beta(heig_config* cfg, const char* beta) {
  if (!cfg || !beta) return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "null argument");
  try {
    cfg->cfg.beta = hgpu::parse_rational(beta);
    return HEIG_OK;
  } catch (const std::exception& e) {
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, e.what());
  }
}

heig_status heig_config_set_precision_bits(heig_config* cfg, long k_bits) {
  if (!cfg || k_bits < 0)
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "precision must be >= 0");
  cfg->cfg.k_bits = k_bits;
  return HEIG_OK;
}

heig_status heig_config_set_workers(heig_config* cfg, long workers) {
  if (!cfg || workers < 1)
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "workers must be >= 1");
  cfg->cfg.workers = workers;
  return HEIG_OK;
}

heig_status heig_config_set_net_bandwidth(heig_config* cfg,
                                          const char* bytes_per_second) {
  if (!cfg || !bytes_per_second)
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "null argument");
  const std::string s(bytes_per_second);
  if (s == "inf") {
    cfg->cfg.net_bandwidth = std::numeric_limits<double>::infinity();
    return HEIG_OK;
  }
  try {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size() || !(v > 0) || std::isnan(v))
      return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "bandwidth must be > 0 or inf");
    cfg->cfg.net_bandwidth = v;
    return HEIG_OK;
  } catch (const std::exception&) {
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "bandwidth must be > 0 or inf");
  }
}

heig_status heig_config_set_net_latency_ms(heig_config* cfg, double ms) {
  if (!cfg || ms < 0 || std::isnan(ms))
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "latency must be >= 0");
  cfg->cfg.net_latency_ms = ms;
  return HEIG_OK;
}

heig_status heig_config_set_verify(heig_config* cfg, int enabled) {
  if (!cfg) return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "null config");
  cfg->cfg.verify = enabled != 0;
  return HEIG_OK;
}

heig_status heig_config_set_matrix_dump_path(heig_config* cfg, const char* path) {
  if (!cfg || !path) return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "null argument");
  cfg->cfg.dump_path = path;
  return HEIG_OK;
}

heig_status heig_run(const heig_config* cfg, heig_result** result_out) {
  if (!cfg || !result_out)
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, "null argument");
  *result_out = nullptr;
  try {
    hgpu::RunResult res = hgpu::run(cfg->cfg);
    auto* out = new heig_result{std::move(res), {}};
    out->beta_str = out->res.beta.str();
    *result_out = out;
    return HEIG_OK;
  } catch (const hgpu::InvalidConfig& e) {
    return heig_fail(HEIG_ERR_INVALID_ARGUMENT, e.what());
  } catch (const hgpu::PrecisionCap& e) {
    return heig_fail(HEIG_ERR_PRECISION_CAP, e.what());
  } catch (const hgpu::Refuted& e) {
    return heig_fail(HEIG_ERR_REFUTED, e.what());
  } catch (const std::exception& e) {
    return heig_fail(HEIG_ERR_INTERNAL, e.what());
  }
}

void heig_result_free(heig_result* res) { delete res; }
long heig_result_n(const heig_result* r) { return r->res.n; }
const char* heig_result_beta(const heig_result* r) { return r->beta_str.c_str(); }
long heig_result_k_bits(const heig_result* r) { return r->res.k_bits; }
long heig_result_kv_bits(const heig_result* r) { return r->res.kv_bits; }
long heig_result_workers(const heig_result* r) { return r->res.workers; }
long heig_result_iterations(const heig_result* r) { return r->res.iterations; }
int heig_result_verified(const heig_result* r) { return r->res.verified ? 1 : 0; }
const char* heig_result_eigenvalue(const heig_result* r) { return r->res.eigenvalue.c_str(); }
const char* heig_result_condition_lower_bound(const heig_result* r) {
  return r->res.condition_lower_bound.c_str();
}
const char* heig_result_diagnosis(const heig_result* r) { return r->res.diagnosis.c_str(); }
double heig_result_total_seconds(const heig_result* r) { return r->res.total_s; }
double heig_result_compute_seconds(const heig_result* r) { return r->res.compute_s; }
double heig_result_net_wait_seconds(const heig_result* r) { return r->res.net_s; }
double heig_result_div_seconds(const heig_result* r) { return r->res.div_s; }
char* heig_result_to_json(const heig_result* r) { return hgpu::dup_string(hgpu::to_json(r->res)); }
char* heig_result_summary(const heig_result* r) { return hgpu::dup_string(hgpu::summary(r->res)); }
void heig_string_free(char* s) { std::free(s); }
const char* heig_last_error(void) { return hgpu::t_heig_error.c_str(); }

}  // extern "C"
