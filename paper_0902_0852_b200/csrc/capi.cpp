// extern "C" boundary of libhgpu (include/hgpu.h).  Exceptions never cross
// it: every status-returning entry point maps hgpu::Error (and anything else)
// to a status and a thread-local message, like the reference's C ABI does
// (/root/reference/proj/src/capi.cpp:24-35, :118-139).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <fstream>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/hgpu.h"
#include "engine.h"
#include "host/bigz.h"

struct hgpu_matrix {
  std::unique_ptr<hgpu::Matrix> impl;
};
struct hgpu_factor {
  hgpu::FactorResult res;
};

namespace {

thread_local std::string g_last_error;
thread_local long g_last_pivot = -1;

template <typename F>
hgpu_status guarded(F&& f) {
  try {
    f();
    return HGPU_OK;
  } catch (const hgpu::Error& e) {
    g_last_error = e.what();
    if (e.status == HGPU_ERR_ZERO_PIVOT) g_last_pivot = e.pivot;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return HGPU_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HGPU_ERR_INTERNAL;
  }
}

hgpu::HostInt make_int(int32_t size, const uint32_t* limbs) {
  hgpu::HostInt h;
  const int len = size < 0 ? -size : size;
  if (len && !limbs) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null limbs");
  h.limbs.assign(limbs, limbs + len);
  while (!h.limbs.empty() && h.limbs.back() == 0) h.limbs.pop_back();
  h.size = h.limbs.empty() ? 0 : (size < 0 ? -1 : 1) * (int)h.limbs.size();
  return h;
}

}  // namespace

namespace hgpu {
Matrix* matrix_impl(hgpu_matrix* m) { return m ? m->impl.get() : nullptr; }
void set_last_error(const std::string& s, long pivot) {
  g_last_error = s;
  if (pivot >= 0) g_last_pivot = pivot;
}
}  // namespace hgpu

extern "C" {

const char* hgpu_version(void) { return "hgpu 0.1 (sm_100a)"; }
const char* hgpu_last_error(void) { return g_last_error.c_str(); }
long hgpu_last_zero_pivot(void) { return g_last_pivot; }

int hgpu_block_owner(long block_index, int world) {
  return world < 1 ? 0 : hgpu::block_owner(block_index, world);
}

hgpu_status hgpu_trim_pool(int device) {
  return guarded([&] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(pool, 0) != cudaSuccess)
      throw hgpu::Error(HGPU_ERR_CUDA, "cannot trim the device memory pool");
  });
}

hgpu_status hgpu_matrix_new(long n, long frac_bits, const int32_t* strip_sizes,
                            const uint32_t* strip_limbs, int device,
                            hgpu_matrix** out) {
  return guarded([&] {
    if (!out || !strip_sizes)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 1 || n > 100000)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "order out of range");
    auto m = std::make_unique<hgpu_matrix>();
    m->impl = std::make_unique<hgpu::Matrix>((int)n, (int)frac_bits,
                                             strip_sizes, strip_limbs, device);
    *out = m.release();
  });
}

hgpu_status hgpu_matrix_new_group(long n, long frac_bits,
                                  const int32_t* strip_sizes,
                                  const uint32_t* strip_limbs, const int* devices,
                                  int world, hgpu_matrix** out) {
  return guarded([&] {
    if (!out || !strip_sizes || !devices || world < 1 || world > 64)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "bad argument");
    if (n < 1 || n > 100000)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "order out of range");
    auto m = std::make_unique<hgpu_matrix>();
    m->impl = std::make_unique<hgpu::Matrix>((int)n, (int)frac_bits, strip_sizes,
                                             strip_limbs, devices[0]);
    m->impl->make_group(std::vector<int>(devices, devices + world));
    *out = m.release();
  });
}

hgpu_status hgpu_matrix_new_from_dump(const char* path, int device, hgpu_matrix** out,
                                      long* n_out, long* frac_bits_out) {
  return guarded([&] {
    if (!path || !out) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    std::ifstream is(path);
    if (!is) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, std::string("cannot open dump file: ") + path);
    // load_matrix_dump (hankel_matrix.cpp:65-87)
    std::vector<int32_t> sizes;
    std::vector<uint32_t> limbs, one;
    long frac_bits = 0;
    std::string line;
    while (std::getline(is, line)) {
      if (line.empty()) continue;
      std::istringstream ls(line);
      std::string s_tok, hex_tok, fb_tok;
      ls >> s_tok >> hex_tok >> fb_tok;
      if (s_tok.rfind("s=", 0) != 0 || hex_tok.rfind("hex=", 0) != 0 ||
          fb_tok.rfind("fracbits=", 0) != 0)
        throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "matrix dump line: " + line);
      long s = 0;
      try {
        s = std::stol(s_tok.substr(2));
        frac_bits = std::stol(fb_tok.substr(9));
      } catch (const std::exception&) {
        throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "matrix dump line: " + line);
      }
      if (s != (long)sizes.size())
        throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT,
                          "matrix dump out of order at s=" + std::to_string(s));
      hgpu::Z z;
      if (__gmpz_set_str(z.p(), hex_tok.c_str() + 4, 16) != 0)
        throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "matrix dump line: " + line);
      sizes.push_back(z.to_limbs(one));
      limbs.insert(limbs.end(), one.begin(), one.end());
    }
    if (sizes.empty() || sizes.size() % 2 == 0)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "matrix dump must hold 2n-1 anti-diagonals");
    const long n = (long)(sizes.size() + 1) / 2;
    if (n > 100000 || frac_bits < 2 || frac_bits > (1L << 24))
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "matrix dump: order or fracbits out of range");
    if (n_out) *n_out = n;
    if (frac_bits_out) *frac_bits_out = frac_bits;
    if (limbs.empty()) limbs.push_back(0u);
    auto m = std::make_unique<hgpu_matrix>();
    m->impl = std::make_unique<hgpu::Matrix>((int)n, (int)frac_bits, sizes.data(), limbs.data(),
                                             device);
    *out = m.release();
  });
}

hgpu_status hgpu_matrix_dump(const hgpu_matrix* m, const char* path) {
  return guarded([&] {
    if (!m || !path) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    std::ofstream os(path);
    if (!os) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, std::string("cannot open dump file: ") + path);
    // dump_matrix (hankel_matrix.cpp:52-57)
    const int n = m->impl->order();
    for (int s = 0; s < 2 * n - 1; ++s) {
      const hgpu::HostInt& h = m->impl->strip_entry(s);
      os << "s=" << s << " hex=" << hgpu::Z::from_limbs(h.size, h.limbs.data()).hex()
         << " fracbits=" << m->impl->frac_bits() << "\n";
    }
    if (!os) throw hgpu::Error(HGPU_ERR_INTERNAL, std::string("write failed: ") + path);
  });
}

int hgpu_matrix_world(const hgpu_matrix* m) { return m ? m->impl->world() : 0; }

void hgpu_matrix_free(hgpu_matrix* m) { delete m; }

hgpu_status hgpu_interval_matrix_new(long n, long frac_bits,
                                     const int32_t* lo_sizes,
                                     const uint32_t* lo_limbs,
                                     const int32_t* hi_sizes,
                                     const uint32_t* hi_limbs, int device,
                                     hgpu_matrix** out) {
  return guarded([&] {
    if (!out || !lo_sizes || !hi_sizes)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 1 || n > 100000)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "order out of range");
    auto m = std::make_unique<hgpu_matrix>();
    m->impl = std::make_unique<hgpu::Matrix>((int)n, (int)frac_bits, lo_sizes,
                                             lo_limbs, device);
    m->impl->set_interval_hi(hi_sizes, hi_limbs);
    *out = m.release();
  });
}

hgpu_status hgpu_ldlt_interval(hgpu_matrix* m, int32_t xlo_size,
                               const uint32_t* xlo_limbs, int32_t xhi_size,
                               const uint32_t* xhi_limbs, long x_frac_bits,
                               unsigned flags, hgpu_factor** out) {
  return guarded([&] {
    if (!m || !out) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    if (x_frac_bits != m->impl->frac_bits())
      throw hgpu::Error(HGPU_ERR_PRECISION_MISMATCH,
                        "fractional precision mismatch");
    auto f = std::make_unique<hgpu_factor>();
    f->res = m->impl->factor_interval(make_int(xlo_size, xlo_limbs),
                                      make_int(xhi_size, xhi_limbs), flags);
    *out = f.release();
  });
}

hgpu_status hgpu_factor_pivot_hi(const hgpu_factor* f, long p, int32_t* size,
                                 const uint32_t** limbs) {
  return guarded([&] {
    if (!f || !size || !limbs || !f->res.interval || p < 0 ||
        p >= (long)f->res.pivots_hi.size())
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "bad pivot index");
    *size = f->res.pivots_hi[p].size;
    *limbs = f->res.pivots_hi[p].limbs.data();
  });
}

hgpu_status hgpu_factor_det_hi(const hgpu_factor* f, int32_t* size,
                               const uint32_t** limbs) {
  return guarded([&] {
    if (!f || !size || !limbs || !f->res.interval || !f->res.have_det)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "no folded interval det");
    *size = f->res.det_hi.size;
    *limbs = f->res.det_hi.limbs.data();
  });
}

int hgpu_factor_det_sign(const hgpu_factor* f) {
  return f && f->res.interval ? f->res.det_sign : 0;
}

hgpu_status hgpu_nccl_unique_id(unsigned char out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess)
      throw hgpu::Error(HGPU_ERR_COMM, "ncclGetUniqueId failed");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

hgpu_status hgpu_matrix_set_comm(hgpu_matrix* m, int rank, int world,
                                 const unsigned char nccl_id[128]) {
  return guarded([&] {
    if (!m) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null matrix");
    m->impl->set_comm(rank, world, nccl_id);
  });
}

hgpu_status hgpu_matrix_set_strip(hgpu_matrix* m, const int32_t* strip_sizes,
                                  const uint32_t* strip_limbs) {
  return guarded([&] {
    if (!m || !strip_sizes) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    m->impl->set_strip(strip_sizes, strip_limbs);
  });
}

hgpu_status hgpu_matrix_set_capture_rows(hgpu_matrix* m, long rows) {
  return guarded([&] {
    if (!m || rows < 0) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "bad argument");
    m->impl->set_capture_rows((int)std::min<long>(rows, 1L << 30));
  });
}

hgpu_status hgpu_ldlt_factor(hgpu_matrix* m, int32_t x_size,
                             const uint32_t* x_limbs, long x_frac_bits,
                             unsigned flags, hgpu_factor** out) {
  return guarded([&] {
    if (!m || !out) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    auto f = std::make_unique<hgpu_factor>();
    hgpu::HostInt x = make_int(x_size, x_limbs);
    f->res = m->impl->factor_checked(x, x_frac_bits, flags);
    *out = f.release();
  });
}

long hgpu_factor_order(const hgpu_factor* f) { return f ? f->res.n : 0; }
long hgpu_factor_frac_bits(const hgpu_factor* f) { return f ? f->res.K : 0; }

hgpu_status hgpu_factor_pivot(const hgpu_factor* f, long p, int32_t* size,
                              const uint32_t** limbs) {
  return guarded([&] {
    if (!f || !size || !limbs || p < 0 || p >= (long)f->res.pivots.size())
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "bad pivot index");
    *size = f->res.pivots[p].size;
    *limbs = f->res.pivots[p].limbs.data();
  });
}

hgpu_status hgpu_factor_ratio(const hgpu_factor* f, long p, long r,
                              int32_t* size, const uint32_t** limbs) {
  return guarded([&] {
    if (!f || !size || !limbs)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    if (!f->res.have_ratios)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "ratios not captured");
    if (p < 0 || p >= (long)f->res.ratios.size() || r <= p || r >= f->res.capture_rows)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "bad ratio index");
    const hgpu::HostInt& h = f->res.ratios[p][r - p - 1];
    *size = h.size;
    *limbs = h.limbs.data();
  });
}

hgpu_status hgpu_factor_det(const hgpu_factor* f, int32_t* size,
                            const uint32_t** limbs) {
  return guarded([&] {
    if (!f || !size || !limbs)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null argument");
    if (!f->res.have_det)
      throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "determinant not folded");
    *size = f->res.det.size;
    *limbs = f->res.det.limbs.data();
  });
}

double hgpu_factor_device_ms(const hgpu_factor* f) {
  return f ? f->res.device_ms : 0.0;
}

hgpu_status hgpu_factor_update_stats(const hgpu_factor* f, long* launches,
                                     double* ms, double* products) {
  return guarded([&] {
    if (!f) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null factor");
    if (launches) *launches = f->res.update_launches;
    if (ms) *ms = f->res.update_ms;
    if (products) *products = f->res.update_products;
  });
}

double hgpu_factor_net_ms(const hgpu_factor* f) { return f ? f->res.net_ms : 0.0; }

long long hgpu_factor_launches(const hgpu_factor* f) {
  return f ? f->res.launches : 0;
}

void hgpu_factor_free(hgpu_factor* f) { delete f; }

hgpu_status hgpu_matrix_plan(const hgpu_matrix* m, int* nprimes, int* length,
                             int* digit_bits, int* cap_limbs,
                             double* workspace_bytes) {
  return guarded([&] {
    if (!m) throw hgpu::Error(HGPU_ERR_INVALID_ARGUMENT, "null matrix");
    const hgpu::Plan& P = m->impl->plan_or_build();
    if (nprimes) *nprimes = P.np;
    if (length) *length = P.L;
    if (digit_bits) *digit_bits = P.w;
    if (cap_limbs) *cap_limbs = P.cap;
    if (workspace_bytes) *workspace_bytes = P.workspace_bytes();
  });
}

}  // extern "C"
