// Interval LDL^T on the GPU (ldlt_det_interval, ldlt.cpp:79-152; SURVEY §8
// f1) and the reference's certification step on top of it
// (verify_eigenvalue, verify.cpp:8-42).
//
// Every workspace entry is the interval [W.lo, W.hi], two transforms (W_ and
// W2_).  Per stage p, on one stream (no lookahead; the interval path is a
// certification step, run twice per eigenvalue):
//   col      W[.][p] -= interval products of the panel's earlier stages
//   extract  V.lo = floor(W.lo / 2^k2), V.hi = ceil(W.hi / 2^k2)  (k_extract
//            round 1/2), pivots [W.lo, W.hi][p][p]; classes of the V bounds;
//            ZeroPivot(p) when [V.lo, V.hi][p] contains zero (ldlt.cpp:110)
//   recip    one reciprocal per divisor bound |V.lo[p]|, |V.hi[p]|
//   divide   R.lo = floor(min corner), R.hi = ceil(max corner)  (IvDiv)
//   update   W.lo -= max corner, W.hi -= min corner  (k_update_iv)
// The determinant interval is folded on the host with the reference's
// FixedInterval::mul semantics (4 corners, outward rounding) when asked;
// otherwise only its sign is derived from the pivot intervals, with an exact
// fold whenever a conservative magnitude bound cannot rule out a zero bound.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "engine.h"
#include "host/bigz.h"

namespace hgpu {

namespace {

template <class T>
T* ialloc(size_t count) {
  return static_cast<T*>(dev_alloc(std::max<size_t>(count, 1) * sizeof(T)));
}

void ifree(void* p) { dev_free(p); }

void ck(cudaError_t e) {
  if (e != cudaSuccess) throw Error(HGPU_ERR_CUDA, cudaGetErrorString(e));
}

int bits_of(const HostInt& h) {
  if (h.limbs.empty()) return 0;
  return 32 * ((int)h.limbs.size() - 1) + (32 - __builtin_clz(h.limbs.back()));
}

Z to_z(const HostInt& h) { return Z::from_limbs(h.size, h.limbs.data()); }

HostInt from_z(const Z& z) {
  HostInt h;
  h.size = z.to_limbs(h.limbs);
  return h;
}

Z fdiv_2exp(const Z& a, unsigned long k) {
  Z r;
  __gmpz_fdiv_q_2exp(r.p(), a.p(), k);
  return r;
}

Z cdiv_2exp(const Z& a, unsigned long k) {
  Z r;
  __gmpz_cdiv_q_2exp(r.p(), a.p(), k);
  return r;
}

// log2 |m| for m != 0 (double precision, for the conservative sign bound)
double log2_abs(const HostInt& h) {
  if (h.limbs.empty()) return -INFINITY;
  const int n = (int)h.limbs.size();
  double top = (double)h.limbs[n - 1];
  if (n >= 2) top = top * 4294967296.0 + (double)h.limbs[n - 2];
  const int used = n >= 2 ? 2 : 1;
  return std::log2(top) + 32.0 * (n - used);
}

}  // namespace

void Matrix::set_interval_hi(const int32_t* sizes, const uint32_t* limbs) {
  if (world_ != 1)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "interval mode runs on one rank");
  strip_hi_.assign(2 * n_ - 1, HostInt{});
  const uint32_t* src = limbs;
  for (int s = 0; s < 2 * n_ - 1; ++s) {
    HostInt& h = strip_hi_[s];
    const int len = std::abs(sizes[s]);
    h.limbs.assign(src, src + len);
    src += len;
    while (!h.limbs.empty() && h.limbs.back() == 0) h.limbs.pop_back();
    h.size = h.limbs.empty() ? 0 : (sizes[s] < 0 ? -1 : 1) * (int)h.limbs.size();
    strip_bits_ = std::max(strip_bits_, bits_of(h));
    // bounds in order (FixedInterval's constructor, fixed_interval.cpp:7-13)
    if (cmp(to_z(strip_[s]), to_z(h)) > 0)
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "interval bounds out of order");
  }
  interval_ = true;
  release();  // the plan depends on both bounds
}

void Matrix::build_interval() {
  const Plan& P = plan_;
  const DevPlan& D = dp_;
  const size_t NW = (size_t)D.NW;
  const int kb = P.kb;
  const int ns = 2 * n_ - 1;
  W2_ = ialloc<uint32_t>((size_t)std::max<long long>(P.entries, 1) * NW);
  strip2_hdr_ = ialloc<int>(ns);
  strip2_limbs_ = ialloc<uint32_t>((size_t)ns * P.cap);
  {
    std::vector<int> hdr(ns);
    std::vector<uint32_t> lim((size_t)ns * P.cap, 0);
    for (int s = 0; s < ns; ++s) {
      if ((int)strip_hi_[s].limbs.size() > P.cap)
        throw Error(HGPU_ERR_CAPACITY, "strip entry exceeds limb capacity");
      hdr[s] = strip_hi_[s].size;
      std::copy(strip_hi_[s].limbs.begin(), strip_hi_[s].limbs.end(),
                lim.begin() + (size_t)s * P.cap);
    }
    ck(cudaMemcpy(strip2_hdr_, hdr.data(), ns * sizeof(int),
                  cudaMemcpyHostToDevice));
    ck(cudaMemcpy(strip2_limbs_, lim.data(), lim.size() * 4,
                  cudaMemcpyHostToDevice));
  }
  that2_ = ialloc<uint32_t>((size_t)ns * NW);
  xhat2_ = ialloc<uint32_t>(NW);
  x2_hdr_ = ialloc<int>(1);
  x2_limbs_ = ialloc<uint32_t>(P.cap);
  ck(launch_fwd_ints(D, IntBuf{strip2_hdr_, strip2_limbs_}, 0, that2_, 0, ns, 0,
                     nullptr, err_, stream_));
  vhdr2_ = ialloc<int>((size_t)kb * n_);
  rhdr2_ = ialloc<int>((size_t)kb * n_);
  vlimbs2_ = ialloc<uint32_t>((size_t)kb * n_ * P.cap);
  rlimbs2_ = ialloc<uint32_t>((size_t)kb * n_ * P.cap);
  vhat2_ = ialloc<uint32_t>((size_t)kb * n_ * NW);
  rhat2_ = ialloc<uint32_t>((size_t)kb * n_ * NW);
  phdr2_ = ialloc<int>(n_);
  plimbs2_ = ialloc<uint32_t>((size_t)n_ * P.cap);
  ybuf2_ = ialloc<uint32_t>((size_t)P.ycap);
  ys2_ = ialloc<int>(4);
  clsv_ = ialloc<int8_t>((size_t)kb * n_);
  clsr_ = ialloc<int8_t>((size_t)kb * n_);
  ivgate_ = ialloc<int>(4);
  int herr[kErrWords];
  ck(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, stream_));
  ck(cudaStreamSynchronize(stream_));
  if (herr[kErrCapacity])
    throw Error(HGPU_ERR_CAPACITY, "strip does not fit the transform plan");
}

void Matrix::release_interval() {
  for (void* p : {(void*)W2_, (void*)that2_, (void*)xhat2_, (void*)strip2_hdr_,
                  (void*)strip2_limbs_, (void*)x2_hdr_, (void*)x2_limbs_,
                  (void*)vhdr2_, (void*)rhdr2_, (void*)phdr2_, (void*)vlimbs2_,
                  (void*)rlimbs2_, (void*)plimbs2_, (void*)vhat2_,
                  (void*)rhat2_, (void*)ybuf2_, (void*)ys2_, (void*)clsv_,
                  (void*)clsr_, (void*)ivgate_})
    ifree(p);
  ivgate_ = nullptr;
  W2_ = that2_ = xhat2_ = strip2_limbs_ = x2_limbs_ = vlimbs2_ = rlimbs2_ =
      plimbs2_ = vhat2_ = rhat2_ = ybuf2_ = nullptr;
  strip2_hdr_ = x2_hdr_ = vhdr2_ = rhdr2_ = phdr2_ = ys2_ = nullptr;
  clsv_ = clsr_ = nullptr;
}

void Matrix::run_interval(const HostInt& xlo, const HostInt& xhi,
                          unsigned flags, FactorResult& res) {
  const Plan& P = plan_;
  const DevPlan& D = dp_;
  cudaStream_t st = stream_;
  const int n = n_, kb = P.kb;
  const size_t NW = (size_t)D.NW;
  res.interval = true;
  // shifts: W.lo's diagonal loses x.hi, W.hi's loses x.lo (ldlt.cpp:96-97)
  for (const HostInt* h : {&xlo, &xhi})
    if ((int)h->limbs.size() > P.cap)
      throw Error(HGPU_ERR_CAPACITY, "shift exceeds limb capacity");
  {
    std::vector<uint32_t> a(P.cap, 0), b(P.cap, 0);
    std::copy(xhi.limbs.begin(), xhi.limbs.end(), a.begin());
    std::copy(xlo.limbs.begin(), xlo.limbs.end(), b.begin());
    ck(cudaMemcpyAsync(x_limbs_, a.data(), P.cap * 4, cudaMemcpyHostToDevice, st));
    ck(cudaMemcpyAsync(x_hdr_, &xhi.size, 4, cudaMemcpyHostToDevice, st));
    ck(cudaMemcpyAsync(x2_limbs_, b.data(), P.cap * 4, cudaMemcpyHostToDevice, st));
    ck(cudaMemcpyAsync(x2_hdr_, &xlo.size, 4, cudaMemcpyHostToDevice, st));
    ck(cudaStreamSynchronize(st));  // a, b live on this frame
  }
  const int herr0[kErrWords] = {INT_MAX, 0, 0, 0};
  ck(cudaMemcpyAsync(err_, herr0, sizeof(herr0), cudaMemcpyHostToDevice, st));
  ck(cudaMemsetAsync(stats_, 0xff, 3 * (size_t)n * sizeof(int), st));
  const long long launches0 = kernel_launch_count();
  ck(cudaEventRecord(ev0_, st));
  ck(launch_fwd_ints(D, IntBuf{x_hdr_, x_limbs_}, 0, xhat_, 0, 1, 0, nullptr,
                     err_, st));
  ck(launch_fwd_ints(D, IntBuf{x2_hdr_, x2_limbs_}, 0, xhat2_, 0, 1, 0, nullptr,
                     err_, st));
  ck(launch_init_w(D, that_, xhat_, colbase_, W_, st));
  ck(launch_init_w(D, that2_, xhat2_, colbase_, W2_, st));

  int* maxbitsV = stats_;
  int* maxdegV = stats_ + n;
  int* maxdegR = stats_ + 2 * n;
  IntBuf vlo{vhdr_, vlimbs_}, vhi{vhdr2_, vlimbs2_};
  IntBuf rlo{rhdr_, rlimbs_}, rhi{rhdr2_, rlimbs2_};
  IntBuf plo{phdr_, plimbs_}, phi{phdr2_, plimbs2_};
  const long long slot_stride = (long long)n * NW;
  // Panels whose V and R bounds are all positive (the common case: Hankel
  // moment matrices are totally positive) take the tiled point kernels with
  // the operand bounds swapped -- W.lo -= V.hi R.hi, W.hi -= V.lo R.lo, the
  // max / min corners for positive intervals -- and the selecting kernel
  // otherwise.  ivgate_ = {INT_MAX, nonpositive-seen, 0, 0} reads as an error
  // word for the point kernels (they skip when it is set) and as the gate of
  // k_update_iv (it runs only when it is set).
  {
    const int g[4] = {INT_MAX, 0, 0, 0};
    ck(cudaMemcpyAsync(ivgate_, g, sizeof(g), cudaMemcpyHostToDevice, st));
    ck(cudaStreamSynchronize(st));
  }
  int* nonpos = ivgate_ + kErrCapacity;
  auto iv_update = [&](int s_end, int c_begin, int c_end, bool col) {
    if (s_end <= 0) return;
    if (col) {
      ck(launch_update_col(D, W_, colbase_, vhat2_, rhat2_, slot_stride, s_end,
                           c_begin, c_begin, n, ivgate_, st));
      ck(launch_update_col(D, W2_, colbase_, vhat_, rhat_, slot_stride, s_end,
                           c_begin, c_begin, n, ivgate_, st));
    } else {
      ck(launch_update(D, P.tile, W_, colbase_, vhat2_, rhat2_, slot_stride,
                       s_end, c_begin, c_end, ivgate_, st));
      ck(launch_update(D, P.tile, W2_, colbase_, vhat_, rhat_, slot_stride,
                       s_end, c_begin, c_end, ivgate_, st));
    }
    ck(launch_update_iv(D, W_, W2_, colbase_, vhat_, vhat2_, rhat_, rhat2_,
                        clsv_, clsr_, 0, s_end, c_begin, c_end, c_begin, nonpos,
                        err_, st));
  };
  const int nblocks = (n + kb - 1) / kb;
  for (int b = 0; b < nblocks; ++b) {
    const int p0 = b * kb, p1 = std::min(n, p0 + kb);
    const long long row0set = 0;  // one slot set: no lookahead here
    ck(cudaMemsetAsync(nonpos, 0, sizeof(int), st));
    for (int p = p0; p < p1; ++p) {
      const int s = p - p0;
      const long long row0 = row0set + (long long)s * n;
      // column p receives the panel's earlier stages (left-looking)
      iv_update(s, p, p + 1, true);
      ck(launch_extract(D, W_, colbase_, p, p, n, vlo, row0, plo, maxbitsV,
                        vhat_, maxdegV, err_, st, 1));
      ck(launch_extract(D, W2_, colbase_, p, p, n, vhi, row0, phi, maxbitsV,
                        vhat2_, maxdegV, err_, st, 2));
      ck(launch_iv_classify(vlo, vhi, row0, p, n, clsv_, p, 1, n, err_, nonpos,
                            st));
      if (p == n - 1) break;
      ck(launch_recip(D, vlo, row0 + p, maxbitsV, p, plo, 0, ybuf_, ys_,
                      rscratch_, recip_global_ ? 1 : 0, err_, st));
      ck(launch_recip(D, vhi, row0 + p, maxbitsV, p, phi, 0, ybuf2_, ys2_,
                      rscratch_, recip_global_ ? 1 : 0, err_, st));
      IvDiv ivl{1, vhi, ybuf2_, ys2_};
      ck(launch_divide(D, vlo, row0, p, p + 1, n, ybuf_, ys_, rlo, row0, rhat_,
                       maxdegR + p, dscratch_, div_global_ ? 1 : 0, err_, st,
                       &ivl));
      IvDiv ivh{2, vhi, ybuf2_, ys2_};
      ck(launch_divide(D, vlo, row0, p, p + 1, n, ybuf_, ys_, rhi, row0, rhat2_,
                       maxdegR + p, dscratch_, div_global_ ? 1 : 0, err_, st,
                       &ivh));
      ck(launch_iv_classify(rlo, rhi, row0, p + 1, n, clsr_, p, 0, n, err_,
                            nonpos, st));
    }
    // trailing update of the panel's stages on every column to its right
    const int nsl = std::min(kb, n - 1 - p0);
    if (p1 < n && nsl > 0) iv_update(nsl, p1, n, false);
  }
  ck(launch_validate(D, maxdegV, maxdegR, n - 1, err_, st));
  ck(cudaEventRecord(ev1_, st));
  res.launches = kernel_launch_count() - launches0;
  int herr[kErrWords];
  ck(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, ev0_, ev1_));
  res.device_ms = ms;
  if (herr[kErrCapacity] & kCapStraddle)
    throw Error(HGPU_ERR_INTERVAL_STRADDLE,
                "interval LDL^T: a column-value bound and a ratio bound both "
                "contain zero");
  if (herr[kErrCapacity]) {
    Error e(HGPU_ERR_CAPACITY, "transform capacity exceeded (flags " +
                                   std::to_string(herr[kErrCapacity]) + ")");
    e.cap_flags = herr[kErrCapacity];
    throw e;
  }
  if (herr[kErrZeroPivot] != INT_MAX) {
    Error e(HGPU_ERR_ZERO_PIVOT,
            "zero pivot at column " + std::to_string(herr[kErrZeroPivot]) +
                " with " + std::to_string(K_) + " fractional bits");
    e.pivot = herr[kErrZeroPivot];
    throw e;
  }
  if (herr[kErrInternal])
    throw Error(HGPU_ERR_INTERNAL, "exactness self-check failed (flags " +
                                       std::to_string(herr[kErrInternal]) + ")");
  // pivot intervals to the host
  std::vector<int> hl(n), hh(n);
  std::vector<uint32_t> ll((size_t)n * P.cap), lh((size_t)n * P.cap);
  ck(cudaMemcpy(hl.data(), phdr_, n * 4, cudaMemcpyDeviceToHost));
  ck(cudaMemcpy(hh.data(), phdr2_, n * 4, cudaMemcpyDeviceToHost));
  ck(cudaMemcpy(ll.data(), plimbs_, ll.size() * 4, cudaMemcpyDeviceToHost));
  ck(cudaMemcpy(lh.data(), plimbs2_, lh.size() * 4, cudaMemcpyDeviceToHost));
  res.pivots.assign(n, HostInt{});
  res.pivots_hi.assign(n, HostInt{});
  for (int p = 0; p < n; ++p) {
    res.pivots[p].size = hl[p];
    res.pivots[p].limbs.assign(ll.begin() + (size_t)p * P.cap,
                               ll.begin() + (size_t)p * P.cap + std::abs(hl[p]));
    res.pivots_hi[p].size = hh[p];
    res.pivots_hi[p].limbs.assign(lh.begin() + (size_t)p * P.cap,
                                  lh.begin() + (size_t)p * P.cap + std::abs(hh[p]));
  }
  // determinant interval: FixedInterval::mul over the pivots
  // (fixed_interval.cpp: 4 corners, floor / ceil at K)
  auto exact_fold = [&]() {
    Z lo = pow2((unsigned long)K_), hi = lo;
    for (int p = 0; p < n; ++p) {
      const Z a = to_z(res.pivots[p]), bb = to_z(res.pivots_hi[p]);
      const Z c1 = lo * a, c2 = lo * bb, c3 = hi * a, c4 = hi * bb;
      const Z* mn = &c1;
      const Z* mx = &c1;
      for (const Z* c : {&c2, &c3, &c4}) {
        if (cmp(*c, *mn) < 0) mn = c;
        if (cmp(*c, *mx) > 0) mx = c;
      }
      Z nlo = fdiv_2exp(*mn, (unsigned long)K_);
      Z nhi = cdiv_2exp(*mx, (unsigned long)K_);
      lo = std::move(nlo);
      hi = std::move(nhi);
    }
    res.det = from_z(lo);
    res.det_hi = from_z(hi);
    res.have_det = true;
    res.det_sign = lo.sgn() > 0 ? 1 : (hi.sgn() < 0 ? -1 : 0);
    res.det_exact_zero = lo.sgn() == 0 && hi.sgn() == 0;
  };
  if (flags & HGPU_FOLD) {
    exact_fold();
    return;
  }
  // sign only: every pivot interval sign-definite and |det| bounded away
  // from the rounding floor (log2 of the fixed-point magnitude stays >= 4)
  // means the exact fold has the product of the pivot signs; otherwise fold.
  int sgn = 1;
  double lg = 0;  // log2 of a lower bound of |det| / 2^K
  bool sure = true;
  for (int p = 0; p < n && sure; ++p) {
    const HostInt& a = res.pivots[p];
    const HostInt& bb = res.pivots_hi[p];
    if (a.size > 0) {
      lg += log2_abs(a) - K_;
    } else if (bb.size < 0) {
      sgn = -sgn;
      lg += log2_abs(bb) - K_;
    } else {
      sure = false;
    }
    lg -= 1e-9;  // floor: (x - 1ulp) stays >= x (1 - 2^-lg) at lg >= 4
    if (lg + K_ < 4.0 + 64.0) sure = false;
  }
  if (sure) {
    res.det_sign = sgn;
  } else {
    exact_fold();
  }
}

FactorResult Matrix::factor_interval(const HostInt& xlo, const HostInt& xhi,
                                     unsigned flags) {
  if (!interval_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "not an interval matrix");
  ck(cudaSetDevice(device_));
  if (cmp(to_z(xlo), to_z(xhi)) > 0)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "interval bounds out of order");
  int min_logL = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (!W_ || (min_logL && plan_.logL < min_logL)) build(min_logL);
    try {
      FactorResult res;
      res.n = n_;
      res.K = K_;
      run_interval(xlo, xhi, flags, res);
      return res;
    } catch (const Error& e) {
      if (e.status != HGPU_ERR_CAPACITY) throw;
      min_logL = plan_.logL + 1;
      release();
    }
  }
  throw Error(HGPU_ERR_CAPACITY, "values outgrew every transform plan");
}

}  // namespace hgpu
