// Host side of the B200 LDL^T engine (see engine.h).
#include "engine.h"

#include <cublas_v2.h>
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>

namespace hgpu {

namespace {

#define CU(expr)                                                           \
  do {                                                                     \
    cudaError_t e_ = (expr);                                               \
    if (e_ != cudaSuccess)                                                 \
      throw Error(HGPU_ERR_CUDA, std::string(#expr) + ": " +               \
                                     cudaGetErrorString(e_));              \
  } while (0)

#define NC(expr)                                                           \
  do {                                                                     \
    ncclResult_t r_ = (expr);                                              \
    if (r_ != ncclSuccess)                                                 \
      throw Error(HGPU_ERR_COMM, std::string(#expr) + ": " +               \
                                     ncclGetErrorString(r_));              \
  } while (0)

using u64 = unsigned long long;
using u128 = unsigned __int128;

u64 powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = (u128)r * b % m;
    b = (u128)b * b % m;
    e >>= 1;
  }
  return r;
}
u64 invmod(u64 a, u64 m) { return powmod(a % m, m - 2, m); }  // m prime

int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

double log2_u128(u128 v) {
  return std::log2((double)(u64)(v >> 64) * 18446744073709551616.0 +
                   (double)(u64)v);
}

// ---- SM partition (green contexts) ---------------------------------------
// The pivot chain (one-row update, extraction, reciprocal, one-row division)
// is a sequence of single-CTA, latency-bound kernels: on an SM shared with
// trailing-update CTAs (which keep the IMAD pipe ~80 % busy) every one of its
// dependent instructions waits for issue, and each launch first queues for a
// free slot.  The chain therefore runs on a reserved group of SMs (a green
// context) and the trailing update on the rest.  Driver entry points are
// fetched through the runtime, so the library does not link libcuda.
// HGPU_SM_SPLIT=<chain SMs>[:<panel stream on a (chain group) | b (update
// group) | p (primary context, every SM)>], "0" disables.
struct GreenSplit {
  bool ok = false;
  int chain_sms = 0, rest_sms = 0;
  CUgreenCtx ga = nullptr, gb = nullptr;
};

GreenSplit make_green_split(int device, int want) {
  GreenSplit g;
  if (want <= 0) return g;
  auto sym = [](const char* name) -> void* {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return fn;
  };
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*,
                             CUdevResource*, unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  auto get_res = (GetRes)sym("cuDeviceGetDevResource");
  auto split = (Split)sym("cuDevSmResourceSplitByCount");
  auto gen = (GenDesc)sym("cuDevResourceGenerateDesc");
  auto create = (Create)sym("cuGreenCtxCreate");
  if (!get_res || !split || !gen || !create) return g;
  CUdevResource all, grp, rest;
  if (get_res((CUdevice)device, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return g;
  unsigned ng = 1;
  if (split(&grp, &ng, &all, &rest, 0, (unsigned)want) != CUDA_SUCCESS || ng != 1)
    return g;
  CUdevResourceDesc da, db;
  if (gen(&da, &grp, 1) != CUDA_SUCCESS || gen(&db, &rest, 1) != CUDA_SUCCESS) return g;
  if (create(&g.ga, da, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      create(&g.gb, db, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return g;
  g.chain_sms = (int)grp.sm.smCount;
  g.rest_sms = (int)rest.sm.smCount;
  g.ok = true;
  return g;
}

// One split per (device, group size) for the process (green contexts are
// kept alive).
const GreenSplit& green_split(int device, int want) {
  static std::mutex mu;
  static std::vector<std::pair<long long, GreenSplit>> cache;
  std::lock_guard<std::mutex> lk(mu);
  const long long key = ((long long)device << 32) | (unsigned)want;
  for (auto& e : cache)
    if (e.first == key) return e.second;
  cache.emplace_back(key, make_green_split(device, want));
  return cache.back().second;
}

cudaStream_t green_stream(CUgreenCtx g, int priority) {
  using SCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuGreenCtxStreamCreate", &fn, cudaEnableDefault, &q) !=
          cudaSuccess || q != cudaDriverEntryPointSuccess)
    throw Error(HGPU_ERR_CUDA, "cuGreenCtxStreamCreate unavailable");
  CUstream s = nullptr;
  if (((SCreate)fn)(&s, g, CU_STREAM_NON_BLOCKING, priority) != CUDA_SUCCESS)
    throw Error(HGPU_ERR_CUDA, "cuGreenCtxStreamCreate failed");
  return (cudaStream_t)s;
}

template <typename T>
T* dalloc(size_t count) {
  if (count == 0) count = 1;
  return static_cast<T*>(dev_alloc(count * sizeof(T)));
}

void dfree(void* p) { dev_free(p); }

}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  CU(cudaDeviceGetDefaultMemPool(&pool, dev));
  static thread_local int configured = -1;
  if (configured != dev) {
    uint64_t keep = UINT64_MAX;  // keep freed blocks in the pool
    CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured = dev;
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, 0);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    CU(cudaDeviceSynchronize());
    CU(cudaMemPoolTrimTo(pool, 0));
    e = cudaMallocFromPoolAsync(&p, bytes, pool, 0);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(HGPU_ERR_CUDA, std::string("device allocation failed: ") +
                                   cudaGetErrorString(e));
  }
  // the legacy stream orders the allocation; our streams are non-blocking
  CU(cudaStreamSynchronize(0));
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  cudaDeviceSynchronize();  // no stream may still use it
  cudaFreeAsync(p, 0);
}

// Device memory dalloc can still hand out: free memory plus the blocks the
// stream-ordered pool keeps after frees (the release threshold is infinite).
size_t device_available(int device) {
  size_t fr = 0, tot = 0;
  CU(cudaMemGetInfo(&fr, &tot));
  cudaMemPool_t pool;
  uint64_t resv = 0, used = 0;
  CU(cudaDeviceGetDefaultMemPool(&pool, device));
  CU(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &resv));
  CU(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return fr + (resv > used ? (size_t)(resv - used) : 0);
}

int block_owner(long block, int world) {
  // reflected round-robin, assignment.hpp:15-23, over column blocks
  const long r = block % (2L * world);
  return (int)(r < world ? r : 2L * world - 1 - r);
}

// ---- in-process rank group ------------------------------------------------
// The reference's workers (ldlt.cpp:205-311) share one ColumnChannel
// (channel.hpp:31-56): the owner of a column publishes it, the others await
// it, and a failing worker poisons the channel so nobody waits forever
// (ldlt.cpp:181-188).  Here a rank is a Matrix on some device, a "column" is
// a panel of kb columns, publishing is a CUDA event recorded after the
// panel on the owner's panel stream, and awaiting is a host wait for that
// record (never a device-side spin), after which the receiver's stream waits
// on the event and its k_fwd_ints launches read the owner's integers
// directly (peer loads over NVLink when the ranks are on different GPUs).
const std::string kPeerFailed = "a peer rank failed: ";

struct PeerGroup {
  int world = 1;
  std::vector<Matrix*> ranks;
  std::mutex mu;
  std::condition_variable cv;
  long long run = 0;  // factorisation in progress (all ranks)
  bool poisoned = false;
  std::string why;
  std::vector<cudaEvent_t> ready_ev;   // [panel]: the owner's event
  std::vector<long long> ready_run;    // run that recorded it
  std::vector<cudaEvent_t> pulled_ev;  // [panel * world + rank]
  std::vector<long long> pulled_run;
  // end-of-run merge of the error words (min pivot index, OR of flags)
  long long merge_run = -1;
  int arrived = 0;
  int merged[kErrWords];

  template <class Pred>
  void wait(std::unique_lock<std::mutex>& lk, Pred pred) {
    cv.wait(lk, [&] { return poisoned || pred(); });
    if (!pred()) throw Error(HGPU_ERR_COMM, kPeerFailed + why);
  }
  void poison(const std::string& w) {
    std::lock_guard<std::mutex> lk(mu);
    if (!poisoned) why = w;
    poisoned = true;
    cv.notify_all();
  }
};

Plan choose_plan(int n, int K, int bits, int min_logL) {
  Plan best;
  long long best_cost = LLONG_MAX;
  for (int np = 2; np <= 4; ++np) {
    u128 Q = 1;
    for (int j = 0; j < np; ++j) Q *= kPrimes[j];
    const double log2_quarter = log2_u128(Q) - 2.0;
    for (int logL = std::max(5, min_logL); logL <= 17; ++logL) {
      const int L = 1 << logL;
      // L digits of w bits must hold any product, with two digits spare
      const int w = (bits + 1 + (L - 2) - 1) / (L - 2);
      if (w > 48) continue;  // digits are handled in 64-bit words
      if (w < 4) continue;
      // n stages x (L/2 overlapping terms) x (2^w-1)^2 (+ slack) < Q/4
      const double lb = std::log2((double)n + 1) + std::log2((double)L / 2 + 1) +
                        2.0 * w + 0.1;
      if (lb >= log2_quarter) continue;
      const long long cost = (long long)np * L;
      if (cost < best_cost) {
        best_cost = cost;
        best.np = np;
        best.L = L;
        best.logL = logL;
        best.w = w;
      }
      break;  // larger L at this np only costs more
    }
  }
  if (best_cost == LLONG_MAX)
    throw Error(HGPU_ERR_CAPACITY, "no transform plan fits the value sizes");
  best.n = n;
  best.K = K;
  // pieces of a CRT coefficient (32*np-bit two's complement): one spare for
  // the sign, but the top piece's shift must stay inside the 128-bit value
  best.T = (32 * best.np + best.w - 1) / best.w + 1;
  if (best.w * (best.T - 1) >= 128) --best.T;
  best.cap = (best.w * (best.L + best.T) + 31) / 32 + 2;
  best.ycap = best.cap + (K / 2) / 32 + 8;
  return best;
}

// Prime constants, Garner constants and the twiddle tables (host copy:
// Shoup forward/inverse pairs, then the Montgomery forms) of plan P.
static std::vector<uint32_t> transform_tables(DevPlan& D, const Plan& P) {
  const size_t npl = (size_t)P.np * P.L;
  D.Lmax = P.L;
  for (int j = 0; j < P.np; ++j) {
    const u64 q = kPrimes[j];
    PrimeConsts& c = D.pc[j];
    c.q = (uint32_t)q;
    // -q^-1 mod 2^32 by Newton
    uint32_t inv = 1;
    for (int i = 0; i < 6; ++i) inv *= 2u - (uint32_t)q * inv;
    c.qneg = (uint32_t)(0u - inv);
    c.r32 = (uint32_t)((1ULL << 32) % q);
    c.r32s = shoup_companion(c.r32, (uint32_t)q);
    c.r64 = (uint32_t)((u128)c.r32 * c.r32 % q);
    c.one_s = shoup_companion(1u, (uint32_t)q);
    const u64 il = invmod(P.L, q);
    D.invL[j] = (uint32_t)il;
    D.invLp[j] = shoup_companion((uint32_t)il, (uint32_t)q);
  }
  const u64 q0 = kPrimes[0], q1 = kPrimes[1], q2 = kPrimes[2];
  D.g1 = (uint32_t)invmod(q0 % q1, q1);
  D.g1p = shoup_companion(D.g1, (uint32_t)q1);
  D.g2 = (uint32_t)invmod((u128)q0 * q1 % q2, q2);
  D.g2p = shoup_companion(D.g2, (uint32_t)q2);
  D.q0m2 = (uint32_t)(q0 % q2);
  D.q0m2p = shoup_companion(D.q0m2, (uint32_t)q2);
  D.q01 = q0 * q1;
  if (P.np == 4) {
    const u64 q3 = kPrimes[3];
    const u128 q012 = (u128)q0 * q1 * q2;
    D.g3 = (uint32_t)invmod((u64)(q012 % q3), q3);
    D.g3p = shoup_companion(D.g3, (uint32_t)q3);
    D.q0m3 = (uint32_t)(q0 % q3);
    D.q0m3p = shoup_companion(D.q0m3, (uint32_t)q3);
    D.q01m3 = (uint32_t)((u128)q0 * q1 % q3);
    D.q01m3p = shoup_companion(D.q01m3, (uint32_t)q3);
    D.q012lo = (u64)q012;
    D.q012hi = (u64)(q012 >> 64);
  }
  u128 Q = 1;
  for (int j = 0; j < P.np; ++j) Q *= kPrimes[j];
  const u128 H = (Q + 1) / 2;
  D.Qlo = (u64)Q;
  D.Qhi = (u64)(Q >> 64);
  D.Hlo = (u64)H;
  D.Hhi = (u64)(H >> 64);

  // twiddles: T[m+i] = w^{(L/2m) bitrev_m(i)}, w a primitive L-th root
  std::vector<uint32_t> tab(4 * (size_t)P.np * P.L, 0);
  for (int j = 0; j < P.np; ++j) {
    const u64 q = kPrimes[j];
    const u64 wL = powmod(kPrimRoots[j], (q - 1) / P.L, q);
    uint32_t* tw = &tab[(0 * P.np + j) * (size_t)P.L];
    uint32_t* twp = &tab[(1 * P.np + j) * (size_t)P.L];
    uint32_t* itw = &tab[(2 * P.np + j) * (size_t)P.L];
    uint32_t* itwp = &tab[(3 * P.np + j) * (size_t)P.L];
    for (int lm = 0; (1 << lm) < P.L; ++lm) {
      const int m = 1 << lm;
      for (int i = 0; i < m; ++i) {
        const u64 e = (u64)(P.L / (2 * m)) * bitrev(i, lm);
        const u64 v = powmod(wL, e, q);
        const u64 iv = invmod(v, q);
        tw[m + i] = (uint32_t)v;
        twp[m + i] = shoup_companion((uint32_t)v, (uint32_t)q);
        itw[m + i] = (uint32_t)iv;
        itwp[m + i] = shoup_companion((uint32_t)iv, (uint32_t)q);
      }
    }
  }
  // Montgomery-form copies (w 2^32 mod q) for the radix-16 transforms
  tab.resize(6 * npl, 0);
  for (int j = 0; j < P.np; ++j) {
    const u64 q = kPrimes[j];
    for (int k = 1; k < P.L; ++k) {
      tab[4 * npl + j * (size_t)P.L + k] =
          (uint32_t)(((u128)tab[0 * npl + j * (size_t)P.L + k] << 32) % q);
      tab[5 * npl + j * (size_t)P.L + k] =
          (uint32_t)(((u128)tab[2 * npl + j * (size_t)P.L + k] << 32) % q);
    }
  }
  return tab;
}

// Transform plan of the solve's AXPY: 32-bit digits (a digit is a limb, so
// the conversions are word copies), the shortest length holding a product
// of `bits` bits with two digits spare, and the fewest primes keeping n
// products of L/2 overlapping digit pairs below Q/4.
Plan solve_plan(int n, int K, int bits) {
  Plan P;
  P.w = 32;
  P.logL = 5;
  while (32LL * ((1 << P.logL) - 2) < (long long)bits + 1) ++P.logL;
  if (P.logL > kMaxLogL) throw Error(HGPU_ERR_CAPACITY, "solve transform too long");
  P.L = 1 << P.logL;
  for (P.np = 2; P.np <= kMaxPrimes; ++P.np) {
    u128 Q = 1;
    for (int j = 0; j < P.np; ++j) Q *= kPrimes[j];
    const double lb = std::log2((double)n + 1) + std::log2((double)P.L / 2 + 1) + 64.1;
    if (lb < log2_u128(Q) - 2.0) break;
  }
  if (P.np > kMaxPrimes) throw Error(HGPU_ERR_CAPACITY, "no solve transform plan fits");
  P.n = n;
  P.K = K;
  P.T = (32 * P.np + P.w - 1) / P.w + 1;
  if (P.w * (P.T - 1) >= 128) --P.T;
  P.cap = (P.w * (P.L + P.T) + 31) / 32 + 2;
  P.ycap = P.cap + (K / 2) / 32 + 8;
  return P;
}

void Matrix::parse_strip(const int32_t* sizes, const uint32_t* limbs) {
  strip_.assign(2 * n_ - 1, HostInt{});
  strip_bits_ = 0;
  const uint32_t* src = limbs;
  for (int s = 0; s < 2 * n_ - 1; ++s) {
    HostInt& h = strip_[s];
    h.size = sizes[s];
    const int len = std::abs(sizes[s]);
    h.limbs.assign(src, src + len);
    src += len;
    while (!h.limbs.empty() && h.limbs.back() == 0) h.limbs.pop_back();
    h.size = h.limbs.empty() ? 0 : (sizes[s] < 0 ? -1 : 1) * (int)h.limbs.size();
    const int b = h.limbs.empty()
                      ? 0
                      : 32 * ((int)h.limbs.size() - 1) +
                            (32 - __builtin_clz(h.limbs.back()));
    strip_bits_ = std::max(strip_bits_, b);
  }
}

// A new strip of the same order and precision (e.g. the next matrix of a
// sweep, or the same moments re-sent): when it fits the current transform
// plan, only the strip's integers are re-sent and re-transformed by the next
// factorisation; otherwise the matrix is rebuilt there.
void Matrix::set_strip(const int32_t* sizes, const uint32_t* limbs) {
  if (interval_) throw Error(HGPU_ERR_INVALID_ARGUMENT, "interval matrices keep their bounds");
  CU(cudaSetDevice(device_));
  parse_strip(sizes, limbs);
  const bool keep = (W_ || ws_released_) && [&] {
    const Plan q = choose_plan(n_, K_, strip_bits_ + 64, 0);
    return q.np == plan_.np && q.L == plan_.L && q.w == plan_.w && q.cap <= plan_.cap;
  }();
  if (keep)
    strip_dirty_ = true;
  else
    release();
  for (auto& pm : peers_) pm->set_strip(sizes, limbs);
}

Matrix::Matrix(int n, int K, const int32_t* sizes, const uint32_t* limbs,
               int device)
    : n_(n), K_(K), device_(device) {
  if (n < 1) throw Error(HGPU_ERR_INVALID_ARGUMENT, "order must be >= 1");
  if (K < 2 || K % 2 != 0)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "frac_bits must be even and >= 2");
  parse_strip(sizes, limbs);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(HGPU_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= ndev)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad device index");
  CU(cudaSetDevice(device_));
  {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    int want = 0;  // off by default: measured slower at config 3
    char panel = 'a';
    if (const char* e = std::getenv("HGPU_SM_SPLIT")) {
      want = std::atoi(e);
      if (const char* c = std::strchr(e, ':')) panel = c[1];
    }
    const GreenSplit& g = green_split(device_, want);
    if (g.ok) {
      split_ga_ = (void*)g.ga;
      split_gb_ = (void*)g.gb;
      // bulk stream on the large group, pivot chain on the reserved SMs;
      // the panel stream where HGPU_SM_SPLIT places it
      stream_ = green_stream(g.gb, 0);
      stream_helper_ = green_stream(g.ga, hi);
      stream_far_ = green_stream(g.gb, hi);
      if (panel == 'b')
        stream_panel_ = green_stream(g.gb, hi);
      else if (panel == 'a')
        stream_panel_ = green_stream(g.ga, hi);
      else
        CU(cudaStreamCreateWithPriority(&stream_panel_, cudaStreamNonBlocking, hi));
      chain_sms_ = g.chain_sms;
    } else {
      CU(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
      CU(cudaStreamCreateWithPriority(&stream_panel_, cudaStreamNonBlocking, hi));
      CU(cudaStreamCreateWithPriority(&stream_helper_, cudaStreamNonBlocking, hi));
      // far rows one priority level below the chain and the near rows
      // (HGPU_FAR_PRIO levels below): a freed SM slot goes to a near-row CTA first
      int fo = 0;  // measured equal at 0, 1, 2 (profiles/r02/sweep_prio_r02.txt)
      if (const char* e = std::getenv("HGPU_FAR_PRIO")) fo = std::max(0, std::atoi(e));
      far_prio_ = std::min(lo, hi + fo);
      CU(cudaStreamCreateWithPriority(&stream_far_, cudaStreamNonBlocking, far_prio_));
    }
  }
  {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // with an SM split every other stream lives on the large group, so the
    // reserved SMs run the pivot chain alone (primary-context streams would
    // still reach them)
    const bool excl = split_gb_ != nullptr;
    if (excl)
      stream_upd1_ = green_stream((CUgreenCtx)split_gb_, hi);
    else
      CU(cudaStreamCreateWithPriority(&stream_upd1_, cudaStreamNonBlocking, hi));
    // HGPU_UPD_SMS=k: the deferred update runs on k SMs only (green context)
    int upd_sms = 0;
    if (const char* e = std::getenv("HGPU_UPD_SMS")) upd_sms = std::atoi(e);
    const GreenSplit& gu = green_split(device_, upd_sms);
    if (gu.ok)
      stream_upd2_ = green_stream(gu.ga, lo);
    else if (excl)
      stream_upd2_ = green_stream((CUgreenCtx)split_gb_, lo);
    else {
      // HGPU_UPD_PRIO=k: the deferred update k levels above the lowest
      // priority (experiment: 0, the lowest, measured best)
      int up = 0;
      if (const char* e = std::getenv("HGPU_UPD_PRIO")) up = std::max(0, std::atoi(e));
      CU(cudaStreamCreateWithPriority(&stream_upd2_, cudaStreamNonBlocking, std::max(hi, lo - up)));
    }
  }
  CU(cudaEventCreate(&ev0_));
  CU(cudaEventCreate(&ev1_));
  if (const char* e = std::getenv("HGPU_DEFER")) defer_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("HGPU_FUSED_PIVOT")) fused_pivot_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_SOLVE_TC")) solve_tc_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_SOLVE_NTT")) solve_ntt_ = std::atoi(e);
  if (const char* e = std::getenv("HGPU_FAR_SUB")) far_sub_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("HGPU_EDF")) edf_h_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("HGPU_EDF_RUN")) edf_run_ = std::max(1, std::min(8, std::atoi(e)));
  if (const char* e = std::getenv("HGPU_FLUSH_AHEAD")) flush_ahead_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("HGPU_FLUSH_BATCH")) flush_batch_ = std::max(1, std::min(8, std::atoi(e)));
  if (const char* e = std::getenv("HGPU_PRE_ENTRY")) pre_entry_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_NEXT_ROW")) next_row_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_UPDATE_TC")) update_tc_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_COL_EXTRACT")) col_extract_ = std::atoi(e);
  if (const char* e = std::getenv("HGPU_LOOKAHEAD")) lookahead_ = std::atoi(e);
  {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (split_gb_) {
      // the pivot entry's early stages gate k_pivot: on the chain's SMs
      stream_pre_ = green_stream((CUgreenCtx)split_ga_, hi);
      stream_next_ = green_stream((CUgreenCtx)split_gb_, hi);
    } else {
      CU(cudaStreamCreateWithPriority(&stream_pre_, cudaStreamNonBlocking, hi));
      CU(cudaStreamCreateWithPriority(&stream_next_, cudaStreamNonBlocking, hi));
    }
    // the near rows' early stages: beside the panel stream (with an SM split
    // on the large group, where the panel's near rows run)
    if (split_gb_)
      stream_pre2_ = green_stream((CUgreenCtx)split_gb_, hi);
    else
      CU(cudaStreamCreateWithPriority(&stream_pre2_, cudaStreamNonBlocking, hi));
  }
  if (const char* e = std::getenv("HGPU_PRE_NEAR")) pre_near_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_LAG_FAR")) lag_far_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("HGPU_PRE_LHAT")) pre_lhat_ = std::atoi(e) != 0;
  if (!split_gb_) {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&stream_lhat_, cudaStreamNonBlocking, lo));
    CU(cudaEventCreateWithFlags(&lhat_ev_, cudaEventDisableTiming));
  }
  if (!split_gb_) {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&stream_join_, cudaStreamNonBlocking, hi));
  }
  if (const char* e = std::getenv("HGPU_PIVOT_SEGS")) pivot_segs_ = std::max(1, std::min(6, std::atoi(e)));
  if (const char* e = std::getenv("HGPU_FAR_LANES"))
    far_lanes_ = std::max(1, std::min(kMaxFarLanes, std::atoi(e)));
  {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    far_streams_[0] = stream_far_;
    for (int l = 1; l < kMaxFarLanes; ++l) {
      if (split_gb_)
        far_streams_[l] = green_stream((CUgreenCtx)split_gb_, hi);
      else
        CU(cudaStreamCreateWithPriority(&far_streams_[l], cudaStreamNonBlocking, far_prio_));
    }
    for (int l = 0; l < kMaxFarLanes; ++l)
      CU(cudaEventCreateWithFlags(&far_ev_[l], cudaEventDisableTiming));
  }
  if (const char* e = std::getenv("HGPU_NEAR")) near_rows_ = std::max(2, std::atoi(e));
  if (const char* e = std::getenv("HGPU_RATIO_GEMM")) ratio_gemm_ = std::atoi(e);
  if (ratio_gemm_)
    for (int i = 0; i < 2; ++i)
      if (cublasCreate((cublasHandle_t*)&blas_[i]) != CUBLAS_STATUS_SUCCESS)
        throw Error(HGPU_ERR_CUDA, "cublasCreate failed");
}

Matrix::~Matrix() {
  cudaSetDevice(device_);
  release();
  if (strip_stage_) cudaFreeHost(strip_stage_);
  if (comm_) ncclCommDestroy((ncclComm_t)comm_);
  for (cudaEvent_t e : uev_) cudaEventDestroy(e);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  for (cudaEvent_t e : pev_) cudaEventDestroy(e);
  for (cudaEvent_t e : sev_) cudaEventDestroy(e);
  for (cudaEvent_t e : edf_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : pre_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : sn_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : grp_ready_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : grp_pulled_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : net_ev_) cudaEventDestroy(e);
  if (stream_next_) cudaStreamDestroy(stream_next_);
  if (stream_pre_) cudaStreamDestroy(stream_pre_);
  if (stream_pre2_) cudaStreamDestroy(stream_pre2_);
  if (stream_join_) cudaStreamDestroy(stream_join_);
  if (stream_lhat_) cudaStreamDestroy(stream_lhat_);
  if (lhat_ev_) cudaEventDestroy(lhat_ev_);
  for (cudaEvent_t e : lag_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : pre2_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : tl_pool_) cudaEventDestroy(e);
  for (void* h : blas_)
    if (h) cublasDestroy((cublasHandle_t)h);
  if (tc_blas_) cublasDestroy((cublasHandle_t)tc_blas_);
  for (int l = 1; l < kMaxFarLanes; ++l)
    if (far_streams_[l]) cudaStreamDestroy(far_streams_[l]);
  for (cudaEvent_t e : far_ev_)
    if (e) cudaEventDestroy(e);
  if (stream_far_) cudaStreamDestroy(stream_far_);
  if (stream_upd1_) cudaStreamDestroy(stream_upd1_);
  if (stream_upd2_) cudaStreamDestroy(stream_upd2_);
  if (stream_helper_) cudaStreamDestroy(stream_helper_);
  if (stream_panel_) cudaStreamDestroy(stream_panel_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Matrix::release() {
  for (void* p : {(void*)tw_, (void*)W_, (void*)that_, (void*)xhat_,
                  (void*)colbase_, (void*)strip_hdr_, (void*)strip_limbs_,
                  (void*)x_hdr_, (void*)x_limbs_, (void*)vhdr_, (void*)vlimbs_,
                  (void*)rhdr_, (void*)rlimbs_, (void*)vhat_, (void*)rhat_,
                  (void*)phdr_, (void*)plimbs_, (void*)ybuf_, (void*)rscratch_,
                  (void*)dscratch_, (void*)dscratch2_, (void*)dscratch3_, (void*)ys_,
                  (void*)vdig_, (void*)rg_t_[0], (void*)rg_t_[1], (void*)rg_c_[0],
                  (void*)rg_c_[1], (void*)rg_ws_[0], (void*)rg_ws_[1],
                  (void*)stats_, (void*)err_})
    dfree(p);
  release_interval();
  // inverse-iteration state (sized by the plan's capacity); a resident
  // start vector survives a re-plan through a host copy
  if (start_resident_ && svhdr_) {
    try {
      const int n = n_, Wv = sWv_;
      std::vector<int> hdr((size_t)n);
      std::vector<uint32_t> lim((size_t)n * Wv);
      CU(cudaMemcpy(hdr.data(), svhdr_, hdr.size() * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(lim.data(), svlimbs_, lim.size() * 4, cudaMemcpyDeviceToHost));
      saved_start_.assign(n, HostInt{});
      for (int i = 0; i < n; ++i) {
        saved_start_[i].size = hdr[i];
        saved_start_[i].limbs.assign(lim.begin() + (size_t)i * Wv,
                                     lim.begin() + (size_t)i * Wv + std::abs(hdr[i]));
      }
    } catch (const Error&) {
      saved_start_.clear();
    }
  }
  start_resident_ = have_y_ = false;
  dfree(lhat_err_);
  lhat_err_ = nullptr;
  lhat_pre_for_ = -1;
  for (void* p : {(void*)rq_prod_, (void*)rq_out_, (void*)rq_scr_, (void*)rq_colsum_,
                  (void*)rq_sign_})
    dfree(p);
  rq_prod_ = rq_out_ = rq_scr_ = nullptr;
  rq_colsum_ = nullptr;
  rq_sign_ = nullptr;
  rq_maxlen_ = rq_grid_ = 0;
  for (void* p : {(void*)lhdr_, (void*)llimbs_, (void*)svhdr_, (void*)svlimbs_,
                  (void*)sacc_, (void*)sgscr_, (void*)spair_hdr_,
                  (void*)spair_limbs_, (void*)sbits_, (void*)sybuf_,
                  (void*)srscr_, (void*)sdscr_, (void*)sys_})
    dfree(p);
  for (void* q : {(void*)rdig_col_, (void*)rdig_row_, (void*)tc_t_, (void*)tc_c_,
                  (void*)tc_acc_, (void*)tc_ws_, (void*)stw_, (void*)lhat_tab_, (void*)acch_,
                  (void*)sxhat_})
    dfree(q);
  for (uint32_t* c : lhat_chunks_) dfree(c);
  lhat_chunks_.clear();
  lhat_tab_ = nullptr;
  stw_ = acch_ = sxhat_ = nullptr;
  sdp_bits_ = sdp_xbits_ = 0;
  lhat_for_ = -1;
  rdig_col_ = rdig_row_ = tc_t_ = tc_ws_ = nullptr;
  tc_c_ = nullptr;
  tc_acc_ = nullptr;
  tc_kr_ = tc_mc_ = 0;
  rdig_for_ = -1;
  lhdr_ = svhdr_ = spair_hdr_ = sbits_ = sys_ = nullptr;
  llimbs_ = svlimbs_ = sacc_ = sgscr_ = spair_limbs_ = sybuf_ = srscr_ =
      sdscr_ = nullptr;
  have_L_ = false;
  tw_ = W_ = that_ = xhat_ = nullptr;
  colbase_ = nullptr;
  strip_hdr_ = x_hdr_ = vhdr_ = rhdr_ = phdr_ = ys_ = stats_ = err_ = nullptr;
  strip_limbs_ = x_limbs_ = vlimbs_ = rlimbs_ = vhat_ = rhat_ = plimbs_ =
      ybuf_ = rscratch_ = dscratch_ = dscratch2_ = dscratch3_ = nullptr;
  vdig_ = rg_t_[0] = rg_t_[1] = nullptr;
  rg_ws_[0] = rg_ws_[1] = nullptr;
  rg_c_[0] = rg_c_[1] = nullptr;
  rg_kd_ = rg_ncols_ = 0;
  plan_ = Plan{};
}

void Matrix::set_comm(int rank, int world, const unsigned char* id) {
  if (world < 1 || rank < 0 || rank >= world)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad rank/world");
  if (group_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "matrix already belongs to an in-process group");
  CU(cudaSetDevice(device_));
  if (comm_) {
    ncclCommDestroy((ncclComm_t)comm_);
    comm_ = nullptr;
  }
  rank_ = rank;
  world_ = world;
  if (world > 1) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c;
    NC(ncclCommInitRank(&c, world, uid, rank));
    comm_ = c;
  }
  release();  // ownership changes the workspace layout
}

void Matrix::make_group(const std::vector<int>& devices) {
  const int W = (int)devices.size();
  if (W < 1 || devices[0] != device_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "group devices must start with the matrix's device");
  if (comm_ || group_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "matrix already belongs to a rank group");
  if (interval_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "interval matrices run on one rank");
  if (W == 1) return;
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  for (int d : devices)
    if (d < 0 || d >= ndev) throw Error(HGPU_ERR_INVALID_ARGUMENT, "bad device index");
  // receivers load the owner's integers directly: peer access both ways
  for (int a : devices)
    for (int b : devices) {
      if (a == b) continue;
      int ok = 0;
      CU(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok)
        throw Error(HGPU_ERR_COMM, "no peer access from device " + std::to_string(a) +
                                       " to device " + std::to_string(b));
      CU(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        (void)cudaGetLastError();
      else
        CU(e);
      // the buffers come from device b's stream-ordered pool (dev_alloc):
      // pool memory is mapped on a peer only through cudaMemPoolSetAccess
      // (cudaDeviceEnablePeerAccess covers cudaMalloc memory alone); the
      // access applies to the pool's existing and future allocations
      cudaMemPool_t pool;
      CU(cudaDeviceGetDefaultMemPool(&pool, b));
      cudaMemAccessDesc desc{};
      desc.location.type = cudaMemLocationTypeDevice;
      desc.location.id = a;
      desc.flags = cudaMemAccessFlagsProtReadWrite;
      CU(cudaMemPoolSetAccess(pool, &desc, 1));
    }
  CU(cudaSetDevice(device_));
  std::vector<int32_t> sz;
  std::vector<uint32_t> lb;
  for (const HostInt& h : strip_) {
    sz.push_back(h.size);
    lb.insert(lb.end(), h.limbs.begin(), h.limbs.end());
  }
  auto g = std::make_shared<PeerGroup>();
  g->world = W;
  g->ranks.push_back(this);
  peers_.clear();
  for (int r = 1; r < W; ++r) {
    peers_.push_back(std::make_unique<Matrix>(n_, K_, sz.data(), lb.data(), devices[r]));
    g->ranks.push_back(peers_.back().get());
  }
  for (int r = 0; r < W; ++r) {
    Matrix* m = g->ranks[r];
    CU(cudaSetDevice(m->device_));
    m->release();  // ownership changes the workspace layout
    m->group_ = g;
    m->rank_ = r;
    m->world_ = W;
  }
  CU(cudaSetDevice(device_));
}

void Matrix::group_publish(int b, cudaStream_t st) {
  PeerGroup& g = *group_;
  CU(cudaEventRecord(grp_ready_ev_[b], st));
  std::lock_guard<std::mutex> lk(g.mu);
  g.ready_ev[b] = grp_ready_ev_[b];
  g.ready_run[b] = grp_run_;
  g.cv.notify_all();
}

Matrix* Matrix::group_await(int b, int owner, cudaStream_t st) {
  PeerGroup& g = *group_;
  cudaEvent_t e;
  {
    std::unique_lock<std::mutex> lk(g.mu);
    g.wait(lk, [&] { return g.ready_run[b] == grp_run_; });
    e = g.ready_ev[b];
  }
  CU(cudaStreamWaitEvent(st, e, 0));
  return g.ranks[owner];
}

void Matrix::group_pulled(int b, cudaStream_t st) {
  PeerGroup& g = *group_;
  CU(cudaEventRecord(grp_pulled_ev_[b], st));
  std::lock_guard<std::mutex> lk(g.mu);
  g.pulled_ev[(size_t)b * g.world + rank_] = grp_pulled_ev_[b];
  g.pulled_run[(size_t)b * g.world + rank_] = grp_run_;
  g.cv.notify_all();
}

void Matrix::group_wait_pulled(int b, cudaStream_t st) {
  PeerGroup& g = *group_;
  for (int r = 0; r < g.world; ++r) {
    if (r == rank_) continue;
    const size_t i = (size_t)b * g.world + r;
    cudaEvent_t e;
    {
      std::unique_lock<std::mutex> lk(g.mu);
      g.wait(lk, [&] { return g.pulled_run[i] == grp_run_; });
      e = g.pulled_ev[i];
    }
    CU(cudaStreamWaitEvent(st, e, 0));
  }
}

void Matrix::group_merge_err(int* herr) {
  PeerGroup& g = *group_;
  std::unique_lock<std::mutex> lk(g.mu);
  if (g.merge_run != grp_run_) {
    g.merge_run = grp_run_;
    g.arrived = 0;
    g.merged[0] = INT_MAX;
    for (int k = 1; k < kErrWords; ++k) g.merged[k] = 0;
  }
  g.merged[kErrZeroPivot] = std::min(g.merged[kErrZeroPivot], herr[kErrZeroPivot]);
  for (int k = 1; k < kErrWords; ++k) g.merged[k] |= herr[k];
  ++g.arrived;
  g.cv.notify_all();
  g.wait(lk, [&] { return g.arrived == g.world; });
  for (int k = 0; k < kErrWords; ++k) herr[k] = g.merged[k];
}

// ldlt_det_parallel over the group (ldlt.cpp:315-341): one host thread per
// rank runs the same panel schedule on its own columns; the plan and the
// capacity retries are decided for all ranks together.
FactorResult Matrix::factor_group(const HostInt& x, unsigned flags) {
  PeerGroup& g = *group_;
  const int W = g.world;
  int min_logL = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    for (Matrix* m : g.ranks) {
      CU(cudaSetDevice(m->device_));
      if (m->ws_released_) m->reclaim_workspace();
      if (!m->W_ || (min_logL && m->plan_.logL < min_logL)) m->build(min_logL);
    }
    CU(cudaSetDevice(device_));
    const int nblocks = (n_ + plan_.kb - 1) / plan_.kb;
    {
      std::lock_guard<std::mutex> lk(g.mu);
      ++g.run;
      g.poisoned = false;
      g.why.clear();
      g.ready_ev.assign(nblocks + 1, nullptr);
      g.ready_run.assign(nblocks + 1, -1);
      g.pulled_ev.assign((size_t)(nblocks + 1) * W, nullptr);
      g.pulled_run.assign((size_t)(nblocks + 1) * W, -1);
    }
    std::vector<FactorResult> res(W);
    std::vector<std::exception_ptr> errs(W);
    auto body = [&](int r) {
      Matrix* m = g.ranks[r];
      try {
        CU(cudaSetDevice(m->device_));
        res[r].n = n_;
        res[r].K = K_;
        // rank 0 holds every pivot and (for captures / KEEP_L) reads the
        // other ranks' ratio columns in place
        const unsigned f = r == 0 ? flags : (flags & HGPU_PROFILE);
        m->run(x, f, res[r]);
      } catch (const std::exception& e) {
        errs[r] = std::current_exception();
        g.poison(std::string("rank ") + std::to_string(r) + ": " + e.what());
      }
    };
    std::vector<std::thread> th;
    for (int r = 1; r < W; ++r) th.emplace_back(body, r);
    body(0);
    for (std::thread& t : th) t.join();
    CU(cudaSetDevice(device_));
    // the first failure that is not a consequence of another rank's
    std::exception_ptr first;
    for (int r = 0; r < W && !first; ++r) {
      if (!errs[r]) continue;
      try {
        std::rethrow_exception(errs[r]);
      } catch (const Error& e) {
        if (std::string(e.what()).rfind(kPeerFailed, 0) != 0) first = errs[r];
      } catch (...) {
        first = errs[r];
      }
    }
    for (int r = 0; r < W && !first; ++r)
      if (errs[r]) first = errs[r];
    if (!first) {
      FactorResult out = std::move(res[0]);
      for (int r = 1; r < W; ++r) {
        out.device_ms = std::max(out.device_ms, res[r].device_ms);
        out.launches += res[r].launches;
        out.update_launches += res[r].update_launches;
        out.update_ms += res[r].update_ms;
        out.update_products += res[r].update_products;
        out.net_ms += res[r].net_ms;
      }
      return out;
    }
    try {
      std::rethrow_exception(first);
    } catch (const Error& e) {
      if (e.status != HGPU_ERR_CAPACITY) throw;
      if (e.cap_flags == kCapAmax && recip_bound_) {
        for (Matrix* m : g.ranks) m->recip_bound_ = false;
        continue;
      }
      min_logL = plan_.logL + 1;
      for (Matrix* m : g.ranks) {
        CU(cudaSetDevice(m->device_));
        m->release();
      }
      CU(cudaSetDevice(device_));
    }
  }
  throw Error(HGPU_ERR_CAPACITY, "values outgrew every transform plan");
}

// Panel slot sets (V/R integers and transforms): two for the lookahead (the
// interval path: one), 2 + deferral depth (HGPU_DEFER), or one per panel for
// the EDF schedule, fewer when the device memory would not hold them beside
// the workspace.
void Matrix::alloc_slots() {
  const Plan& P = plan_;
  const size_t NW = (size_t)dp_.NW;
  const int kb = P.kb;
  size_t nsets = 1;
  if (!interval_) {
    const int nblocks = (n_ + kb - 1) / kb;
    nsets = edf_h_ > 0 ? (size_t)nblocks + 1 : 2 + (size_t)std::max(0, defer_);
    const double per_set = (double)kb * n_ * (2.0 * NW + 2.0 * P.cap + 2.0) * 4.0;
    const size_t free_b = device_available(device_);
    // share of the free memory the slot sets may take (the rest is for the L
    // store and the solve buffers of an inverse iteration); HGPU_SLOT_SETS
    // forces a count (tests of the reuse path on small matrices)
    double frac = 0.6;
    if (const char* e = std::getenv("HGPU_SLOT_FRAC")) frac = std::min(0.9, std::max(0.1, std::atof(e)));
    while (nsets > 2 && per_set * nsets > frac * (double)free_b) --nsets;
    if (const char* e = std::getenv("HGPU_SLOT_SETS"))
      nsets = std::min(nsets, (size_t)std::max(2, std::atoi(e)));
  }
  nsets_ = (int)nsets;
  vhdr_ = dalloc<int>(nsets * kb * n_);
  rhdr_ = dalloc<int>(nsets * kb * n_);
  vlimbs_ = dalloc<uint32_t>(nsets * kb * n_ * P.cap);
  rlimbs_ = dalloc<uint32_t>(nsets * kb * n_ * P.cap);
  vhat_ = dalloc<uint32_t>(nsets * kb * n_ * NW);
  rhat_ = dalloc<uint32_t>(nsets * kb * n_ * NW);
  ws_released_ = false;
}

// The transform-domain solve needs the L-entry transforms of the whole factor
// (ne x NW words); at configs 4/5 they do not fit beside the factorisation's
// workspace.  The solves never touch W or the slot sets, so they are handed
// back to the pool for the solves and taken again by the next factorisation
// (whose L-entry transforms are recomputed anyway).
void Matrix::release_workspace() {
  for (void* q : {(void*)W_, (void*)vhdr_, (void*)rhdr_, (void*)vlimbs_, (void*)rlimbs_,
                  (void*)vhat_, (void*)rhat_})
    dfree(q);
  W_ = vlimbs_ = rlimbs_ = vhat_ = rhat_ = nullptr;
  vhdr_ = rhdr_ = nullptr;
  ws_released_ = true;
}

void Matrix::reclaim_workspace() {
  release_solve_transforms();
  W_ = dalloc<uint32_t>((size_t)std::max<long long>(plan_.entries, 1) * dp_.NW);
  alloc_slots();
  ws_released_ = false;
}

void Matrix::release_solve_transforms() {
  dfree(stw_);
  dfree(lhat_tab_);
  for (uint32_t* c : lhat_chunks_) dfree(c);
  lhat_chunks_.clear();
  dfree(acch_);
  dfree(sxhat_);
  stw_ = acch_ = sxhat_ = nullptr;
  lhat_tab_ = nullptr;
  sdp_bits_ = sdp_xbits_ = 0;
  lhat_for_ = -1;
}

void Matrix::build(int min_logL) {
  release();
  // PD bound: every workspace entry and every product V_p[c] R_p[r] is
  // bounded by the largest diagonal moment (plus the shift); 64 bits margin.
  plan_ = choose_plan(n_, K_, strip_bits_ + 64, min_logL);
  Plan& P = plan_;
  // panel width (experiment knob: 16, 32 or 64 columns; 32 measured best)
  if (const char* e = std::getenv("HGPU_KB")) {
    const int v = std::atoi(e);
    if (v == 16 || v == 32 || v == 64) P.kb = v;
  }
  // ownership: column blocks of kb columns, reflected round-robin
  const int nblocks = (n_ + P.kb - 1) / P.kb;
  owned_blocks_.clear();
  colbase_h_.assign(n_, -1);
  long long entries = 0;
  for (int b = 0; b < nblocks; ++b) {
    if (block_owner(b, world_) != rank_) continue;
    owned_blocks_.push_back(b);
    for (int c = b * P.kb; c < std::min(n_, (b + 1) * P.kb); ++c) {
      colbase_h_[c] = entries;
      entries += n_ - c;
    }
  }
  P.entries = entries;

  DevPlan& D = dp_;
  D = DevPlan{};
  D.n = n_;
  D.K = K_;
  D.k2 = K_ / 2;
  D.np = P.np;
  D.logL = P.logL;
  D.L = P.L;
  D.w = P.w;
  D.T = P.T;
  D.cap = P.cap;
  D.ycap = P.ycap;
  D.NW = P.np * P.L;
  std::vector<uint32_t> tab = transform_tables(D, P);
  const size_t npl = (size_t)P.np * P.L;
  tw_ = dalloc<uint32_t>(tab.size());
  CU(cudaMemcpy(tw_, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
  D.tw = tw_;
  D.twp = tw_ + npl;
  D.itw = tw_ + 2 * npl;
  D.itwp = tw_ + 3 * npl;
  D.twm = tw_ + 4 * npl;
  D.itwm = tw_ + 5 * npl;
  {
    // stage the tables in SMEM when the extraction CTA still fits twice
    const size_t words = 3 * npl + 2 * (size_t)(P.L + P.T) + P.cap + 64;
    D.tw_smem = words * 4 <= 110 * 1024 ? 1 : 0;
    int dev = 0, nsm = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int per_sm = 3;
    if (const char* g = std::getenv("HGPU_GRID")) per_sm = std::max(1, std::atoi(g));
    D.grid_cap = per_sm * nsm;
    // HGPU_RECIP_FAST=0: the original reciprocal; 1: the latency-lean body (same
    // Y bit for bit); 3 (default): its first levels on the register ladder
    D.recip_fast = 3;
    if (const char* rf = std::getenv("HGPU_RECIP_FAST")) D.recip_fast = std::atoi(rf);
    if (const char* dbg = std::getenv("HGPU_DEBUG")) D.debug = std::atoi(dbg);
#ifndef HGPU_TIMING_EXPERIMENTS
    // bits that skip work (512: the deferred update, 16384 / 32768: the
    // solve's pointwise / critical work) exist for timing experiments only
    // and give wrong results: a production build ignores them
    D.debug &= ~(512 | 16384 | 32768);
#endif
  }

  CU(configure_kernels(D, &div_smem_, &div_global_, &recip_global_));
  if (update_tc_) CU(configure_update_tc());

  const size_t NW = (size_t)D.NW;
  const int kb = P.kb;
  W_ = dalloc<uint32_t>((size_t)std::max<long long>(entries, 1) * NW);
  colbase_ = dalloc<long long>(n_);
  CU(cudaMemcpy(colbase_, colbase_h_.data(), n_ * sizeof(long long),
                cudaMemcpyHostToDevice));
  // strip + x as limb integers, and their transforms
  const int ns = 2 * n_ - 1;
  strip_hdr_ = dalloc<int>(ns);
  strip_limbs_ = dalloc<uint32_t>((size_t)ns * P.cap);
  {
    std::vector<int> hdr(ns);
    std::vector<uint32_t> lim((size_t)ns * P.cap, 0);
    for (int s = 0; s < ns; ++s) {
      if ((int)strip_[s].limbs.size() > P.cap)
        throw Error(HGPU_ERR_CAPACITY, "strip entry exceeds limb capacity");
      hdr[s] = strip_[s].size;
      std::copy(strip_[s].limbs.begin(), strip_[s].limbs.end(),
                lim.begin() + (size_t)s * P.cap);
    }
    CU(cudaMemcpy(strip_hdr_, hdr.data(), ns * sizeof(int),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(strip_limbs_, lim.data(), lim.size() * 4,
                  cudaMemcpyHostToDevice));
  }
  that_ = dalloc<uint32_t>((size_t)ns * NW);
  xhat_ = dalloc<uint32_t>(NW);
  x_hdr_ = dalloc<int>(1);
  x_limbs_ = dalloc<uint32_t>(P.cap);
  err_ = dalloc<int>(kErrWords);
  {
    const int init[kErrWords] = {INT_MAX, 0, 0, 0};
    CU(cudaMemcpy(err_, init, sizeof(init), cudaMemcpyHostToDevice));
  }
  CU(launch_fwd_ints(D, IntBuf{strip_hdr_, strip_limbs_}, 0, that_, 0, ns, 0,
                     nullptr, err_, stream_));
  int herr[kErrWords];
  CU(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, stream_));
  CU(cudaStreamSynchronize(stream_));
  if (herr[kErrCapacity])
    throw Error(HGPU_ERR_CAPACITY, "strip does not fit the transform plan");

  alloc_slots();
  phdr_ = dalloc<int>(n_);
  plimbs_ = dalloc<uint32_t>((size_t)n_ * P.cap);
  // reciprocals in a ring of kYRing stage sets: the far-row divisions of
  // stage p may lag the pivot chain by up to a panel
  ybuf_ = dalloc<uint32_t>(kYRing * (size_t)P.ycap);
  ys_ = dalloc<int>(4 * kYRing);
  rscratch_ = dalloc<uint32_t>(recip_scratch_words(D));
  if (div_global_) {
    dscratch_ = dalloc<uint32_t>((size_t)D.grid_cap * divide_smem_words(D));
    dscratch2_ = dalloc<uint32_t>((size_t)D.grid_cap * divide_smem_words(D));
    dscratch3_ = dalloc<uint32_t>((size_t)D.grid_cap * divide_smem_words(D));
  }
  stats_ = dalloc<int>(3 * (size_t)n_);
  if (ratio_gemm_ && !interval_) {
    // ratio GEMM operands, sized for the PD bounds of any shift whose
    // diagonal stays within strip_bits_ + 64 bits (run() checks its own)
    const int db = strip_bits_ + 64;
    rg_kd_ = ratio_gemm_kd(db);
    rg_ncols_ = ratio_gemm_ncols(db);
    vdig_ = dalloc<uint8_t>((size_t)n_ * rg_kd_);
    for (int i = 0; i < 2; ++i) {
      rg_t_[i] = dalloc<uint8_t>((size_t)rg_ncols_ * rg_kd_);
      rg_c_[i] = dalloc<int32_t>((size_t)n_ * rg_ncols_);
      rg_ws_[i] = dalloc<uint8_t>(kBlasWorkspace);
      if (cublasSetWorkspace((cublasHandle_t)blas_[i], rg_ws_[i], kBlasWorkspace) !=
          CUBLAS_STATUS_SUCCESS)
        throw Error(HGPU_ERR_CUDA, "cublasSetWorkspace failed");
    }
  }
  if (interval_) build_interval();
}

// 7-bit digit columns of |V| (K of the ratio GEMM) and quotient columns (M)
// for diagonal entries of at most db bits: |V| <= dmax + 3 - k2 bits (PD
// bound, k_recip's amax), and the columns needed above K0d are
// (e + 282) / 7 + 3 with e <= (db + 1) / 2 + k2 + 5 (k_ratio_finish checks
// every row against its actual operands).
int Matrix::ratio_gemm_kd(int db) const {
  const int vb = std::min(db + 3 - K_ / 2, 32 * plan_.cap - K_ / 2);
  return ((vb + 6) / 7 + 15) & ~15;
}
int Matrix::ratio_gemm_ncols(int db) const {
  const int e = (db + 1) / 2 + K_ / 2 + 5;
  return ((e + 282) / 7 + 3 + 15) & ~15;
}

void Matrix::ratio_gemm(int which, int p, int r_begin, int r_end, IntBuf vint,
                        long long row0, const uint32_t* yb, const int* yss,
                        IntBuf rint, int* maxdegR, uint32_t* dscr,
                        cudaStream_t s) {
  const DevPlan& D = dp_;
  r_begin = std::max(r_begin, p + 1);
  const int rows = r_end - r_begin;
  if (rows <= 0) return;
  cublasHandle_t h = (cublasHandle_t)blas_[which];
  CU(launch_toeplitz(D, yb, yss, rg_kd_, rg_ncols_, rg_t_[which], err_, s));
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS)
    throw Error(HGPU_ERR_CUDA, "cublasSetStream failed");
  const int32_t one = 1, zero = 0;
  const cublasStatus_t bs = cublasGemmEx(
      h, CUBLAS_OP_T, CUBLAS_OP_N, rg_ncols_, rows, rg_kd_, &one, rg_t_[which],
      CUDA_R_8I, rg_kd_, vdig_ + (size_t)r_begin * rg_kd_, CUDA_R_8I, rg_kd_,
      &zero, rg_c_[which], CUDA_R_32I, rg_ncols_, CUBLAS_COMPUTE_32I,
      CUBLAS_GEMM_DEFAULT);
  if (bs != CUBLAS_STATUS_SUCCESS)
    throw Error(HGPU_ERR_CUDA, "int8 ratio GEMM failed (cublas status " +
                                   std::to_string((int)bs) + ")");
  CU(launch_ratio_finish(D, vint, row0, p, r_begin, r_end, yb, yss,
                         rg_c_[which], rg_ncols_, rint, row0, rhat_, maxdegR,
                         dscr, div_global_ ? 1 : 0, err_, s));
}

void Matrix::panel_broadcast(int owner, int p0, int ns, long long row0,
                             cudaStream_t st) {
  if (world_ == 1 || !comm_) return;
  ncclComm_t c = (ncclComm_t)comm_;
  const Plan& P = plan_;
  // stage p = p0 + s: V_p[r] for r >= p and R_p[r] for r > p (the rows below
  // p are unused), each at the slot's cap stride -- ns (n - p) rows instead
  // of the whole slot set.  The error words are not broadcast: every rank
  // keeps its own flags until the end-of-run reduction (run()).
  NC(ncclGroupStart());
  for (int s = 0; s < ns; ++s) {
    const int p = p0 + s;
    const long long r0 = row0 + (long long)s * n_ + p;
    const size_t rows = (size_t)(n_ - p);
    NC(ncclBroadcast(vhdr_ + r0, vhdr_ + r0, rows, ncclInt32, owner, c, st));
    NC(ncclBroadcast(rhdr_ + r0, rhdr_ + r0, rows, ncclInt32, owner, c, st));
    NC(ncclBroadcast(vlimbs_ + r0 * P.cap, vlimbs_ + r0 * P.cap, rows * P.cap, ncclUint32,
                     owner, c, st));
    NC(ncclBroadcast(rlimbs_ + r0 * P.cap, rlimbs_ + r0 * P.cap, rows * P.cap, ncclUint32,
                     owner, c, st));
  }
  NC(ncclBroadcast(phdr_ + p0, phdr_ + p0, ns, ncclInt32, owner, c, st));
  NC(ncclBroadcast(plimbs_ + (size_t)p0 * P.cap, plimbs_ + (size_t)p0 * P.cap,
                   (size_t)ns * P.cap, ncclUint32, owner, c, st));
  for (int k = 0; k < 3; ++k)
    NC(ncclBroadcast(stats_ + (size_t)k * n_ + p0, stats_ + (size_t)k * n_ + p0,
                     ns, ncclInt32, owner, c, st));
  NC(ncclGroupEnd());
}

void Matrix::run(const HostInt& x, unsigned flags, FactorResult& res) {
  const auto t_run0 = std::chrono::steady_clock::now();
  const Plan& P = plan_;
  const DevPlan& D = dp_;
  cudaStream_t st = stream_;       // trailing updates (bulk)
  cudaStream_t sp = stream_panel_; // panel factorisation (critical path)
  const int n = n_, kb = P.kb;
  const size_t NW = (size_t)D.NW;
  const long long slot_stride = (long long)n * NW;

  // x -> transform
  if ((int)x.limbs.size() > P.cap)
    throw Error(HGPU_ERR_CAPACITY, "shift exceeds limb capacity");
  {
    std::vector<uint32_t> xl(P.cap, 0);
    std::copy(x.limbs.begin(), x.limbs.end(), xl.begin());
    CU(cudaMemcpyAsync(x_limbs_, xl.data(), P.cap * 4, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(x_hdr_, &x.size, 4, cudaMemcpyHostToDevice, st));
  }
  int herr0[kErrWords] = {INT_MAX, 0, 0, 0};
  CU(cudaMemcpyAsync(err_, herr0, sizeof(herr0), cudaMemcpyHostToDevice, st));
  if (strip_dirty_) {
    // set_strip: the new moments into the plan's strip buffers and their
    // transforms (a capacity overflow raises the flag checked below)
    const int ns = 2 * n_ - 1;
    // pinned staging (kept): hdr words, then cap-strided limbs
    const size_t words = (size_t)ns + (size_t)ns * P.cap;
    if (strip_stage_words_ < words) {
      if (strip_stage_) cudaFreeHost(strip_stage_);
      strip_stage_ = nullptr;
      CU(cudaHostAlloc((void**)&strip_stage_, words * 4, cudaHostAllocDefault));
      strip_stage_words_ = words;
    }
    int* hdr = reinterpret_cast<int*>(strip_stage_);
    uint32_t* lim = strip_stage_ + ns;
    for (int s2 = 0; s2 < ns; ++s2) {
      if ((int)strip_[s2].limbs.size() > P.cap)
        throw Error(HGPU_ERR_CAPACITY, "strip entry exceeds limb capacity");
      hdr[s2] = strip_[s2].size;
      uint32_t* dst = lim + (size_t)s2 * P.cap;
      const size_t len = strip_[s2].limbs.size();
      std::memcpy(dst, strip_[s2].limbs.data(), len * 4);
      std::memset(dst + len, 0, (P.cap - len) * 4);
    }
    CU(cudaMemcpyAsync(strip_hdr_, hdr, ns * sizeof(int), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(strip_limbs_, lim, (size_t)ns * P.cap * 4, cudaMemcpyHostToDevice, st));
    CU(launch_fwd_ints(D, IntBuf{strip_hdr_, strip_limbs_}, 0, that_, 0, ns, 0, nullptr, err_,
                       st));
    strip_dirty_ = false;
  }
  CU(cudaMemsetAsync(stats_, 0xff, 3 * (size_t)n * sizeof(int), st));  // -1
  const long long launches0 = kernel_launch_count();
  if (group_) {
    std::lock_guard<std::mutex> lk(group_->mu);
    grp_run_ = group_->run;
  }
  CU(cudaEventRecord(ev0_, st));
  CU(launch_fwd_ints(D, IntBuf{x_hdr_, x_limbs_}, 0, xhat_, 0, 1, 0, nullptr,
                     err_, st));
  CU(launch_init_w(D, that_, xhat_, colbase_, W_, st));

  int* maxbitsV = stats_;
  int* maxdegV = stats_ + n;
  int* maxdegR = stats_ + 2 * n;
  IntBuf vint{vhdr_, vlimbs_}, rint{rhdr_, rlimbs_}, piv{phdr_, plimbs_};
  const bool capture = flags & HGPU_CAPTURE;
  have_L_ = false;
  if ((flags & HGPU_KEEP_L) && !lhdr_) {
    const size_t nl = (size_t)n * (n - 1) / 2;
    const auto ta = std::chrono::steady_clock::now();
    lhdr_ = dalloc<int>(std::max<size_t>(nl, 1));
    llimbs_ = dalloc<uint32_t>(std::max<size_t>(nl, 1) * P.cap);
    if (std::getenv("HGPU_HOST_TRACE"))
      std::fprintf(stderr, "L store: %.1f MB allocated in %.3f ms\n", nl * (double)P.cap * 4 / 1e6,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta)
                       .count());
  }
  const bool profile = flags & HGPU_PROFILE;
  // capture limit (hgpu_matrix_set_capture_rows): stages and rows < crow
  const int crow = capture_rows_ > 0 ? std::min(n, capture_rows_) : n;
  if (capture) {
    res.ratios.assign(crow > 0 ? crow - 1 : 0, {});
    res.have_ratios = true;
    res.capture_rows = crow;
  }
  std::vector<int> hr_hdr;
  std::vector<uint32_t> hr_limbs;
  size_t uev_used = 0;
  const int nblocks = (n + kb - 1) / kb;
  while ((int)pev_.size() < 4 * nblocks + 4) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pev_.push_back(e);
  }
  // events: panel_done[b], next_ready[b] (panel b's columns fully updated),
  // trail_done[b] (slot set of panel b released)
  if (world_ > 1)
    while ((int)net_ev_.size() < 2 * nblocks + 2) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      net_ev_.push_back(e);
    }
  std::vector<int> net_panels;
  if (group_)
    for (auto* evs : {&grp_ready_ev_, &grp_pulled_ev_})
      while ((int)evs->size() < nblocks + 1) {
        cudaEvent_t e;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs->push_back(e);
      }
  cudaEvent_t* panel_done = pev_.data();
  cudaEvent_t* next_ready = pev_.data() + nblocks + 1;
  cudaEvent_t* trail_done = pev_.data() + 2 * nblocks + 2;
  // rest_done[b]: the deferred part of panel b's trailing update (stream su2)
  cudaEvent_t* rest_done = pev_.data() + 3 * nblocks + 3;

  // slot set of panel b: rows [set*kb*n, ...) of Vint/Rint/Vhat/Rhat
  const int nsets = nsets_;
  auto set_row0 = [&](int b) { return (long long)(b % nsets) * kb * n; };
  // Trailing update of panel b, by band j (columns
  // [j kb, (j+1) kb)):
  //   j = b+1          at the end of panel b on su1 (gates panel b+1),
  //   b+2 <= j <= b+s  caught up on su1 at the start of panel j-1, while
  //                    panel j-1 factorises (band j is idle then),
  //   j >= b+1+s       at the end of panel b on su2, lowest priority.
  // su2's update of panel b may lag up to s panels: early panels (much
  // trailing work, short pivot chain) hand work to late ones (little work,
  // the chain alone).  Band j is touched by su2 up to panel j-1-s, then by
  // su1, which waits for rest_done[j-1-s] first.  Slot sets are reused after
  // nsets = s + 2 panels.
  const int sdef = std::max(1, nsets - 2);
  cudaStream_t su1 = stream_upd1_, su2 = stream_upd2_;
  // EDF schedule of the trailing update (edf_h_ = H > 0): the update of band
  // j by panel b' (U(b',j)) is due at panel j.  su1 runs U(b, b+1) at the
  // end of panel b; every other pair goes to su2 in deadline order: at the
  // end of panel b, all pending pairs with j <= b + H + 1, by band and then
  // panel, one launch each.  Far bands are not touched before they come
  // within H panels, so old panels' far work never blocks a near band (the
  // FIFO trap of one launch per panel).  band_ev[j]: su2's last launch on
  // band j (su1 waits for it); edf_next[b']: next band of panel b' to queue.
  const bool edf = edf_h_ > 0 && nsets >= 3;
  std::vector<int> edf_next(nblocks, INT_MAX);
  std::vector<cudaEvent_t> band_ev(nblocks + 1, nullptr);
  size_t edf_used = 0;
  auto edf_event = [&]() {
    while (edf_ev_.size() <= edf_used) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      edf_ev_.push_back(e);
    }
    return edf_ev_[edf_used++];
  };
  const char* tl_path = std::getenv("HGPU_TIMELINE");
  tl_.clear();
  tl_used_ = 0;
  // kinds: 0 col(pivot) 1 extract(pivot) 2 recip 3 col(rest) 4 extract(rest)
  //        5 divide 6 col(all) 7 extract(all) 8 update(next panel) 9 update(rest)
  auto TL = [&](int kind, int p, cudaStream_t s, auto&& launch) {
    if (!tl_path) {
      CU(launch());
      return;
    }
    while (tl_pool_.size() < tl_used_ + 2) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      tl_pool_.push_back(e);
    }
    cudaEvent_t a = tl_pool_[tl_used_], b = tl_pool_[tl_used_ + 1];
    tl_used_ += 2;
    CU(cudaEventRecord(a, s));
    CU(launch());
    CU(cudaEventRecord(b, s));
    tl_.push_back({kind, p, a, b});
  };
  // rows: the whole lower part (r_lo < 0), rows below r_hi only (r_lo < 0,
  // r_hi >= 0), or the rectangle [r_lo, r_hi) (r_lo >= c_end)
  auto timed_update = [&](int b, int nslots, int c_begin, int c_end,
                          cudaStream_t us, int kind, int s0 = 0, int r_lo = -1,
                          int r_hi = -1) {
    if (c_begin >= c_end || nslots <= 0) return;
    if (r_lo >= 0 && r_lo >= r_hi) return;
    if (profile) {
      while (uev_.size() < uev_used + 2) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        uev_.push_back(e);
      }
      CU(cudaEventRecord(uev_[uev_used], us));
    }
    const long long r0 = set_row0(b) + (long long)s0 * n;  // stage s0 of the panel
    const bool tc = update_tc_ && c_end - c_begin <= 32 && nslots <= 256 && D.NW % 4 == 0 &&
                    D.L % 4 == 0 && r_lo < 0 && r_hi < 0;
    TL(kind, b, us, [&] {
      if (tc)
        return launch_update_tc(D, W_, colbase_, vhat_ + r0 * NW, rhat_ + r0 * NW, slot_stride,
                                nslots, c_begin, c_end, err_, us);
      if (r_lo >= 0)
        return launch_update_rect(D, W_, colbase_, vhat_ + r0 * NW, rhat_ + r0 * NW,
                                  slot_stride, nslots, c_begin, c_end, r_lo, r_hi, err_, us);
      return launch_update(D, P.tile, W_, colbase_, vhat_ + r0 * NW,
                           rhat_ + r0 * NW, slot_stride, nslots, c_begin, c_end,
                           err_, us, r_hi);
    });
    if (profile) {
      CU(cudaEventRecord(uev_[uev_used + 1], us));
      uev_used += 2;
      double pairs = 0;
      const int rb_ = r_lo >= 0 ? r_lo : 0, re_ = r_hi >= 0 ? std::min(n, r_hi) : n;
      for (int c = c_begin; c < c_end; ++c) pairs += std::max(0, re_ - std::max(c, rb_));
      res.update_products += pairs * nslots * (double)NW;
      ++res.update_launches;
    }
  };
  // trailing update of panel b restricted to owned columns in [lo, hi)
  // (stages [s0, s0 + ns) of the panel; ns < 0: all from s0)
  auto trailing = [&](int b, int lo, int hi, cudaStream_t us, int kind, int s0 = 0,
                      int ns = -1) {
    const int p0 = b * kb;
    const int nsl = ns >= 0 ? ns : std::min(kb, n - 1 - p0) - s0;
    if (nsl <= 0) return;
    int run_begin = -1, run_end = -1;
    auto flush = [&]() {
      if (run_begin >= 0 && run_begin < run_end)
        timed_update(b, nsl, run_begin, run_end, us, kind, s0);
      run_begin = run_end = -1;
    };
    for (int ob : owned_blocks_) {
      const int c0 = std::max(lo, ob * kb), c1 = std::min(hi, (ob + 1) * kb);
      if (c0 >= c1) continue;
      if (run_begin >= 0 && c0 == run_end) {
        run_end = c1;
      } else {
        flush();
        run_begin = c0;
        run_end = c1;
      }
    }
    flush();
  };

  // U(bp, j) for the m consecutive panels bp.. on su2 (owned columns of band
  // j): their slot sets are adjacent, so one launch accumulates all 32 m
  // stages (<= 256, the accumulator bound) with one pass over W
  auto edf_enqueue = [&](int bp, int m, int j) {
    const int c0 = j * kb, c1 = std::min(n, (j + 1) * kb);
    if (!(D.debug & 512)) {  // 512: timing experiment only
      for (int ob : owned_blocks_)
        if (ob == j) timed_update(bp, kb * m, c0, c1, su2, 9);
    }
    cudaEvent_t e = edf_event();
    CU(cudaEventRecord(e, su2));
    band_ev[j] = e;
  };
  // all pending panels of band j (edf_next[bp] == j), in runs of <= 8
  // consecutive panels whose slot sets do not wrap
  auto edf_band = [&](int j, int bmax) {
    int bp = 0;
    while (bp <= bmax) {
      if (edf_next[bp] != j) {
        ++bp;
        continue;
      }
      int m = 1;
      while (m < std::min(edf_run_, 256 / kb) && bp + m <= bmax && edf_next[bp + m] == j &&
             (bp % nsets) + m < nsets)
        ++m;
      edf_enqueue(bp, m, j);
      for (int k = 0; k < m; ++k) ++edf_next[bp + k];
      bp += m;
    }
  };
  while ((int)sev_.size() < 4 * n + 4) {  // + panel entry / far join
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sev_.push_back(e);
  }
  cudaStream_t sh = stream_helper_;
  while ((int)sn_ev_.size() < n) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sn_ev_.push_back(e);
  }
  while ((int)pre_ev_.size() < n) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pre_ev_.push_back(e);
  }
  while ((int)lag_ev_.size() < 2 * nblocks + 4) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    lag_ev_.push_back(e);
  }
  while ((int)pre2_ev_.size() < n) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pre2_ev_.push_back(e);
  }
  {
    // bits bound of any diagonal Schur complement W_rr (PD: <= M_rr - x)
    int db = 0;
    for (int r = 0; r < n; ++r) {
      const HostInt& d = strip_[2 * r];
      if (!d.limbs.empty())
        db = std::max(db, 32 * ((int)d.limbs.size() - 1) +
                              (32 - __builtin_clz(d.limbs.back())));
    }
    if (!x.limbs.empty())
      db = std::max(db, 32 * ((int)x.limbs.size() - 1) +
                            (32 - __builtin_clz(x.limbs.back())));
    dmax_bits_ = db + 1;
  }
  CU(cudaEventRecord(next_ready[0], st));  // init done
  CU(cudaStreamWaitEvent(su1, next_ready[0], 0));
  CU(cudaStreamWaitEvent(su2, next_ready[0], 0));
  // lagged far rows (see engine.h): single rank, EDF order, plain near path
  const bool lag_ok = lag_far_ && edf && world_ == 1 && !group_ && !capture && !lookahead_ &&
                      stream_join_ && near_rows_ >= kb && P.tile == 16 && D.NW % 32 == 0 &&
                      !update_tc_;
  bool prev_lag = false;  // panel b-1 left band b's far rows to lag_ev_[2b+1]
  int edf_flushed = 0;    // panels [0, edf_flushed) have had all their bands enqueued
  // L-entry transforms during the factorisation: a solve plan with its own
  // chunk store exists (not borrowing the workspace), single rank
  const bool pre_lhat_on = pre_lhat_ && (flags & HGPU_KEEP_L) && solve_ntt_ && sdp_bits_ > 0 &&
                           !lhat_chunks_.empty() && lhat_tab_ && stream_lhat_ && world_ == 1 &&
                           !group_ && !interval_;
  if (pre_lhat_on) {
    if (!lhat_err_) lhat_err_ = dalloc<int>(kErrWords);
    const int z[kErrWords] = {INT_MAX, 0, 0, 0};
    CU(cudaMemcpyAsync(lhat_err_, z, sizeof(z), cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(lhat_ev_, st));
    CU(cudaStreamWaitEvent(stream_lhat_, lhat_ev_, 0));
  }
  lhat_pre_for_ = -1;
  for (int b = 0; b < nblocks; ++b) {
    const int p0 = b * kb, p1 = std::min(n, p0 + kb), ns = p1 - p0;
    const int owner = block_owner(b, world_);
    bool lag = false;       // this panel ends without its lanes >= 1
    const long long row0set = set_row0(b);
    // stages of this panel already applied to band b+1 (sub-panel lookahead)
    int la_done = 0;
    // ---- panel b on the high-priority streams
    CU(cudaStreamWaitEvent(sp, next_ready[b], 0));
    // slot set reuse: su1's last use of panel b - nsets precedes next_ready[b]
    if (edf && nsets <= nblocks) {
      // EDF with reused slot sets: a panel whose set comes up for reuse gets
      // all its remaining bands (it is "flushed").  Flushing at the reuse
      // stalls the chain for the whole flush; instead the oldest pending
      // panels are flushed flush_ahead_ panels early, several per launch
      // (adjacent slot sets, one pass over W per band), and the panel stream
      // only waits for the event of the set it actually reuses.
      const int fa = std::min(flush_ahead_, std::max(0, nsets - 3));
      const int need = std::min(b, b - nsets + 1 + fa);  // panels < need are flushed
      if (need > edf_flushed) {
        const int upto = std::max(need, std::min(b - 2, edf_flushed + flush_batch_));
        int bp = edf_flushed;
        while (bp < upto) {
          int m = 1;
          while (m < std::min(edf_run_, 256 / kb) && bp + m < upto &&
                 edf_next[bp + m] == edf_next[bp] && (bp % nsets) + m < nsets)
            ++m;
          for (int j = edf_next[bp]; j < nblocks; ++j) edf_enqueue(bp, m, j);
          for (int k2 = 0; k2 < m; ++k2) {
            edf_next[bp + k2] = INT_MAX;
            CU(cudaEventRecord(rest_done[bp + k2], su2));
          }
          bp += m;
        }
        edf_flushed = upto;
      }
      if (b >= nsets) CU(cudaStreamWaitEvent(sp, rest_done[b - nsets], 0));
    } else if (!edf && b >= nsets) {
      CU(cudaStreamWaitEvent(sp, rest_done[b - nsets], 0));
    }
    // catch-up of band b+1 with panels [b+1-s, b-1] on su1 (after su2's
    // last touch of the band, panel b-s), overlapping panel b
    if (!edf && p1 < n) {
      if (b - sdef >= 0) CU(cudaStreamWaitEvent(su1, rest_done[b - sdef], 0));
      for (int bb = std::max(0, b + 1 - sdef); bb <= b - 1; ++bb)
        trailing(bb, p1, std::min(n, p1 + kb), su1, 13);
    }
    if (owner == rank_ && group_) {
      // group: the receivers of the last panel this rank wrote into the same
      // slot set must have pulled it (read its integers) before it is reused
      for (int bb = b - nsets; bb >= 0; bb -= nsets)
        if (block_owner(bb, world_) == rank_) {
          group_wait_pulled(bb, sp);
          break;
        }
    }
    if (owner == rank_) {
      // Per stage p three chains run concurrently:
      //   sh (critical): col(pivot p) -> extract(pivot p) -> recip(p) ->
      //                  R_p[p+1] (one row)          [-> stage p+1 pivot]
      //   sp (near):     col, extract, R_p for rows p+1 < r < near_end
      //   sf (far):      col, extract, R_p for rows r >= near_end
      // The pivot chain reads only near rows (row p+2 at stage p feeds the
      // stage-(p+1) divide, and so on inside the window), so the far rows run
      // behind it on their own stream and only have to be done before the
      // trailing update of the panel.  near_end = p0 + near_rows_.
      // Events (per stage): sev_[4p] extract(near p) done, sev_[4p+1]
      // recip(p) done, sev_[4p+2] near divide(p) done, sev_[4p+3] chain done.
      const int near_end = std::min(n, p0 + std::max(near_rows_, kb + 2));
      const bool far = near_end < n && recip_bound_;
      // ratio GEMM for this run's operand bounds (else k_divide)
      const bool rg_ok = ratio_gemm_ && rg_kd_ > 0 &&
                         ratio_gemm_kd(dmax_bits_) <= rg_kd_ &&
                         ratio_gemm_ncols(dmax_bits_) <= rg_ncols_;
      const bool rg_near = rg_ok && (ratio_gemm_ & 2);
      const bool rg_far = rg_ok && (ratio_gemm_ & 1);
      bool chain_started = false;
      // far lanes (one when the divisions use global scratch or the GEMM)
      const int nlanes = (div_global_ || rg_far) ? 1 : far_lanes_;
      // next-row stream (HGPU_NEXT_ROW): the chain's next row apart from the
      // bulk near rows (fused chain, shared-memory divisions, >= 3 near rows)
      const bool nr = next_row_ && fused_pivot_ && !div_global_ && !rg_near &&
                      (far ? near_end : n) - p0 >= 3 && recip_bound_;
      // far rows' in-panel update in sub-panels of fsub stages (0: plain
      // left-looking); needs the far rows below the panel's columns
      const int fsub = (far_sub_ > 0 && near_end >= p1 && D.NW % 32 == 0) ? far_sub_ : 0;
      // near rows' early stages on the pre stream (plain near path only)
      const bool pre_near_on = pre_near_ && !nr && !(col_extract_ & 1) && fused_pivot_ &&
                               recip_bound_;
      // rows of lane 0 when the other lanes lag: the next panel's near rows
      const int mid = std::min(n, p1 + near_rows_);
      lag = lag_ok && far && nlanes >= 2 && !div_global_ && !rg_far && p1 < n && near_end < mid;
      if (far) {
        CU(cudaEventRecord(sev_[4 * n + 1], sp));
        for (int l = 0; l < nlanes; ++l) {
          CU(cudaStreamWaitEvent(far_streams_[l], sev_[4 * n + 1], 0));
          // band b's far rows took panel b-1 after the chain moved on
          if (prev_lag) CU(cudaStreamWaitEvent(far_streams_[l], lag_ev_[2 * b + 1], 0));
        }
      } else if (prev_lag) {
        CU(cudaStreamWaitEvent(sp, lag_ev_[2 * b + 1], 0));
      }
      for (int p = p0; p < p1; ++p) {
        const int s = p - p0;
        const long long row0 = row0set + (long long)s * n;
        const uint32_t* vh = vhat_ + row0set * NW;
        const uint32_t* rh = rhat_ + row0set * NW;
        uint32_t* yb = ybuf_ + (size_t)(p % kYRing) * P.ycap;
        int* yss = ys_ + (p % kYRing) * 4;
        if (recip_bound_ && p < n - 1) {
          if (!chain_started) {
            // the helper stream enters the panel where the panel stream is
            CU(cudaEventRecord(sev_[4 * n], sp));
            CU(cudaStreamWaitEvent(sh, sev_[4 * n], 0));
            chain_started = true;
          } else if (nr) {
            // next-row stream: V_{p-1}[p] and R_{p-2}[p] come from sn(p-1),
            // V^_{p-2}[p] from the bulk extraction (p-2) and older ratios
            // from the bulk divisions (p-3)
            CU(cudaStreamWaitEvent(sh, sn_ev_[p - 1], 0));
            if (p - 2 >= p0) CU(cudaStreamWaitEvent(sh, sev_[4 * (p - 2)], 0));
            if (p - 3 >= p0) CU(cudaStreamWaitEvent(sh, sev_[4 * (p - 3) + 2], 0));
          } else {
            // pivot entry of column p needs V_{p-1}[p] (extract(near p-1))
            // and R_{p-2}[p] (near divide(p-2)); R_{p-1}[p] is on sh already
            CU(cudaStreamWaitEvent(sh, sev_[4 * (p - 1)], 0));
            if (p - 2 >= p0) CU(cudaStreamWaitEvent(sh, sev_[4 * (p - 2) + 2], 0));
          }
          if (fused_pivot_) {
            // R_{p-1}[p] (inside the panel), pivot-entry update, extraction
            // and reciprocal in one CTA
            PivotDiv pd{};
            pd.recip_words = std::min<long long>(
                (long long)recip_scratch_words(D), recip_words_bound(D, dmax_bits_, pivot_segs_));
            if (D.recip_fast)
              pd.recip_words = std::min<long long>(
                  (long long)recip_scratch_words(D),
                  std::max(pd.recip_words, recip_fast_words_bound(D, dmax_bits_)));
            if (p > p0) {
              pd.on = 1;
              pd.vrow0 = row0 - n;  // stage p-1 of this panel's slot set
              pd.Ybuf = ybuf_ + (size_t)((p - 1) % kYRing) * P.ycap;
              pd.ys = ys_ + ((p - 1) % kYRing) * 4;
              pd.rint = rint;
              pd.rhat = rhat_;
              pd.maxdegR = maxdegR + (p - 1);
              pd.dscr = dscratch_;
              pd.use_dscr = div_global_ ? 1 : 0;
            }
            // stages [p0, p-1) of the pivot entry W[p][p] ahead of the chain,
            // on their own stream with 32 CTAs (k_pivot's single CTA is
            // latency-bound on those reads); k_pivot applies stage p-1
            int s_first = 0;
            if (pre_entry_ && s >= 2) {
              if (nr) {
                // stages <= p-2 of W[p][p]: R_{p-2}[p] from sn(p-1), older
                // ratios from the bulk divisions (p-3), V^_{p-2}[p] from the
                // bulk extraction (p-2)
                CU(cudaStreamWaitEvent(stream_pre_, sn_ev_[p - 1], 0));
                CU(cudaStreamWaitEvent(stream_pre_, sev_[4 * (p - 2)], 0));
                if (p - 3 >= p0)
                  CU(cudaStreamWaitEvent(stream_pre_, sev_[4 * (p - 3) + 2], 0));
              } else {
                CU(cudaStreamWaitEvent(stream_pre_, sev_[4 * (p - 2) + 2], 0));
              }
              TL(16, p, stream_pre_, [&] {
                return launch_update_col(D, W_, colbase_, vh, rh, slot_stride, s - 1,
                                         p, p, p + 1, err_, stream_pre_);
              });
              CU(cudaEventRecord(pre_ev_[p], stream_pre_));
              CU(cudaStreamWaitEvent(sh, pre_ev_[p], 0));
              s_first = s - 1;
            }
            TL(2, p, sh, [&] {
              return launch_pivot(D, W_, colbase_, vh + s_first * slot_stride,
                                  rh + s_first * slot_stride, slot_stride, s - s_first, p,
                                  vint, row0, piv, maxbitsV, vhat_, maxdegV,
                                  dmax_bits_, yb, yss, rscratch_,
                                  recip_global_ ? 1 : 0, err_, sh, pd);
            });
          } else {
            TL(0, p, sh, [&] {
              return launch_update_col(D, W_, colbase_, vh, rh, slot_stride, s,
                                       p, p, p + 1, err_, sh);
            });
            TL(1, p, sh, [&] {
              return launch_extract(D, W_, colbase_, p, p, p + 1, vint, row0,
                                    piv, maxbitsV, vhat_, maxdegV, err_, sh);
            });
            TL(2, p, sh, [&] {
              return launch_recip(D, vint, row0 + p, maxbitsV, p, piv,
                                  dmax_bits_, yb, yss, rscratch_,
                                  recip_global_ ? 1 : 0, err_, sh);
            });
          }
          CU(cudaEventRecord(sev_[4 * p + 1], sh));
          const int rn = far ? near_end : n;
          if (nr) {
            // sn(p): row p+1 of column p, which the chain needs next --
            // (i) R_{p-1}[p+1], (ii) its entry update with stages [p0, p),
            // (iii) its extraction -- off the bulk near rows' stream
            cudaStream_t sn = stream_next_;
            if (s == 0) {
              CU(cudaEventRecord(sev_[4 * n + 3], sp));  // panel entry
              CU(cudaStreamWaitEvent(sn, sev_[4 * n + 3], 0));
            }
            if (s >= 1) {
              CU(cudaStreamWaitEvent(sn, sev_[4 * (p - 1) + 1], 0));  // Y_{p-1}
              CU(cudaStreamWaitEvent(sn, sev_[4 * (p - 1)], 0));      // V_{p-1}[p+1]
              if (s >= 2) CU(cudaStreamWaitEvent(sn, sev_[4 * (p - 2) + 2], 0));
              TL(17, p, sn, [&] {
                return launch_divide(D, vint, row0 - n, p - 1, p + 1, p + 2,
                                     ybuf_ + (size_t)((p - 1) % kYRing) * P.ycap,
                                     ys_ + ((p - 1) % kYRing) * 4, rint, row0 - n, rhat_,
                                     maxdegR + (p - 1), dscratch_, 0, err_, sn);
              });
              TL(17, p, sn, [&] {
                return launch_update_col(D, W_, colbase_, vh, rh, slot_stride, s,
                                         p, p + 1, p + 2, err_, sn);
              });
            }
            TL(17, p, sn, [&] {
              return launch_extract(D, W_, colbase_, p, p + 1, p + 2, vint, row0,
                                    piv, maxbitsV, vhat_, maxdegV, err_, sn, 0,
                                    rg_near ? vdig_ : nullptr, rg_kd_);
            });
            CU(cudaEventRecord(sn_ev_[p], sn));
            // bulk near rows [p+2, rn): V^_{p-1}[p] comes from sn(p-1)
            if (s >= 1) CU(cudaStreamWaitEvent(sp, sn_ev_[p - 1], 0));
          }
          // near rows of column p on the panel stream (rows > p)
          const int rb = nr ? p + 2 : p + 1;
          if (col_extract_ & 1) {
            TL(4, p, sp, [&] {
              return launch_col_extract(D, W_, colbase_, vh, rh, slot_stride, s, p, rb, rn,
                                        vint, row0, piv, maxbitsV, vhat_, maxdegV, err_, sp,
                                        rg_near ? vdig_ : nullptr, rg_kd_);
            });
          } else {
            // stages [p0, p-2] arrived ahead of time on the pre stream (below,
            // enqueued at stage p-2): only stage p-1 is left
            int s0 = 0;
            if (pre_near_on && s >= 2 && rb < rn) {
              CU(cudaStreamWaitEvent(sp, pre2_ev_[p], 0));
              s0 = s - 1;
            }
            TL(3, p, sp, [&] {
              return launch_update_col(D, W_, colbase_, vh + s0 * slot_stride,
                                       rh + s0 * slot_stride, slot_stride, s - s0,
                                       p, rb, rn, err_, sp);
            });
            TL(4, p, sp, [&] {
              return launch_extract(D, W_, colbase_, p, rb, rn, vint, row0,
                                    piv, maxbitsV, vhat_, maxdegV, err_, sp, 0,
                                    rg_near ? vdig_ : nullptr, rg_kd_);
            });
          }
          CU(cudaEventRecord(sev_[4 * p], sp));
          // R_p[p+1] on the chain (it only needs V_p[p+1] besides the pivot):
          // inside the next stage's k_pivot, except at the panel's last stage
          // (the trailing update reads it)
          CU(cudaStreamWaitEvent(sh, nr ? sn_ev_[p] : sev_[4 * p], 0));
          if (!fused_pivot_ || p + 1 == p1 || p + 1 == n - 1) {
            TL(5, p, sh, [&] {
              return launch_divide(D, vint, row0, p, p + 1, p + 2, yb, yss,
                                   rint, row0, rhat_, maxdegR + p, dscratch_,
                                   div_global_ ? 1 : 0, err_, sh);
            });
          }
          CU(cudaEventRecord(sev_[4 * p + 3], sh));
          // R_p[p+1 < r < rn] on the panel stream
          CU(cudaStreamWaitEvent(sp, sev_[4 * p + 1], 0));
          if (rg_near) {
            TL(5, p, sp, [&] {
              ratio_gemm(0, p, p + 2, rn, vint, row0, yb, yss, rint, maxdegR + p,
                         dscratch2_, sp);
              return cudaSuccess;
            });
          } else {
            // with sn, row p+2 of stage p is sn(p+1)'s first task (inside
            // the panel)
            const int db0 = (nr && p + 1 < p1 && p + 1 < n - 1) ? p + 3 : p + 2;
            TL(5, p, sp, [&] {
              return launch_divide(D, vint, row0, p, db0, rn, yb, yss, rint,
                                   row0, rhat_, maxdegR + p, dscratch2_,
                                   div_global_ ? 1 : 0, err_, sp);
            });
          }
          CU(cudaEventRecord(sev_[4 * p + 2], sp));
          if (pre_near_on && p + 2 < p1 && p + 3 < rn) {
            // column c = p + 2: every stage up to p is now complete for the
            // near rows (R^_p from the division just enqueued, V^_p[c] from
            // the extraction before it); it takes them on the pre stream
            // while the panel stream works on column p + 1
            const int c = p + 2;
            CU(cudaStreamWaitEvent(stream_pre2_, sev_[4 * p + 2], 0));
            TL(18, c, stream_pre2_, [&] {
              return launch_update_col(D, W_, colbase_, vh, rh, slot_stride, s + 1, c, c + 1,
                                       rn, err_, stream_pre2_);
            });
            CU(cudaEventRecord(pre2_ev_[c], stream_pre2_));
          }
          if (far) {
            // far rows: column p receives stages [p0, p) (V^_s[p] of the
            // near rows, extract(near p-1) done; their own R^_s on the lane's
            // stream), then extraction and, once recip(p) is done, the
            // ratios.  The far rows are split into lanes on separate streams
            // so that one lane's division overlaps another's extraction.
            for (int l = 0; l < nlanes; ++l) {
              cudaStream_t fs = far_streams_[l];
              int lo = near_end + (int)((long long)(n - near_end) * l / nlanes);
              int hi = near_end + (int)((long long)(n - near_end) * (l + 1) / nlanes);
              if (lag) {
                // lane 0: [near_end, mid); lanes 1..: [mid, n) in equal parts
                lo = l == 0 ? near_end : mid + (int)((long long)(n - mid) * (l - 1) / (nlanes - 1));
                hi = l == 0 ? mid : mid + (int)((long long)(n - mid) * l / (nlanes - 1));
              }
              if (lo >= hi) continue;
              if (p > p0) CU(cudaStreamWaitEvent(fs, sev_[4 * (p - 1)], 0));
              if (nr && p > p0) CU(cudaStreamWaitEvent(fs, sn_ev_[p - 1], 0));
              // column p receives the stages of its own sub-panel [ps, p);
              // earlier sub-panels arrived by the rank-fsub updates below
              const int ps = fsub > 0 ? p0 + (s / fsub) * fsub : p0;
              if (col_extract_ & 2) {
                TL(11, p, fs, [&] {
                  return launch_col_extract(D, W_, colbase_, vh + (ps - p0) * slot_stride,
                                            rh + (ps - p0) * slot_stride, slot_stride, p - ps,
                                            p, lo, hi, vint, row0, piv, maxbitsV, vhat_,
                                            maxdegV, err_, fs, rg_far ? vdig_ : nullptr,
                                            rg_kd_);
                });
              } else {
                TL(10, p, fs, [&] {
                  return launch_update_col(D, W_, colbase_, vh + (ps - p0) * slot_stride,
                                           rh + (ps - p0) * slot_stride, slot_stride,
                                           p - ps, p, lo, hi, err_, fs);
                });
                TL(11, p, fs, [&] {
                  return launch_extract(D, W_, colbase_, p, lo, hi, vint, row0,
                                        piv, maxbitsV, vhat_, maxdegV, err_, fs, 0,
                                        rg_far ? vdig_ : nullptr, rg_kd_);
                });
              }
              CU(cudaStreamWaitEvent(fs, sev_[4 * p + 1], 0));
              if (rg_far) {
                TL(12, p, fs, [&] {
                  ratio_gemm(1, p, lo, hi, vint, row0, yb, yss, rint,
                             maxdegR + p, dscratch3_, fs);
                  return cudaSuccess;
                });
              } else {
                TL(12, p, fs, [&] {
                  return launch_divide(D, vint, row0, p, lo, hi, yb, yss, rint,
                                       row0, rhat_, maxdegR + p, dscratch3_,
                                       div_global_ ? 1 : 0, err_, fs);
                });
              }
              if (fsub > 0 && (s + 1) % fsub == 0 && p + 1 < p1) {
                // the finished sub-panel [p+1-fsub, p] on the panel's
                // remaining columns of these rows, one tiled pass (R^ read
                // once per tile instead of once per column); needs V^_p of
                // those columns (near extract of stage p)
                CU(cudaStreamWaitEvent(fs, sev_[4 * p], 0));
                if (nr) CU(cudaStreamWaitEvent(fs, sn_ev_[p], 0));
                const int sb0 = p + 1 - fsub - p0;
                TL(14, p, fs, [&] {
                  return launch_update_rect(D, W_, colbase_, vh + sb0 * slot_stride,
                                            rh + sb0 * slot_stride, slot_stride, fsub,
                                            p + 1, p1, lo, hi, err_, fs);
                });
              }
            }
          }
          if (lookahead_ && edf && far && !nr && fsub > 0 && (s + 1) % fsub == 0 &&
              p + 1 < p1 && p1 < n) {
            // sub-panel lookahead: stages [p+1-fsub, p] of this panel onto band
            // b+1 now, on su1 (idle during the panel), so the panel boundary
            // only waits for the last sub-panel's share of U(b, b+1).  Band
            // b+1's rows are near rows (near divide of stage p) or far rows
            // (each lane's launches up to stage p); su2 last touched the band
            // at the end of panel b-1 (band_ev)
            // (lookahead_ 2: on su2 at the lowest priority, after the band's
            // pending deadline-ordered work, instead of su1)
            cudaStream_t lu = lookahead_ == 2 ? su2 : su1;
            CU(cudaStreamWaitEvent(lu, sev_[4 * p + 2], 0));
            for (int l = 0; l < nlanes; ++l) {
              CU(cudaEventRecord(far_ev_[l], far_streams_[l]));
              CU(cudaStreamWaitEvent(lu, far_ev_[l], 0));
            }
            if (lu == su1 && la_done == 0 && band_ev[b + 1])
              CU(cudaStreamWaitEvent(su1, band_ev[b + 1], 0));
            trailing(b, p1, std::min(n, p1 + kb), lu, 15, la_done, fsub);
            la_done += fsub;
            if (lu == su2) {
              cudaEvent_t e = edf_event();
              CU(cudaEventRecord(e, su2));
              band_ev[b + 1] = e;  // su1's share at the panel end waits for it
            }
          }
          if (p + 1 == p1 || p + 1 == n - 1) {
            // join: the next step on sp needs R_p[p+1] as well
            CU(cudaStreamWaitEvent(sp, sev_[4 * p + 3], 0));
            if (nr) CU(cudaStreamWaitEvent(sp, sn_ev_[p], 0));
            if (far)
              for (int l = 0; l < nlanes; ++l) {
                CU(cudaEventRecord(far_ev_[l], far_streams_[l]));
                // (lagging lanes join on the join stream after the panel)
                if (!lag || l == 0) CU(cudaStreamWaitEvent(sp, far_ev_[l], 0));
              }
          }
        } else {
          // left-looking inside the panel: column p receives stages [p0, p)
          TL(6, p, sp, [&] {
            return launch_update_col(D, W_, colbase_, vh, rh, slot_stride, s,
                                     p, p, n, err_, sp);
          });
          // W[r][p] -> V_p[r] (+ its transform for rows r > p)
          TL(7, p, sp, [&] {
            return launch_extract(D, W_, colbase_, p, p, n, vint, row0, piv,
                                  maxbitsV, vhat_, maxdegV, err_, sp);
          });
          if (p == n - 1) break;
          TL(2, p, sp, [&] {
            return launch_recip(D, vint, row0 + p, maxbitsV, p, piv, 0, yb,
                                yss, rscratch_, recip_global_ ? 1 : 0, err_,
                                sp);
          });
          // R_p[r] (+ its Montgomery-form transform)
          TL(5, p, sp, [&] {
            return launch_divide(D, vint, row0, p, p + 1, n, yb, yss, rint,
                                 row0, rhat_, maxdegR + p, dscratch_,
                                 div_global_ ? 1 : 0, err_, sp);
          });
        }
      }
    }
    // the panel's integers on every rank: NCCL broadcast into the local slot
    // set, or (in-process group) read from the owner's slot set in place
    IntBuf src_v = vint, src_r = rint;
    long long src_row0 = row0set;
    if (world_ > 1 && owner != rank_) {
      CU(cudaEventRecord(net_ev_[2 * b], sp));
      net_panels.push_back(b);
    }
    if (group_) {
      if (owner == rank_) {
        group_publish(b, sp);
      } else {
        const Matrix* o = group_await(b, owner, sp);
        src_v = IntBuf{o->vhdr_, o->vlimbs_};
        src_r = IntBuf{o->rhdr_, o->rlimbs_};
        src_row0 = o->slot_row0(b);
        // the panel's pivots (fold) and stage statistics (k_validate)
        CU(cudaMemcpyAsync(phdr_ + p0, o->phdr_ + p0, ns * sizeof(int), cudaMemcpyDefault, sp));
        CU(cudaMemcpyAsync(plimbs_ + (size_t)p0 * P.cap, o->plimbs_ + (size_t)p0 * P.cap,
                           (size_t)ns * P.cap * 4, cudaMemcpyDefault, sp));
        for (int k = 0; k < 3; ++k)
          CU(cudaMemcpyAsync(stats_ + (size_t)k * n + p0, o->stats_ + (size_t)k * n + p0,
                             ns * sizeof(int), cudaMemcpyDefault, sp));
      }
    } else {
      panel_broadcast(owner, p0, ns, row0set, sp);
    }
    if (owner != rank_ && p1 < n) {
      // transforms of the rows this rank's columns need (rows >= p1); in a
      // group these launches are the transfer: they load the owner's limbs
      for (int s = 0; s < ns; ++s) {
        const long long row0 = row0set + (long long)s * n;
        const long long srow = src_row0 + (long long)s * n;
        CU(launch_fwd_ints(D, src_v, srow + p1, vhat_, row0 + p1, n - p1, 0,
                           nullptr, err_, sp));
        CU(launch_fwd_ints(D, src_r, srow + p1, rhat_, row0 + p1, n - p1, 1,
                           nullptr, err_, sp));
      }
    }
    if (world_ > 1 && owner != rank_) CU(cudaEventRecord(net_ev_[2 * b + 1], sp));
    if (lag) {
      // early: chain, near rows and lane 0; done: every lane (join stream)
      CU(cudaEventRecord(lag_ev_[2 * b], sp));
      CU(cudaStreamWaitEvent(stream_join_, lag_ev_[2 * b], 0));
      for (int l = 1; l < kMaxFarLanes; ++l)
        CU(cudaStreamWaitEvent(stream_join_, far_ev_[l], 0));
      CU(cudaEventRecord(panel_done[b], stream_join_));
    } else {
      CU(cudaEventRecord(panel_done[b], sp));
    }
    if (flags & HGPU_KEEP_L) {
      // the panel's ratio columns into the packed L store: off the panel
      // stream (2 ns copies per panel) when there is a join stream and the
      // slot set is not reused before the end (every panel has its own)
      cudaStream_t ks = (stream_join_ && nsets > nblocks && !group_) ? stream_join_ : sp;
      if ((ks != sp) != lag) CU(cudaStreamWaitEvent(ks, panel_done[b], 0));
      keep_panel_L(p0, ns, src_row0, ks, src_r);
      if (pre_lhat_on) {
        // this panel's entries of the packed L store (contiguous: stages
        // p0 .. p1-1), transformed in the solve plan while the factorisation
        // goes on
        const long long e0 = (long long)p0 * (n - 1) - (long long)p0 * (p0 - 1) / 2;
        const int pe = std::min(p1, n - 1);
        const long long e1 = (long long)pe * (n - 1) - (long long)pe * (pe - 1) / 2;
        CU(cudaEventRecord(lhat_ev_, ks));
        CU(cudaStreamWaitEvent(stream_lhat_, lhat_ev_, 0));
        CU(launch_solve_rhat(sdp_, P.cap, IntBuf{lhdr_, llimbs_}, e1 - e0, lhat_store(),
                             dp_.grid_cap, lhat_err_, stream_lhat_, e0));
        kernel_launch_count_add(1);
      }
    }
    if (capture) {
      const int nsr = std::min(ns, crow - 1 - p0);
      if (nsr > 0) {
        hr_hdr.resize((size_t)nsr * n);
        hr_limbs.resize((size_t)nsr * n * P.cap);
        CU(cudaMemcpyAsync(hr_hdr.data(), src_r.hdr + src_row0, hr_hdr.size() * 4,
                           cudaMemcpyDefault, sp));
        CU(cudaMemcpyAsync(hr_limbs.data(), src_r.limbs + src_row0 * P.cap,
                           hr_limbs.size() * 4, cudaMemcpyDefault, sp));
        CU(cudaStreamSynchronize(sp));
        for (int s = 0; s < nsr; ++s) {
          const int p = p0 + s;
          auto& colv = res.ratios[p];
          colv.resize(crow - p - 1);
          for (int r = p + 1; r < crow; ++r) {
            const size_t idx = (size_t)s * n + r;
            HostInt& h = colv[r - p - 1];
            h.size = hr_hdr[idx];
            const int len = std::abs(h.size);
            h.limbs.assign(hr_limbs.begin() + idx * P.cap,
                           hr_limbs.begin() + idx * P.cap + len);
          }
        }
      }
    }
    if (group_ && owner != rank_) group_pulled(b, sp);
    // ---- trailing update of panel b on the bulk stream: the next panel's
    // columns first (they gate panel b+1), then everything to their right,
    // which overlaps panel b+1's factorisation
    if (!lag) CU(cudaStreamWaitEvent(su1, panel_done[b], 0));
    CU(cudaStreamWaitEvent(su2, panel_done[b], 0));
    if (edf) {
      if (lag) {
        // band b+1: the next panel's near rows now (they gate panel b+1), the
        // rows below once the lagging lanes are done (they gate panel b+1's
        // far lanes, lag_ev_[2(b+1)+1])
        const int p2 = std::min(n, p1 + kb), mid = std::min(n, p1 + near_rows_);
        const int nsl = std::min(kb, n - 1 - p0);
        CU(cudaStreamWaitEvent(su1, lag_ev_[2 * b], 0));
        if (band_ev[b + 1]) CU(cudaStreamWaitEvent(su1, band_ev[b + 1], 0));
        timed_update(b, nsl, p1, p2, su1, 8, 0, -1, mid);
        CU(cudaEventRecord(next_ready[b + 1], su1));
        CU(cudaStreamWaitEvent(su1, panel_done[b], 0));
        timed_update(b, nsl, p1, p2, su1, 8, 0, mid, n);
        CU(cudaEventRecord(lag_ev_[2 * (b + 1) + 1], su1));
      } else {
      if (p1 < n) {
        const int p2 = std::min(n, p1 + kb);
        if (band_ev[b + 1]) CU(cudaStreamWaitEvent(su1, band_ev[b + 1], 0));
        trailing(b, p1, p2, su1, 8, la_done);  // what the lookahead left
      }
      CU(cudaEventRecord(next_ready[b + 1], su1));
      }
      edf_next[b] = b + 2;
      const int jmax = std::min(nblocks - 1, b + edf_h_ + 1);
      for (int j = b + 2; j <= jmax; ++j) edf_band(j, b);
    } else if (p1 < n) {
      const int p2 = std::min(n, p1 + kb);
      trailing(b, p1, p2, su1, 8);
      CU(cudaEventRecord(next_ready[b + 1], su1));
      const int pr = std::min(n, (b + 1 + sdef) * kb);
      if (!(D.debug & 512)) trailing(b, pr, n, su2, 9);  // 512: timing experiment only
    } else {
      CU(cudaEventRecord(next_ready[b + 1], su1));
    }
    if (!edf) CU(cudaEventRecord(rest_done[b], su2));
    prev_lag = lag;
  }
  // join the panel and update streams back into the bulk stream
  CU(cudaEventRecord(panel_done[nblocks], sp));
  CU(cudaStreamWaitEvent(st, panel_done[nblocks], 0));
  if (stream_join_) {
    CU(cudaEventRecord(lag_ev_[2 * nblocks + 2], stream_join_));
    CU(cudaStreamWaitEvent(st, lag_ev_[2 * nblocks + 2], 0));
  }
  CU(cudaEventRecord(trail_done[0], su1));
  CU(cudaStreamWaitEvent(st, trail_done[0], 0));
  CU(cudaEventRecord(trail_done[1], su2));
  CU(cudaStreamWaitEvent(st, trail_done[1], 0));
  CU(launch_validate(D, maxdegV, maxdegR, n - 1, err_, st));
  CU(cudaEventRecord(ev1_, st));
  res.launches = kernel_launch_count() - launches0;

  if (comm_ && world_ > 1) {
    // every rank raised its own flags (its transforms, its updates): the
    // factorisation's status is the first zero pivot and the union of flags
    ncclComm_t c = (ncclComm_t)comm_;
    NC(ncclGroupStart());
    NC(ncclAllReduce(err_, err_, 1, ncclInt32, ncclMin, c, st));
    NC(ncclAllReduce(err_ + 1, err_ + 1, kErrWords - 1, ncclInt32, ncclMax, c, st));
    NC(ncclGroupEnd());
  }
  int herr[kErrWords];
  // (the copy into pageable memory below returns when it is done, i.e. at
  // the end of the device work: the enqueue time is taken before it)
  const auto t_enq = std::chrono::steady_clock::now();
  CU(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, st));
  int lherr[kErrWords] = {INT_MAX, 0, 0, 0};
  if (pre_lhat_on) {
    // (after ev1_: the tail of the L-entry transforms is not factorisation time)
    CU(cudaEventRecord(lhat_ev_, stream_lhat_));
    CU(cudaStreamWaitEvent(st, lhat_ev_, 0));
    CU(cudaMemcpyAsync(lherr, lhat_err_, sizeof(lherr), cudaMemcpyDeviceToHost, st));
  }
  CU(cudaStreamSynchronize(st));
  if (pre_lhat_on && have_L_ && !lherr[kErrCapacity] && !lherr[kErrInternal])
    lhat_pre_for_ = factor_serial_;
  if (group_) group_merge_err(herr);
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, ev0_, ev1_));
  res.device_ms = ms;
  if (std::getenv("HGPU_HOST_TRACE"))
    std::fprintf(stderr, "factor: host enqueue %.3f ms, device %.3f ms, wall %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t_enq - t_run0).count(), ms,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                           t_run0).count());
  if (tl_path) {
    if (FILE* f = std::fopen(tl_path, "a")) {
      std::fprintf(f, "# factorisation n=%d K=%d device_ms=%.3f\n", n, K_, ms);
      for (const TlRec& t : tl_) {
        float a = 0, b2 = 0;
        CU(cudaEventElapsedTime(&a, ev0_, t.a));
        CU(cudaEventElapsedTime(&b2, ev0_, t.b));
        std::fprintf(f, "%d,%d,%.4f,%.4f\n", t.kind, t.p, a, b2);
      }
      std::fclose(f);
    }
  }
  for (int b : net_panels) {
    float t = 0;
    CU(cudaEventElapsedTime(&t, net_ev_[2 * b], net_ev_[2 * b + 1]));
    res.net_ms += t;
  }
  if (profile) {
    for (size_t i = 0; i < uev_used; i += 2) {
      float t = 0;
      CU(cudaEventElapsedTime(&t, uev_[i], uev_[i + 1]));
      res.update_ms += t;
    }
  }
  if (herr[kErrCapacity]) {
    Error e(HGPU_ERR_CAPACITY,
            "transform capacity exceeded (flags " +
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
  // pivots to host
  std::vector<int> ph(n);
  std::vector<uint32_t> pl((size_t)n * P.cap);
  CU(cudaMemcpy(ph.data(), phdr_, n * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(pl.data(), plimbs_, pl.size() * 4, cudaMemcpyDeviceToHost));
  res.pivots.resize(n);
  for (int p = 0; p < n; ++p) {
    res.pivots[p].size = ph[p];
    const int len = std::abs(ph[p]);
    res.pivots[p].limbs.assign(pl.begin() + (size_t)p * P.cap,
                               pl.begin() + (size_t)p * P.cap + len);
  }
  if (flags & HGPU_FOLD) fold(res);
}

// R_p[r] for the panel's stages (rows r > p) into the packed L store.
void Matrix::keep_panel_L(int p0, int ns, long long row0set, cudaStream_t st,
                          IntBuf srcb) {
  const Plan& P = plan_;
  const int n = n_;
  for (int s = 0; s < ns; ++s) {
    const int p = p0 + s;
    if (p >= n - 1) break;
    const long long src = row0set + (long long)s * n + p + 1;
    const long long dst = (long long)p * (n - 1) - (long long)p * (p - 1) / 2;
    const size_t rows = (size_t)(n - p - 1);
    CU(cudaMemcpyAsync(lhdr_ + dst, srcb.hdr + src, rows * 4, cudaMemcpyDefault, st));
    CU(cudaMemcpyAsync(llimbs_ + dst * P.cap, srcb.limbs + src * P.cap,
                       rows * P.cap * 4, cudaMemcpyDefault, st));
  }
  have_L_ = true;
  ++factor_serial_;
}

std::vector<HostInt> Matrix::solve(const std::vector<HostInt>& u,
                                   long long* launches) {
  set_start(u);
  return solve_resident(launches, true);
}

// Solves with the right-hand side already in the solve buffer's u rows
// (set_start, or rescale_start after an earlier solve); y stays on the
// device (rows 3n..4n) and is copied back only on request.
std::vector<HostInt> Matrix::solve_resident(long long* launches, bool download) {
  if (!start_resident_ && !saved_start_.empty()) {
    // a re-plan released the solve buffers: the start vector comes back
    const std::vector<HostInt> u = std::move(saved_start_);
    saved_start_.clear();
    set_start(u);
  }
  if (!start_resident_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "solve_resident needs a start vector (set_start)");
  // tensor-core AXPY (HGPU_SOLVE_TC=1) once an earlier solve has recorded
  // the operand widths; any capacity flag reruns the solve on the integer path
  // (the u rows are never written by a solve, so a rerun reads the same u)
  if (solve_ntt_) {
    try {
      return solve_impl(launches, 2, download);
    } catch (const Error& e) {
      if (e.status != HGPU_ERR_CAPACITY || solve_ntt_ == 2) throw;
      sdp_bits_ = 0;  // re-plan from the widths the integer path records
      lhat_for_ = -1;
    }
  }
  if (solve_tc_ && solve_xlimbs_ > 0) {
    try {
      return solve_impl(launches, 1, download);
    } catch (const Error& e) {
      if (e.status != HGPU_ERR_CAPACITY) throw;
      solve_xlimbs_ = 0;
    }
  }
  return solve_impl(launches, 0, download);
}

void Matrix::ensure_solve_buffers() {
  if (svhdr_) return;
  const Plan& P = plan_or_build();
  const int n = n_;
  CU(cudaSetDevice(device_));
  sWv_ = 2 * P.cap + 8;
  sWa_ = P.cap + sWv_ + 2;
  svhdr_ = dalloc<int>(4 * (size_t)n);
  svlimbs_ = dalloc<uint32_t>(4 * (size_t)n * sWv_);
  sacc_ = dalloc<uint32_t>((size_t)n * sWa_);
  spair_hdr_ = dalloc<int>(2 * (size_t)n);
  spair_limbs_ = dalloc<uint32_t>(2 * (size_t)n * sWv_);
  bool axpy_global = false;
  CU(configure_solve_kernels(P.cap, sWv_, sWa_, &axpy_global));
  if (axpy_global)
    sgscr_ = dalloc<uint32_t>((size_t)dp_.grid_cap *
                              solve_axpy_smem_words(sWv_, P.cap, sWv_, sWa_));
}

// The right-hand side u (n signed limb vectors) into the solve buffer.
void Matrix::set_start(const std::vector<HostInt>& u) {
  if (world_ != 1 && !(group_ && rank_ == 0))
    throw Error(HGPU_ERR_INVALID_ARGUMENT,
                "solve runs on a single rank (or rank 0 of an in-process group)");
  if ((int)u.size() != n_) throw Error(HGPU_ERR_INVALID_ARGUMENT, "start vector length");
  ensure_solve_buffers();
  const int n = n_, Wv = sWv_;
  cudaStream_t st = stream_;
  CU(cudaSetDevice(device_));
  std::vector<int> hdr((size_t)n, 0);
  std::vector<uint32_t> lim((size_t)n * Wv, 0);
  for (int i = 0; i < n; ++i) {
    if ((int)u[i].limbs.size() > Wv)
      throw Error(HGPU_ERR_CAPACITY, "start vector entry too large");
    hdr[i] = u[i].size;
    std::copy(u[i].limbs.begin(), u[i].limbs.end(), lim.begin() + (size_t)i * Wv);
  }
  CU(cudaMemcpyAsync(svhdr_, hdr.data(), hdr.size() * 4, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(svlimbs_, lim.data(), lim.size() * 4, cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));
  start_resident_ = true;
  have_y_ = false;
  saved_start_.clear();
}

namespace {
// M + 2 two's-complement limbs -> sign and magnitude
HostInt from_twos(const uint32_t* w, int words) {
  HostInt h;
  const bool neg = (w[words - 1] & 0x80000000u) != 0;
  h.limbs.assign(w, w + words);
  if (neg) {
    uint64_t c = 1;
    for (uint32_t& x : h.limbs) {
      c += (uint64_t)(uint32_t)~x;
      x = (uint32_t)c;
      c >>= 32;
    }
  }
  while (!h.limbs.empty() && h.limbs.back() == 0) h.limbs.pop_back();
  h.size = neg ? -(int)h.limbs.size() : (int)h.limbs.size();
  return h;
}
}  // namespace

// num = y.u and den = y.y of the last solve, exact, on the device
// (rq_kernels.cu); ybits = max_i bits(|y_i|), which fixes the next scaling.
void Matrix::rayleigh(HostInt& num, HostInt& den, long& ybits, long long* launches) {
  if (!have_y_) throw Error(HGPU_ERR_INVALID_ARGUMENT, "rayleigh needs a solve");
  const int n = n_, Wv = sWv_;
  cudaStream_t st = stream_;
  CU(cudaSetDevice(device_));
  const int maxlen = std::max(1, std::max(last_ulimbs_, last_ylimbs_));
  const int M = 2 * maxlen;
  if (maxlen > rq_maxlen_) {
    dfree(rq_prod_);
    dfree(rq_colsum_);
    dfree(rq_out_);
    dfree(rq_scr_);
    rq_scr_ = nullptr;
    const int cap = maxlen + maxlen / 8 + 8;  // room for the iterates to grow
    if (!rq_sign_) rq_sign_ = dalloc<int>(2 * (size_t)n);
    rq_prod_ = dalloc<uint32_t>(2 * (size_t)n * 2 * cap);
    rq_colsum_ = dalloc<long long>(2 * (size_t)2 * cap);
    rq_out_ = dalloc<uint32_t>(2 * ((size_t)2 * cap + 2));
    bool global = false;
    CU(configure_rq_kernels(cap, &global));
    rq_grid_ = n;
    if (global) {
      rq_grid_ = std::min(n, 2 * 148);
      rq_scr_ = dalloc<uint32_t>((size_t)rq_grid_ * rq_products_words(cap));
    }
    rq_maxlen_ = cap;
  }
  // the shared-memory layout follows the operands actually met (maxlen), the
  // global scratch the allocation (rq_maxlen_)
  const int lay = rq_scr_ ? rq_maxlen_ : maxlen;
  const int Ml = 2 * lay;
  (void)M;
  IntBuf vecs{svhdr_, svlimbs_};
  int herr0[kErrWords] = {INT_MAX, 0, 0, 0};
  CU(cudaMemcpyAsync(err_, herr0, sizeof(herr0), cudaMemcpyHostToDevice, st));
  CU(launch_rq_products(vecs, 3 * n, 0, n, Wv, lay, rq_prod_, rq_sign_, rq_scr_, rq_grid_,
                        err_, st));
  CU(launch_rq_reduce(rq_prod_, rq_sign_, n, Ml, rq_colsum_, rq_out_, st));
  CU(launch_int_bits_batch(vecs, 3 * n, 1, Wv, n, sbits_, st));
  if (launches) *launches += 4;
  std::vector<uint32_t> out(2 * ((size_t)Ml + 2));
  std::vector<int> bits((size_t)n);
  int herr[kErrWords];
  CU(cudaMemcpyAsync(out.data(), rq_out_, out.size() * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(bits.data(), sbits_, bits.size() * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (herr[kErrCapacity])
    throw Error(HGPU_ERR_INTERNAL, "Rayleigh-quotient layout smaller than its operands");
  num = from_twos(out.data(), Ml + 2);
  den = from_twos(out.data() + Ml + 2, Ml + 2);
  ybits = 0;
  for (int i = 0; i < n; ++i) ybits = std::max<long>(ybits, bits[i]);
}

// u <- y 2^-sh (tdiv_2exp for sh > 0): the next start vector, on the device.
void Matrix::rescale_start(long sh, long long* launches) {
  if (!have_y_) throw Error(HGPU_ERR_INVALID_ARGUMENT, "rescale_start needs a solve");
  const int n = n_, Wv = sWv_;
  cudaStream_t st = stream_;
  CU(cudaSetDevice(device_));
  IntBuf vecs{svhdr_, svlimbs_};
  int herr0[kErrWords] = {INT_MAX, 0, 0, 0};
  CU(cudaMemcpyAsync(err_, herr0, sizeof(herr0), cudaMemcpyHostToDevice, st));
  CU(launch_rq_rescale(vecs, 3 * n, 0, n, Wv, (int)sh, err_, st));
  if (launches) *launches += 1;
  int herr[kErrWords];
  CU(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (herr[kErrCapacity]) throw Error(HGPU_ERR_CAPACITY, "rescaled start vector too large");
  have_y_ = false;
}

std::vector<HostInt> Matrix::solve_impl(long long* launches, int mode, bool download) {
  const bool tc = mode == 1, ntt = mode == 2;
  const auto t_start = std::chrono::steady_clock::now();
  if (!have_L_)
    throw Error(HGPU_ERR_INVALID_ARGUMENT, "solve needs a HGPU_KEEP_L factorisation");
  if (world_ != 1 && !(group_ && rank_ == 0))
    throw Error(HGPU_ERR_INVALID_ARGUMENT,
                "solve runs on a single rank (or rank 0 of an in-process group)");
  const Plan& P = plan_;
  const int n = n_, k2 = K_ / 2;
  cudaStream_t st = stream_;
  CU(cudaSetDevice(device_));
  ensure_solve_buffers();
  // division plan: the LDL^T plan with integer capacity Wv (k_recip/k_divide
  // over pairs (piv_p, z_p 2^k2), scratch in global memory, no transform),
  // batched over all n pairs on gridDim.y
  DevPlan D2 = dp_;
  D2.n = 2;
  D2.cap = sWv_;
  D2.ycap = sWv_ + k2 / 32 + 8;
  D2.tw_smem = 0;
  D2.grid_cap = 1;
  D2.bat_vrow = 2;
  D2.bat_rrow = 1;
  D2.bat_ys = 4;
  D2.bat_mb = 1;
  D2.bat_ybuf = D2.ycap;
  D2.bat_scr = (long long)recip_scratch_words(D2);
  if (!sybuf_) {
    sybuf_ = dalloc<uint32_t>((size_t)n * D2.ycap);
    sys_ = dalloc<int>(4 * (size_t)n);
    sbits_ = dalloc<int>((size_t)n);
    srscr_ = dalloc<uint32_t>((size_t)n * D2.bat_scr);
    sdscr_ = dalloc<uint32_t>((size_t)n * (divide_smem_words(D2) + 64));
  }
  const int Wv = sWv_, Wa = sWa_;
  // tensor-core AXPY operands (digits of the L entries once per factorisation)
  int kr = 0, mc = 0;
  if (tc) {
    const long long ne = (long long)n * (n - 1) / 2;
    if (rdig_for_ != factor_serial_) {
      std::vector<int> bits(std::max<long long>(ne, 1));
      int* dbits = dalloc<int>(std::max<long long>(ne, 1));
      CU(launch_int_bits_batch(IntBuf{lhdr_, llimbs_}, 0, 1, P.cap, (int)ne, dbits, st));
      CU(cudaMemcpyAsync(bits.data(), dbits, ne * 4, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      dfree(dbits);
      int mb = 1;
      for (long long i = 0; i < ne; ++i) mb = std::max(mb, bits[i]);
      const int need_kr = ((mb + 6) / 7 + 15) & ~15;
      if (need_kr > tc_kr_ || !rdig_col_) {
        dfree(rdig_col_);
        dfree(rdig_row_);
        rdig_col_ = dalloc<uint8_t>((size_t)ne * need_kr);
        rdig_row_ = dalloc<uint8_t>((size_t)ne * need_kr);
        tc_kr_ = need_kr;
      }
      CU(launch_solve_rdig(n, P.cap, IntBuf{lhdr_, llimbs_}, tc_kr_, rdig_col_, rdig_row_,
                           err_, st));
      rdig_for_ = factor_serial_;
    }
    kr = tc_kr_;
    const int xd = ((32 * (solve_xlimbs_ + solve_xlimbs_ / 16 + 8)) + 6) / 7;
    mc = (kr + xd + 15) & ~15;
    if (mc > tc_mc_) {
      dfree(tc_t_);
      dfree(tc_c_);
      dfree(tc_acc_);
      tc_t_ = dalloc<uint8_t>((size_t)mc * kr);
      tc_c_ = dalloc<int32_t>((size_t)n * mc);
      tc_acc_ = dalloc<long long>((size_t)n * mc);
      tc_mc_ = mc;
    }
    mc = tc_mc_;
    int ok = 0;
    CU(configure_solve_tc(Wv, Wa, mc, &ok));
    if (!ok) throw Error(HGPU_ERR_CAPACITY, "tensor-core solve operands exceed shared memory");
    if (!tc_blas_) {
      if (cublasCreate((cublasHandle_t*)&tc_blas_) != CUBLAS_STATUS_SUCCESS)
        throw Error(HGPU_ERR_CUDA, "cublasCreate failed");
      tc_ws_ = dalloc<uint8_t>(kBlasWorkspace);
      if (cublasSetWorkspace((cublasHandle_t)tc_blas_, tc_ws_, kBlasWorkspace) !=
          CUBLAS_STATUS_SUCCESS)
        throw Error(HGPU_ERR_CUDA, "cublasSetWorkspace failed");
    }
    if (cublasSetStream((cublasHandle_t)tc_blas_, st) != CUBLAS_STATUS_SUCCESS)
      throw Error(HGPU_ERR_CUDA, "cublasSetStream failed");
  }
  // transform-domain AXPY: plan for |R| < 2^mbR and |x| < 2^xb, transforms
  // of every L entry once per factorisation
  const long long ne = (long long)n * (n - 1) / 2;
  int xbmax = 0;
  if (ntt) {
    if (lhat_for_ != factor_serial_) {
      std::vector<int> bits(std::max<long long>(ne, 1));
      int* dbits = dalloc<int>(std::max<long long>(ne, 1));
      CU(launch_int_bits_batch(IntBuf{lhdr_, llimbs_}, 0, 1, P.cap, (int)ne, dbits, st));
      CU(cudaMemcpyAsync(bits.data(), dbits, ne * 4, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      dfree(dbits);
      int mb = 1;
      for (long long i = 0; i < ne; ++i) mb = std::max(mb, bits[i]);
      const int xb = 32 * std::max(P.cap, solve_xlimbs_ + 16);
      // a plan made for wider operands stays exact; re-plan when the operands
      // outgrow it (or shrink by enough to matter)
      const bool fits = sdp_bits_ > 0 && xb <= sdp_xbits_ && mb + sdp_xbits_ <= sdp_bits_ &&
                        mb + sdp_xbits_ + 4096 > sdp_bits_;
      if (fits && lhat_pre_for_ == factor_serial_) {
        // transformed during the factorisation in this very plan
        lhat_for_ = factor_serial_;
      } else {
      if (!fits) {
        // bits of one product; choose_plan adds the column count n to the
        // coefficient bound and keeps two spare digits
        const Plan SP = solve_plan(n, K_, mb + xb);
        dfree(stw_);
        dfree(lhat_tab_);
        for (uint32_t* c : lhat_chunks_) dfree(c);
        lhat_chunks_.clear();
        dfree(acch_);
        dfree(sxhat_);
        stw_ = acch_ = sxhat_ = nullptr;
        lhat_tab_ = nullptr;
        // nothing describes the freed buffers any more; an allocation failure
        // below leaves the solve unplanned and reports a capacity failure, so
        // solve() falls back to the schoolbook AXPY
        sdp_bits_ = sdp_xbits_ = 0;
        lhat_for_ = -1;
        auto unplan = [&]() { release_solve_transforms(); };
        try {
        DevPlan S{};
        S.n = n;
        S.K = K_;
        S.k2 = k2;
        S.np = SP.np;
        S.logL = SP.logL;
        S.L = SP.L;
        S.w = SP.w;
        S.T = SP.T;
        S.cap = SP.cap;
        S.ycap = SP.ycap;
        S.NW = SP.np * SP.L;
        const std::vector<uint32_t> tab = transform_tables(S, SP);
        const size_t npl = (size_t)SP.np * SP.L;
        stw_ = dalloc<uint32_t>(tab.size());
        CU(cudaMemcpy(stw_, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
        S.tw = stw_;
        S.twp = stw_ + npl;
        S.itw = stw_ + 2 * npl;
        S.itwp = stw_ + 3 * npl;
        S.twm = stw_ + 4 * npl;
        S.itwm = stw_ + 5 * npl;
        S.tw_smem = 0;
        S.grid_cap = dp_.grid_cap;
        S.debug = dp_.debug;
        int ok = 0;
        CU(configure_solve_ntt(S, P.cap, Wv, Wa, &ok));
        size_t fr = device_available(device_);
        const size_t need = ((size_t)ne + n + 2) * S.NW * 4;
        if (ok && need + (1ull << 30) > fr && W_ && !interval_) {
          // the factorisation's workspace is idle during the solves
          CU(cudaStreamSynchronize(st));
          release_workspace();
          fr = device_available(device_);
        }
        if (!ok || need + (1ull << 30) > fr)
          throw Error(HGPU_ERR_CAPACITY, "transform-domain solve does not fit");
        // chunks of <= 256 MB: a warm pool serves them from the blocks the
        // factorisation's slot sets returned (one 16 GB block would map
        // fresh memory, ~0.5 s)
        lhat_shift_ = 0;
        while ((2ull << lhat_shift_) * S.NW * 4 <= (256ull << 20)) ++lhat_shift_;
        const long long per = 1LL << lhat_shift_;
        const long long nch = (std::max<long long>(ne, 1) + per - 1) / per;
        for (long long c = 0; c < nch; ++c)
          lhat_chunks_.push_back(dalloc<uint32_t>((size_t)per * S.NW));
        lhat_tab_ = dalloc<uint32_t*>(nch);
        CU(cudaMemcpy(lhat_tab_, lhat_chunks_.data(), nch * sizeof(uint32_t*),
                      cudaMemcpyHostToDevice));
        acch_ = dalloc<uint32_t>((size_t)n * S.NW);
        sxhat_ = dalloc<uint32_t>(2 * (size_t)S.NW);
        sdp_ = S;
        sdp_bits_ = mb + xb;
        sdp_xbits_ = xb;
        } catch (const Error& e) {
          unplan();
          if (e.status != HGPU_ERR_CUDA) throw;
          throw Error(HGPU_ERR_CAPACITY,
                      std::string("transform-domain solve allocation failed: ") + e.what());
        }
      }
      CU(launch_solve_rhat(sdp_, P.cap, IntBuf{lhdr_, llimbs_}, ne, lhat_store(), dp_.grid_cap, err_,
                           st));
      lhat_for_ = factor_serial_;
      }
    }
    xbmax = sdp_xbits_;
  }
  // C[t][k'] = sum_i B[t][i] T[k'][i] for `rows` targets (int8 -> int32)
  auto tc_gemm = [&](const uint8_t* B, int rows) {
    const int32_t one = 1, zero = 0;
    const cublasStatus_t bs = cublasGemmEx(
        (cublasHandle_t)tc_blas_, CUBLAS_OP_T, CUBLAS_OP_N, mc, rows, kr, &one, tc_t_,
        CUDA_R_8I, kr, B, CUDA_R_8I, kr, &zero, tc_c_, CUDA_R_32I, mc,
        CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
    if (bs != CUBLAS_STATUS_SUCCESS)
      throw Error(HGPU_ERR_CUDA, "solve GEMM failed (cublas status " +
                                     std::to_string((int)bs) + ")");
  };
  IntBuf vecs{svhdr_, svlimbs_};
  IntBuf pairs{spair_hdr_, spair_limbs_};
  IntBuf L{lhdr_, llimbs_};
  const int U = 0, Z = n, Wq = 2 * n, Y = 3 * n;
  // (the z | w | y headers are rewritten by the solve's own kernels)
  CU(cudaMemsetAsync(svhdr_ + n, 0, 3 * (size_t)n * sizeof(int), st));
  // the AXPY's shared-memory layout at full operand capacities (measured:
  // layouts sized to the operands actually met let the block scheduler pack
  // more CTAs per SM and ran slower on this grid)
  const int capX = Wv, capC = P.cap;
  const int sgrid = dp_.grid_cap;
  long long nl = 0;
  int herr[kErrWords];
  std::vector<int> vh(4 * (size_t)n);
  std::vector<uint32_t> yl(download ? (size_t)n * Wv : 0);
  {
    int herr0[kErrWords] = {INT_MAX, 0, 0, 0};
    CU(cudaMemcpyAsync(err_, herr0, sizeof(herr0), cudaMemcpyHostToDevice, st));
    // pivots into the even rows of the pair buffer
    CU(cudaMemcpy2DAsync(spair_hdr_, 2 * sizeof(int), phdr_, sizeof(int),
                         sizeof(int), n, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemsetAsync(spair_limbs_, 0, 2 * (size_t)n * Wv * 4, st));
    CU(cudaMemcpy2DAsync(spair_limbs_, 2 * (size_t)Wv * 4, plimbs_,
                         (size_t)P.cap * 4, (size_t)P.cap * 4, n,
                         cudaMemcpyDeviceToDevice, st));
    // forward: z_p = u_p - tdiv_2exp(acc_p, k2); acc_r += R_p[r] z_p (r > p)
    CU(cudaMemsetAsync(sacc_, 0, (size_t)n * Wa * 4, st));
    // (each step also finishes the next row, so one launch per step)
    CU(launch_solve_finish(Wv, Wa, k2, sacc_,
                           Finish{vecs, U, vecs, Z, pairs, 1, k2}, err_, st));
    ++nl;
    if (tc) CU(cudaMemsetAsync(tc_acc_, 0, (size_t)n * mc * 8, st));
    const int SNW = sdp_.NW;
    // one resident CTA per SM (the critical CTA's shared memory): block 0
    // plus one pointwise CTA on every other SM
    int nsm = 148;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device_));
    const int ntt_grid = std::max(1, nsm - 1);
    if (ntt) {
      CU(cudaMemsetAsync(acch_, 0, (size_t)n * SNW * 4, st));
      CU(launch_solve_xhat(sdp_, vecs, Z, Wv, sxhat_, xbmax, err_, st));
      ++nl;
    }
    for (int p = 0; p + 1 < n; ++p) {
      const Finish f{vecs, U + p + 1, vecs, Z + p + 1, pairs, 2 * (p + 1) + 1, k2};
      if (ntt) {
        CU(launch_solve_ntt(sdp_, n, Wv, Wa, k2, lhat_store(), sxhat_ + (size_t)(p & 1) * SNW,
                            sxhat_ + (size_t)((p + 1) & 1) * SNW, acch_, p, 0, f, ntt_grid, xbmax,
                            err_, st));
        ++nl;
        continue;
      }
      if (tc) {
        CU(launch_solve_toeplitz(vecs, Z + p, Wv, kr, mc, tc_t_, err_, st));
        tc_gemm(rdig_col_ + (size_t)((long long)p * (n - 1) - (long long)p * (p - 1) / 2) * kr,
                n - 1 - p);
        CU(launch_solve_acc_tc(n, Wv, Wa, k2, L, vecs, Z + p, p, 0, tc_c_, mc, tc_acc_, f,
                               sgrid, err_, st));
        nl += 3;
        continue;
      }
      CU(launch_solve_axpy(n, P.cap, Wv, Wa, k2, L, vecs, Z + p, p, 0, sacc_, f,
                           capX, capC, sgscr_, sgrid, err_, st));
      ++nl;
    }
    // diagonal: w_p = tdiv(z_p 2^K, piv_p) with the LDL^T division kernels,
    // all n independent divisions in one batched launch each
    CU(launch_int_bits_batch(pairs, 1, 2, Wv, n, sbits_, st));
    CU(launch_recip_batch(D2, pairs, 0, sbits_, sybuf_, sys_, srscr_, n, err_, st));
    CU(launch_divide_batch(D2, pairs, 0, sybuf_, sys_, vecs, Wq - 1, sdscr_, n,
                           err_, st));
    nl += 3;
    // back: y_r = w_r - tdiv_2exp(acc'_r, k2); acc'_q += R_q[r] y_r (q < r)
    CU(cudaMemsetAsync(sacc_, 0, (size_t)n * Wa * 4, st));
    CU(launch_solve_finish(Wv, Wa, k2, sacc_ + (size_t)(n - 1) * Wa,
                           Finish{vecs, Wq + n - 1, vecs, Y + n - 1, vecs, 0, 0},
                           err_, st));
    ++nl;
    if (tc) CU(cudaMemsetAsync(tc_acc_, 0, (size_t)n * mc * 8, st));
    if (ntt) {
      CU(cudaMemsetAsync(acch_, 0, (size_t)n * SNW * 4, st));
      CU(launch_solve_xhat(sdp_, vecs, Y + n - 1, Wv, sxhat_, xbmax, err_, st));
      ++nl;
    }
    for (int r = n - 1; r >= 1; --r) {
      const Finish f{vecs, Wq + r - 1, vecs, Y + r - 1, vecs, 0, 0};
      if (ntt) {
        const int par = (n - 1 - r) & 1;
        CU(launch_solve_ntt(sdp_, n, Wv, Wa, k2, lhat_store(), sxhat_ + (size_t)par * SNW,
                            sxhat_ + (size_t)(par ^ 1) * SNW, acch_, r, 1, f, ntt_grid, xbmax,
                            err_, st));
        ++nl;
        continue;
      }
      if (tc) {
        CU(launch_solve_toeplitz(vecs, Y + r, Wv, kr, mc, tc_t_, err_, st));
        tc_gemm(rdig_row_ + (size_t)((long long)r * (r - 1) / 2) * kr, r);
        CU(launch_solve_acc_tc(n, Wv, Wa, k2, L, vecs, Y + r, r, 1, tc_c_, mc, tc_acc_, f,
                               sgrid, err_, st));
        nl += 3;
        continue;
      }
      CU(launch_solve_axpy(n, P.cap, Wv, Wa, k2, L, vecs, Y + r, r, 1, sacc_, f,
                           capX, capC, sgscr_, sgrid, err_, st));
      ++nl;
    }
    CU(cudaMemcpyAsync(herr, err_, sizeof(herr), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(vh.data(), svhdr_, vh.size() * 4, cudaMemcpyDeviceToHost, st));
    if (download)
      CU(cudaMemcpyAsync(yl.data(), svlimbs_ + (size_t)Y * Wv, yl.size() * 4,
                         cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  if (launches) *launches += nl;
  if (herr[kErrCapacity])
    throw Error(HGPU_ERR_CAPACITY, "solve capacity exceeded (flags " +
                                       std::to_string(herr[kErrCapacity]) + ")");
  if (herr[kErrInternal])
    throw Error(HGPU_ERR_INTERNAL, "solve exactness self-check failed");
  if (herr[kErrZeroPivot] != INT_MAX)
    throw Error(HGPU_ERR_INTERNAL, "zero divisor in the diagonal solve");
  if (std::getenv("HGPU_SOLVE_TRACE")) {
    int mx[4] = {0, 0, 0, 0};
    for (int v = 0; v < 4; ++v)
      for (int i = 0; i < n; ++i) mx[v] = std::max(mx[v], std::abs(vh[(size_t)v * n + i]));
    std::fprintf(stderr, "solve mode %d %.3f ms; limbs: u %d z %d w %d y %d (Wv %d, R cap %d)\n",
                 mode,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                           t_start).count(),
                 mx[0], mx[1], mx[2], mx[3], Wv, P.cap);
  }
  {
    int mx = 0;
    for (int i = 0; i < n; ++i)
      mx = std::max(mx, std::max(std::abs(vh[(size_t)Z + i]), std::abs(vh[(size_t)Y + i])));
    solve_xlimbs_ = std::max(solve_xlimbs_, mx);
  }
  last_ulimbs_ = last_ylimbs_ = 0;
  for (int i = 0; i < n; ++i) {
    last_ulimbs_ = std::max(last_ulimbs_, std::abs(vh[(size_t)U + i]));
    last_ylimbs_ = std::max(last_ylimbs_, std::abs(vh[(size_t)Y + i]));
  }
  have_y_ = true;
  if (!download) return {};
  std::vector<int> yh(vh.begin() + Y, vh.begin() + Y + n);
  std::vector<HostInt> y(n);
  for (int i = 0; i < n; ++i) {
    y[i].size = yh[i];
    const int len = std::abs(yh[i]);
    y[i].limbs.assign(yl.begin() + (size_t)i * Wv, yl.begin() + (size_t)i * Wv + len);
  }
  return y;
}

void Matrix::fold(FactorResult& res) {
  const Plan& P = plan_;
  const int n = n_;
  std::vector<int> plen(n);
  int neg = 0;
  long long nx = K_ / 32 + 1, xcap = nx;
  for (int p = 0; p < n; ++p) {
    plen[p] = std::abs(res.pivots[p].size);
    neg ^= res.pivots[p].size < 0;
    nx = nx + plen[p] - K_ / 32;
    xcap = std::max(xcap, nx);
  }
  xcap += 2;
  uint32_t* X0 = dalloc<uint32_t>(xcap);
  uint32_t* X1 = dalloc<uint32_t>(xcap);
  uint32_t* col = dalloc<uint32_t>(3 * (size_t)(xcap + P.cap));
  const size_t nch = (size_t)(xcap + P.cap) / 2048 + 4;
  uint32_t* cf = dalloc<uint32_t>(nch);
  int* cc = dalloc<int>(nch);
  long long launches = 0;
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  CU(cudaEventRecord(a, stream_));
  const long long nfin = fold_pivots_device(plimbs_, plen.data(), n, P.cap, K_,
                                            X0, X1, xcap, col, cf, cc,
                                            stream_, &launches);
  CU(cudaEventRecord(b, stream_));
  std::vector<uint32_t> hx(std::max<long long>(nfin, 0));
  if (nfin > 0)
    CU(cudaMemcpyAsync(hx.data(), X0, nfin * 4, cudaMemcpyDeviceToHost, stream_));
  CU(cudaStreamSynchronize(stream_));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  for (void* p : {(void*)X0, (void*)X1, (void*)col, (void*)cf, (void*)cc}) dfree(p);
  CU(cudaGetLastError());
  if (nfin < 0) throw Error(HGPU_ERR_INTERNAL, "fold buffer too small");
  while (!hx.empty() && hx.back() == 0) hx.pop_back();
  res.det.limbs = std::move(hx);
  res.det.size = res.det.limbs.empty() ? 0 : (neg ? -1 : 1) * (int)res.det.limbs.size();
  res.have_det = true;
  res.fold_ms = ms;
  res.launches += launches;
}

FactorResult Matrix::factor(const HostInt& x, unsigned flags) {
  if (group_) {
    if (rank_ != 0)
      throw Error(HGPU_ERR_INVALID_ARGUMENT, "a group is driven by its rank 0");
    return factor_group(x, flags);
  }
  CU(cudaSetDevice(device_));
  if (ws_released_) reclaim_workspace();
  FactorResult res;
  res.n = n_;
  res.K = K_;
  // plans escalate only on a capacity failure (non-PD shifts can outgrow
  // the PD bound); every rank sees the same flags, so all escalate together
  int min_logL = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (!W_ || (min_logL && plan_.logL < min_logL)) {
      const auto tb = std::chrono::steady_clock::now();
      build(min_logL);
      if (std::getenv("HGPU_HOST_TRACE")) {
        CU(cudaDeviceSynchronize());
        std::fprintf(stderr, "build: %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               tb)
                         .count());
      }
    }
    try {
      res = FactorResult{};
      res.n = n_;
      res.K = K_;
      run(x, flags, res);
      return res;
    } catch (const Error& e) {
      if (e.status != HGPU_ERR_CAPACITY) throw;
      if (e.cap_flags == kCapAmax && recip_bound_) {
        recip_bound_ = false;  // non-PD sizes: exact per-stage maxima
        continue;
      }
      min_logL = plan_.logL + 1;
      release();
    }
  }
  throw Error(HGPU_ERR_CAPACITY, "values outgrew every transform plan");
}

}  // namespace hgpu
