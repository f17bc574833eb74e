// Trailing update on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// The same operation as k_update_tiled (ldlt.cpp:65-71 in the transform
// domain): for a band of columns c and every row r >= c,
//   W[r][c][t] -= REDC( sum_s Rhat_s[r][t] * Vhat_s[c][t] )   mod q_t,
// for all NW = np*L words t, over nslots <= 256 stages s.  For one word t
// this is a small matrix product, C_t = A_t B_t^T with A_t[r][s] = Rhat and
// B_t[c][s] = Vhat, batched over t.  The residues are < 2^28, so each is four
// unsigned bytes, and
//   a * b = sum_{i,j} a_i b_j 2^{8(i+j)}:
// 16 int8 GEMMs per word, accumulated exactly in s32 by digit-sum d = i+j
// (7 TMEM accumulators; each <= 4 * 256 * 255^2 < 2^31), then recombined as
// sum_d acc_d (2^{8d} mod q) < 2^58 and reduced with the update's own REDC
// (reduce_sum64), so the result is bit-identical to the IMAD kernel's.
//
// CTA tile: 128 rows x 16 band columns x 4 consecutive words, K = 32 stages
// per step.  All 256 threads load the step's residues (16-byte vectors of 4
// words), transpose them into byte planes in the canonical K-major layout
// ([16-stage half][row][16 bytes]), one thread issues the 64 MMAs
// (M=128, N=16, K=32) and commits them to an mbarrier; the planes are double
// buffered so the next step's loads overlap the tensor-core work.  The
// epilogue reads the accumulators with tcgen05.ld (warp w reads TMEM lanes
// 32 (w % 4) ..), recombines, reduces and read-modify-writes W four words
// (16 bytes) at a time.
#include <cuda_runtime.h>

#include <cstdint>

#include "ldlt_kernels.cuh"
#include "modarith.cuh"

namespace hgpu {

long long kernel_launch_count_add(long long k);

namespace {

constexpr int kRows = 128;  // MMA M: rows r per CTA
constexpr int kCols = 16;   // MMA N: band columns per CTA
constexpr int kTB = 4;      // words t per CTA (one 16-byte vector)
constexpr int kK = 32;      // stages per MMA step (int8 K)
constexpr int kThreads = 256;
constexpr int kAPlane = 2 * kRows * 16;  // bytes of one A byte-plane tile
constexpr int kBPlane = 2 * kCols * 16;
constexpr int kABuf = kTB * 4 * kAPlane;  // 64 KB
constexpr int kBBuf = kTB * 4 * kBPlane;  // 8 KB
constexpr int kBuf = kABuf + kBBuf;
constexpr int kTmemCols = 512;  // kTB * 7 * kCols = 448 used

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, no swizzle: core matrices of 8 rows x 16 bytes (rows 16 bytes
// apart), 8-row groups sbo bytes apart, the two 16-byte K halves lbo apart
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// instruction descriptor: D s32, A and B u8, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// byte i of each of four words, packed (word v -> byte v)
__device__ __forceinline__ uint32_t plane4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                           int i) {
  const uint32_t lo = __byte_perm(w0, w1, (uint32_t)(i | ((4 + i) << 4)));
  const uint32_t hi = __byte_perm(w2, w3, (uint32_t)(i | ((4 + i) << 4)));
  return __byte_perm(lo, hi, 0x5410);
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
k_update_tc(const __grid_constant__ DevPlan P, uint32_t* W, const long long* colbase, const uint32_t* Vhat,
            const uint32_t* Rhat, long long row_stride_slot, int nslots, int c_begin,
            int c_end, int nchalf, const int* err) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  (void)err;  // no early exit: the CTA's barriers and TMEM allocation need every thread
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * kTB;
  const int ch = blockIdx.y % nchalf, rt = blockIdx.y / nchalf;
  const int c0 = c_begin + ch * kCols;
  const int r0 = c_begin + rt * kRows;
  if (r0 + kRows - 1 < c0) return;  // tile above the diagonal
  const long long NW = P.NW;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  const int nk = (nslots + kK - 1) / kK;
  // A: 128 rows x 8 stage quads, B: 16 columns x 8 quads = 1152 items, at
  // most kItems per thread; a step's residues are loaded into registers one
  // step ahead (software pipeline), so HBM latency overlaps the previous
  // step's transpose and MMAs
  constexpr int kItems = ((kRows + kCols) * 8 + kThreads - 1) / kThreads;
  uint4 cur[kItems][4], nxt[kItems][4];
  auto load_step = [&](int kk, uint4 (*w)[4]) {
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int it = tid + u * kThreads;
      const int q = it & 7, row = it >> 3;
      const bool isA = row < kRows;
      const int idx = isA ? r0 + row : c0 + (row - kRows);
      const bool valid = it < (kRows + kCols) * 8 && (isA ? idx < P.n : idx < c_end);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int s = kk * kK + 4 * q + v;
        if (valid && s < nslots) {
          const uint32_t* src =
              (isA ? Rhat : Vhat) + s * row_stride_slot + (long long)idx * NW + t0;
          w[u][v] = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
          w[u][v] = make_uint4(0, 0, 0, 0);
        }
      }
    }
  };
  load_step(0, cur);
  for (int kk = 0; kk < nk; ++kk) {
    const int buf = kk & 1;
    uint8_t* A = smem + buf * kBuf;
    uint8_t* B = A + kABuf;
    if (kk + 1 < nk) load_step(kk + 1, nxt);
    // the MMAs of step kk-2 read this buffer
    if (kk >= 2) mbar_wait(smem_u32(&mbar[buf]), ((kk - 2) >> 1) & 1);
#pragma unroll
    for (int u = 0; u < kItems; ++u) {
      const int it = tid + u * kThreads;
      if (it >= (kRows + kCols) * 8) break;
      const int q = it & 7, row = it >> 3;
      const bool isA = row < kRows;
      uint8_t* base = isA ? A + (q >> 2) * (kRows * 16) + row * 16 + (q & 3) * 4
                          : B + (q >> 2) * (kCols * 16) + (row - kRows) * 16 + (q & 3) * 4;
      const int plane = isA ? kAPlane : kBPlane;
      const uint4* w = cur[u];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        *reinterpret_cast<uint32_t*>(base + (0 * 4 + i) * plane) =
            plane4(w[0].x, w[1].x, w[2].x, w[3].x, i);
        *reinterpret_cast<uint32_t*>(base + (1 * 4 + i) * plane) =
            plane4(w[0].y, w[1].y, w[2].y, w[3].y, i);
        *reinterpret_cast<uint32_t*>(base + (2 * 4 + i) * plane) =
            plane4(w[0].z, w[1].z, w[2].z, w[3].z, i);
        *reinterpret_cast<uint32_t*>(base + (3 * 4 + i) * plane) =
            plane4(w[0].w, w[1].w, w[2].w, w[3].w, i);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t id = idesc_u8(kRows, kCols);
#pragma unroll 1
      for (int t = 0; t < kTB; ++t) {
        uint32_t started = 0;  // accumulators of this word written in step 0
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int d = i + j;
            const uint64_t da = umma_desc(smem_u32(A + (t * 4 + i) * kAPlane), kRows * 16, 128);
            const uint64_t db = umma_desc(smem_u32(B + (t * 4 + j) * kBPlane), kCols * 16, 128);
            const uint32_t acc = (kk > 0 || ((started >> d) & 1)) ? 1u : 0u;
            started |= 1u << d;
            const uint32_t dst = tmem + (uint32_t)((t * 7 + d) * kCols);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dst),
                "l"(da), "l"(db), "r"(id), "r"(acc));
          }
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&mbar[buf])));
    }
#pragma unroll
    for (int u = 0; u < kItems; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cur[u][v] = nxt[u][v];
  }
  // the last step's commit covers every earlier MMA (they complete in order)
  mbar_wait(smem_u32(&mbar[(nk - 1) & 1]), ((nk - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: warp w -> TMEM lanes (rows) 32 (w % 4) .. +31, columns 8 (w / 4) .. +7
  const int quad = warp & 3, chalf = warp >> 2;
  const int row = r0 + quad * 32 + lane;
  const PrimeConsts pc = P.pc[t0 / P.L];
  uint32_t wd[7];
  {
    uint64_t x = 1;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      wd[d] = (uint32_t)x;
      x = (x << 8) % pc.q;
    }
  }
  uint32_t res[kTB][8];
#pragma unroll
  for (int t = 0; t < kTB; ++t) {
    uint64_t y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = 0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      uint32_t v[8];
      const uint32_t taddr =
          tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)((t * 7 + d) * kCols + 8 * chalf);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 8; ++c) y[c] += (uint64_t)v[c] * wd[d];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) res[t][c] = reduce_sum64(y[c], pc);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int col = c0 + 8 * chalf + c;
    if (col >= c_end || row < col || row >= P.n) continue;
    uint4* dst = reinterpret_cast<uint4*>(W + (colbase[col] + (row - col)) * NW + t0);
    uint4 o = *dst;
    auto sub = [&](uint32_t a, uint32_t b) { return a >= b ? a - b : a + pc.q - b; };
    o.x = sub(o.x, res[0][c]);
    o.y = sub(o.y, res[1][c]);
    o.z = sub(o.z, res[2][c]);
    o.w = sub(o.w, res[3][c]);
    *dst = o;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols));
}

size_t update_tc_smem_bytes() { return 2 * (size_t)kBuf; }

cudaError_t configure_update_tc() {
  return cudaFuncSetAttribute(k_update_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)update_tc_smem_bytes());
}

// The lower triangle r >= c of the band [c_begin, c_end) (rows up to n).
// Needs NW % 4 == 0 (16-byte words groups inside one prime) and nslots <= 256.
cudaError_t launch_update_tc(const DevPlan& P, uint32_t* W, const long long* colbase,
                             const uint32_t* Vhat, const uint32_t* Rhat,
                             long long row_stride_slot, int nslots, int c_begin, int c_end,
                             const int* err, cudaStream_t st) {
  if (c_begin >= c_end || nslots <= 0) return cudaSuccess;
  if (nslots > 256 || P.NW % kTB != 0 || P.L % kTB != 0) return cudaErrorInvalidValue;
  const int nchalf = (c_end - c_begin + kCols - 1) / kCols;
  const int nrt = (P.n - c_begin + kRows - 1) / kRows;
  dim3 grid(P.NW / kTB, nrt * nchalf);
  kernel_launch_count_add(1);
  k_update_tc<<<grid, kThreads, update_tc_smem_bytes(), st>>>(
      P, W, colbase, Vhat, Rhat, row_stride_slot, nslots, c_begin, c_end, nchalf, err);
  return cudaGetLastError();
}

}  // namespace hgpu
