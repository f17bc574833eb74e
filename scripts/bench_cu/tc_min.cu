// Minimal tcgen05.mma kind::i8 check: one CTA, D[128x32] (s32, TMEM) =
// A[128x32] (u8, K-major) x B[32x32]^T (u8, K-major), against the CPU.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major, no swizzle: ((8,m),2):((16B, SBO), LBO)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                      // D: s32
         | (0u << 7) | (0u << 10)       // A, B: u8
         | (0u << 15) | (0u << 16)      // K-major
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void k_tc_min(const uint8_t* A, const uint8_t* B, int32_t* D) {
  __shared__ __align__(128) uint8_t sA[2 * 128 * 16];
  __shared__ __align__(128) uint8_t sB[2 * 32 * 16];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  // layout [half][row][16 B]
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    const int r = e / 32, k = e % 32;
    sA[(k / 16) * 128 * 16 + r * 16 + (k % 16)] = A[r * 32 + k];
  }
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e / 32, k = e % 32;
    sB[(k / 16) * 32 * 16 + r * 16 + (k % 16)] = B[r * 32 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // generic-proxy smem writes -> visible to the async (tensor) proxy
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da = make_desc(smem_u32(sA), 128 * 16, 8 * 16);
    const uint64_t db = make_desc(smem_u32(sB), 32 * 16, 8 * 16);
    const uint32_t id = idesc_i8(128, 32);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < 32; ++c) D[row * 32 + c] = (int32_t)v[c];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  uint8_t hA[128 * 32], hB[32 * 32];
  srand(1);
  for (auto& x : hA) x = rand() & 255;
  for (auto& x : hB) x = rand() & 255;
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, 128 * 32 * 4);
  k_tc_min<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  int32_t hD[128 * 32];
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 32; ++c) {
      int32_t s = 0;
      for (int k = 0; k < 32; ++k) s += (int32_t)hA[r * 32 + k] * hB[c * 32 + k];
      if (s != hD[r * 32 + c] && bad++ < 5) printf("r %d c %d: want %d got %d\n", r, c, s, hD[r * 32 + c]);
    }
  printf("%s; %d mismatches\n", cudaGetErrorString(e), bad);
  return bad != 0;
}
