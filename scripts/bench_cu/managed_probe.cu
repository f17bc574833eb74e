// Managed-memory oversubscription probe: allocate G GB of managed memory,
// sweep it from the GPU forwards then backwards (chunked, with prefetch),
// report GB/s per sweep.  usage: managed_probe <GB> <chunk_MB> <prefetch 0/1>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CU(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void touch(uint4* p, size_t n, unsigned add) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    v.x += add; v.y += add; v.z += add; v.w += add;
    p[i] = v;
  }
}
int main(int argc, char** argv) {
  const size_t gb = argc > 1 ? atol(argv[1]) : 200;
  const size_t chunk = (argc > 2 ? atol(argv[2]) : 1024) << 20;
  const int pf = argc > 3 ? atoi(argv[3]) : 1;
  size_t fr, tot;
  CU(cudaMemGetInfo(&fr, &tot));
  printf("device free %.1f GB of %.1f GB\n", fr / 1e9, tot / 1e9);
  const size_t bytes = gb << 30;
  char* p;
  CU(cudaMallocManaged(&p, bytes));
  CU(cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, 0));
  cudaStream_t st, st2;
  CU(cudaStreamCreate(&st));
  CU(cudaStreamCreate(&st2));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t nch = (bytes + chunk - 1) / chunk;
  for (int sweep = 0; sweep < 4; ++sweep) {
    CU(cudaEventRecord(a, st));
    for (size_t k = 0; k < nch; ++k) {
      const size_t c = (sweep & 1) ? nch - 1 - k : k;
      const size_t off = c * chunk, len = bytes - off < chunk ? bytes - off : chunk;
      if (pf) CU(cudaMemPrefetchAsync(p + off, len, 0, st));
      touch<<<148 * 8, 256, 0, st>>>((uint4*)(p + off), len / 16, 1u);
    }
    CU(cudaEventRecord(b, st));
    CU(cudaStreamSynchronize(st));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("sweep %d (%s): %.2f s, %.1f GB/s\n", sweep, (sweep & 1) ? "backward" : "forward", ms / 1e3, bytes / 1e6 / ms);
    fflush(stdout);
  }
  return 0;
}
