// Probe: split the SMs into two green contexts, launch runtime-API kernels on
// a stream of each (no context switch on the host), and record which SMs the
// CTAs ran on.  Build: nvcc -arch=sm_100a -o /tmp/gp scripts/green_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <set>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void k_smid(int* out, long long spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

int main(int argc, char** argv) {
  const int chain_sms = argc > 1 ? atoi(argv[1]) : 16;
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  CUdevResource grp, rest;
  unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(&grp, &ng, &all, &rest, 0, chain_sms));
  printf("group SMs %u, remaining %u\n", grp.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc da, db;
  CK(cuDevResourceGenerateDesc(&da, &grp, 1));
  CK(cuDevResourceGenerateDesc(&db, &rest, 1));
  CUgreenCtx ga, gb;
  CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb;
  int lo, hi;
  RK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, hi));
  CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  int *oa, *ob;
  const int na = 4 * chain_sms, nb = 8 * 148;
  RK(cudaMalloc(&oa, na * 4));
  RK(cudaMalloc(&ob, nb * 4));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  // cross-context event dependency: b waits for a
  RK(cudaEventRecord(e0, (cudaStream_t)sa));
  k_smid<<<na, 128, 0, (cudaStream_t)sa>>>(oa, 2000000);
  RK(cudaGetLastError());
  RK(cudaEventRecord(e1, (cudaStream_t)sa));
  k_smid<<<nb, 128, 0, (cudaStream_t)sb>>>(ob, 2000000);
  RK(cudaGetLastError());
  RK(cudaStreamWaitEvent((cudaStream_t)sb, e1, 0));
  k_smid<<<1, 32, 0, (cudaStream_t)sb>>>(ob, 10);
  RK(cudaDeviceSynchronize());
  float ms;
  RK(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<int> ha(na), hb(nb);
  RK(cudaMemcpy(ha.data(), oa, na * 4, cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(hb.data(), ob, nb * 4, cudaMemcpyDeviceToHost));
  std::set<int> sa_set(ha.begin(), ha.end()), sb_set(hb.begin(), hb.end());
  int overlap = 0;
  for (int s : sa_set) overlap += sb_set.count(s);
  printf("stream A: %zu distinct SMs, stream B: %zu distinct SMs, overlap %d, A kernel %.3f ms\n",
         sa_set.size(), sb_set.size(), overlap, ms);
  // a plain (primary-context) stream still sees every SM
  cudaStream_t sp;
  RK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
  k_smid<<<nb, 128, 0, sp>>>(ob, 100000);
  RK(cudaStreamSynchronize(sp));
  RK(cudaMemcpy(hb.data(), ob, nb * 4, cudaMemcpyDeviceToHost));
  std::set<int> sp_set(hb.begin(), hb.end());
  printf("primary stream: %zu distinct SMs\n", sp_set.size());
  return 0;
}
