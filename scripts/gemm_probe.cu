// Probe: int8 x int8 -> int32 GEMM throughput (cublasGemmEx, TN) at the
// shapes of the batched ratio product C = T(Y)^T V:
// M = quotient columns, K = digits of V, N = rows of the stage.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gp scripts/gemm_probe.cu -lcublas
#include <cublas_v2.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

int main() {
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) { printf("no cublas\n"); return 1; }
  const int M = 3104, K = 4192;
  const int Ns[] = {1000, 512, 256, 128, 64, 32};
  int8_t *A, *B;
  int32_t* C;
  cudaMalloc(&A, (size_t)M * K);
  cudaMalloc(&B, (size_t)K * 1000);
  cudaMalloc(&C, (size_t)M * 1000 * 4);
  std::vector<int8_t> ha((size_t)M * K), hb((size_t)K * 1000);
  for (size_t i = 0; i < ha.size(); ++i) ha[i] = (int8_t)((i * 2654435761u >> 13) & 127);
  for (size_t i = 0; i < hb.size(); ++i) hb[i] = (int8_t)((i * 40503u >> 7) & 127);
  cudaMemcpy(A, ha.data(), ha.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb.data(), hb.size(), cudaMemcpyHostToDevice);
  const int32_t one = 1, zero = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int N : Ns) {
    auto run = [&] {
      return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, CUDA_R_8I, K, B,
                          CUDA_R_8I, K, &zero, C, CUDA_R_32I, M, CUBLAS_COMPUTE_32I,
                          CUBLAS_GEMM_DEFAULT);
    };
    cublasStatus_t s = run();
    if (s != CUBLAS_STATUS_SUCCESS) { printf("N=%d status %d\n", N, (int)s); continue; }
    cudaDeviceSynchronize();
    const int reps = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / reps;
    printf("M=%d N=%d K=%d: %.1f us, %.1f TOPS\n", M, N, K, us, 2.0 * M * N * K / us * 1e-6);
  }
  // spot check one entry
  std::vector<int32_t> hc((size_t)M * 32);
  cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, M, 32, K, &one, A, CUDA_R_8I, K, B, CUDA_R_8I, K,
               &zero, C, CUDA_R_32I, M, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
  cudaMemcpy(hc.data(), C, hc.size() * 4, cudaMemcpyDeviceToHost);
  long long ref = 0;
  const int i = 77, j = 5;
  for (int k = 0; k < K; ++k) ref += (long long)ha[(size_t)i * K + k] * hb[(size_t)j * K + k];
  printf("check C[%d][%d] = %d, ref %lld\n", i, j, hc[(size_t)j * M + i], ref);
  return 0;
}
