// k_update_tc (tensor cores) against k_update_tiled (IMAD) on the same
// random residues: bit-identical W, and the time of one band-run launch at
// config-3 shapes (NW = 4 x 1024 words, 8 panels = 256 stages).
//   tc_update_bench [n] [c_begin] [nslots]
#include "../../paper_0902_0852_b200/csrc/ldlt_kernels.cu"
#include "../../paper_0902_0852_b200/csrc/tc_update.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace hgpu;

static uint32_t inv_neg(uint32_t q) {  // -q^{-1} mod 2^32
  uint32_t x = 1;
  for (int i = 0; i < 5; ++i) x *= 2 - q * x;
  return (uint32_t)(0u - x);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1000;
  const int c_begin = argc > 2 ? atoi(argv[2]) : 288;
  const int nslots = argc > 3 ? atoi(argv[3]) : 256;
  const int c_end = std::min(n, c_begin + 32);
  DevPlan P{};
  P.n = n; P.np = 4; P.L = 1024; P.logL = 10; P.NW = 4096;
  const uint32_t qs[4] = {268369921u, 268361729u, 268271617u, 268238849u};  // < 2^28, odd
  for (int j = 0; j < 4; ++j) {
    P.pc[j].q = qs[j];
    P.pc[j].qneg = inv_neg(qs[j]);
    P.pc[j].r32 = (uint32_t)((1ull << 32) % qs[j]);
  }
  const long long NW = P.NW;
  // W entries for columns [c_begin, c_end), rows r >= c; V/R slot rows: nslots x n
  std::vector<long long> cb(n, -1);
  long long entries = 0;
  for (int c = c_begin; c < c_end; ++c) cb[c] = entries, entries += n - c;
  std::mt19937_64 rng(7);
  auto fill = [&](std::vector<uint32_t>& v) {
    for (size_t e = 0; e < v.size(); ++e) v[e] = (uint32_t)(rng() % qs[(e % NW) / P.L]);
  };
  std::vector<uint32_t> hW(entries * NW), hV((size_t)nslots * n * NW), hR((size_t)nslots * n * NW);
  fill(hW); fill(hV); fill(hR);
  uint32_t *W1, *W2, *V, *R;
  long long* dcb;
  int* err;
  cudaMalloc(&W1, hW.size() * 4); cudaMalloc(&W2, hW.size() * 4);
  cudaMalloc(&V, hV.size() * 4); cudaMalloc(&R, hR.size() * 4);
  cudaMalloc(&dcb, n * 8); cudaMalloc(&err, 16);
  cudaMemcpy(W1, hW.data(), hW.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(W2, hW.data(), hW.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(V, hV.data(), hV.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(R, hR.data(), hR.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dcb, cb.data(), n * 8, cudaMemcpyHostToDevice);
  int e0[4] = {INT_MAX, 0, 0, 0};
  cudaMemcpy(err, e0, 16, cudaMemcpyHostToDevice);
  size_t ds = 0; bool dg = false, rg = false;
  P.K = 64; P.k2 = 32; P.cap = 4; P.ycap = 8; P.T = 3; P.w = 29;
  configure_kernels(P, &ds, &dg, &rg);
  if (configure_update_tc() != cudaSuccess) { printf("configure_update_tc failed\n"); return 1; }
  const long long stride = (long long)n * NW;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float t_imad = 0, t_tc = 0;
  cudaEventRecord(a);
  launch_update(P, 16, W1, dcb, V, R, stride, nslots, c_begin, c_end, err, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&t_imad, a, b);
  cudaEventRecord(a);
  cudaError_t le = launch_update_tc(P, W2, dcb, V, R, stride, nslots, c_begin, c_end, err, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&t_tc, a, b);
  cudaError_t se = cudaDeviceSynchronize();
  std::vector<uint32_t> o1(hW.size()), o2(hW.size());
  cudaMemcpy(o1.data(), W1, o1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o2.data(), W2, o2.size() * 4, cudaMemcpyDeviceToHost);
  long long bad = 0, changed = 0;
  for (size_t e = 0; e < o1.size(); ++e) {
    if (o1[e] != o2[e] && bad++ < 5) printf("word %zu: imad %u tc %u (was %u)\n", e, o1[e], o2[e], hW[e]);
    changed += o1[e] != hW[e];
  }
  // timing: repeat (W keeps changing; both kernels see the same work)
  float best_i = 1e9, best_t = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    float ms;
    cudaEventRecord(a);
    launch_update(P, 16, W1, dcb, V, R, stride, nslots, c_begin, c_end, err, 0);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); best_i = std::min(best_i, ms);
    cudaEventRecord(a);
    launch_update_tc(P, W2, dcb, V, R, stride, nslots, c_begin, c_end, err, 0);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); best_t = std::min(best_t, ms);
  }
  double pairs = 0;
  for (int c = c_begin; c < c_end; ++c) pairs += n - c;
  const double prods = pairs * nslots * NW;
  printf("n=%d band [%d,%d) nslots=%d: %lld/%zu words differ (%lld changed); launch %s, sync %s\n", n,
         c_begin, c_end, nslots, bad, o1.size(), changed, cudaGetErrorString(le), cudaGetErrorString(se));
  printf("IMAD k_update_tiled %.3f ms (%.2f Tprod/s)   TC k_update_tc %.3f ms (%.2f Tprod/s)   speed-up %.2fx\n",
         best_i, prods / best_i / 1e9, best_t, prods / best_t / 1e9, best_i / best_t);
  return bad != 0;
}
