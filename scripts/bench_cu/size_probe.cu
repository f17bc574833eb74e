#include "../../paper_0902_0852_b200/csrc/ldlt_kernels.cu"
using namespace hgpu;
__global__ void __launch_bounds__(512) k_rf_only(DevPlan P, IntBuf vint, long long prow, const int* maxbitsV, int p,
                          IntBuf piv, int dmax_bits, uint32_t* Ybuf, int* ys, int* err) {
  extern __shared__ uint32_t sm_dyn[];
  recip_fast_body(P, vint, prow, maxbitsV, p, piv, dmax_bits, Ybuf, ys, sm_dyn, err);
}
__global__ void __launch_bounds__(512) k_old_only(DevPlan P, IntBuf vint, long long prow, const int* maxbitsV, int p,
                          IntBuf piv, int dmax_bits, uint32_t* Ybuf, int* ys, int* err) {
  recip_body(P, vint, prow, maxbitsV, p, piv, dmax_bits, Ybuf, ys, nullptr, 0, err, 0);
}
