// FP64 pipe peak probe: MEASURED_PEAKS.json carries HBM and bf16 figures
// only, so bench.py measures the DFMA roofline denominator on the same GPU
// in the same run with this kernel (8 independent FMA chains per thread).
#include "common.cuh"

namespace {
__global__ void __launch_bounds__(256) k_fp64_probe(double *out, int64_t iters, double a) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  const double b = 1e-12;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;   // never true; keeps the chains live
}
}  // namespace

// flops = blocks * 256 * iters * 8 * 8 * 2
extern "C" int hoi_fp64_probe(double *out, int64_t iters, int32_t blocks, void *stream) {
  HOI_CHECK_ARG(out && iters > 0 && blocks > 0, "hoi_fp64_probe: bad args");
  k_fp64_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters, 0.999999);
  return hoib::check_launch("k_fp64_probe");
}
