// Fixed-order per-n-plet kernels, orders 13..16 (see eval_kernels.cuh).
#include "eval_kernels.cuh"

namespace hoib {

int launch_eval_k13_16(const EvalArgs &A, int K, cudaStream_t s) {
  upload_binomials();
  switch (K) {
    case 13:
      return launch_one<13, true, true, true>(A, K, s);
    case 14:
      return launch_one<14, true, true, true>(A, K, s);
    case 15:
      return launch_one<15, true, true, true>(A, K, s);
    case 16:
      return launch_one<16, true, true, true>(A, K, s);
    default:
      return -1;
  }
}

}  // namespace hoib
