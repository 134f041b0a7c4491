// Fixed-order per-n-plet kernels, orders 1..12 (see eval_kernels.cuh).
#include "eval_kernels.cuh"

namespace hoib {

int launch_eval_k1_12(const EvalArgs &A, int K, cudaStream_t s) {
  upload_binomials();
  switch (K) {
    case 1:
      return launch_one<1, true, true, true>(A, K, s);
    case 2:
      return launch_one<2, true, true, true>(A, K, s);
    case 3:
      return launch_one<3, true, true, true>(A, K, s);
    case 4:
      return launch_one<4, true, true, true>(A, K, s);
    case 5:
      return launch_one<5, true, true, true>(A, K, s);
    case 6:
      return launch_one<6, true, true, true>(A, K, s);
    case 7:
      return launch_one<7, true, true, true>(A, K, s);
    case 8:
      return launch_one<8, true, true, true>(A, K, s);
    case 9:
      return launch_one<9, true, true, true>(A, K, s);
    case 10:
      return launch_one<10, true, true, true>(A, K, s);
    case 11:
      return launch_one<11, true, true, true>(A, K, s);
    case 12:
      return launch_one<12, true, true, true>(A, K, s);
    default:
      return -1;
  }
}

}  // namespace hoib
