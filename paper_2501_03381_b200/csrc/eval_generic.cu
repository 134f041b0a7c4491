// Runtime-order per-n-plet kernels (orders without a fixed instantiation,
// K <= 64; local-memory triangle).
#include "eval_kernels.cuh"

namespace hoib {

int launch_eval_generic(const EvalArgs &A, int K, cudaStream_t s) {
  upload_binomials();
  if (K <= 16) return launch_one<16, false>(A, K, s);
  if (K <= 24) return launch_one<24, false>(A, K, s);
  if (K <= 32) return launch_one<32, false>(A, K, s);
  if (K <= 48) return launch_one<48, false>(A, K, s);
  return launch_one<64, false>(A, K, s);
}

}  // namespace hoib
