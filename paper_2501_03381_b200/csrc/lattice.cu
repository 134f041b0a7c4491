// Engine 2: subset-lattice engine for exhaustive scans (placeholder until
// the lattice kernels land; hoi_scan_full falls back to engine 1).
#include "common.cuh"

namespace hoib {
int lattice_ws_bytes(int N, int D, size_t *bytes) {
  (void)N; (void)D;
  *bytes = 0;
  return fail(HOI_INVALID_ARG, "lattice engine not built yet");
}
int scan_full_lattice(const double *, const double *, int, int, int, int, int, int64_t, int64_t,
                      double *, int32_t *, void *, size_t, cudaStream_t) {
  return fail(HOI_INVALID_ARG, "lattice engine not built yet");
}
}  // namespace hoib
namespace hoib {
bool lattice_available() { return false; }
}
