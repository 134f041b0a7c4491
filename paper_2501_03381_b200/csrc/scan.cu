// hoi_scan_full: engine selection for exhaustive full-output scans.
#include "common.cuh"

namespace hoib {
int scan_full_percell(const double *corr, const double *sdiag, const double *eta, int kstride,
                      int N, int D, int kmin, int kmax, int64_t g_begin, int64_t g_end,
                      double *out, int32_t *err_count, int64_t *err_coords, int err_cap,
                      cudaStream_t s);
int lattice_ws_bytes(int N, int D, size_t *bytes);
bool lattice_available();
bool lattice_supports(int N);
int scan_full_lattice(const double *corr, const double *eta, int kstride, int N, int D, int kmin,
                      int kmax, int64_t g_begin, int64_t g_end, double *out, int32_t *err_count,
                      void *ws, size_t ws_bytes, cudaStream_t s);
}  // namespace hoib

using namespace hoib;

extern "C" int hoi_scan_full(const double *corr, const double *sdiag, const double *eta,
                             int32_t kstride, int32_t N, int32_t D, int32_t kmin, int32_t kmax,
                             int64_t g_begin, int64_t g_end, int32_t engine, double *out,
                             int32_t *err_count, int64_t *err_coords, int32_t err_cap, void *ws,
                             size_t *ws_bytes, void *stream) {
  HOI_CHECK_ARG(N >= 1 && N <= 64 && D >= 1 && kmin >= 1 && kmin <= kmax && kmax <= N,
                "hoi_scan_full: bad order range");
  uint64_t total = 0;
  for (int k = kmin; k <= kmax; ++k) {
    uint64_t c = host_binom(N, k);
    HOI_CHECK_ARG(c != UINT64_MAX && total + c >= total, "hoi_scan_full: n-plet count overflows");
    total += c;
  }
  HOI_CHECK_ARG(g_begin >= 0 && g_begin <= g_end && (uint64_t)g_end <= total,
                "hoi_scan_full: bad rank range");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_scan_full: bias table too short");
  if (engine == 0) engine = lattice_available() && lattice_supports(N) ? 2 : 1;
  HOI_CHECK_ARG(engine >= 0 && engine <= 2, "hoi_scan_full: engine must be 0 (auto), 1 or 2");
  if (engine == 2) {
    size_t need = 0;
    int st = lattice_ws_bytes(N, D, &need);
    if (st) return st;
    if (ws == nullptr) {
      HOI_CHECK_ARG(ws_bytes != nullptr, "hoi_scan_full: ws_bytes is NULL");
      *ws_bytes = need;
      return HOI_OK;
    }
    if (!ws_bytes || *ws_bytes < need) return fail(HOI_CAPACITY, "hoi_scan_full: workspace too small");
    HOI_CHECK_ARG(corr && out && err_count, "hoi_scan_full: null pointer");
    return scan_full_lattice(corr, eta, kstride, N, D, kmin, kmax, g_begin, g_end, out, err_count,
                             ws, *ws_bytes, (cudaStream_t)stream);
  }
  if (ws == nullptr && ws_bytes) {
    *ws_bytes = 0;
    return HOI_OK;
  }
  HOI_CHECK_ARG(corr && out && err_count, "hoi_scan_full: null pointer");
  return scan_full_percell(corr, sdiag, eta, kstride, N, D, kmin, kmax, g_begin, g_end, out,
                           err_count, err_coords, err_cap, (cudaStream_t)stream);
}
