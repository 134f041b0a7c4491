// Host-side helpers: thread-local error string, launch counter, binomials.
#include "common.cuh"

#include <mutex>
#include <vector>

namespace hoib {

static thread_local std::string t_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { t_err = msg; }

int fail(int code, const std::string &msg) {
  t_err = msg;
  return code;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HOI_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
  return HOI_OK;
}

uint64_t host_binom(int n, int m) {
  if (m < 0 || n < 0 || m > n) return 0;
  // Pascal with saturation
  static std::vector<uint64_t> tab;
  static std::once_flag once;
  std::call_once(once, [] {
    tab.assign(kBinomN * kBinomN, 0);
    for (int i = 0; i < kBinomN; ++i) {
      tab[i * kBinomN] = 1;
      for (int j = 1; j <= i; ++j) {
        uint64_t a = tab[(i - 1) * kBinomN + j - 1];
        uint64_t b = (j <= i - 1) ? tab[(i - 1) * kBinomN + j] : 0;
        uint64_t s = a + b;
        tab[i * kBinomN + j] = (s < a || a == UINT64_MAX || b == UINT64_MAX) ? UINT64_MAX : s;
      }
    }
  });
  return tab[n * kBinomN + m];
}

void fill_binomials(uint64_t *h) {
  for (int n = 0; n < kBinomN; ++n)
    for (int m = 0; m < kBinomN; ++m) h[n * kBinomN + m] = host_binom(n, m);
}

}  // namespace hoib

extern "C" {

int hoi_version(void) { return 100; }

const char *hoi_last_error(void) { return hoib::t_err.c_str(); }

int64_t hoi_launch_count(void) { return hoib::g_launches.load(); }

}
