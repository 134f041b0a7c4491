// Device reducers over full-output planes (ref:scanner.py:50-137).
#include "common.cuh"

namespace hoib {
namespace {

constexpr int kHistSmemBins = 4096;

// numpy.histogram with explicit edges after np.clip(v, lo, hi): bin i counts
// e_i <= x < e_{i+1}, the last bin is closed; NaN is dropped
// (searchsorted-based path numpy takes for an edge array).
__global__ void k_hist(const double *__restrict__ vals, int64_t n, int D, int bins, double lo,
                       double hi, const double *__restrict__ edges,
                       unsigned long long *__restrict__ counts) {
  extern __shared__ unsigned char smem[];
  double *e = reinterpret_cast<double *>(smem);
  unsigned int *h = reinterpret_cast<unsigned int *>(e + bins + 1);
  const bool local = bins <= kHistSmemBins;
  for (int i = threadIdx.x; i <= bins; i += blockDim.x) e[i] = edges[i];
  if (local)
    for (int i = threadIdx.x; i < bins * D; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t total = n * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double x = vals[t];
    if (x != x) continue;
    x = x < lo ? lo : (x > hi ? hi : x);
    if (x < e[0] || x > e[bins]) continue;
    // number of interior edges e_1..e_{bins-1} that are <= x
    int a = 1, b = bins;  // search in [1, bins)
    while (a < b) {
      int m = (a + b) >> 1;
      if (e[m] <= x) a = m + 1; else b = m;
    }
    int bin = a - 1;
    int d = (int)(t % D);
    if (local)
      atomicAdd(&h[d * bins + bin], 1u);
    else
      atomicAdd(&counts[(int64_t)d * bins + bin], 1ull);
  }
  if (local) {
    __syncthreads();
    for (int i = threadIdx.x; i < bins * D; i += blockDim.x)
      if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
  }
}

__global__ void k_topk_filter(const double *__restrict__ vals, int64_t n, int D, int d,
                              double sign, const double *__restrict__ thresh,
                              int64_t *__restrict__ cand, unsigned long long *__restrict__ count,
                              int64_t cap) {
  const double th = *thresh;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    double v = sign * vals[p * D + d];
    if (v <= th) {
      unsigned long long slot = atomicAdd(count, 1ull);
      if ((int64_t)slot < cap) cand[slot] = p;
    }
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace
}  // namespace hoib

using namespace hoib;

extern "C" int hoi_histogram(const double *vals, int64_t n, int32_t D, int32_t bins, double lo,
                             double hi, const double *edges, int64_t *counts, void *stream) {
  HOI_CHECK_ARG(vals && edges && counts && bins >= 1 && D >= 1 && n >= 0, "hoi_histogram: bad args");
  bool local = bins <= kHistSmemBins && (int64_t)bins * D <= kHistSmemBins * 2;
  size_t shm = sizeof(double) * (bins + 1) + (local ? sizeof(unsigned int) * bins * D : 0);
  if (!local) {
    // force the global-atomics path by passing a bin count the kernel treats as non-local
  }
  int blocks = 4 * sm_count();
  cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(shm + 1024));
  if (local) {
    k_hist<<<blocks, 256, shm, (cudaStream_t)stream>>>(vals, n, D, bins, lo, hi, edges,
                                                       reinterpret_cast<unsigned long long *>(counts));
  } else {
    return fail(HOI_INVALID_ARG, "hoi_histogram: bins * D too large");
  }
  return check_launch("k_hist");
}

extern "C" int hoi_topk_filter(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                               const double *thresh, int64_t *cand, int64_t *cand_count,
                               int64_t cand_cap, void *stream) {
  HOI_CHECK_ARG(vals && thresh && cand && cand_count && d >= 0 && d < D, "hoi_topk_filter: bad args");
  k_topk_filter<<<8 * sm_count(), 256, 0, (cudaStream_t)stream>>>(
      vals, n, D, d, sign, thresh, cand, reinterpret_cast<unsigned long long *>(cand_count), cand_cap);
  return check_launch("k_topk_filter");
}
