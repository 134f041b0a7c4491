// Engine 1 host side: dispatch, unranking, mask compaction and the C ABI.
// The per-unit kernels live in eval_kernels.cuh (see there).
#include <cstdlib>

#include "eval_kernels.cuh"

namespace hoib {

int launch_eval(const EvalArgs &A, int K, cudaStream_t s) {
  if (K < 1 || K > 64) return fail(HOI_INVALID_ARG, "order > 64 is not supported");
  int st = -1;
  if (K <= 12) {
    st = launch_eval_pipe(A, K, s);            // large-N index batches (gather-pipelined)
    if (st < 0) st = launch_eval_k1_12(A, K, s);
  }
  else if (K <= 16) st = launch_eval_k13_16(A, K, s);
  else if (K <= 32) {
    st = launch_eval_hybrid(A, K, s);          // K <= 23: bordered LDL^T (eval_hybrid.cu)
    if (st < 0) st = launch_eval_group(A, K, s);   // G threads per unit (eval_group.cu)
  }
  return st >= 0 ? st : launch_eval_generic(A, K, s);
}

// ------------------------------------------------------------ unranking --
__global__ void k_unrank(int N, int kmin, int kmax, int64_t g0, int64_t count,
                         int32_t *__restrict__ idx_out, int32_t *__restrict__ order_out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  uint64_t g = (uint64_t)(g0 + t);
  int k = kmin;
  while (k < kmax && g >= binom(N, k)) {
    g -= binom(N, k);
    ++k;
  }
  int s[64];
  unrank_lex(g, k, N, s);
  int32_t *row = idx_out + t * kmax;
  for (int i = 0; i < kmax; ++i) row[i] = i < k ? s[i] : -1;
  if (order_out) order_out[t] = k;
}

__global__ void k_unrank_list(int N, int kmin, int kmax, const int64_t *__restrict__ ranks,
                              int64_t count, int32_t *__restrict__ idx_out,
                              int32_t *__restrict__ order_out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  uint64_t g = (uint64_t)ranks[t];
  int k = kmin;
  while (k < kmax && g >= binom(N, k)) {
    g -= binom(N, k);
    ++k;
  }
  int s[64];
  unrank_lex(g, k, N, s);
  int32_t *row = idx_out + t * kmax;
  for (int i = 0; i < kmax; ++i) row[i] = i < k ? s[i] : -1;
  if (order_out) order_out[t] = k;
}

// -------------------------------------------------------- mask compaction --
// Rows are bucketed by order (popcount over W words); the per-order
// kernels take orders <= 64, so orders above land in the last bucket and
// are refused.
constexpr int kMaskOrders = 72;
__global__ void k_mask_orders(const uint64_t *__restrict__ masks, int W, int64_t B,
                              int32_t *__restrict__ order, int32_t *__restrict__ hist) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  int k = 0;
  for (int w = 0; w < W; ++w) k += __popcll(masks[b * W + w]);
  order[b] = k;
  atomicAdd(&hist[k < kMaskOrders - 1 ? k : kMaskOrders - 1], 1);   // last slot: order > 64
}

__global__ void k_mask_scatter(const uint64_t *__restrict__ masks, int W, int N, int64_t B,
                               const int32_t *__restrict__ order, int32_t *__restrict__ cursor,
                               int32_t *__restrict__ idx_sorted, int64_t *__restrict__ row_map) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  int k = order[b];
  int pos = atomicAdd(&cursor[k], 1);
  int32_t *row = idx_sorted + (int64_t)pos * N;
  int c = 0;
  for (int w = 0; w < W; ++w) {
    uint64_t m = masks[b * W + w];
    while (m) {
      int bit = __ffsll((long long)m) - 1;
      row[c++] = w * 64 + bit;
      m &= m - 1;
    }
  }
  row_map[pos] = b;
}

}  // namespace hoib

using namespace hoib;

extern "C" int hoi_eval_indices(const double *corr, const double *sdiag, const double *eta,
                                int32_t kstride, int32_t N, int32_t D, const int32_t *idx,
                                int64_t B, int32_t K, double *out, double *logdet,
                                double *invdiag, int32_t *err_count, int64_t *err_coords,
                                int32_t err_cap, void *stream) {
  HOI_CHECK_ARG(corr && idx && err_count && N >= 1 && D >= 1 && B >= 0, "hoi_eval_indices: bad args");
  HOI_CHECK_ARG(K >= 1 && K <= 64 && K <= N, "hoi_eval_indices: bad order");
  HOI_CHECK_ARG(!eta || kstride > K, "hoi_eval_indices: bias table too short");
  EvalArgs A{};
  A.src = corr; A.sdiag = sdiag; A.eta = eta; A.kstride = kstride;
  A.N = N; A.D = D; A.mats = 0; A.idx = idx; A.idx_stride = K; A.row_map = nullptr;
  A.B = B; A.r0 = 0; A.out = out; A.plane = B * (int64_t)D; A.out_row0 = 0;
  A.logdet = logdet; A.invdiag = invdiag; A.inv_n = 0;
  A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
  return launch_eval(A, K, (cudaStream_t)stream);
}

extern "C" int hoi_eval_indices_into(const double *corr, const double *sdiag, const double *eta,
                                     int32_t kstride, int32_t N, int32_t D, const int32_t *idx,
                                     int64_t B, int32_t K, double *out, int64_t out_plane,
                                     int32_t *err_count, int64_t *err_coords, int32_t err_cap,
                                     void *stream) {
  HOI_CHECK_ARG(corr && idx && out && err_count && N >= 1 && D >= 1 && B >= 0 &&
                    out_plane >= B * (int64_t)D,
                "hoi_eval_indices_into: bad args");
  HOI_CHECK_ARG(K >= 1 && K <= 64 && K <= N, "hoi_eval_indices_into: bad order");
  HOI_CHECK_ARG(!eta || kstride > K, "hoi_eval_indices_into: bias table too short");
  EvalArgs A{};
  A.src = corr; A.sdiag = sdiag; A.eta = eta; A.kstride = kstride;
  A.N = N; A.D = D; A.mats = 0; A.idx = idx; A.idx_stride = K; A.row_map = nullptr;
  A.B = B; A.r0 = 0; A.out = out; A.plane = out_plane; A.out_row0 = 0;
  A.logdet = nullptr; A.invdiag = nullptr; A.inv_n = 0;
  A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
  return launch_eval(A, K, (cudaStream_t)stream);
}

extern "C" int hoi_eval_indices_fp32(const double *corr, const float *corr32,
                                     const double *sdiag, const double *eta, int32_t kstride,
                                     int32_t N, int32_t D, const int32_t *idx, int64_t B,
                                     int32_t K, double *out, int32_t *err_count,
                                     int64_t *err_coords, int32_t err_cap, void *stream) {
  HOI_CHECK_ARG(corr && corr32 && idx && err_count && out && N >= 1 && D >= 1 && B >= 0,
                "hoi_eval_indices_fp32: bad args");
  HOI_CHECK_ARG(K >= 1 && K <= 64 && K <= N, "hoi_eval_indices_fp32: bad order");
  HOI_CHECK_ARG(!eta || kstride > K, "hoi_eval_indices_fp32: bias table too short");
  EvalArgs A{};
  A.src = corr; A.src32 = corr32; A.fp32 = 1; A.sdiag = sdiag; A.eta = eta; A.kstride = kstride;
  A.N = N; A.D = D; A.mats = 0; A.idx = idx; A.idx_stride = K; A.row_map = nullptr;
  A.B = B; A.r0 = 0; A.out = out; A.plane = B * (int64_t)D; A.out_row0 = 0;
  A.logdet = nullptr; A.invdiag = nullptr; A.inv_n = 0;
  A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
  return launch_eval(A, K, (cudaStream_t)stream);
}

extern "C" int hoi_logdet_invdiag(const double *mats, int64_t M, int32_t K, double *logdet,
                                  double *invdiag, int32_t *err_count, int64_t *err_coords,
                                  int32_t err_cap, void *stream) {
  HOI_CHECK_ARG(mats && err_count && K >= 1 && K <= 64 && M >= 0, "hoi_logdet_invdiag: bad args");
  EvalArgs A{};
  A.src = mats; A.sdiag = nullptr; A.eta = nullptr; A.kstride = 0;
  A.N = K; A.D = 1; A.mats = 1; A.idx = nullptr; A.idx_stride = 0; A.row_map = nullptr;
  A.B = M; A.r0 = 0; A.out = nullptr; A.plane = M; A.out_row0 = 0;
  A.logdet = logdet; A.invdiag = invdiag; A.inv_n = 0;
  A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
  return launch_eval(A, K, (cudaStream_t)stream);
}

extern "C" int hoi_eval_masks(const double *corr, const double *sdiag, const double *eta,
                              int32_t kstride, int32_t N, int32_t D, const uint64_t *masks,
                              int32_t W, int64_t B, double *out, double *logdet,
                              double *invdiag, int32_t *err_count, int64_t *err_coords,
                              int32_t err_cap, void *stream) {
  HOI_CHECK_ARG(corr && masks && err_count && N >= 1 && N <= 64 * W && D >= 1,
                "hoi_eval_masks: bad args");
  if (B == 0) return HOI_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // compaction workspace (stream-ordered allocation; mask batches are not
  // the exhaustive hot path)
  int32_t *order = nullptr, *hist = nullptr, *idx_sorted = nullptr;
  int64_t *row_map = nullptr;
  size_t bytes = sizeof(int32_t) * (B + 2 * 72) + sizeof(int32_t) * B * N + sizeof(int64_t) * B;
  char *ws = nullptr;
  if (stream_alloc((void **)&ws, bytes + 64, s) != cudaSuccess)
    return fail(HOI_CUDA_ERROR, "hoi_eval_masks: allocation failed");
  row_map = reinterpret_cast<int64_t *>(ws);
  order = reinterpret_cast<int32_t *>(row_map + B);
  hist = order + B;
  int32_t *cursor = hist + 72;
  idx_sorted = cursor + 72;
  cudaMemsetAsync(hist, 0, sizeof(int32_t) * 144, s);
  int st = HOI_OK;
  k_mask_orders<<<grid_for(B, 256), 256, 0, s>>>(masks, W, B, order, hist);
  if ((st = check_launch("k_mask_orders"))) goto done;
  {
    int32_t h[72];
    cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (h[0] != 0) {
      st = fail(HOI_INVALID_ARG, "hoi_eval_masks: empty mask row");
      goto done;
    }
    for (int k = 65; k < kMaskOrders; ++k)
      if (h[k] != 0) {
        st = fail(HOI_INVALID_ARG, "hoi_eval_masks: mask rows of order > 64 are not supported");
        goto done;
      }
    int32_t off[72];
    int acc = 0;
    for (int k = 0; k < 72; ++k) { off[k] = acc; acc += h[k]; }
    cudaMemcpyAsync(cursor, off, sizeof(off), cudaMemcpyHostToDevice, s);
    k_mask_scatter<<<grid_for(B, 256), 256, 0, s>>>(masks, W, N, B, order, cursor, idx_sorted, row_map);
    if ((st = check_launch("k_mask_scatter"))) goto done;
    for (int k = 1; k <= N && k <= 64 && !st; ++k) {
      if (h[k] == 0) continue;
      HOI_CHECK_ARG(!eta || kstride > k, "hoi_eval_masks: bias table too short");
      EvalArgs A{};
      A.src = corr; A.sdiag = sdiag; A.eta = eta; A.kstride = kstride;
      A.N = N; A.D = D; A.mats = 0; A.idx = idx_sorted + (int64_t)off[k] * N; A.idx_stride = N;
      A.row_map = row_map + off[k]; A.B = h[k]; A.r0 = 0; A.out = out; A.plane = B * (int64_t)D;
      A.out_row0 = 0; A.logdet = logdet; A.invdiag = invdiag; A.inv_n = N;
      A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
      st = launch_eval(A, k, s);
    }
  }
done:
  cudaFreeAsync(ws, s);
  return st;
}

extern "C" int hoi_unrank(int32_t N, int32_t kmin, int32_t kmax, int64_t g_begin, int64_t count,
                          int32_t *idx_out, int32_t *order_out, void *stream) {
  HOI_CHECK_ARG(N >= 1 && N <= 64 && kmin >= 1 && kmin <= kmax && kmax <= N && idx_out,
                "hoi_unrank: bad args");
  upload_binomials();
  k_unrank<<<grid_for(count, 128), 128, 0, (cudaStream_t)stream>>>(N, kmin, kmax, g_begin, count,
                                                                   idx_out, order_out);
  return check_launch("k_unrank");
}

extern "C" int hoi_unrank_list(int32_t N, int32_t kmin, int32_t kmax, const int64_t *ranks,
                               int64_t count, int32_t *idx_out, int32_t *order_out, void *stream) {
  HOI_CHECK_ARG(N >= 1 && N <= 64 && kmin >= 1 && kmin <= kmax && kmax <= N && idx_out && ranks,
                "hoi_unrank_list: bad args");
  if (count == 0) return HOI_OK;
  upload_binomials();
  k_unrank_list<<<grid_for(count, 128), 128, 0, (cudaStream_t)stream>>>(N, kmin, kmax, ranks, count,
                                                                         idx_out, order_out);
  return check_launch("k_unrank_list");
}

namespace hoib {
// Engine 1 over a global rank range: one launch per order segment.
int scan_full_percell(const double *corr, const double *sdiag, const double *eta, int kstride,
                      int N, int D, int kmin, int kmax, int64_t g_begin, int64_t g_end,
                      double *out, int32_t *err_count, int64_t *err_coords, int err_cap,
                      cudaStream_t s) {
  upload_binomials();
  int64_t off = 0;
  const int64_t plane = (g_end - g_begin) * (int64_t)D;
  for (int k = kmin; k <= kmax; ++k) {
    int64_t c = (int64_t)host_binom(N, k);
    int64_t lo = off > g_begin ? off : g_begin;
    int64_t hi = (off + c) < g_end ? (off + c) : g_end;
    if (lo < hi) {
      EvalArgs A{};
      A.src = corr; A.sdiag = sdiag; A.eta = eta; A.kstride = kstride;
      A.N = N; A.D = D; A.mats = 0; A.idx = nullptr; A.idx_stride = 0; A.row_map = nullptr;
      A.B = hi - lo; A.r0 = (uint64_t)(lo - off); A.out = out; A.plane = plane;
      A.out_row0 = lo - g_begin; A.logdet = nullptr; A.invdiag = nullptr; A.inv_n = 0;
      A.err_count = err_count; A.err_coords = err_coords; A.err_cap = err_cap;
      int st = launch_eval(A, k, s);
      if (st) return st;
    }
    off += c;
  }
  return HOI_OK;
}
}  // namespace hoib
