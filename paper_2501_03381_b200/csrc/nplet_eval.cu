// Engine 1: per-(n-plet, dataset) evaluation.
//
// One thread owns one (n-plet, dataset) unit.  For K <= kMaxRegK the K x K
// packed lower triangle lives in registers (K is a template parameter and
// every loop is fully unrolled, so all indices are compile-time); larger K
// use the same code with a runtime K (local memory).
//
// Per unit:  gather R_S from the L2-resident correlation matrix (dataset
// index fastest, so the D units of one n-plet read one cache line) ->
// square-root-free LDL^T (log det = sum log d_j) -> in-place inverse of the
// unit lower factor U = L^-1 -> inverse diagonal (R_S^-1)_jj =
// sum_i U_ij^2 / d_i (every leave-one-out determinant is
// det(R_S) * (R_S^-1)_jj, ref:nplet_engine.py:267-273) -> fused epilogue
// writing only tc, dtc, o, s (ref:measures.py:41-81).
//
// In the correlation form the per-variable log Sigma_jj terms cancel from
// every measure, so with l = log det R_S and lam = sum_j log (R_S^-1)_jj:
//   tc  = -l/2                 - k*eta1 + eta_k
//   dtc = (l + lam)/2          + (k-1)*eta_k - k*eta_{k-1}
//   o   = -l - lam/2           - k*eta1 - (k-2)*eta_k + k*eta_{k-1}
//   s   = tc + dtc
// (eta = finite-sample bias, ref:nplet_engine.py:295-321).
//
// Failure handling mirrors ref:nplet_engine.py:237-264: a non-positive (or
// NaN) pivot triggers one retry of that matrix with Sigma_S + eps*I,
// eps = 1e-10 * trace(Sigma_S) / k; a second failure records (row, dataset).
#include "common.cuh"

namespace hoib {

constexpr int kMaxRegK = 12;

struct EvalArgs {
  const double *src;       // corr (N,N,D)  or matrix stack (M,K,K) when mats
  const double *sdiag;     // (D,N) covariance diagonal or nullptr
  const double *eta;       // (D,kstride) or nullptr
  int kstride;
  int N, D;
  int mats;                // 1: raw matrix stack mode
  const int32_t *idx;      // (B, idx_stride) or nullptr -> unrank
  int64_t idx_stride;
  const int64_t *row_map;  // output row of input row b, or nullptr
  int64_t B;
  uint64_t r0;             // unrank: local lexicographic rank of row 0
  double *out;             // 4 planes, plane stride `plane`
  int64_t plane;
  int64_t out_row0;
  double *logdet;          // (rows, D) or nullptr
  double *invdiag;         // (rows, D, K) or scattered (rows, D, inv_n)
  int inv_n;               // 0: dense K layout, >0: scatter by variable id
  int32_t *err_count;
  int64_t *err_coords;
  int err_cap;
};

#define TRI(i, j) ((i) * ((i) + 1) / 2 + (j))

__device__ __forceinline__ void unrank_lex(uint64_t r, int K, int N, int *s) {
  int c = 0;
  for (int p = 0; p < K; ++p) {
    while (c < N) {
      uint64_t b = binom(N - 1 - c, K - 1 - p);
      if (b <= r) {
        r -= b;
        ++c;
      } else {
        break;
      }
    }
    s[p] = c++;
  }
}

template <int KT, bool FIXED>
__device__ __forceinline__ void load_matrix(const EvalArgs &A, int64_t b, int d, int K,
                                            const int (&s)[KT], double (&a)[KT * (KT + 1) / 2],
                                            bool jitter) {
  if (A.mats) {
    const double *m = A.src + (int64_t)b * K * K;
    double tr = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j <= i; ++j) a[TRI(i, j)] = m[i * K + j];
      tr += m[i * K + i];
    }
    if (jitter) {
      double eps = 1e-10 * tr / (double)K;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        a[TRI(i, i)] += eps;
      }
    }
    return;
  }
  const int N = A.N, D = A.D;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const double *row = A.src + ((int64_t)s[i] * N) * D + d;
#pragma unroll
    for (int j = 0; j <= i; ++j) a[TRI(i, j)] = __ldg(row + (int64_t)s[j] * D);
  }
  if (jitter) {
    double tr = 0.0;
    if (A.sdiag) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        tr += A.sdiag[(int64_t)d * N + s[i]];
      }
    } else {
      tr = (double)K;
    }
    double eps = 1e-10 * tr / (double)K;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      double sc = A.sdiag ? A.sdiag[(int64_t)d * N + s[i]] : 1.0;
      a[TRI(i, i)] += eps / sc;
    }
  }
}

// LDL^T + unit-triangular inverse + inverse diagonal.  Returns false on a
// non-positive / NaN pivot.  cs[j] = (M^-1)_jj; l = log det M; lam = sum log cs.
template <int KT, bool FIXED>
__device__ __forceinline__ bool ldl_invdiag(double (&a)[KT * (KT + 1) / 2], int K,
                                            double (&cs)[KT], double &l, double &lam) {
  double dinv[KT];
  double col[KT];
  LogProd pd;
  pd.init();
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double dj = a[TRI(j, j)];
    if (!(dj > 0.0)) return false;
    pd.mul(dj);
    if ((j & 7) == 7) pd.renorm();
    double r = 1.0 / dj;
    dinv[j] = r;
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      col[i] = a[TRI(i, j)];
      a[TRI(i, j)] = col[i] * r;
    }
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double lij = a[TRI(i, j)];
#pragma unroll
      for (int m = j + 1; m <= i; ++m) a[TRI(i, m)] = fma(-lij, col[m], a[TRI(i, m)]);
    }
  }
  pd.renorm();
  // U = L^-1 (unit lower), column by column, in place.
#pragma unroll
  for (int j = 0; j < K; ++j) {
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double acc = a[TRI(i, j)];
#pragma unroll
      for (int m = j + 1; m < i; ++m) acc = fma(a[TRI(i, m)], a[TRI(m, j)], acc);
      a[TRI(i, j)] = -acc;
    }
  }
  LogProd pl;
  pl.init();
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double sacc = dinv[j];
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double u = a[TRI(i, j)];
      sacc = fma(u * u, dinv[i], sacc);
    }
    cs[j] = sacc;
    pl.mul(sacc);
    if ((j & 7) == 7) pl.renorm();
  }
  pl.renorm();
  l = pd.log_value();
  lam = pl.log_value();
  return true;
}

template <int KT, bool FIXED>
__device__ __forceinline__ void eval_unit(const EvalArgs &A, int64_t b, int d, int kdyn) {
  const int K = FIXED ? KT : kdyn;
  int s[KT];
  if (!A.mats) {
    if (A.idx) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        s[i] = A.idx[b * A.idx_stride + i];
      }
    } else {
      unrank_lex(A.r0 + (uint64_t)b, K, A.N, s);
    }
  }
  double a[KT * (KT + 1) / 2];
  double cs[KT];
  double l = 0.0, lam = 0.0;
  load_matrix<KT, FIXED>(A, b, d, K, s, a, false);
  bool ok = ldl_invdiag<KT, FIXED>(a, K, cs, l, lam);
  if (!ok) {
    load_matrix<KT, FIXED>(A, b, d, K, s, a, true);
    ok = ldl_invdiag<KT, FIXED>(a, K, cs, l, lam);
  }
  const int64_t ob = A.row_map ? A.row_map[b] : A.out_row0 + b;
  const int64_t o = ob * A.D + d;
  if (!ok) {
    int slot = atomicAdd(A.err_count, 1);
    if (slot < A.err_cap) {
      A.err_coords[2 * slot] = ob;
      A.err_coords[2 * slot + 1] = d;
    }
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    if (A.out) {
#pragma unroll
      for (int q = 0; q < 4; ++q) A.out[q * A.plane + o] = nan;
    }
    if (A.logdet) A.logdet[o] = nan;
    return;
  }
  if (A.out) {
    double tc, dtc, oi;
    const double kd = (double)K;
    if (A.eta) {
      const double *e = A.eta + (int64_t)d * A.kstride;
      const double e1 = e[1], ek = e[K], ek1 = e[K - 1];
      tc = -0.5 * l - kd * e1 + ek;
      dtc = 0.5 * (l + lam) + (kd - 1.0) * ek - kd * ek1;
      oi = -l - 0.5 * lam - kd * e1 - (kd - 2.0) * ek + kd * ek1;
    } else {
      tc = -0.5 * l;
      dtc = 0.5 * (l + lam);
      oi = -l - 0.5 * lam;
    }
    A.out[o] = tc;
    A.out[A.plane + o] = dtc;
    A.out[2 * A.plane + o] = oi;
    A.out[3 * A.plane + o] = tc + dtc;
  }
  if (A.logdet || A.invdiag) {
    // Sigma-space values (entropy_terms compat): log det Sigma_S =
    // l + sum log sigma_j, (Sigma_S^-1)_jj = (R_S^-1)_jj / sigma_j.
    double ld = l;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double sg = (!A.mats && A.sdiag) ? A.sdiag[(int64_t)d * A.N + s[j]] : 1.0;
      if (!A.mats && A.sdiag) ld += log(sg);
      if (A.invdiag) {
        double v = cs[j] / sg;
        if (A.inv_n > 0)
          A.invdiag[o * A.inv_n + s[j]] = v;
        else
          A.invdiag[o * K + j] = v;
      }
    }
    if (A.logdet) A.logdet[o] = ld;
  }
}

template <int KT, bool FIXED>
__global__ void __launch_bounds__(128) k_eval(const EvalArgs A, int kdyn) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= A.B * A.D) return;
  const int64_t b = t / A.D;
  const int d = (int)(t - b * A.D);
  eval_unit<KT, FIXED>(A, b, d, kdyn);
}

template <int KT, bool FIXED>
static int launch_one(const EvalArgs &A, int K, cudaStream_t s) {
  int64_t n = A.B * (int64_t)A.D;
  if (n == 0) return HOI_OK;
  k_eval<KT, FIXED><<<grid_for(n, 128), 128, 0, s>>>(A, K);
  return check_launch("k_eval");
}

int launch_eval(const EvalArgs &A, int K, cudaStream_t s) {
  switch (K) {
#define HOI_CASE(k) \
  case k:           \
    return launch_one<k, true>(A, K, s);
    HOI_CASE(1) HOI_CASE(2) HOI_CASE(3) HOI_CASE(4) HOI_CASE(5) HOI_CASE(6)
    HOI_CASE(7) HOI_CASE(8) HOI_CASE(9) HOI_CASE(10) HOI_CASE(11) HOI_CASE(12)
#undef HOI_CASE
    default:
      break;
  }
  if (K <= 16) return launch_one<16, false>(A, K, s);
  if (K <= 24) return launch_one<24, false>(A, K, s);
  if (K <= 32) return launch_one<32, false>(A, K, s);
  if (K <= 48) return launch_one<48, false>(A, K, s);
  if (K <= 64) return launch_one<64, false>(A, K, s);
  return fail(HOI_INVALID_ARG, "order > 64 is not supported");
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
__global__ void k_mask_orders(const uint64_t *__restrict__ masks, int W, int64_t B,
                              int32_t *__restrict__ order, int32_t *__restrict__ hist) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  int k = 0;
  for (int w = 0; w < W; ++w) k += __popcll(masks[b * W + w]);
  order[b] = k;
  atomicAdd(&hist[k], 1);
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
  HOI_CHECK_ARG(N <= 64, "hoi_eval_masks: N > 64 is not supported");
  if (B == 0) return HOI_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // compaction workspace (stream-ordered allocation; mask batches are not
  // the exhaustive hot path)
  int32_t *order = nullptr, *hist = nullptr, *idx_sorted = nullptr;
  int64_t *row_map = nullptr;
  size_t bytes = sizeof(int32_t) * (B + 2 * 72) + sizeof(int32_t) * B * N + sizeof(int64_t) * B;
  char *ws = nullptr;
  if (cudaMallocAsync((void **)&ws, bytes + 64, s) != cudaSuccess)
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
    int32_t off[72];
    int acc = 0;
    for (int k = 0; k < 72; ++k) { off[k] = acc; acc += h[k]; }
    cudaMemcpyAsync(cursor, off, sizeof(off), cudaMemcpyHostToDevice, s);
    k_mask_scatter<<<grid_for(B, 256), 256, 0, s>>>(masks, W, N, B, order, cursor, idx_sorted, row_map);
    if ((st = check_launch("k_mask_scatter"))) goto done;
    for (int k = 1; k <= N && !st; ++k) {
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
