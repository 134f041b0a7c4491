// Gaussian copula (per-column stable rank -> normal quantile grid) and the
// FP64 covariance / correlation forms.
//
// Reference behaviour: rank_columns / copula_transform / estimate_covariance
// (ref:copula_core.py:155-189).  Ranks are ordinal with ties broken by row
// (scipy rankdata method='ordinal'), z = ndtri(rank / (T + 1)) -- the grid
// is computed on the host with scipy so z is bit-identical to the reference.
#include "common.cuh"

#include <algorithm>

namespace hoib {
namespace {

constexpr int kSortThreads = 1024;
constexpr int kMaxChunk = 8192;   // 8192 * (8 + 4) B = 96 KB of shared memory

__device__ __forceinline__ bool before(uint64_t ka, int ra, uint64_t kb, int rb) {
  return ka < kb || (ka == kb && ra < rb);
}

// One CTA sorts one chunk of one column by (value, row): bitonic network in
// shared memory.  When the column fits a single chunk the sorted position is
// the final 0-based rank and z is written directly; otherwise the sorted
// chunk is stored for the merge-rank pass.
__global__ void __launch_bounds__(kSortThreads)
k_rank_chunk(const double *__restrict__ x, int64_t T, int N, int chunk, int pad,
             const double *__restrict__ qgrid, int64_t *__restrict__ ranks,
             double *__restrict__ z, uint64_t *__restrict__ ws_keys,
             int *__restrict__ ws_rows) {
  extern __shared__ unsigned char smem[];
  uint64_t *key = reinterpret_cast<uint64_t *>(smem);
  int *row = reinterpret_cast<int *>(key + pad);
  const int col = blockIdx.x;                 // d * N + j
  const int d = col / N, j = col - d * N;
  const int c = blockIdx.y;
  const int64_t t0 = (int64_t)c * chunk;
  const int n_here = (int)((int64_t)chunk < T - t0 ? (int64_t)chunk : T - t0);
  const double *xc = x + (int64_t)d * T * N + j;
  for (int i = threadIdx.x; i < pad; i += blockDim.x) {
    if (i < n_here) {
      key[i] = orderable_key(xc[(t0 + i) * N]);
      row[i] = (int)(t0 + i);
    } else {
      key[i] = ~0ull;
      row[i] = 0x7fffffff;
    }
  }
  __syncthreads();
  for (int size = 2; size <= pad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < pad; i += blockDim.x) {
        int p = i ^ stride;
        if (p > i) {
          bool up = (i & size) == 0;
          uint64_t ki = key[i], kp = key[p];
          int ri = row[i], rp = row[p];
          bool swap = up ? before(kp, rp, ki, ri) : before(ki, ri, kp, rp);
          if (swap) {
            key[i] = kp; key[p] = ki;
            row[i] = rp; row[p] = ri;
          }
        }
      }
      __syncthreads();
    }
  }
  if (ws_keys == nullptr) {            // single chunk: final ranks
    for (int i = threadIdx.x; i < n_here; i += blockDim.x) {
      int t = row[i];
      int64_t o = ((int64_t)d * T + t) * N + j;
      if (ranks) ranks[o] = i + 1;
      z[o] = qgrid[i];
    }
  } else {
    int64_t base = (int64_t)col * ((T + chunk - 1) / chunk) * chunk + t0;
    for (int i = threadIdx.x; i < n_here; i += blockDim.x) {
      ws_keys[base + i] = key[i];
      ws_rows[base + i] = row[i];
    }
  }
}

// Merge rank for multi-chunk columns: an element's rank counts, in every
// other sorted chunk, the elements that precede it -- key <= own key in
// earlier chunks (smaller rows), key < own key in later chunks.
__global__ void k_rank_merge(int64_t T, int N, int D, int chunk, int nchunks,
                             const double *__restrict__ qgrid,
                             const uint64_t *__restrict__ ws_keys,
                             const int *__restrict__ ws_rows,
                             int64_t *__restrict__ ranks, double *__restrict__ z) {
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t per_col = (int64_t)nchunks * chunk;
  if (gid >= (int64_t)D * N * per_col) return;
  int64_t col = gid / per_col;
  int64_t within = gid - col * per_col;
  int c = (int)(within / chunk);
  int pos = (int)(within - (int64_t)c * chunk);
  int64_t t0 = (int64_t)c * chunk;
  if (t0 + pos >= T) return;
  const uint64_t *kc = ws_keys + col * per_col;
  uint64_t k = kc[within];
  int64_t r = pos;
  for (int o = 0; o < nchunks; ++o) {
    if (o == c) continue;
    int64_t lo_t = (int64_t)o * chunk;
    int len = (int)((int64_t)chunk < T - lo_t ? (int64_t)chunk : T - lo_t);
    const uint64_t *a = kc + lo_t;
    int lo = 0, hi = len;
    if (o < c) {       // upper_bound
      while (lo < hi) { int m = (lo + hi) >> 1; if (a[m] <= k) lo = m + 1; else hi = m; }
    } else {           // lower_bound
      while (lo < hi) { int m = (lo + hi) >> 1; if (a[m] < k) lo = m + 1; else hi = m; }
    }
    r += lo;
  }
  int d = (int)(col / N), j = (int)(col - (int64_t)d * N);
  int t = ws_rows[col * per_col + within];
  int64_t out = ((int64_t)d * T + t) * N + j;
  if (ranks) ranks[out] = r + 1;
  z[out] = qgrid[r];
}

__global__ void k_col_mean(const double *__restrict__ z, int64_t T, int N, int D,
                           double *__restrict__ mean) {
  // one warp per (d, j)
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= D * N) return;
  int d = w / N, j = w - d * N;
  const double *zc = z + (int64_t)d * T * N + j;
  double s = 0.0;
  for (int64_t t = lane; t < T; t += 32) s += zc[t * N];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) mean[w] = s / (double)T;
}

// X^T X on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): one 32 x 32
// output tile per CTA (upper tiles only), its two 32-sample centred panels
// staged in shared memory; 8 warps x 2 of the 16 8x8 sub-tiles, 8 MMA
// k-steps of 4 samples per panel, FP64 accumulation throughout.  The value
// of (i, j) is written to (i, j) and (j, i), so the covariance is exactly
// symmetric (the reference symmetrises with 0.5 (S + S^T),
// ref:copula_core.py:187-189).
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256)
k_cov(const double *__restrict__ z, const double *__restrict__ mean, int64_t T,
      int N, double *__restrict__ cov) {
  __shared__ double A[32][33];
  __shared__ double B[32][33];
  int nt = (N + 31) / 32;
  int tile = blockIdx.x, d = blockIdx.y;
  // decode upper-triangular tile index
  int ti = 0, rem = tile;
  while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
  int tj = ti + rem;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int lane = tx, warp = ty;
  const double *zd = z + (int64_t)d * T * N;
  const double *md = mean + (int64_t)d * N;
  const int ci = ti * 32 + tx, cj = tj * 32 + tx;
  const double mi = ci < N ? md[ci] : 0.0, mj = cj < N ? md[cj] : 0.0;
  // warp -> sub-tile row block rb, column blocks cb0, cb0 + 1
  const int rb = warp >> 1, cb0 = (warp & 1) * 2;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t t0 = 0; t0 < T; t0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      int64_t t = t0 + r;
      bool ok = t < T;
      A[r][tx] = (ok && ci < N) ? zd[t * N + ci] - mi : 0.0;
      B[r][tx] = (ok && cj < N) ? zd[t * N + cj] - mj : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int r = 4 * kk + (lane & 3);
      const double a = A[r][rb * 8 + (lane >> 2)];                 // A^T fragment (8 x 4, row)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double b = B[r][(cb0 + c) * 8 + (lane >> 2)];        // B fragment (4 x 8, col)
        dmma_8x8x4(acc[c][0], acc[c][1], a, b);
      }
    }
    __syncthreads();
  }
  const double inv = 1.0 / (double)(T - 1);
  double *cd = cov + (int64_t)d * N * N;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = ti * 32 + rb * 8 + (lane >> 2);
      const int j = tj * 32 + (cb0 + c) * 8 + 2 * (lane & 3) + h;
      if (i < N && j < N && (ti < tj || i <= j)) {
        const double v = acc[c][h] * inv;
        cd[(int64_t)i * N + j] = v;
        cd[(int64_t)j * N + i] = v;
      }
    }
  }
}

__global__ void k_corr(const double *__restrict__ cov, int N, int D,
                       double *__restrict__ corr, double *__restrict__ sdiag) {
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)N * N * D;
  if (gid >= total) return;
  int d = (int)(gid % D);
  int64_t ij = gid / D;
  int i = (int)(ij / N), j = (int)(ij - (int64_t)i * N);
  const double *cd = cov + (int64_t)d * N * N;
  double v;
  if (i == j) {
    v = 1.0;
    sdiag[(int64_t)d * N + i] = cd[(int64_t)i * N + i];
  } else {
    double ri = 1.0 / sqrt(cd[(int64_t)i * N + i]);
    double rj = 1.0 / sqrt(cd[(int64_t)j * N + j]);
    double rr = (i < j) ? ri * rj : rj * ri;     // same operand order both ways
    v = cd[(int64_t)i * N + j] * rr;
  }
  corr[gid] = v;
}

}  // namespace
}  // namespace hoib

using namespace hoib;

extern "C" int hoi_rank_copula(const double *x, int64_t T, int32_t N, int32_t D,
                               const double *qgrid, int64_t *ranks, double *z,
                               void *ws, size_t *ws_bytes, void *stream) {
  HOI_CHECK_ARG(T >= 1 && N >= 1 && D >= 1, "hoi_rank_copula: bad shape");
  HOI_CHECK_ARG(T < (int64_t)1 << 31, "hoi_rank_copula: T too large");
  int chunk = kMaxChunk;
  int nchunks = (int)((T + chunk - 1) / chunk);
  if (nchunks == 1) {
    chunk = 1;
    while (chunk < T) chunk <<= 1;
  }
  size_t need = 0;
  if (nchunks > 1) {
    size_t elems = (size_t)D * N * nchunks * chunk;
    need = elems * sizeof(uint64_t) + elems * sizeof(int) + 256;
  }
  if (ws == nullptr) {
    HOI_CHECK_ARG(ws_bytes != nullptr, "hoi_rank_copula: ws_bytes is NULL");
    *ws_bytes = need;
    return HOI_OK;
  }
  if (ws_bytes && *ws_bytes < need) return fail(HOI_CAPACITY, "hoi_rank_copula: workspace too small");
  HOI_CHECK_ARG(x && qgrid && z, "hoi_rank_copula: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  int pad = chunk;
  size_t shm = (size_t)pad * (sizeof(uint64_t) + sizeof(int));
  cudaFuncSetAttribute(k_rank_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  uint64_t *wk = nullptr;
  int *wr = nullptr;
  if (nchunks > 1) {
    size_t elems = (size_t)D * N * nchunks * chunk;
    wk = reinterpret_cast<uint64_t *>(ws);
    wr = reinterpret_cast<int *>(wk + elems);
  }
  dim3 grid((unsigned)(D * N), (unsigned)nchunks);
  int threads = std::min(kSortThreads, std::max(32, pad / 2));
  k_rank_chunk<<<grid, threads, shm, s>>>(x, T, N, chunk, pad, qgrid, ranks, z, wk, wr);
  int st = check_launch("k_rank_chunk");
  if (st) return st;
  if (nchunks > 1) {
    int64_t n = (int64_t)D * N * nchunks * chunk;
    k_rank_merge<<<grid_for(n, 256), 256, 0, s>>>(T, N, D, chunk, nchunks, qgrid, wk, wr, ranks, z);
    st = check_launch("k_rank_merge");
  }
  return st;
}

extern "C" int hoi_covariance(const double *z, int64_t T, int32_t N, int32_t D,
                              double *cov, void *stream) {
  HOI_CHECK_ARG(T >= 2 && N >= 1 && D >= 1 && z && cov, "hoi_covariance: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  double *mean = nullptr;
  if (stream_alloc((void **)&mean, sizeof(double) * D * N, s) != cudaSuccess)
    return fail(HOI_CUDA_ERROR, "hoi_covariance: cudaMallocAsync failed");
  k_col_mean<<<grid_for((int64_t)D * N * 32, 256), 256, 0, s>>>(z, T, N, D, mean);
  int st = check_launch("k_col_mean");
  if (!st) {
    int nt = (N + 31) / 32;
    dim3 grid((unsigned)(nt * (nt + 1) / 2), (unsigned)D);
    k_cov<<<grid, 256, 0, s>>>(z, mean, T, N, cov);
    st = check_launch("k_cov");
  }
  cudaFreeAsync(mean, s);
  return st;
}

extern "C" int hoi_correlation(const double *cov, int32_t N, int32_t D, double *corr,
                               double *sdiag, void *stream) {
  HOI_CHECK_ARG(N >= 1 && D >= 1 && cov && corr && sdiag, "hoi_correlation: bad args");
  int64_t n = (int64_t)N * N * D;
  k_corr<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cov, N, D, corr, sdiag);
  return check_launch("k_corr");
}
