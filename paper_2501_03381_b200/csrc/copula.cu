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

// Data layout.  The reference's matrices are samples x variables (T, N),
// row-major, so a column -- the unit of the rank transform -- is strided by
// N.  Every kernel here works on the column-major copy (D, N, T): one tiled
// shared-memory transpose reads the data coalesced, the rank sort then loads
// its column contiguously, writes its T copula values into one contiguous
// column (scattered only within those 8T bytes, merged in L2), and the
// covariance streams contiguous column panels.  The (T, N) outputs of the
// row-major entry points are one more transpose.

// (D, R, C) -> (D, C, R) through 32 x 32 shared tiles (conflict-free, +1 pad).
template <typename V>
__global__ void __launch_bounds__(256) k_transpose(const V *__restrict__ in, int64_t R, int64_t C,
                                                   V *__restrict__ out) {
  __shared__ V tile[32][33];
  const int64_t d = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const V *src = in + d * R * C;
  V *dst = out + d * R * C;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    if (r < R && c < C) tile[i][tx] = src[r * C + c];
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + tx;
    if (r < R && c < C) dst[c * R + r] = tile[tx][i];
  }
}

template <typename V>
static void transpose(const V *in, int64_t R, int64_t C, int D, V *out, cudaStream_t s) {
  dim3 grid((unsigned)((C + 31) / 32), (unsigned)((R + 31) / 32), (unsigned)D);
  k_transpose<V><<<grid, 256, 0, s>>>(in, R, C, out);
}

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
k_rank_chunk(const double *__restrict__ xt, int64_t T, int N, int chunk, int pad,
             const double *__restrict__ qgrid, int64_t *__restrict__ ranks,
             double *__restrict__ z, uint64_t *__restrict__ ws_keys,
             int *__restrict__ ws_rows) {
  extern __shared__ unsigned char smem[];
  uint64_t *key = reinterpret_cast<uint64_t *>(smem);
  int *row = reinterpret_cast<int *>(key + pad);
  const int col = blockIdx.x;                 // d * N + j (column-major layout)
  const int c = blockIdx.y;
  const int64_t t0 = (int64_t)c * chunk;
  const int n_here = (int)((int64_t)chunk < T - t0 ? (int64_t)chunk : T - t0);
  const double *xc = xt + (int64_t)col * T;   // the column, contiguous
  for (int i = threadIdx.x; i < pad; i += blockDim.x) {
    if (i < n_here) {
      key[i] = orderable_key(xc[t0 + i]);
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
      int64_t o = (int64_t)col * T + t;
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
  int t = ws_rows[col * per_col + within];
  int64_t out = col * T + t;
  if (ranks) ranks[out] = r + 1;
  z[out] = qgrid[r];
}

// Column means of the column-major (D, N, T) copy: one 256-thread CTA per
// column, strided partial sums combined in a fixed tree (deterministic).
__global__ void __launch_bounds__(256) k_col_mean(const double *__restrict__ z, int64_t T,
                                                  double *__restrict__ mean) {
  __shared__ double red[8];
  const double *zc = z + (int64_t)blockIdx.x * T;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < T; t += 256) s += zc[t];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
    mean[blockIdx.x] = a / (double)T;
  }
}

// X^T X on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): one 32 x 32
// output tile per CTA (upper tiles only), its two 32-sample centred panels
// staged in shared memory from the column-major copy (lanes along t:
// coalesced), 8 warps x 2 of the 16 8x8 sub-tiles, 8 MMA k-steps of 4
// samples per panel, FP64 accumulation throughout.  Split over T (grid.z =
// S slices of the 32-sample panels) so small N still fills the GPU -- at
// cfg4 (N = 30, one tile) 63 CTAs of one panel each instead of one CTA
// walking all 63 -- the slices' partial tiles are summed in a fixed order by
// k_cov_reduce (deterministic).  The value of (i, j) is written to (i, j)
// and (j, i), so the covariance is exactly symmetric (the reference
// symmetrises with 0.5 (S + S^T), ref:copula_core.py:187-189).
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tile_of(int tile, int nt, int &ti, int &tj) {
  ti = 0;
  int rem = tile;
  while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
  tj = ti + rem;
}

__global__ void __launch_bounds__(256)
k_cov(const double *__restrict__ zt, const double *__restrict__ mean, int64_t T,
      int N, int S, double *__restrict__ cov, double *__restrict__ part) {
  __shared__ double A[32][33];
  __shared__ double B[32][33];
  const int nt = (N + 31) / 32;
  const int tile = blockIdx.x, d = blockIdx.y, sl = blockIdx.z;
  int ti, tj;
  tile_of(tile, nt, ti, tj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int lane = tx, warp = ty;
  const double *zd = zt + (int64_t)d * N * T;
  const double *md = mean + (int64_t)d * N;
  const int rb = warp >> 1, cb0 = (warp & 1) * 2;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int64_t npan = (T + 31) / 32;
  const int64_t p0 = npan * sl / S, p1 = npan * (sl + 1) / S;
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t t = p * 32 + tx;
    for (int c = ty; c < 32; c += 8) {
      const int ci = ti * 32 + c, cj = tj * 32 + c;
      A[tx][c] = (t < T && ci < N) ? zd[(int64_t)ci * T + t] - md[ci] : 0.0;
      B[tx][c] = (t < T && cj < N) ? zd[(int64_t)cj * T + t] - md[cj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int r = 4 * kk + (lane & 3);
      const double av = A[r][rb * 8 + (lane >> 2)];                // A^T fragment (8 x 4, row)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double bv = B[r][(cb0 + c) * 8 + (lane >> 2)];       // B fragment (4 x 8, col)
        dmma_8x8x4(acc[c][0], acc[c][1], av, bv);
      }
    }
    __syncthreads();
  }
  const double inv = 1.0 / (double)(T - 1);
  double *cd = cov + (int64_t)d * N * N;
  double *pt = part ? part + (((int64_t)sl * gridDim.y + d) * gridDim.x + tile) * 1024 : nullptr;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = rb * 8 + (lane >> 2), lj = (cb0 + c) * 8 + 2 * (lane & 3) + h;
      if (pt) {
        pt[li * 32 + lj] = acc[c][h];
        continue;
      }
      const int i = ti * 32 + li, j = tj * 32 + lj;
      if (i < N && j < N && (ti < tj || i <= j)) {
        const double v = acc[c][h] * inv;
        cd[(int64_t)i * N + j] = v;
        cd[(int64_t)j * N + i] = v;
      }
    }
  }
}

// Sum of the S slices' partial tiles, slice 0 first (fixed order), scaled
// by 1/(T-1) and mirrored: one thread per tile entry, the S slice loads
// independent (issued together), the adds in slice order.
__global__ void __launch_bounds__(1024)
k_cov_reduce(const double *__restrict__ part, int64_t T, int N, int D, int S, int ntiles,
             double *__restrict__ cov) {
  const int tile = blockIdx.x, d = blockIdx.y;
  const int nt = (N + 31) / 32;
  int ti, tj;
  tile_of(tile, nt, ti, tj);
  const int e = threadIdx.x;
  const int li = e >> 5, lj = e & 31;
  const int i = ti * 32 + li, j = tj * 32 + lj;
  if (!(i < N && j < N && (ti < tj || i <= j))) return;
  const double *p = part + ((int64_t)d * ntiles + tile) * 1024 + e;
  const int64_t step = (int64_t)D * ntiles * 1024;
  double v = 0.0;
  int sl = 0;
  for (; sl + 8 <= S; sl += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(p + (sl + u) * step);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += x[u];
  }
  for (; sl < S; ++sl) v += __ldg(p + sl * step);
  v *= 1.0 / (double)(T - 1);
  double *cd = cov + (int64_t)d * N * N;
  cd[(int64_t)i * N + j] = v;
  cd[(int64_t)j * N + i] = v;
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

namespace {
// Sort chunk per column: at most kMaxChunk (shared memory), and small
// enough that the D*N columns give ~2 CTAs per SM (a 2000-sample column of
// the 30-variable headline system is 8 chunks of 256, not one 2048-wide
// bitonic network per column on 30 SMs); a column that fits one chunk is
// ranked directly, otherwise k_rank_merge combines its sorted chunks.
void pick_chunk(int64_t T, int64_t cols, int &chunk, int &nchunks) {
  int64_t want = (2 * 148 + cols - 1) / cols;                 // chunks per column
  int64_t per = (T + want - 1) / want;
  chunk = 256;
  while (chunk < per && chunk < kMaxChunk) chunk <<= 1;
  if (chunk >= T) {                                           // one chunk: pad to 2^k >= T
    chunk = 1;
    while (chunk < T) chunk <<= 1;
  }
  nchunks = (int)((T + chunk - 1) / chunk);
}

// Column-major rank + copula (x already (D, N, T)); ranks_t / z_t (D, N, T).
int rank_copula_cols(const double *xt, int64_t T, int N, int D, const double *qgrid,
                     int64_t *ranks_t, double *z_t, char *merge_ws, cudaStream_t s) {
  int chunk, nchunks;
  pick_chunk(T, (int64_t)N * D, chunk, nchunks);
  const int pad = chunk;
  const size_t shm = (size_t)pad * (sizeof(uint64_t) + sizeof(int));
  cudaFuncSetAttribute(k_rank_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  uint64_t *wk = nullptr;
  int *wr = nullptr;
  if (nchunks > 1) {
    const size_t elems = (size_t)D * N * nchunks * chunk;
    wk = reinterpret_cast<uint64_t *>(merge_ws);
    wr = reinterpret_cast<int *>(wk + elems);
  }
  dim3 grid((unsigned)(D * N), (unsigned)nchunks);
  const int threads = std::min(kSortThreads, std::max(32, pad / 2));
  k_rank_chunk<<<grid, threads, shm, s>>>(xt, T, N, chunk, pad, qgrid, ranks_t, z_t, wk, wr);
  int st = check_launch("k_rank_chunk");
  if (st) return st;
  if (nchunks > 1) {
    const int64_t n = (int64_t)D * N * nchunks * chunk;
    k_rank_merge<<<grid_for(n, 256), 256, 0, s>>>(T, N, D, chunk, nchunks, qgrid, wk, wr,
                                                  ranks_t, z_t);
    st = check_launch("k_rank_merge");
  }
  return st;
}

size_t merge_bytes(int64_t T, int N, int D) {
  int chunk, nchunks;
  pick_chunk(T, (int64_t)N * D, chunk, nchunks);
  if (nchunks == 1) return 0;
  const size_t elems = (size_t)D * N * nchunks * chunk;
  return ((elems * (sizeof(uint64_t) + sizeof(int)) + 255) & ~(size_t)255);
}

size_t col_bytes(int64_t T, int N, int D) {
  return (((size_t)D * N * T * sizeof(double)) + 255) & ~(size_t)255;
}
}  // namespace

extern "C" int hoi_rank_copula_cols(const double *x, int64_t T, int32_t N, int32_t D,
                                    const double *qgrid, int64_t *ranks_t, double *z_t, void *ws,
                                    size_t *ws_bytes, void *stream) {
  HOI_CHECK_ARG(T >= 1 && N >= 1 && D >= 1, "hoi_rank_copula_cols: bad shape");
  HOI_CHECK_ARG(T < (int64_t)1 << 31, "hoi_rank_copula_cols: T too large");
  const size_t need = col_bytes(T, N, D) + merge_bytes(T, N, D);
  if (ws == nullptr) {
    HOI_CHECK_ARG(ws_bytes != nullptr, "hoi_rank_copula_cols: ws_bytes is NULL");
    *ws_bytes = need;
    return HOI_OK;
  }
  if (ws_bytes && *ws_bytes < need) return fail(HOI_CAPACITY, "hoi_rank_copula_cols: workspace too small");
  HOI_CHECK_ARG(x && qgrid && z_t, "hoi_rank_copula_cols: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  double *xt = reinterpret_cast<double *>(ws);
  transpose<double>(x, T, N, D, xt, s);
  int st = check_launch("k_transpose");
  if (st) return st;
  return rank_copula_cols(xt, T, N, D, qgrid, ranks_t, z_t,
                          reinterpret_cast<char *>(ws) + col_bytes(T, N, D), s);
}

extern "C" int hoi_rank_copula(const double *x, int64_t T, int32_t N, int32_t D,
                               const double *qgrid, int64_t *ranks, double *z,
                               void *ws, size_t *ws_bytes, void *stream) {
  HOI_CHECK_ARG(T >= 1 && N >= 1 && D >= 1, "hoi_rank_copula: bad shape");
  HOI_CHECK_ARG(T < (int64_t)1 << 31, "hoi_rank_copula: T too large");
  // [xt | z_t | ranks_t | merge]
  const size_t cb = col_bytes(T, N, D);
  const size_t rb = ((size_t)D * N * T * sizeof(int64_t) + 255) & ~(size_t)255;
  const size_t need = 2 * cb + rb + merge_bytes(T, N, D);
  if (ws == nullptr) {
    HOI_CHECK_ARG(ws_bytes != nullptr, "hoi_rank_copula: ws_bytes is NULL");
    *ws_bytes = need;
    return HOI_OK;
  }
  if (ws_bytes && *ws_bytes < need) return fail(HOI_CAPACITY, "hoi_rank_copula: workspace too small");
  HOI_CHECK_ARG(x && qgrid && z, "hoi_rank_copula: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  char *w = reinterpret_cast<char *>(ws);
  double *xt = reinterpret_cast<double *>(w);
  double *zt = reinterpret_cast<double *>(w + cb);
  int64_t *rt = ranks ? reinterpret_cast<int64_t *>(w + 2 * cb) : nullptr;
  transpose<double>(x, T, N, D, xt, s);
  int st = rank_copula_cols(xt, T, N, D, qgrid, rt, zt, w + 2 * cb + rb, s);
  if (st) return st;
  transpose<double>(zt, N, T, D, z, s);
  if (rt) transpose<int64_t>(rt, N, T, D, ranks, s);
  return check_launch("k_transpose");
}

// Covariance of column-major z_t (D, N, T).
extern "C" int hoi_covariance_cols(const double *z_t, int64_t T, int32_t N, int32_t D,
                                   double *cov, void *stream) {
  HOI_CHECK_ARG(T >= 2 && N >= 1 && D >= 1 && z_t && cov, "hoi_covariance_cols: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = (N + 31) / 32;
  const int ntiles = nt * (nt + 1) / 2;
  const int64_t npan = (T + 31) / 32;
  // slices of T so that the grid covers ~2 CTAs per SM
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t S = (2 * (int64_t)sms + (int64_t)ntiles * D - 1) / ((int64_t)ntiles * D);
  if (S > npan) S = npan;
  if (S < 1) S = 1;
  double *mean = nullptr, *part = nullptr;
  const size_t pbytes = S > 1 ? sizeof(double) * 1024 * (size_t)S * D * ntiles : 0;
  if (stream_alloc((void **)&mean, sizeof(double) * D * N + pbytes, s) != cudaSuccess)
    return fail(HOI_CUDA_ERROR, "hoi_covariance: cudaMallocAsync failed");
  if (S > 1) part = mean + (size_t)D * N;
  k_col_mean<<<(unsigned)(D * N), 256, 0, s>>>(z_t, T, mean);
  int st = check_launch("k_col_mean");
  if (!st) {
    k_cov<<<dim3((unsigned)ntiles, (unsigned)D, (unsigned)S), 256, 0, s>>>(z_t, mean, T, N, (int)S,
                                                                           cov, part);
    st = check_launch("k_cov");
  }
  if (!st && S > 1) {
    k_cov_reduce<<<dim3((unsigned)ntiles, (unsigned)D), 1024, 0, s>>>(part, T, N, D, (int)S,
                                                                      ntiles, cov);
    st = check_launch("k_cov_reduce");
  }
  cudaFreeAsync(mean, s);
  return st;
}

extern "C" int hoi_covariance(const double *z, int64_t T, int32_t N, int32_t D,
                              double *cov, void *stream) {
  HOI_CHECK_ARG(T >= 2 && N >= 1 && D >= 1 && z && cov, "hoi_covariance: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  double *zt = nullptr;
  if (stream_alloc((void **)&zt, sizeof(double) * (size_t)D * N * T, s) != cudaSuccess)
    return fail(HOI_CUDA_ERROR, "hoi_covariance: cudaMallocAsync failed");
  transpose<double>(z, T, N, D, zt, s);
  int st = check_launch("k_transpose");
  if (!st) st = hoi_covariance_cols(zt, T, N, D, cov, stream);
  cudaFreeAsync(zt, s);
  return st;
}

extern "C" int hoi_correlation(const double *cov, int32_t N, int32_t D, double *corr,
                               double *sdiag, void *stream) {
  HOI_CHECK_ARG(N >= 1 && D >= 1 && cov && corr && sdiag, "hoi_correlation: bad args");
  int64_t n = (int64_t)N * N * D;
  k_corr<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cov, N, D, corr, sdiag);
  return check_launch("k_corr");
}
