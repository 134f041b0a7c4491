// Device reducers over full-output planes (ref:scanner.py:50-137).
#include "common.cuh"

#include <vector>

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

// Radix-select histogram: the `bits`-wide digit (<= 12) at `shift` of the
// orderable key of sign*vals[p*D+d] over the elements whose already
// resolved key bits equal `prefix` (masked by `hi_mask`).  The digit is
// masked to `bits`: the last round of a 64-bit select is 4 bits wide at
// shift 0, and bits 4..11 there are part of the resolved prefix.
constexpr int kHistUnroll = 8;   // loads in flight per thread in the select / filter passes
constexpr int kRadixBits = 12;
constexpr int kRadixBins = 1 << kRadixBits;

__global__ void __launch_bounds__(512)
k_radix_hist(const double *__restrict__ vals, int64_t n, int D, int d, double sign,
             uint64_t prefix, uint64_t hi_mask, int shift, int bits,
             unsigned long long *__restrict__ counts) {
  __shared__ unsigned int h[kRadixBins];
  const uint64_t digit_mask = (1ull << bits) - 1;
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int cur = -1;
  unsigned run = 0;     // run-length aggregation (see k_radix_hist_multi)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += kHistUnroll * stride) {
    double v[kHistUnroll];   // independent loads in flight (see k_radix_hist_multi)
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t pp = p + u * stride;
      v[u] = pp < n ? __ldcs(vals + pp * D + d) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      if (p + u * stride >= n) break;
      const uint64_t key = orderable_key(sign * v[u]);
      if ((key & hi_mask) != prefix) continue;
      const int b = (int)((key >> shift) & digit_mask);
      if (b == cur) {
        ++run;
      } else {
        if (run) atomicAdd(&h[cur], run);
        cur = b;
        run = 1;
      }
    }
  }
  if (run) atomicAdd(&h[cur], run);
  __syncthreads();
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x)
    if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

__global__ void k_key_filter(const double *__restrict__ vals, int64_t n, int D, int d, double sign,
                             uint64_t key_max, int64_t *__restrict__ cand,
                             unsigned long long *__restrict__ count, int64_t cap) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += kHistUnroll * stride) {
    double v[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t pp = p + u * stride;
      v[u] = pp < n ? __ldcs(vals + pp * D + d) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t pp = p + u * stride;
      if (pp >= n) break;
      if (orderable_key(sign * v[u]) <= key_max) {
        unsigned long long slot = atomicAdd(count, 1ull);
        if ((int64_t)slot < cap) cand[slot] = pp;
      }
    }
  }
}

// Multi-dataset radix select (all D datasets of a plane in lockstep):
// 8-bit digits, per-dataset histograms in shared memory (D <= 64).
constexpr int kMBits = 8;
constexpr int kMBins = 1 << kMBits;

// One dataset per lane slot (t % D), warp-private D x 256 histograms in
// shared memory: lanes of a warp cover 32 consecutive (row, dataset)
// elements, so at most ceil(32 / D)-way contention, none across warps.
// Consecutive hits to the same bin are counted in a register first (the
// leading digits put almost every value in a handful of bins).
__global__ void k_radix_hist_multi(const double *__restrict__ vals, int64_t n, int D, double sign,
                                   const uint64_t *__restrict__ prefix,
                                   const uint64_t *__restrict__ hi_mask,
                                   const int *__restrict__ live, int shift,
                                   unsigned long long *__restrict__ counts) {
  extern __shared__ unsigned int hm[];
  // one histogram per block (D x 256 counters): with run-length aggregation
  // the shared atomics are rare (round 1: long runs of one bin; later rounds:
  // most keys fail the prefix), so per-warp copies only cost occupancy
  const int bins = D * kMBins;
  for (int i = threadIdx.x; i < bins; i += blockDim.x) hm[i] = 0;
  __syncthreads();
  unsigned int *my = hm;
  const int64_t total = n * D;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;     // a multiple of D
  const int d = (int)(t0 % D);
  if (live[d]) {
    const uint64_t pre = prefix[d], msk = hi_mask[d];
    int cur = -1;
    unsigned run = 0;
    // kHistUnroll independent loads in flight per thread before any is
    // binned: one load per iteration left the pass latency-bound (0.77 TB/s
    // on cfg5's 512 MB, round-2 ncu)
    for (int64_t t = t0; t < total; t += kHistUnroll * stride) {
      double v[kHistUnroll];
#pragma unroll
      for (int u = 0; u < kHistUnroll; ++u) {
        const int64_t tt = t + u * stride;
        v[u] = tt < total ? __ldcs(vals + tt) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kHistUnroll; ++u) {
        if (t + u * stride >= total) break;
        const uint64_t key = orderable_key(sign * v[u]);
        if ((key & msk) != pre) continue;
        const int b = (int)((key >> shift) & (kMBins - 1));
        if (b == cur) {
          ++run;
        } else {
          if (run) atomicAdd(&my[d * kMBins + cur], run);
          cur = b;
          run = 1;
        }
      }
    }
    if (run) atomicAdd(&my[d * kMBins + cur], run);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x) {
    const unsigned v = hm[i];
    if (v) atomicAdd(&counts[i], (unsigned long long)v);
  }
}

__global__ void k_key_filter_multi(const double *__restrict__ vals, int64_t n, int D, double sign,
                                   const uint64_t *__restrict__ key_max, int64_t *__restrict__ cand,
                                   unsigned long long *__restrict__ count, int64_t cap) {
  // blockDim.x is a multiple of D (see the launch): every thread keeps one
  // dataset, and its row advances by stride / D per step (no 64-bit division)
  const int64_t total = n * D;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int d = (int)(t0 % D);
  const uint64_t km = key_max[d];
  const int64_t rstep = stride / D;
  int64_t row = t0 / D;
  for (int64_t t = t0; t < total; t += kHistUnroll * stride, row += kHistUnroll * rstep) {
    double v[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t tt = t + u * stride;
      v[u] = tt < total ? __ldcs(vals + tt) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      if (t + u * stride >= total) break;
      if (orderable_key(sign * v[u]) <= km) {
        const unsigned long long slot = atomicAdd(&count[d], 1ull);
        if ((int64_t)slot < cap) cand[(int64_t)d * cap + slot] = row + u * rstep;
      }
    }
  }
}

// numpy's float64 sum of n contiguous values (np.add.reduce / mean's
// summation, numpy/_core/src/umath/loops_utils.h pairwise_sum): sequential
// below 8 elements, 8 interleaved accumulators combined as a tree up to 128,
// halves (rounded down to a multiple of 8) above.  Matching it to the bit
// keeps the optimisers' energies -- and so their beam tie-breaks and
// annealing decisions -- identical to the reference's.  Every add is an
// explicit __dadd_rn, so nothing is contracted into an FMA.
template <typename Get>
__device__ double np_pairwise_sum(const Get &get, int i0, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, get(i0 + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(i0 + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], get(i0 + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, get(i0 + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(get, i0, n2), np_pairwise_sum(get, i0 + n2, n - n2));
}

// Optimiser objective per row of a (B, D) plane (ref:optimizers.py:74-102),
// every sum in the order numpy takes it in the reference:
//  mode 0: vals.mean(axis=1) -- vals is a C-ordered HoiBatch plane, so the
//          reduction runs along contiguous rows: np_pairwise_sum;
//  mode 1: paired Cohen's d over (cond_a[i], cond_b[i]) --
//          diff = vals[:, cond_a] - vals[:, cond_b] is built by list
//          indexing, which numpy lays out column-major, so diff.mean(axis=1)
//          and diff.std(axis=1, ddof=1) reduce along a strided axis with the
//          row index innermost: plain sequential sums;
//          energy = mean(diff) / std(diff).
// energy = sign * aggregate (sign -1 for direction 'min').  A zero or
// non-finite pair standard deviation sets *degenerate.
__global__ void k_objective(const double *__restrict__ vals, int64_t B, int D, int mode,
                            const int *__restrict__ ca, const int *__restrict__ cb, int np,
                            double sign, double *__restrict__ energy, int *__restrict__ degenerate) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B;
       b += (int64_t)gridDim.x * blockDim.x) {
    const double *row = vals + b * D;
    double agg;
    if (mode == 0) {
      agg = np_pairwise_sum([&](int i) { return row[i]; }, 0, D) / (double)D;
    } else {
      double sum = 0.0;
      for (int i = 0; i < np; ++i) sum = __dadd_rn(sum, row[ca[i]] - row[cb[i]]);
      const double mean = sum / (double)np;
      double ss = 0.0;
      for (int i = 0; i < np; ++i) {
        const double x = (row[ca[i]] - row[cb[i]]) - mean;
        ss = __dadd_rn(ss, __dmul_rn(x, x));      // numpy squares, then sums
      }
      const double sd = sqrt(ss / (double)(np - 1));
      if (!(sd > 0.0) || !isfinite(sd)) atomicExch(degenerate, 1);
      agg = mean / sd;
    }
    energy[b] = sign * agg;
  }
}

// 21-feature accumulator (ref:scanner.py:205-287), device part.  Pass 1:
// thread t (grid stride a multiple of D, so one dataset per thread) walks
// its rows in increasing rank order and keeps partials; pass 2: one CTA
// per dataset merges that dataset's partials in a fixed order
// (deterministic).  Fields per thread / per dataset:
//  0 pair count, 1 sum tc (pairs), 2 sum tc^2 (pairs), 3 count (order >= 3),
//  4..7 sum tc dtc o s, 8..11 max, 12..15 min, 16 first rank of the o max,
//  17 first rank of the o min, 18 count o < 0.
constexpr int kFeat = 19;

__global__ void k_features_partial(const double *__restrict__ out, int64_t rows, int D,
                                   int64_t plane, int64_t g0, int64_t pair_begin,
                                   int64_t pair_end, double *__restrict__ part) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double f[kFeat];
  for (int i = 0; i < kFeat; ++i) f[i] = 0.0;
  for (int m = 0; m < 4; ++m) {
    f[8 + m] = -INFINITY;
    f[12 + m] = INFINITY;
  }
  f[16] = f[17] = -1.0;
  const int64_t total = rows * D;
  for (int64_t t = t0; t < total; t += stride) {
    const int64_t r = t / D;
    const int64_t g = g0 + r;
    const double tc = out[t], dtc = out[plane + t], o = out[2 * plane + t], sv = out[3 * plane + t];
    if (g >= pair_begin && g < pair_end) {
      f[0] += 1.0;
      f[1] += tc;
      f[2] += tc * tc;
      continue;
    }
    const double v[4] = {tc, dtc, o, sv};
    f[3] += 1.0;
    for (int m = 0; m < 4; ++m) {
      f[4 + m] += v[m];
      if (v[m] > f[8 + m]) {
        f[8 + m] = v[m];
        if (m == 2) f[16] = (double)g;
      }
      if (v[m] < f[12 + m]) {
        f[12 + m] = v[m];
        if (m == 2) f[17] = (double)g;
      }
    }
    if (o < 0.0) f[18] += 1.0;
  }
  double *p = part + t0 * kFeat;
  for (int i = 0; i < kFeat; ++i) p[i] = f[i];
}

// Merge partial p into f: sums add; max / min keep the larger / smaller
// value, and for o an equal value keeps the smaller first-attainment rank,
// so the merge is associative and commutative (order-independent).
__device__ __forceinline__ void feat_merge(double *f, const double *p) {
  for (int i = 0; i < 8; ++i) f[i] += p[i];
  for (int m = 0; m < 4; ++m) {
    if (p[8 + m] > f[8 + m] ||
        (m == 2 && p[8 + m] == f[8 + m] && p[16] >= 0 && (f[16] < 0 || p[16] < f[16]))) {
      f[8 + m] = p[8 + m];
      if (m == 2) f[16] = p[16];
    }
    if (p[12 + m] < f[12 + m] ||
        (m == 2 && p[12 + m] == f[12 + m] && p[17] >= 0 && (f[17] < 0 || p[17] < f[17]))) {
      f[12 + m] = p[12 + m];
      if (m == 2) f[17] = p[17];
    }
  }
  f[18] += p[18];
}

// One CTA per dataset: thread i merges partials d + D*(i + 256 j) in j order,
// then a fixed shared-memory tree -- the same summation order every run.
constexpr int kFeatRed = 256;
__global__ void __launch_bounds__(kFeatRed)
k_features_reduce(const double *__restrict__ part, int64_t nthreads, int D,
                  double *__restrict__ feat) {
  __shared__ double sh[kFeatRed * kFeat];
  const int d = blockIdx.x, i = threadIdx.x;
  double f[kFeat];
  for (int q = 0; q < kFeat; ++q) f[q] = 0.0;
  for (int m = 0; m < 4; ++m) {
    f[8 + m] = -INFINITY;
    f[12 + m] = INFINITY;
  }
  f[16] = f[17] = -1.0;
  for (int64_t t = d + (int64_t)D * i; t < nthreads; t += (int64_t)D * kFeatRed) {
    double p[kFeat];
    for (int q = 0; q < kFeat; ++q) p[q] = part[t * kFeat + q];
    feat_merge(f, p);
  }
  for (int q = 0; q < kFeat; ++q) sh[i * kFeat + q] = f[q];
  __syncthreads();
  for (int h = kFeatRed / 2; h > 0; h >>= 1) {
    if (i < h) {
      for (int q = 0; q < kFeat; ++q) f[q] = sh[i * kFeat + q];
      feat_merge(f, sh + (i + h) * kFeat);
      for (int q = 0; q < kFeat; ++q) sh[i * kFeat + q] = f[q];
    }
    __syncthreads();
  }
  if (i < kFeat) feat[(int64_t)d * kFeat + i] = sh[i];
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

// Exact candidate set for a top-k: the positions whose key sign*v is among
// the k smallest, plus every position tied with or close to the k-th key
// (all of the k-th key's final radix bucket, at most `bucket_cap` extra).
// A 12-bit radix select narrows the threshold bucket until it holds at most
// bucket_cap elements (or the key is fully resolved); one filter pass then
// collects key <= bucket end.  Synchronous (reads back small histograms).
extern "C" int hoi_topk_select(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                               int64_t k, int64_t bucket_cap, int64_t *cand, int64_t cand_cap,
                               int64_t *h_count, void *ws, void *stream) {
  HOI_CHECK_ARG(vals && cand && h_count && ws && d >= 0 && d < D && k >= 1 && n >= 0,
                "hoi_topk_select: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long *counts = reinterpret_cast<unsigned long long *>(ws);
  unsigned long long *ccount = counts + kRadixBins;
  std::vector<unsigned long long> h(kRadixBins);
  uint64_t prefix = 0, hi_mask = 0;
  int64_t need = k < n ? k : n;
  uint64_t key_max = ~0ull;
  int blocks = 4 * sm_count();
  if (need < n) {
    for (int shift = 64 - kRadixBits; shift > -kRadixBits; shift -= kRadixBits) {
      int sh = shift < 0 ? 0 : shift;
      int bits = shift < 0 ? kRadixBits + shift : kRadixBits;
      cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * kRadixBins, s);
      k_radix_hist<<<blocks, 512, 0, s>>>(vals, n, D, d, sign, prefix, hi_mask, sh, bits, counts);
      int st = check_launch("k_radix_hist");
      if (st) return st;
      cudaMemcpyAsync(h.data(), counts, sizeof(unsigned long long) * kRadixBins,
                      cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      int64_t acc = 0;
      int b = 0;
      for (; b < (1 << bits); ++b) {
        if (acc + (int64_t)h[b] >= need) break;
        acc += (int64_t)h[b];
      }
      need -= acc;
      prefix |= (uint64_t)b << sh;
      hi_mask |= (uint64_t)((1 << bits) - 1) << sh;
      key_max = prefix | (sh ? ((1ull << sh) - 1) : 0ull);
      if ((int64_t)h[b] <= bucket_cap || sh == 0) break;
    }
  }
  cudaMemsetAsync(ccount, 0, sizeof(unsigned long long), s);
  k_key_filter<<<8 * sm_count(), 256, 0, s>>>(vals, n, D, d, sign, key_max, cand, ccount, cand_cap);
  int st = check_launch("k_key_filter");
  if (st) return st;
  unsigned long long c = 0;
  cudaMemcpyAsync(&c, ccount, sizeof(c), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  *h_count = (int64_t)c;
  return HOI_OK;
}

// hoi_topk_select for every dataset of a (n, D) plane at once (D <= 64):
// candidates of dataset d go to cand[d * cand_cap ...], their count to
// h_counts[d] (HOST).  ws: device workspace of at least
// D * 256 + 4 * D + 64 uint64.  Synchronous.
// One radix round's bookkeeping for every live dataset, on the device (the
// host used to read the histograms back after every round: three syncs and
// round trips per cfg5 TopK): find the bucket holding the need-th key,
// narrow the prefix, and retire the dataset once that bucket holds at most
// bucket_cap keys (or the last digit is resolved).
__global__ void k_radix_step_multi(const unsigned long long *__restrict__ counts, int D, int shift,
                                   int64_t bucket_cap, uint64_t *prefix, uint64_t *mask,
                                   uint64_t *keymax, int64_t *need, int *live) {
  const int d = threadIdx.x;
  if (d >= D || !live[d]) return;
  const unsigned long long *hd = counts + (size_t)d * kMBins;
  const int64_t nd = need[d];
  int64_t acc = 0;
  int b = 0;
  for (; b < kMBins - 1; ++b) {
    if (acc + (int64_t)hd[b] >= nd) break;
    acc += (int64_t)hd[b];
  }
  need[d] = nd - acc;
  const uint64_t pre = prefix[d] | ((uint64_t)b << shift);
  prefix[d] = pre;
  mask[d] |= (uint64_t)(kMBins - 1) << shift;
  keymax[d] = pre | (shift ? ((1ull << shift) - 1) : 0ull);
  if ((int64_t)hd[b] <= bucket_cap || shift == 0) live[d] = 0;
}

extern "C" int hoi_topk_select_multi(const double *vals, int64_t n, int32_t D, double sign,
                                     int64_t k, int64_t bucket_cap, int64_t *cand,
                                     int64_t cand_cap, int64_t *h_counts, void *ws,
                                     void *stream) {
  HOI_CHECK_ARG(vals && cand && h_counts && ws && D >= 1 && D <= 64 && k >= 1 && n >= 0,
                "hoi_topk_select_multi: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  // ws: counts (D x 256) | prefix | mask | keymax | need (D each) | live
  // (64 int) | candidate counts (D)
  unsigned long long *counts = reinterpret_cast<unsigned long long *>(ws);
  uint64_t *d_prefix = reinterpret_cast<uint64_t *>(counts + (size_t)D * kMBins);
  uint64_t *d_mask = d_prefix + D;
  uint64_t *d_keymax = d_mask + D;
  int64_t *d_need = reinterpret_cast<int64_t *>(d_keymax + D);
  int *d_live = reinterpret_cast<int *>(d_need + D);
  unsigned long long *ccount = reinterpret_cast<unsigned long long *>(d_live + 64);
  {
    std::vector<uint64_t> init((size_t)4 * D);
    for (int d = 0; d < D; ++d) {
      init[d] = 0;                                  // prefix
      init[D + d] = 0;                              // mask
      init[2 * D + d] = ~0ull;                      // keymax
      init[3 * D + d] = (uint64_t)(k < n ? k : n);  // need
    }
    std::vector<int> live(64, 0);
    for (int d = 0; d < D; ++d) live[d] = k < n ? 1 : 0;
    cudaMemcpyAsync(d_prefix, init.data(), sizeof(uint64_t) * 4 * D, cudaMemcpyHostToDevice, s);
    // (pageable sources: staged before the calls return, so the vectors may
    // go out of scope)
    cudaMemcpyAsync(d_live, live.data(), sizeof(int) * 64, cudaMemcpyHostToDevice, s);
  }
  // 256-thread blocks (a multiple of D: one dataset per thread), one
  // D x 256 histogram each (16 KB at D = 16: 8 blocks, 64 warps per SM);
  // every round is launched, a retired dataset's threads skip their loads
  const int bs = (256 / D) * D;
  const size_t shm = sizeof(unsigned int) * D * kMBins;
  const int blocks = 8 * sm_count();
  cudaFuncSetAttribute(k_radix_hist_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  for (int shift = 64 - kMBits; shift >= 0; shift -= kMBits) {
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * D * kMBins, s);
    k_radix_hist_multi<<<blocks, bs, shm, s>>>(vals, n, D, sign, d_prefix, d_mask, d_live, shift,
                                               counts);
    k_radix_step_multi<<<1, 64, 0, s>>>(counts, D, shift, bucket_cap, d_prefix, d_mask, d_keymax,
                                        d_need, d_live);
    int st = check_launch("k_radix_hist_multi/k_radix_step_multi");
    if (st) return st;
  }
  cudaMemsetAsync(ccount, 0, sizeof(unsigned long long) * D, s);
  k_key_filter_multi<<<8 * sm_count(), bs, 0, s>>>(vals, n, D, sign, d_keymax, cand, ccount,
                                                    cand_cap);
  int st = check_launch("k_key_filter_multi");
  if (st) return st;
  std::vector<unsigned long long> c(D);
  cudaMemcpyAsync(c.data(), ccount, sizeof(unsigned long long) * D, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  for (int d = 0; d < D; ++d) h_counts[d] = (int64_t)c[d];
  return HOI_OK;
}

// The exact k-th smallest orderable key of sign*vals[p*D+d], p < n (full
// 64-bit radix select), written to device memory *key_out; ~0 when n <= k
// (every element qualifies).  Synchronous.
static int topk_key(const double *vals, int64_t n, int32_t D, int32_t d, double sign, int64_t k,
                    int bits_wanted, uint64_t *key_out, void *ws, cudaStream_t s);

extern "C" int hoi_topk_threshold(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                                  int64_t k, uint64_t *key_out, void *ws, void *stream) {
  HOI_CHECK_ARG(vals && key_out && ws && d >= 0 && d < D && k >= 1 && n >= 0,
                "hoi_topk_threshold: bad args");
  return topk_key(vals, n, D, d, sign, k, 64, key_out, ws, (cudaStream_t)stream);
}

// An upper bound of that key after resolving only its top `bits` bits (the
// end of the k-th key's bucket): enough for a filter threshold, with fewer
// synchronous radix rounds (12 bits each).  bits >= 64 is the exact key.
extern "C" int hoi_topk_bound(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                              int64_t k, int32_t bits, uint64_t *key_out, void *ws, void *stream) {
  HOI_CHECK_ARG(vals && key_out && ws && d >= 0 && d < D && k >= 1 && n >= 0 && bits >= 1,
                "hoi_topk_bound: bad args");
  return topk_key(vals, n, D, d, sign, k, bits, key_out, ws, (cudaStream_t)stream);
}

static int topk_key(const double *vals, int64_t n, int32_t D, int32_t d, double sign, int64_t k,
                    int bits_wanted, uint64_t *key_out, void *ws, cudaStream_t s) {
  unsigned long long *counts = reinterpret_cast<unsigned long long *>(ws);
  std::vector<unsigned long long> h(kRadixBins);
  uint64_t prefix = 0, hi_mask = 0;
  uint64_t key = ~0ull;
  int64_t need = k;
  if (n > k) {
    const int blocks = 4 * sm_count();
    for (int shift = 64 - kRadixBits; shift > -kRadixBits; shift -= kRadixBits) {
      const int sh = shift < 0 ? 0 : shift;
      const int bits = shift < 0 ? kRadixBits + shift : kRadixBits;
      cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * kRadixBins, s);
      k_radix_hist<<<blocks, 512, 0, s>>>(vals, n, D, d, sign, prefix, hi_mask, sh, bits, counts);
      int st = check_launch("k_radix_hist");
      if (st) return st;
      cudaMemcpyAsync(h.data(), counts, sizeof(unsigned long long) * kRadixBins,
                      cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      int64_t acc = 0;
      int b = 0;
      for (; b < (1 << bits); ++b) {
        if (acc + (int64_t)h[b] >= need) break;
        acc += (int64_t)h[b];
      }
      need -= acc;
      prefix |= (uint64_t)b << sh;
      hi_mask |= (uint64_t)((1 << bits) - 1) << sh;
      if (sh == 0) break;
      if (64 - sh >= bits_wanted) {               // bound: the end of the bucket
        prefix |= (1ull << sh) - 1;
        break;
      }
    }
    key = prefix;
  }
  cudaMemcpyAsync(key_out, &key, sizeof(key), cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  return HOI_OK;
}

extern "C" int hoi_objective(const double *vals, int64_t B, int32_t D, int32_t mode,
                             const int32_t *cond_a, const int32_t *cond_b, int32_t npairs,
                             double sign, double *energy, int32_t *degenerate, void *stream) {
  HOI_CHECK_ARG(vals && energy && degenerate && B >= 0 && D >= 1 && (mode == 0 || mode == 1),
                "hoi_objective: bad args");
  HOI_CHECK_ARG(mode == 0 || (cond_a && cond_b && npairs >= 2), "hoi_objective: bad pairs");
  if (B == 0) return HOI_OK;
  const int64_t g = (B + 255) / 256;
  k_objective<<<(int)(g < 8 * sm_count() ? g : 8 * sm_count()), 256, 0, (cudaStream_t)stream>>>(
      vals, B, D, mode, cond_a, cond_b, npairs, sign, energy, degenerate);
  return check_launch("k_objective");
}

// Feature partials of a full-output chunk (4 planes of (rows, D), global
// rank of row 0 = g0; rows with global rank in [pair_begin, pair_end) are
// the order-2 pairs): feat (D, 19) doubles, see k_features_partial.
// ws: device workspace of >= 8 * 148 * 256 * 19 doubles.
extern "C" int hoi_features(const double *out, int64_t rows, int32_t D, int64_t g0,
                            int64_t pair_begin, int64_t pair_end, double *feat, void *ws,
                            int64_t ws_doubles, void *stream) {
  HOI_CHECK_ARG(out && feat && ws && D >= 1 && rows >= 0, "hoi_features: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  int bs = (256 / D) * D;                      // a multiple of D: one dataset per thread
  if (bs < D) bs = D;
  // grid sized by the work (>= 32 units per thread), at most 4 CTAs per SM:
  // small chunks must not write and re-read a full grid of partials
  const int64_t want = (rows * (int64_t)D + (int64_t)bs * 32 - 1) / ((int64_t)bs * 32);
  int blocks = (int)(want < 4 * sm_count() ? (want > 0 ? want : 1) : 4 * sm_count());
  if ((int64_t)blocks * bs * kFeat > ws_doubles) blocks = (int)(ws_doubles / ((int64_t)bs * kFeat));
  if (blocks < 1) return fail(HOI_CAPACITY, "hoi_features: workspace too small");
  const int64_t nthreads = (int64_t)blocks * bs;
  k_features_partial<<<blocks, bs, 0, s>>>(out, rows, D, rows * (int64_t)D, g0, pair_begin,
                                           pair_end, reinterpret_cast<double *>(ws));
  int st = check_launch("k_features_partial");
  if (st) return st;
  k_features_reduce<<<D, kFeatRed, 0, s>>>(reinterpret_cast<double *>(ws), nthreads, D, feat);
  return check_launch("k_features_reduce");
}

extern "C" int hoi_topk_filter(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                               const double *thresh, int64_t *cand, int64_t *cand_count,
                               int64_t cand_cap, void *stream) {
  HOI_CHECK_ARG(vals && thresh && cand && cand_count && d >= 0 && d < D, "hoi_topk_filter: bad args");
  k_topk_filter<<<8 * sm_count(), 256, 0, (cudaStream_t)stream>>>(
      vals, n, D, d, sign, thresh, cand, reinterpret_cast<unsigned long long *>(cand_count), cand_cap);
  return check_launch("k_topk_filter");
}

// ------------------------------------------------- exact TopK ordering ----
// The reference's TopK key (ref:scanner.py:75-100) is (sign * value, index
// tuple), ascending: one CTA per dataset sorts that dataset's candidate
// positions (hoi_topk_select_multi's output: the k best keys plus every tie
// at the k-th) by the orderable 64-bit key, equal keys by the lexicographic
// index tuple of their rows (idx, (n, K) int32: a fixed-order batch, so
// tuples have equal length), equal tuples by position (a stable sort of the
// batch order), and writes the first min(k, count) positions.  Bitonic sort
// over a power-of-two padding in shared memory; the tuple comparison only
// runs on exactly equal keys.
constexpr int kOrderMax = 8192;          // candidates per dataset (128 KB of smem)
constexpr int kOrderThreads = 1024;

__device__ __forceinline__ bool topk_less(uint64_t ka, int64_t pa, uint64_t kb, int64_t pb,
                                          const int32_t *__restrict__ idx, int K) {
  if (ka != kb) return ka < kb;
  if (pa == pb) return false;
  if (pa < 0 || pb < 0) return pa >= 0;           // padding (-1) sorts last
  const int32_t *ra = idx + pa * K, *rb = idx + pb * K;
  for (int i = 0; i < K; ++i) {
    const int32_t x = __ldg(ra + i), y = __ldg(rb + i);
    if (x != y) return x < y;
  }
  return pa < pb;
}

__global__ void __launch_bounds__(kOrderThreads)
k_topk_order(const double *__restrict__ vals, int D, double sign, const int64_t *__restrict__ cand,
             int64_t cand_cap, const int64_t *__restrict__ counts, const int32_t *__restrict__ idx,
             int K, int64_t k, int64_t *__restrict__ top_pos) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = blockIdx.x;
  const int c = (int)(counts[d] < cand_cap ? counts[d] : cand_cap);
  int P = 1;
  while (P < c) P <<= 1;
  uint64_t *key = reinterpret_cast<uint64_t *>(smem_raw);
  int64_t *pos = reinterpret_cast<int64_t *>(key + P);
  const int64_t *cd = cand + (int64_t)d * cand_cap;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < c) {
      const int64_t p = cd[i];
      pos[i] = p;
      key[i] = orderable_key(sign * vals[p * D + d]);
    } else {
      pos[i] = -1;
      key[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t ka = key[lo], kb = key[hi];
        const int64_t pa = pos[lo], pb = pos[hi];
        const bool swap = up ? topk_less(kb, pb, ka, pa, idx, K) : topk_less(ka, pa, kb, pb, idx, K);
        if (swap) {
          key[lo] = kb; key[hi] = ka;
          pos[lo] = pb; pos[hi] = pa;
        }
      }
      __syncthreads();
    }
  }
  const int m = (int)(k < c ? k : c);
  for (int i = threadIdx.x; i < k; i += blockDim.x) top_pos[(int64_t)d * k + i] = i < m ? pos[i] : -1;
}

extern "C" int hoi_topk_order(const double *vals, int32_t D, double sign, const int64_t *cand,
                              int64_t cand_cap, const int64_t *counts, const int32_t *idx,
                              int32_t K, int64_t k, int64_t *top_pos, void *stream) {
  HOI_CHECK_ARG(vals && cand && counts && idx && top_pos && D >= 1 && K >= 1 && k >= 1 &&
                cand_cap >= 1 && cand_cap <= kOrderMax, "hoi_topk_order: bad args");
  int P = 1;
  while (P < cand_cap) P <<= 1;
  const size_t shm = (size_t)P * (sizeof(uint64_t) + sizeof(int64_t));
  cudaFuncSetAttribute(k_topk_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  k_topk_order<<<D, kOrderThreads, shm, (cudaStream_t)stream>>>(vals, D, sign, cand, cand_cap,
                                                                 counts, idx, K, k, top_pos);
  return check_launch("k_topk_order");
}
