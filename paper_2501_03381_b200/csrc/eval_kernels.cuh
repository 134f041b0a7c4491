// Engine 1: per-(n-plet, dataset) evaluation.
//
// One thread owns one (n-plet, dataset) unit.  For K <= 16 the K x K
// packed lower triangle lives in registers (K is a template parameter and
// every loop is fully unrolled, so all indices are compile-time; past
// K = 13 the compiler spills the coldest part); K > 16 uses the same code
// with a runtime K (local memory).  Measured on B200 (cfg4 order segments):
// fixed K = 13..16 run 6.4-8.7 TF/s against ~1 for the runtime-K kernel;
// fixed K = 17..22 only reach 1.1-1.8 TF/s (5-21 KB of spills per thread)
// at 5-11 min of compile per 4 orders, so they are not instantiated.  The
// fixed-K instantiations are spread over eval_k*.cu (parallel compile).
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
#pragma once
#include "common.cuh"

namespace hoib {

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
  const float *src32;      // FP32 copy of the correlation (FP32 fast path) or nullptr
  int fp32;                // 1: factorise in FP32 (log products and epilogue in FP64)
};

#define TRI(i, j) ((i) * ((i) + 1) / 2 + (j))

__device__ __forceinline__ void unrank_lex(uint64_t r, int K, int N, int *s) {
  int c = 0;
  for (int p = 0; p < K; ++p) {
    while (c < N) {
      uint64_t b = binom_l1(N - 1 - c, K - 1 - p);
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

// Lexicographic successor of the K-subset s (s not the last one), register
// form: every position is a compile-time slot, the rightmost incrementable
// position p is found with predicates, no runtime-indexed array.
template <int KT>
__device__ __forceinline__ void lex_successor(int (&s)[KT], int K, int N) {
  int p = 0;
#pragma unroll
  for (int q = 0; q < KT; ++q)
    if (q < K && s[q] < N - K + q) p = q;
  int v = 0;
#pragma unroll
  for (int q = 0; q < KT; ++q) {
    if (q == p) v = s[q] + 1;
    if (q >= p && q < K) s[q] = v + (q - p);
  }
}

// src: the correlation matrix (N, N, D) -- global, or the CTA's shared
// copy for small N x N x D -- or the raw matrix stack in mats mode.  The
// correlation form has an exact unit diagonal (k_corr writes 1.0), so only
// the strict lower triangle is gathered.
template <int KT, bool FIXED, typename TM = double>
__device__ __forceinline__ void load_matrix(const EvalArgs &A, const TM *__restrict__ src,
                                            int64_t b, int d, int K,
                                            const int (&s)[KT], TM (&a)[KT * (KT + 1) / 2],
                                            bool jitter) {
  if (A.mats) {   // (FP64 only)
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
    const TM *row = src + (s[i] * N) * D + d;
#pragma unroll
    for (int j = 0; j < i; ++j) a[TRI(i, j)] = row[s[j] * D];
    a[TRI(i, i)] = TM(1);
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
// Rows are updated bottom-up so the unscaled column j stays readable without
// a temporary copy (fewer live registers -> more resident warps); the
// pivot reciprocal: the hardware approximation (~2^-23 relative error)
// refined by one cubic Newton step, e = 1 - x r, r' = r + r (e + e^2): the
// error cubes below double precision (result within an ulp of 1 / x for
// the positive normal pivots that reach it) in 3 dependent DFMA, against
// __drcp_rn's longer correctly rounded sequence with its special-case
// branch.  (A quadratic step, 2 DFMA, leaves ~2^-44 and fails the
// reference's 1e-14 closed-form check on a near-singular 2x2 system.)
__device__ __forceinline__ double pivot_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rcp_rn(double x) { return pivot_rcp(x); }
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }

template <int KT, bool FIXED, bool STORE_CS, typename TM = double>
__device__ __forceinline__ bool ldl_invdiag(TM (&a)[KT * (KT + 1) / 2], int K,
                                            double (&cs)[KT], double &l, double &lam) {
  // the diagonal slot of column j holds 1/d_j once the column is done, so
  // the packed triangle is the only K x K state (fewer live registers)
  // a non-positive pivot is flagged, not branched on: the factorisation is
  // one straight-line block the scheduler can overlap across pivots (the
  // values after a bad pivot are discarded by the caller's retry)
  LogProd pd;
  pd.init();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const TM dj = a[TRI(j, j)];
    bad |= !(dj > TM(0));
    pd.mul((double)dj);
    if ((j & 7) == 7) pd.renorm();
    const TM r = rcp_rn(dj);
    a[TRI(j, j)] = r;
#pragma unroll
    for (int i = K - 1; i > j; --i) {
      const TM lij = a[TRI(i, j)] * r;
#pragma unroll
      for (int m = j + 1; m <= i; ++m) a[TRI(i, m)] = fma(-lij, a[TRI(m, j)], a[TRI(i, m)]);
      a[TRI(i, j)] = lij;
    }
  }
  if (bad) return false;
  pd.renorm();
  // U = L^-1 (unit lower), column by column, in place (diagonal untouched).
#pragma unroll
  for (int j = 0; j < K; ++j) {
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      TM acc = a[TRI(i, j)];
#pragma unroll
      for (int m = j + 1; m < i; ++m) acc = fma(a[TRI(i, m)], a[TRI(m, j)], acc);
      a[TRI(i, j)] = -acc;
    }
  }
  // (M^-1)_jj = sum_i U_ij^2 / d_i
  LogProd pl;
  pl.init();
#pragma unroll
  for (int j = 0; j < K; ++j) {
    TM sacc = a[TRI(j, j)];
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      const TM u = a[TRI(i, j)];
      sacc = fma(u * u, a[TRI(i, i)], sacc);
    }
    if (STORE_CS) cs[j] = (double)sacc;
    pl.mul((double)sacc);
    if ((j & 7) == 7) pl.renorm();
  }
  pl.renorm();
  l = pd.log_value();
  lam = pl.log_value();
  return true;
}

template <int KT, bool FIXED>
__device__ __forceinline__ void unit_indices(const EvalArgs &A, int64_t b, int K, int (&s)[KT]) {
  if (A.mats) return;
  if (A.idx) {
#pragma unroll
    for (int i = 0; i < K; ++i) s[i] = A.idx[b * A.idx_stride + i];
  } else {
    unrank_lex(A.r0 + (uint64_t)b, K, A.N, s);
  }
}

template <int KT, bool FIXED, bool COMPAT>
__device__ __forceinline__ void finish_unit(const EvalArgs &A, int64_t b, int d, int K,
                                            const int (&s)[KT], bool ok, double l, double lam,
                                            const double (&cs)[KT]) {
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
    if (COMPAT && A.logdet) A.logdet[o] = nan;
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
  if (COMPAT) {
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

// The reference's one jitter retry of a failing matrix (rare): out of line,
// so the hot path carries a single copy of the factorisation.
template <int KT, bool FIXED, bool COMPAT>
__device__ __noinline__ void eval_retry(const EvalArgs &A, const double *src, int64_t b, int d,
                                        int K) {
  int s[KT];
  unit_indices<KT, FIXED>(A, b, K, s);
  double a[KT * (KT + 1) / 2];
  double cs[KT];
  double l = 0.0, lam = 0.0;
  load_matrix<KT, FIXED>(A, src, b, d, K, s, a, true);
  const bool ok = ldl_invdiag<KT, FIXED, COMPAT>(a, K, cs, l, lam);
  finish_unit<KT, FIXED, COMPAT>(A, b, d, K, s, ok, l, lam, cs);
}

// TM = float: the FP32 fast path (factorisation in FP32, log products and
// the epilogue in FP64; a failing pivot reruns the unit through the FP64
// path with the reference's jitter rule).
template <int KT, bool FIXED, bool COMPAT, typename TM = double>
__device__ __forceinline__ void eval_unit(const EvalArgs &A, const TM *src, int64_t b, int d,
                                          int kdyn, const int (&s)[KT]) {
  const int K = FIXED ? KT : kdyn;
  TM a[KT * (KT + 1) / 2];
  double cs[KT];
  double l = 0.0, lam = 0.0;
  load_matrix<KT, FIXED, TM>(A, src, b, d, K, s, a, false);
  if (!ldl_invdiag<KT, FIXED, COMPAT, TM>(a, K, cs, l, lam)) {
    if constexpr (sizeof(TM) == sizeof(double))
      eval_retry<KT, FIXED, COMPAT>(A, reinterpret_cast<const double *>(src), b, d, K);
    else
      eval_retry<KT, FIXED, COMPAT>(A, A.src, b, d, K);
    return;
  }
  finish_unit<KT, FIXED, COMPAT>(A, b, d, K, s, true, l, lam, cs);
}

// Register budget per order (min resident CTAs of 128 threads): the
// compiler would otherwise keep every gathered element in flight (190+
// registers at K = 10, 8 warps/SM); capping it trades a little ILP for
// 2-4x the resident warps.
template <int KT>
struct EvalOcc {
  static constexpr int value = KT <= 4 ? 8 : KT <= 8 ? 4 : KT <= 10 ? 3 : KT <= 12 ? 2 : 1;
};

// Grid-stride over (n-plet, dataset) units, dataset fastest.  SMEM: the
// whole correlation matrix (small N x N x D, e.g. 7.2 KB for N = 30) is
// staged once per CTA and gathered from shared memory instead of L1/L2.
template <int KT, bool FIXED, bool COMPAT, bool SMEM, typename TM = double>
__global__ void __launch_bounds__(128, EvalOcc<KT>::value) k_eval(const EvalArgs A, int kdyn) {
  extern __shared__ __align__(16) unsigned char sRraw[];
  TM *sR = reinterpret_cast<TM *>(sRraw);
  const TM *src;
  if constexpr (sizeof(TM) == sizeof(double))
    src = reinterpret_cast<const TM *>(A.src);
  else
    src = reinterpret_cast<const TM *>(A.src32);
  if (SMEM) {
    const int n = A.N * A.N * A.D;
    for (int x = threadIdx.x; x < n; x += blockDim.x) sR[x] = __ldg(src + x);
    __syncthreads();
    src = sR;
  }
  const int64_t units = A.B * A.D;
  const int K = FIXED ? KT : kdyn;
  int s[KT];
  if (!A.idx && !A.mats) {
    // unranking mode (exhaustive segments): each thread takes a contiguous
    // chunk of units (dataset fastest), unranks its first n-plet once and
    // steps to the lexicographic successor -- the per-unit unranking was a
    // serial chain of ~N dependent binomial loads (~20% of k_eval<16>'s
    // stall samples, round-2 ncu).  Stores are per-thread contiguous.
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t per = (units + nth - 1) / nth;
    const int64_t u0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * per;
    const int64_t u1 = u0 + per < units ? u0 + per : units;
    int64_t cur_b = -1;
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t b = u / A.D;
      const int d = (int)(u - b * A.D);
      if (b != cur_b) {
        if (cur_b >= 0) {
          lex_successor<KT>(s, K, A.N);
        } else {
          unrank_lex(A.r0 + (uint64_t)b, K, A.N, s);
        }
        cur_b = b;
      }
      eval_unit<KT, FIXED, COMPAT, TM>(A, src, b, d, kdyn, s);
    }
    return;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < units;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / A.D;
    const int d = (int)(t - b * A.D);
    unit_indices<KT, FIXED>(A, b, K, s);
    eval_unit<KT, FIXED, COMPAT, TM>(A, src, b, d, kdyn, s);
  }
}

constexpr int kEvalSmemMax = 48 * 1024;

template <int KT, bool FIXED, bool COMPAT, bool SMEM, typename TM = double>
static int launch_k(const EvalArgs &A, int K, int64_t n, cudaStream_t s) {
  const int smem = SMEM ? (int)(sizeof(TM) * A.N * A.N * A.D) : 0;
  static thread_local int cap_for = -1, cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cap_for != dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eval<KT, FIXED, COMPAT, SMEM, TM>, 128,
                                                  SMEM ? kEvalSmemMax : 0);
    cap = sms * (per > 0 ? per : 1);
    cap_for = dev;
  }
  const int64_t want = (n + 127) / 128;
  const int grid = (int)(want < cap ? want : cap);
  k_eval<KT, FIXED, COMPAT, SMEM, TM><<<grid, 128, smem, s>>>(A, K);
  return check_launch("k_eval");
}

// WITH_COMPAT: also instantiate the entropy_terms variant (log det and the
// inverse diagonal in Sigma space); large fixed orders route it to the
// runtime-K kernel instead (compile time).
template <int KT, bool FIXED, bool WITH_COMPAT = true, bool WITH_FP32 = false>
static int launch_one(const EvalArgs &A, int K, cudaStream_t s) {
  int64_t n = A.B * (int64_t)A.D;
  if (n == 0) return HOI_OK;
  const bool compat = A.logdet || A.invdiag;
  if constexpr (WITH_FP32) {
    if (A.fp32 && A.src32 && !compat && !A.mats) {
      const bool sm32 = sizeof(float) * A.N * A.N * A.D <= (size_t)kEvalSmemMax;
      return sm32 ? launch_k<KT, FIXED, false, true, float>(A, K, n, s)
                  : launch_k<KT, FIXED, false, false, float>(A, K, n, s);
    }
  }
  const bool smem = !A.mats && sizeof(double) * A.N * A.N * A.D <= (size_t)kEvalSmemMax;
  if (compat) {
    if (!WITH_COMPAT) return -1;
    return smem ? launch_k<KT, FIXED, true, true>(A, K, n, s) : launch_k<KT, FIXED, true, false>(A, K, n, s);
  }
  return smem ? launch_k<KT, FIXED, false, true>(A, K, n, s) : launch_k<KT, FIXED, false, false>(A, K, n, s);
}

// fixed-order dispatchers, one per translation unit (eval_k*.cu); each
// returns -1 when K is not one of its orders or the variant is not built
int launch_eval_k1_12(const EvalArgs &A, int K, cudaStream_t s);
int launch_eval_k13_16(const EvalArgs &A, int K, cudaStream_t s);
int launch_eval_generic(const EvalArgs &A, int K, cudaStream_t s);
int launch_eval_group(const EvalArgs &A, int K, cudaStream_t s);  // 17 <= K <= 32
int launch_eval_pipe(const EvalArgs &A, int K, cudaStream_t s);   // 4 <= K <= 12, R in L2
int launch_eval_hybrid(const EvalArgs &A, int K, cudaStream_t s); // 17 <= K <= 23, FP64 measures

}  // namespace hoib
