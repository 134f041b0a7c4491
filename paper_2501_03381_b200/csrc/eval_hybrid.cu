// Engine 1, orders 17..23: one thread per (n-plet, dataset) unit with a
// bordered LDL^T, so the register file holds only the leading KR x KR block.
//
// A K = 17..23 packed triangle (153-276 doubles) does not fit in 255
// registers: the fixed-K register kernel spills kilobytes per thread and the
// group kernel (eval_group.cu) splits a unit over G threads that exchange
// every column through shared memory.  Here the factorisation is reordered
// so the tail rows never live in registers as a block:
//
//   A = [A11 A12; A21 A22],  A11 = L11 D1 L11^T (registers, right-looking)
//   tail row i:  z = L11^-1 a_i (forward solve), l_i = D1^-1 z (stored to
//                the thread's shared-memory scratch, conflict-free
//                [entry][thread] layout), Schur column
//                c_ii' = a_ii' - z . l_i'  for the tail rows i' <= i
//   C = A22 - L21 D1 L21^T = L22 D2 L22^T (TT = K - KR rows; factorised in
//                the shared scratch too, beside the multipliers)
//   U = L^-1:  U11 = L11^-1, U22 = L22^-1 in place, U21 = -U22 (L21 U11)
//   (R_S^-1)_jj = sum_i U_ij^2 / d_i over both blocks.
//
// The arithmetic is the reference's (ref nplet_engine.py:267-281 restated:
// log det from the pivots, every leave-one-out determinant from
// det(R_S) (R_S^-1)_jj) and ~KR^2 TT extra shared-memory words per unit move
// instead of K^3 / 3 register-resident FMAs' operands.  Measures and the
// failure rule as k_eval (ref measures.py:41-81, nplet_engine.py:237-264): a
// non-positive pivot reruns the unit with the jittered diagonal, a second
// failure records (row, dataset) and writes NaN.
//
// The loops over tail rows are deliberately not unrolled: unrolled, the
// scheduler interleaved the rows and kept all their gathers and partial
// sums live (3-5 KB of spills per thread); rolled, KR = 14 spills ~0.5 KB.
#include "eval_kernels.cuh"

namespace hoib {
namespace {

__device__ __forceinline__ int opaque_zero(double v) {
  int z;
  asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(__double2loint(v)));
  return z;
}

template <int K, int KR, int NT, bool JIT>
__device__ __forceinline__ bool hyb_unit(const double *__restrict__ src, const EvalArgs &A, int d,
                                         const int (&s)[K], double *__restrict__ x, double eps,
                                         double &l, double &lam) {
  constexpr int TT = K - KR;
  const int N = A.N, D = A.D;
  auto R = [&](int i, int j) -> double { return src[(s[i] * N + s[j]) * D + d]; };
  auto DG = [&](int i) -> double {
    if (!JIT) return 1.0;
    const double sc = A.sdiag ? A.sdiag[(int64_t)d * N + s[i]] : 1.0;
    return 1.0 + eps / sc;
  };
  auto X = [&](int t, int m) -> double & { return x[(t * KR + m) * NT]; };
  // tail Schur complement / its factor, packed lower triangle, also scratch
  auto Cs = [&](int t, int u) -> double & { return x[(TT * KR + TRI(t, u)) * NT]; };

  // ---- leading block: right-looking LDL^T in registers (rows bottom-up so
  // the unscaled column stays readable; the diagonal slot ends as 1/d_j)
  double a[KR * (KR + 1) / 2];
#pragma unroll
  for (int i = 0; i < KR; ++i) {
#pragma unroll
    for (int j = 0; j < i; ++j) a[TRI(i, j)] = R(i, j);
    a[TRI(i, i)] = DG(i);
  }
  LogProd pd;
  pd.init();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < KR; ++j) {
    const double dj = a[TRI(j, j)];
    bad |= !(dj > 0.0);
    pd.mul(dj);
    if ((j & 7) == 7) pd.renorm();
    const double r = pivot_rcp(dj);
    a[TRI(j, j)] = r;
#pragma unroll
    for (int i = KR - 1; i > j; --i) {
      const double lij = a[TRI(i, j)] * r;
#pragma unroll
      for (int m = j + 1; m <= i; ++m) a[TRI(i, m)] = fma(-lij, a[TRI(m, j)], a[TRI(i, m)]);
      a[TRI(i, j)] = lij;
    }
  }

  // ---- tail rows: forward solve, multipliers to scratch, Schur complement.
  // Each row's gathers take an opaque zero offset computed from the previous
  // row's result, so the scheduler cannot hoist all K (K - 1) / 2 loads to
  // the top of the unit (they would stay live and spill).
  int dep = opaque_zero(a[TRI(KR - 1, KR - 1)]);
#pragma unroll 1
  for (int t = 0; t < TT; ++t) {
    const int i = KR + t;
    const double *srow = src + dep;
    auto RT = [&](int j) -> double { return srow[(s[i] * N + s[j]) * D + d]; };
    double z[KR];
#pragma unroll
    for (int m = 0; m < KR; ++m) {
      double v = RT(m);
#pragma unroll
      for (int p = 0; p < m; ++p) v = fma(-a[TRI(m, p)], z[p], v);
      z[m] = v;
    }
#pragma unroll 1
    for (int u = 0; u < t; ++u) {
      double v = RT(KR + u);
#pragma unroll
      for (int m = 0; m < KR; ++m) v = fma(-z[m], X(u, m), v);
      Cs(t, u) = v;
    }
    double v = DG(i);
#pragma unroll
    for (int m = 0; m < KR; ++m) {
      const double lm = z[m] * a[TRI(m, m)];
      v = fma(-z[m], lm, v);
      X(t, m) = lm;
    }
    Cs(t, t) = v;
    dep = opaque_zero(v);
  }

  // ---- tail block: LDL^T of the Schur complement
#pragma unroll
  for (int j = 0; j < TT; ++j) {
    const double dj = Cs(j, j);
    bad |= !(dj > 0.0);
    pd.mul(dj);
    if (((KR + j) & 7) == 7) pd.renorm();
    const double r = pivot_rcp(dj);
    Cs(j, j) = r;
#pragma unroll
    for (int i = TT - 1; i > j; --i) {
      const double lij = Cs(i, j) * r;
#pragma unroll
      for (int m = j + 1; m <= i; ++m) Cs(i, m) = fma(-lij, Cs(m, j), Cs(i, m));
      Cs(i, j) = lij;
    }
  }
  if (bad) return false;
  pd.renorm();

  // ---- U11 = L11^-1 and U22 = L22^-1 in place (unit lower, column by column)
#pragma unroll
  for (int j = 0; j < KR; ++j) {
#pragma unroll
    for (int i = j + 1; i < KR; ++i) {
      double acc = a[TRI(i, j)];
#pragma unroll
      for (int m = j + 1; m < i; ++m) acc = fma(a[TRI(i, m)], a[TRI(m, j)], acc);
      a[TRI(i, j)] = -acc;
    }
  }
#pragma unroll
  for (int j = 0; j < TT; ++j) {
#pragma unroll
    for (int i = j + 1; i < TT; ++i) {
      double acc = Cs(i, j);
#pragma unroll
      for (int m = j + 1; m < i; ++m) acc = fma(Cs(i, m), Cs(m, j), acc);
      Cs(i, j) = -acc;
    }
  }
  // ---- W = L21 U11 row by row, over the multipliers in scratch
#pragma unroll 1
  for (int t = 0; t < TT; ++t) {
    double lr[KR];
#pragma unroll
    for (int m = 0; m < KR; ++m) lr[m] = X(t, m);
#pragma unroll
    for (int j = 0; j < KR; ++j) {
      double v = lr[j];
#pragma unroll
      for (int m = j + 1; m < KR; ++m) v = fma(lr[m], a[TRI(m, j)], v);
      X(t, j) = v;
    }
  }
  // ---- (R_S^-1)_jj = sum_i U_ij^2 / d_i; U21 = -U22 W (the sign squares away)
  LogProd pl;
  pl.init();
#pragma unroll
  for (int j = 0; j < KR; ++j) {
    double sacc = a[TRI(j, j)];
#pragma unroll
    for (int i = j + 1; i < KR; ++i) {
      const double u = a[TRI(i, j)];
      sacc = fma(u * u, a[TRI(i, i)], sacc);
    }
    double w[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) w[t] = X(t, j);
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      double u = w[t];
#pragma unroll
      for (int q = 0; q < t; ++q) u = fma(Cs(t, q), w[q], u);
      sacc = fma(u * u, Cs(t, t), sacc);
    }
    pl.mul(sacc);
    if ((j & 7) == 7) pl.renorm();
  }
#pragma unroll
  for (int t = 0; t < TT; ++t) {
    double sacc = Cs(t, t);
#pragma unroll
    for (int i = t + 1; i < TT; ++i) {
      const double u = Cs(i, t);
      sacc = fma(u * u, Cs(i, i), sacc);
    }
    pl.mul(sacc);
    if (((KR + t) & 7) == 7) pl.renorm();
  }
  pl.renorm();
  l = pd.log_value();
  lam = pl.log_value();
  return true;
}

// the reference's one jitter retry (rare): out of line, eps = 1e-10 *
// trace(Sigma_S) / k on the covariance scale (ref nplet_engine.py:237-264)
template <int K, int KR, int NT>
__device__ __noinline__ bool hyb_retry(const double *__restrict__ src, const EvalArgs &A, int d,
                                       const int (&s)[K], double *__restrict__ x, double &l,
                                       double &lam) {
  double tr = 0.0;
  if (A.sdiag) {
#pragma unroll
    for (int i = 0; i < K; ++i) tr += A.sdiag[(int64_t)d * A.N + s[i]];
  } else {
    tr = (double)K;
  }
  return hyb_unit<K, KR, NT, true>(src, A, d, s, x, 1e-10 * tr / (double)K, l, lam);
}

// resident threads per SM the register budget targets (2 CTAs of 128).
// 384 (a 170-register cap, 12 warps/SM with 64-thread CTAs) measured
// 45-53 ms for order 17 against 29.5 at 256: the spills cost more than the
// extra warps hide (scripts/exp_hyb.cu -DHYB_OCC=384 -DHYB_VARIANTS).
#ifndef HYB_OCC
#define HYB_OCC 256
#endif
template <int K, int KR, int NT, bool SMEM>
__global__ void __launch_bounds__(NT, HYB_OCC / NT) k_eval_hyb(const EvalArgs A) {
  constexpr int TT = K - KR;
  extern __shared__ __align__(16) unsigned char hyb_raw[];
  double *x = reinterpret_cast<double *>(hyb_raw) + threadIdx.x;
  const double *src = A.src;
  if (SMEM) {
    double *sR = reinterpret_cast<double *>(hyb_raw) + (TT * KR + TT * (TT + 1) / 2) * NT;
    const int n = A.N * A.N * A.D;
    for (int q = threadIdx.x; q < n; q += blockDim.x) sR[q] = __ldg(A.src + q);
    __syncthreads();
    src = sR;
  }
  const double cs_dummy[K] = {};
  const int64_t units = A.B * A.D;
  int s[K];
  auto unit = [&](int64_t b, int d) {
    double l = 0.0, lam = 0.0;
    bool ok = hyb_unit<K, KR, NT, false>(src, A, d, s, x, 0.0, l, lam);
    if (!ok) ok = hyb_retry<K, KR, NT>(src, A, d, s, x, l, lam);
    finish_unit<K, true, false>(A, b, d, K, s, ok, l, lam, cs_dummy);
  };
  if (!A.idx) {
    // unranking mode: per-thread contiguous chunks, lexicographic successor
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t per = (units + nth - 1) / nth;
    const int64_t u0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * per;
    const int64_t u1 = u0 + per < units ? u0 + per : units;
    int64_t cur_b = -1;
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t b = u / A.D;
      const int d = (int)(u - b * A.D);
      if (b != cur_b) {
        if (cur_b >= 0)
          lex_successor<K>(s, K, A.N);
        else
          unrank_lex(A.r0 + (uint64_t)b, K, A.N, s);
        cur_b = b;
      }
      unit(b, d);
    }
    return;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < units;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / A.D;
    const int d = (int)(t - b * A.D);
#pragma unroll
    for (int i = 0; i < K; ++i) s[i] = A.idx[b * A.idx_stride + i];
    unit(b, d);
  }
}

template <int K, int KR, int NT, bool SMEM>
int launch_hyb_t(const EvalArgs &A, cudaStream_t st) {
  constexpr int TT = K - KR;
  const int smem = (int)((TT * KR + TT * (TT + 1) / 2) * NT * sizeof(double) +
                         (SMEM ? sizeof(double) * A.N * A.N * A.D : 0));
  static thread_local int cap_for = -1, cap = 0, set_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cap_for != dev || smem > set_smem) {
    const int maxs = (int)((TT * KR + TT * (TT + 1) / 2) * NT * sizeof(double)) + kEvalSmemMax;
    cudaFuncSetAttribute(k_eval_hyb<K, KR, NT, SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eval_hyb<K, KR, NT, SMEM>, NT, smem);
    cap = sms * (per > 0 ? per : 1);
    cap_for = dev;
    set_smem = maxs;
  }
  const int64_t n = A.B * (int64_t)A.D;
  const int64_t want = (n + NT - 1) / NT;
  const int grid = (int)(want < cap ? want : cap);
  k_eval_hyb<K, KR, NT, SMEM><<<grid < 1 ? 1 : grid, NT, smem, st>>>(A);
  return check_launch("k_eval_hyb");
}

template <int K, int KR, int NT>
int launch_hyb(const EvalArgs &A, cudaStream_t st) {
  const bool smem = sizeof(double) * A.N * A.N * A.D <= (size_t)kEvalSmemMax;
  return smem ? launch_hyb_t<K, KR, NT, true>(A, st) : launch_hyb_t<K, KR, NT, false>(A, st);
}

}  // namespace

// -1 when the launch is not this kernel's: FP64 measures only (no
// entropy_terms outputs, no raw matrix stacks).  precision="fp32" requests
// run here in FP64 too, as they do on every kernel above order 16, so the
// two precisions give identical values at these orders.
int launch_eval_hybrid(const EvalArgs &A, int K, cudaStream_t s) {
  if (A.mats || A.logdet || A.invdiag || !A.out) return -1;
  if (A.B * (int64_t)A.D == 0) return HOI_OK;
  upload_binomials();
  switch (K) {
    // (KR, threads per CTA) per order, measured on B200 (whole cfg4 orders,
    // ms; the group kernel in brackets): KR = 13 | 14 | 15 for K = 17:
    // 31.6 | 29.5 | 32.8 (71.0); K = 18: 29.0 | 27.0 | 28.6 (52.0); K = 19:
    // 23.6 (KR 13) | 21.4 | 22.9 (42.3); K = 20: KR 14 x 128 threads 15.4,
    // 15 x 128 17.6, 14 x 96 18.8, 13 x 64 20.2 (24.2); K = 21: 16 x 128
    // 11.1, 15 x 96 11.4 (19.2); K = 22: 15 x 64 6.8, 16 x 96 7.0 (8.2).
    // The scratch (TT KR + TT (TT + 1) / 2 doubles per thread) bounds the
    // CTAs per SM; KR = 14 spills ~0.5 KB, which costs less than the
    // bigger tail of a smaller KR.  Orders 14-16 stay on the register
    // kernel (K = 16: 28.8 ms there, 30.4 bordered at KR = 13 or 14).
    case 17: return launch_hyb<17, 14, 128>(A, s);
    case 18: return launch_hyb<18, 14, 128>(A, s);
    case 19: return launch_hyb<19, 14, 128>(A, s);
    case 20: return launch_hyb<20, 14, 128>(A, s);
    case 21: return launch_hyb<21, 16, 128>(A, s);
    case 22: return launch_hyb<22, 15, 64>(A, s);
    case 23: return launch_hyb<23, 16, 64>(A, s);   // 2.73 ms (group 3.03)
    default: return -1;
  }
}

}  // namespace hoib
