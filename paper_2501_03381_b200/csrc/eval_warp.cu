// Engine 1, orders 17..32: one warp per (n-plet, dataset) unit.
//
// Past K = 16 a thread-per-unit register triangle spills (5-21 KB per
// thread at K = 17..22) and the runtime-K kernel runs from local memory
// (~1 TF/s).  Here lane i owns row i of R_S in registers (K doubles):
//
//   LDL^T, right-looking: at step j every lane publishes its column-j entry
//   to a per-warp shared vector, the pivot d_j and the column are read back
//   as broadcasts (128-bit loads), and lane i updates its row
//   a[i][m] -= l_ij a[m][j] for m > j (the upper part of a row is scratch).
//   log det = log prod d_j (LogProd, one log).
//
//   Inverse diagonal: L goes to shared memory (row-padded so rows are
//   16-byte aligned); lane j forward-substitutes column j of U = L^-1
//   (u_i = -sum_{m<i} L_im u_m, broadcast loads of L) and forms
//   (R_S^-1)_jj = sum_i u_i^2 / d_i; lambda = sum_j log (R_S^-1)_jj is a
//   warp sum of one log per lane.
//
// Same failure rule as the thread kernel (ref nplet_engine.py:237-264): a
// non-positive pivot retries the unit once with the jittered diagonal, a
// second failure records (row, dataset) and writes NaN.
#include "eval_kernels.cuh"

namespace hoib {
namespace {

constexpr int kWK = 32;                 // max order handled here
constexpr int kWarps = 8;               // warps per CTA
// row i of L (i entries, padded to even) starts at sum_{t=2..i} (t & ~1):
// 2h^2 for i = 2h, 2h(h+1) for i = 2h+1 (closed form: usable with a runtime i)
__host__ __device__ constexpr int lrow(int i) {
  return (i & 1) ? 2 * (i >> 1) * ((i >> 1) + 1) : 2 * (i >> 1) * (i >> 1);
}

template <int KT>
struct WarpSmem {
  double col[kWarps][KT];
  double dinv[kWarps][KT];
  double L[kWarps][lrow(KT) + 2];
  int idx[kWarps][KT];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// KT: the order bound of this instantiation (K in (KT-4, KT]); every
// per-row loop is unrolled to KT, so KT close to K keeps predicated-off
// slots and registers down.
template <int KT, bool COMPAT, bool SMEM>
__global__ void __launch_bounds__(32 * kWarps, 2) k_eval_warp(const EvalArgs A, int K) {
  extern __shared__ __align__(16) double dynR[];
  __shared__ __align__(16) WarpSmem<KT> sm;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int N = A.N, D = A.D;
  const double *src = A.src;
  if (SMEM) {
    const int n = N * N * D;
    for (int x = threadIdx.x; x < n; x += blockDim.x) dynR[x] = __ldg(A.src + x);
    __syncthreads();
    src = dynR;
  }
  double *col = sm.col[w], *dinv = sm.dinv[w], *Ls = sm.L[w];
  int *sidx = sm.idx[w];
  // each warp takes a contiguous chunk of units (dataset fastest), so in
  // unranking mode it unranks once and then steps to the lexicographic
  // successor (one ballot) instead of unranking every n-plet serially
  const int64_t units = A.B * (int64_t)D;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w;
  const int64_t per = (units + nw - 1) / nw;
  const int64_t u_begin = gw * per, u_end = u_begin + per < units ? u_begin + per : units;
  int64_t cur_b = -1;
  for (int64_t u = u_begin; u < u_end; ++u) {
    const int64_t b = u / D;
    const int d = (int)(u - b * D);
    // ---------------------------------------------------------- indices ----
    if (b != cur_b) {
      if (A.idx) {
        if (lane < K) sidx[lane] = A.idx[b * A.idx_stride + lane];
      } else if (cur_b >= 0 && b == cur_b + 1) {
        // successor: rightmost position p with s[p] < N - K + p is
        // incremented, the positions after it follow consecutively
        const int sv = lane < K ? sidx[lane] : 0;
        const unsigned can = __ballot_sync(0xffffffffu, lane < K && sv < N - K + lane);
        const int p = 31 - __clz(can);
        const int sp = __shfl_sync(0xffffffffu, sv, p);
        __syncwarp();
        if (lane >= p && lane < K) sidx[lane] = sp + 1 + (lane - p);
      } else if (lane == 0) {
        int s[KT];
        uint64_t r = A.r0 + (uint64_t)b;
        int c = 0;
#pragma unroll
        for (int p = 0; p < KT; ++p) {
          if (p < K) {
            while (c < N) {
              const uint64_t bb = binom_l1(N - 1 - c, K - 1 - p);
              if (bb <= r) {
                r -= bb;
                ++c;
              } else {
                break;
              }
            }
            s[p] = c++;
          }
        }
#pragma unroll
        for (int p = 0; p < KT; ++p)
          if (p < K) sidx[p] = s[p];
      }
      cur_b = b;
    }
    __syncwarp();
    const int si = lane < K ? sidx[lane] : 0;
    double sg_lane = 1.0;
    if (A.sdiag && lane < K) sg_lane = A.sdiag[(int64_t)d * N + si];
    bool ok = false;
    double l = 0.0, lam = 0.0, cs = 0.0;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
      // ------------------------------------------------------- gather ----
      double r[KT];
      const double *row = src + (si * N) * D + d;
#pragma unroll
      for (int m = 0; m < KT; ++m) {
        double v = 0.0;
        if (m < K && lane < K) {
          if (m < lane) v = row[sidx[m] * D];
          else if (m == lane) v = 1.0;
        }
        r[m] = v;
      }
      if (attempt == 1) {   // the reference's jitter: Sigma_S + eps I, eps = 1e-10 tr / K
        const double tr = A.sdiag ? warp_sum(lane < K ? sg_lane : 0.0) : (double)K;
        const double eps = 1e-10 * tr / (double)K;
#pragma unroll
        for (int m = 0; m < KT; ++m)
          if (m == lane && lane < K) r[m] += eps / sg_lane;
      }
      // ---------------------------------------------------------- LDL ----
      LogProd pd;
      pd.init();
      bool good = true;
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        if (j < K) {
          if (lane < KT) col[lane] = r[j];   // lanes >= KT own no row
          __syncwarp();
          const double dj = col[j];
          if (!(dj > 0.0)) {
            good = false;
            __syncwarp();
            break;
          }
          pd.mul(dj);
          if ((j & 7) == 7) pd.renorm();
          const double rp = __drcp_rn(dj);
          const double lij = r[j] * rp;
#pragma unroll
          for (int mm = (j + 1) & ~1; mm < KT; mm += 2) {
            if (mm < K) {
              const double2 v = *reinterpret_cast<const double2 *>(col + mm);
              if (mm > j) r[mm] = fma(-lij, v.x, r[mm]);
              if (mm + 1 < K) r[mm + 1] = fma(-lij, v.y, r[mm + 1]);
            }
          }
          r[j] = lij;
          if (lane == j) dinv[j] = rp;
          __syncwarp();
        }
      }
      if (!good) continue;
      pd.renorm();
      l = pd.log_value();
      // ------------------------------------------- L -> shared memory ----
#pragma unroll
      for (int m = 0; m < KT - 1; ++m)
        if (m < lane && lane < K) Ls[lrow(lane) + m] = r[m];
      __syncwarp();
      // ----------------------------- column `lane` of U = L^-1, (R^-1)_jj --
      double uu[KT];
#pragma unroll
      for (int m = 0; m < KT; ++m) uu[m] = (m == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int i = 1; i < KT; ++i) {
        if (i < K) {
          double acc = 0.0;
#pragma unroll
          for (int m = 0; m < i; m += 2) {
            const double2 v = *reinterpret_cast<const double2 *>(Ls + lrow(i) + m);
            acc = fma(v.x, uu[m], acc);
            if (m + 1 < i) acc = fma(v.y, uu[m + 1], acc);
          }
          if (i > lane) uu[i] = -acc;
        }
      }
      double c = 0.0;
#pragma unroll
      for (int i = 0; i < KT; ++i)
        if (i < K) c = fma(uu[i] * uu[i], dinv[i], c);
      cs = c;
      lam = warp_sum(lane < K ? log(c) : 0.0);
      ok = true;
      __syncwarp();
    }
    // ----------------------------------------------------------- output ----
    const int64_t ob = A.row_map ? A.row_map[b] : A.out_row0 + b;
    const int64_t o = ob * D + d;
    if (!ok) {
      if (lane == 0) {
        const int slot = atomicAdd(A.err_count, 1);
        if (slot < A.err_cap) {
          A.err_coords[2 * slot] = ob;
          A.err_coords[2 * slot + 1] = d;
        }
        const double nan = __longlong_as_double(0x7ff8000000000000ll);
        if (A.out)
          for (int q = 0; q < 4; ++q) A.out[q * A.plane + o] = nan;
        if (COMPAT && A.logdet) A.logdet[o] = nan;
      }
      __syncwarp();
      continue;
    }
    if (A.out && lane == 0) {
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
      // Sigma-space values (entropy_terms compat)
      const double lsg = warp_sum(lane < K && A.sdiag ? log(sg_lane) : 0.0);
      if (A.invdiag && lane < K) {
        const double v = cs / sg_lane;
        if (A.inv_n > 0)
          A.invdiag[o * A.inv_n + si] = v;
        else
          A.invdiag[o * K + lane] = v;
      }
      if (A.logdet && lane == 0) A.logdet[o] = l + lsg;
    }
    __syncwarp();
  }
}

template <int KT, bool COMPAT, bool SMEM>
int launch_warp(const EvalArgs &A, int K, cudaStream_t s) {
  const int smem = SMEM ? (int)(sizeof(double) * A.N * A.N * A.D) : 0;
  static thread_local int cap_for = -1, cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cap_for != dev) {
    if (SMEM)
      cudaFuncSetAttribute(k_eval_warp<KT, COMPAT, SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kEvalSmemMax);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eval_warp<KT, COMPAT, SMEM>, 32 * kWarps,
                                                  SMEM ? kEvalSmemMax : 0);
    cap = sms * (per > 0 ? per : 1);
    cap_for = dev;
  }
  const int64_t n = A.B * (int64_t)A.D;
  const int64_t want = (n + kWarps - 1) / kWarps;
  const int grid = (int)(want < cap ? want : cap);
  k_eval_warp<KT, COMPAT, SMEM><<<grid, 32 * kWarps, smem, s>>>(A, K);
  return check_launch("k_eval_warp");
}

template <int KT>
int pick(const EvalArgs &A, int K, bool compat, bool smem, cudaStream_t s) {
  if (compat) return smem ? launch_warp<KT, true, true>(A, K, s) : launch_warp<KT, true, false>(A, K, s);
  return smem ? launch_warp<KT, false, true>(A, K, s) : launch_warp<KT, false, false>(A, K, s);
}

}  // namespace

int launch_eval_warp(const EvalArgs &A, int K, cudaStream_t s) {
  if (K < 17 || K > kWK || A.mats) return -1;
  upload_binomials();
  const int64_t n = A.B * (int64_t)A.D;
  if (n == 0) return HOI_OK;
  const bool compat = A.logdet || A.invdiag;
  const bool smem = sizeof(double) * A.N * A.N * A.D <= (size_t)kEvalSmemMax;
  if (K <= 20) return pick<20>(A, K, compat, smem, s);
  if (K <= 24) return pick<24>(A, K, compat, smem, s);
  if (K <= 28) return pick<28>(A, K, compat, smem, s);
  return pick<32>(A, K, compat, smem, s);
}

}  // namespace hoib
