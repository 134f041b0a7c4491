// Engine 1, orders 17..32: G threads per (n-plet, dataset) unit, 32/G units
// per warp, the whole factorisation in registers with compile-time indices.
//
// Thread t of a group owns rows i = t + G*m (m < M, KT = G*M >= K).  Row
// slot m is stored padded to G*(m+1) columns, so every register index is a
// compile-time (m, column) pair and the thread id only enters predicates and
// shared-memory addresses -- the matrix stays in registers (a packed
// triangle indexed by a runtime row went to local memory).  Orders K < KT
// are padded with identity rows: pivots 1, no updates, log 1 = 0.
//
//   LDL^T, right-looking: step j publishes column j (each thread its rows'
//   entries) to a per-unit shared vector; every thread reads the pivot and
//   the column back as broadcasts and updates a[i][l] -= l_ij a[l][j] for
//   its rows (entries right of a row's diagonal are scratch).
//   W = L^-1 in place, right-looking: step j publishes row j of W (final by
//   then), rows i > j apply w[i][c] -= l_ij w[j][c] and set w[i][j] = -l_ij.
//   (R_S^-1)_cc = sum_i w[i][c]^2 / d_i: per-thread column partials go
//   through shared memory, thread t sums the columns c = t (mod G) it owns.
//
// Work per unit ~ KT^3/3 FMAs spread over G lanes (the warp-per-unit kernel
// issues ~KT^2 warp-wide FMAs per unit with half its lanes idle or on the
// scratch half).  Failure rule as the other kernels (ref
// nplet_engine.py:237-264): a non-positive pivot retries the unit once with
// the jittered diagonal; a second failure records (row, dataset) and writes
// NaN.
#include "eval_kernels.cuh"

namespace hoib {
namespace {

constexpr int kGWarps = 4;   // warps per CTA

template <int G, int M>
struct GrpCore {                       // one per unit (group); 16-byte vector accesses
  double vec[2][G * M + 2];            // broadcast vector, double-buffered by step (pair) parity
  double red[G][G * M];                // column partials of the inverse diagonal; during the
                                       // blocked LDL its first two rows hold column j+1 (even
                                       // row length: 16-byte aligned rows)
  int idx[G * M + ((G * M) & 3 ? 4 - ((G * M) & 3) : 0)];   // variable ids (16-byte multiple)
};
// Unit stride an odd multiple of 16 bytes: the 32/G groups of a warp read
// their broadcast vectors at the same offset, and a stride that is a
// multiple of 128 B put them all on the same banks (an 8-way conflict that
// cost (4,6) a third of its speed).
template <int G, int M>
struct __align__(16) GrpSmem : GrpCore<G, M> {
  char pad[sizeof(GrpCore<G, M>) % 32 == 16 ? 32 : 16];
};

// Control flow is warp-uniform (every group of a warp runs the same unit
// count, attempt count and steps), so group exchanges use full-warp
// __syncwarp() / shuffles: a partial-mask __syncwarp(gmask) lowers to a
// MATCH.ANY + REDUX + VOTE convergence check whose latency was ~23% of the
// (2,9) kernel's stall samples (round-2 ncu, cfg4 order 17).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G, int M, int MINB, bool COMPAT, bool SMEM>
__global__ void __launch_bounds__(32 * kGWarps, MINB) k_eval_grp(const EvalArgs A, int K) {
  constexpr int KT = G * M, U = 32 / G, S = G * M * (M + 1) / 2;
  // LDL^T two columns per broadcast where the extra live values fit in
  // registers; measured on B200 (cfg4 order segments): (2,9) K 17-18
  // 3.2-3.7 -> 4.4-5.2 TF/s, (4,5) K 19-20 +4%; (4,6) and (4,7) run 2-5%
  // slower blocked (more spills), so they keep one column per broadcast.
  constexpr bool kBlocked2 = G == 2 || (G == 4 && M == 5);
  // dynamic shared memory: the groups' exchange slots (sizes above the 48 KB
  // static limit for (2,10)), then the CTA's copy of R in SMEM mode
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  GrpSmem<G, M> *usm = reinterpret_cast<GrpSmem<G, M> *>(dyn_raw);
  double *dynR = reinterpret_cast<double *>(dyn_raw + sizeof(GrpSmem<G, M>) * kGWarps * U);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = lane % G, g = lane / G;
  const int N = A.N, D = A.D;
  const double *src = A.src;
  if (SMEM) {
    const int n = N * N * D;
    for (int x = threadIdx.x; x < n; x += blockDim.x) dynR[x] = __ldg(A.src + x);
    __syncthreads();
    src = dynR;
  }
  GrpSmem<G, M> &sm = usm[w * U + g];
  // each group takes a contiguous chunk of units (dataset fastest): in
  // unranking mode it unranks once, then steps to the lexicographic successor.
  // Every group runs `per` iterations; past its chunk's end it recomputes
  // the last unit and stores nothing (warp-uniform trip count).
  const int64_t units = A.B * (int64_t)D;
  const int64_t ng = (int64_t)gridDim.x * kGWarps * U;
  const int64_t gid = ((int64_t)blockIdx.x * kGWarps + w) * U + g;
  const int64_t per = (units + ng - 1) / ng;
  const int64_t u_begin = gid * per, u_end = u_begin + per < units ? u_begin + per : units;
  int64_t cur_b = -1;
  for (int64_t it = 0; it < per; ++it) {
    const bool valid = u_begin + it < u_end;
    const int64_t u = valid ? u_begin + it : (u_end > u_begin ? u_end - 1 : units - 1);
    const int64_t b = u / D;
    const int d = (int)(u - b * D);
    // ------------------------------------------------------------ indices ----
    const bool fresh = b != cur_b;
    __syncwarp();                              // previous unit's idx reads done
    if (fresh) {
      if (A.idx) {
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (t + G * m < K) sm.idx[t + G * m] = A.idx[b * A.idx_stride + t + G * m];
      } else if (t == 0) {
        if (cur_b >= 0 && b == cur_b + 1) {
          // successor: the rightmost position p with s[p] < N - K + p is
          // incremented, the positions after it follow consecutively
          int p = K - 1;
          while (p > 0 && sm.idx[p] >= N - K + p) --p;
          const int v = sm.idx[p] + 1;
          for (int q = p; q < K; ++q) sm.idx[q] = v + (q - p);
        } else {
          uint64_t r = A.r0 + (uint64_t)b;
          int c = 0;
          for (int p = 0; p < K; ++p) {
            while (c < N) {
              const uint64_t bb = binom_l1(N - 1 - c, K - 1 - p);
              if (bb <= r) {
                r -= bb;
                ++c;
              } else {
                break;
              }
            }
            sm.idx[p] = c++;
          }
        }
      }
      cur_b = b;
    }
    __syncwarp();
    int si[M];
    double sg[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int i = t + G * m;
      si[m] = i < K ? sm.idx[i] : 0;
      sg[m] = (A.sdiag && i < K) ? A.sdiag[(int64_t)d * N + si[m]] : 1.0;
    }
    bool ok = false;
    double l = 0.0, lam = 0.0;
    double inv[M];
    for (int attempt = 0; attempt < 2; ++attempt) {
      // the jitter retry runs for the whole warp when any group needs it;
      // groups that already have their values recompute and discard
      if (attempt == 1 && __all_sync(0xffffffffu, ok)) break;
      // ----------------------------------------------------------- gather ----
      double a[S];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int i = t + G * m;
        const double *row = src + ((int64_t)si[m] * N) * D + d;
#pragma unroll
        for (int c = 0; c < G * (m + 1); ++c) {
          double v = c == i ? 1.0 : 0.0;
          if (c < i && i < K) v = row[(int64_t)sm.idx[c] * D];
          a[G * m * (m + 1) / 2 + c] = v;
        }
      }
      if (attempt == 1) {   // the reference's jitter: Sigma_S + eps I, eps = 1e-10 tr / K
        double tr = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) tr += t + G * m < K ? sg[m] : 0.0;
        tr = A.sdiag ? group_sum<G>(tr) : (double)K;
        const double eps = 1e-10 * tr / (double)K;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int i = t + G * m;
#pragma unroll
          for (int c = 0; c < G * (m + 1); ++c)
            if (c == i && i < K) a[G * m * (m + 1) / 2 + c] += eps / sg[m];
        }
      }
      // -------------------------------------------------------------- LDL ----
      LogProd pd;
      pd.init();
      bool good = true;
      double dinv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) dinv[m] = 1.0;
      if constexpr (kBlocked2) {
        // two columns per broadcast: columns j and j+1 are published as they
        // stand before step j; every thread derives the step-j update of
        // column j+1 (a'[c][j+1] = a[c][j+1] - a[c][j] l_(j+1)j) and applies
        // both rank-1 updates to its rows -- one group sync per two columns.
#pragma unroll
        for (int j = 0; j < KT; j += 2) {
          if (j < K) {
            const bool two = j + 1 < K;
            double *v0 = sm.vec[(j >> 1) & 1];
            double *v1 = sm.red[(j >> 1) & 1];
#pragma unroll
            for (int m = 0; m < M; ++m) {
              const int o = G * m * (m + 1) / 2;
              if (G * (m + 1) > j) v0[t + G * m] = a[o + j];
              if (G * (m + 1) > j + 1) v1[t + G * m] = a[o + j + 1];
            }
            __syncwarp();
            const double dj = v0[j];
            good &= dj > 0.0;   // flagged, not branched on (see ldl_invdiag)
            pd.mul(dj);
            const double rp = pivot_rcp(dj);
            if (t == j % G) dinv[j / G] = rp;
            if (!two) {
#pragma unroll
              for (int m = 0; m < M; ++m) {
                if (G * (m + 1) > j + 1) {
                  const int o = G * m * (m + 1) / 2;
                  const double lij = a[o + j] * rp;
#pragma unroll
                  for (int c = j + 2; c < G * (m + 1); c += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(v0 + c);
                    a[o + c] = fma(-lij, v.x, a[o + c]);
                    a[o + c + 1] = fma(-lij, v.y, a[o + c + 1]);
                  }
                  a[o + j + 1] = fma(-lij, v0[j + 1], a[o + j + 1]);
                  a[o + j] = lij;
                }
              }
              continue;
            }
            const double u = v0[j + 1];              // a[j+1][j]
            const double l10 = u * rp;               // L[j+1][j]
            const double dj1 = fma(-u, l10, v1[j + 1]);
            good &= dj1 > 0.0;   // flagged, not branched on (see ldl_invdiag)
            pd.mul(dj1);
            if ((j & 7) == 6) pd.renorm();
            const double rp1 = pivot_rcp(dj1);
            if (t == (j + 1) % G) dinv[(j + 1) / G] = rp1;
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (G * (m + 1) > j + 1) {             // the slot has rows below j
                const int o = G * m * (m + 1) / 2;
                const double lij = a[o + j] * rp;
                const double li1 = fma(-lij, u, a[o + j + 1]) * rp1;
#pragma unroll
                for (int c = j + 2; c < G * (m + 1); c += 2) {
                  const double2 w0 = *reinterpret_cast<const double2 *>(v0 + c);
                  const double2 w1 = *reinterpret_cast<const double2 *>(v1 + c);
                  const double n0 = fma(-w0.x, l10, w1.x), n1 = fma(-w0.y, l10, w1.y);
                  a[o + c] = fma(-li1, n0, fma(-lij, w0.x, a[o + c]));
                  a[o + c + 1] = fma(-li1, n1, fma(-lij, w0.y, a[o + c + 1]));
                }
                a[o + j] = lij;
                a[o + j + 1] = li1;
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          if (j < K) {
            double *vec = sm.vec[j & 1];
  #pragma unroll
            for (int m = 0; m < M; ++m)
              if (G * (m + 1) > j) vec[t + G * m] = a[G * m * (m + 1) / 2 + j];
            __syncwarp();
            const double dj = vec[j];
            good &= dj > 0.0;   // flagged, not branched on (see ldl_invdiag)
            pd.mul(dj);
            if ((j & 7) == 7) pd.renorm();
            const double rp = pivot_rcp(dj);
            if (t == j % G) dinv[j / G] = rp;
  #pragma unroll
            for (int m = 0; m < M; ++m) {
              if (G * (m + 1) > j + 1) {         // the slot has rows below j
                const int o = G * m * (m + 1) / 2;
                const double lij = a[o + j] * rp;
  #pragma unroll
                for (int c = (j + 1) & ~1; c < G * (m + 1); c += 2) {
                  const double2 v = *reinterpret_cast<const double2 *>(vec + c);
                  if (c > j) a[o + c] = fma(-lij, v.x, a[o + c]);
                  a[o + c + 1] = fma(-lij, v.y, a[o + c + 1]);
                }
                a[o + j] = lij;
              }
            }
          }
        }
        }
      pd.renorm();
      const double lt = pd.log_value();
      __syncwarp();                       // last LDL step's broadcast reads done
      // ------------------------------------------------- W = L^-1 in place ----
#pragma unroll
      for (int j = 1; j < KT; ++j) {
        if (j < K) {
          double *vec = sm.vec[j & 1];
          if (t == j % G) {                    // row j of W is final: publish it
#pragma unroll
            for (int c = 0; c < j; c += 2) {
              const int q = G * (j / G) * (j / G + 1) / 2 + c;
              if (c + 1 < j)
                *reinterpret_cast<double2 *>(vec + c) = make_double2(a[q], a[q + 1]);
              else
                vec[c] = a[q];
            }
          }
          __syncwarp();
#pragma unroll
          for (int m = 0; m < M; ++m) {
            if (G * (m + 1) > j + 1) {
              const int o = G * m * (m + 1) / 2;
              if (t + G * m > j) {
                const double lij = a[o + j];
#pragma unroll
                for (int c = 0; c < j; c += 2) {
                  const double2 v = *reinterpret_cast<const double2 *>(vec + c);
                  a[o + c] = fma(-lij, v.x, a[o + c]);
                  if (c + 1 < j) a[o + c + 1] = fma(-lij, v.y, a[o + c + 1]);
                }
                a[o + j] = -lij;
              }
            }
          }
        }
      }
      // ------------------------------- (R^-1)_cc = sum_i w_ic^2 / d_i ----
#pragma unroll
      for (int c = 0; c < KT; ++c) {
        double p = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (G * (m + 1) > c) {
            const int i = t + G * m;
            const double wv = c < i ? a[G * m * (m + 1) / 2 + c] : (c == i ? 1.0 : 0.0);
            p = fma(wv * wv, dinv[m], p);
          }
        }
        sm.red[t][c] = p;
      }
      __syncwarp();
      // one log per thread of the product of its columns' (R^-1)_cc (each
      // >= 1; LogProd keeps the running product in range), not one per column
      const bool take = good && !ok;
      LogProd lp;
      lp.init();
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int c = t + G * m;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < G; ++q) s += sm.red[q][c];
        if (take) inv[m] = s;
        if (c < K) lp.mul(s);
        if ((m & 7) == 7) lp.renorm();
      }
      lp.renorm();
      const double lamt = group_sum<G>(lp.log_value());
      if (take) {
        l = lt;
        lam = lamt;
        ok = true;
      }
      __syncwarp();
    }
    // ------------------------------------------------------------- output ----
    // (no early exits: the COMPAT group sum below is a full-warp shuffle)
    double lsg = 0.0;
    if (COMPAT) {
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (t + G * m < K && A.sdiag) lsg += log(sg[m]);
      lsg = group_sum<G>(lsg);
    }
    if (valid) {
      const int64_t ob = A.row_map ? A.row_map[b] : A.out_row0 + b;
      const int64_t o = ob * D + d;
      if (!ok) {
        if (t == 0) {
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
      } else {
        if (A.out && t == 0) {
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
          if (A.invdiag) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
              const int c = t + G * m;
              if (c < K) {
                const double v = inv[m] / sg[m];
                if (A.inv_n > 0)
                  A.invdiag[o * A.inv_n + si[m]] = v;
                else
                  A.invdiag[o * K + c] = v;
              }
            }
          }
          if (A.logdet && t == 0) A.logdet[o] = l + lsg;
        }
      }
    }
  }
}

template <int G, int M, int MINB, bool COMPAT, bool SMEM>
int launch_grp(const EvalArgs &A, int K, cudaStream_t s) {
  auto kern = k_eval_grp<G, M, MINB, COMPAT, SMEM>;
  constexpr int kSlots = (int)sizeof(GrpSmem<G, M>) * kGWarps * (32 / G);
  const int smem = kSlots + (SMEM ? (int)(sizeof(double) * A.N * A.N * A.D) : 0);
  static thread_local int cap_for = -1, cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cap_for != dev) {
    const int most = kSlots + (SMEM ? kEvalSmemMax : 0);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * kGWarps, most);
    cap = sms * (per > 0 ? per : 1);
    cap_for = dev;
  }
  constexpr int per_cta = kGWarps * (32 / G);
  const int64_t n = A.B * (int64_t)A.D;
  const int64_t want = (n + per_cta - 1) / per_cta;
  const int grid = (int)(want < cap ? want : cap);
  kern<<<grid, 32 * kGWarps, smem, s>>>(A, K);
  return check_launch("k_eval_grp");
}

template <int G, int M, int MINB>
int pick_grp(const EvalArgs &A, int K, bool compat, bool smem, cudaStream_t s) {
  if (compat)
    return smem ? launch_grp<G, M, MINB, true, true>(A, K, s) : launch_grp<G, M, MINB, true, false>(A, K, s);
  return smem ? launch_grp<G, M, MINB, false, true>(A, K, s) : launch_grp<G, M, MINB, false, false>(A, K, s);
}

}  // namespace

int launch_eval_group(const EvalArgs &A, int K, cudaStream_t s) {
  if (K < 17 || K > 32 || A.mats) return -1;
  upload_binomials();
  const int64_t n = A.B * (int64_t)A.D;
  if (n == 0) return HOI_OK;
  const bool compat = A.logdet || A.invdiag;
  const bool smem = sizeof(double) * A.N * A.N * A.D <= (size_t)kEvalSmemMax;
  // (G, M) per order range, measured on B200 (cfg4 order segments, round 1
  // TF/s): K 17-18 (2,9) 3.2-3.7 | 21-24 (4,6) 3.9-4.9 | 25-28 (4,7) 3.1 (a
  // little spilled, still 20% over (8,4)) | 29-32 (8,4); (8,3) for 21-24 ran
  // 2.7-3.4, the warp-per-unit kernel 0.8-1.5.  Round 2 (segment ms): fewer,
  // fatter threads win while the rows fit -- K 17-18 (2,9) 2.52 vs (4,5)
  // 3.87; K 19-20 (2,10) 3.34 vs (4,5) 4.11 (its exchange slots need the
  // dynamic shared memory above); K 21-22 (2,11) 5.85 vs (4,6) 5.60.
  if (K <= 18) return pick_grp<2, 9, 1>(A, K, compat, smem, s);
  if (K <= 20) return pick_grp<2, 10, 1>(A, K, compat, smem, s);
  if (K <= 24) return pick_grp<4, 6, 1>(A, K, compat, smem, s);
  if (K <= 28) return pick_grp<4, 7, 1>(A, K, compat, smem, s);
  return pick_grp<8, 4, 1>(A, K, compat, smem, s);
}

}  // namespace hoib
