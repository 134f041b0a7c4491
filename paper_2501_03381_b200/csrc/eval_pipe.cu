// Engine 1, batched index mode with the correlation matrix in L2 (large N,
// e.g. BASELINE config 5: N = 400, D = 16, order 10): a gather-pipelined
// variant of k_eval for fixed orders 4..12.
//
// k_eval gathers the K(K-1)/2 off-diagonal entries of R_S straight into
// registers and then factorises, so each warp sits idle for an L2 round
// trip per unit and the register file holds the gathered values in flight
// (168 registers, ~12 warps/SM, FP64 pipe ~49% busy at K = 10).  Here every
// thread streams the NEXT unit's entries into its own shared-memory stage
// with cp.async (8-byte LDGSTS, no registers held) while it factorises the
// current one from the other stage: the L2 latency hides behind a unit of
// FP64 work and the kernel runs FP64-bound at 8 warps/SM (two 128-thread
// CTAs: 2 stages x K(K-1)/2 doubles x 128 threads of shared memory each).
//
// Stage layout [stage][entry][thread]: a warp's 32 threads touch 32
// consecutive doubles per entry (conflict-free).  Threads keep a fixed
// dataset d (grid x 128 is a multiple of D) and walk n-plets b, b + step/D,
// ...; with the dataset index fastest in R (N, N, D), the 16 threads of a
// config-5 n-plet read one 128-byte line per entry.
//
// Arithmetic per unit is k_eval's (ref:nplet_engine.py:267-281 restated as
// LDL^T + unit-triangular inverse + inverse diagonal, ref:measures.py:41-81
// epilogue) with two cheaper non-algorithmic pieces: the pivot reciprocal
// is eval_kernels.cuh's pivot_rcp (MUFU.RCP64H + one quadratic Newton
// step, shared with k_eval and the group kernel), and
// the two log products go through k_eval's LogProd.  A non-positive pivot
// reruns the unit through k_eval's jitter retry (ref:nplet_engine.py:237-264).
#include "eval_kernels.cuh"

namespace hoib {
namespace {

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}



// Table-driven FP64 log (the lattice kernel's fast_log, 256 entries):
// x = 2^e f, j = top 8 bits of f, r = f c_j - 1 in [0, 2^-8), log x =
// e ln2 + L_j + log1p(r) with a degree-8 polynomial; ~12 FP64 instructions
// against ~25 for log().  The table lives in each CTA's shared memory.
__constant__ double2 c_plog[256];

__device__ __forceinline__ double pipe_log(double m, int e_extra, const double2 *tab) {
  const long long b = __double_as_longlong(m);
  const int e = (int)((b >> 52) & 0x7FF) - 1023 + e_extra;
  const int j = (int)((b >> 44) & 0xFF);
  const double f = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  const double2 t = tab[j];
  const double r = fma(f, t.x, -1.0);
  double p = fma(r, -0.125, 0.14285714285714285);
  p = fma(r, p, -0.16666666666666666);
  p = fma(r, p, 0.2);
  p = fma(r, p, -0.25);
  p = fma(r, p, 0.33333333333333331);
  p = fma(r, p, -0.5);
  p = fma(r, p, 1.0);
  const double ed = (double)e;
  return fma(ed, 6.93147180369123816490e-01, fma(ed, 1.90821492927058770002e-10, fma(r, p, t.y)));
}

__device__ __forceinline__ double logprod_value(const LogProd &lp, const double2 *tab) {
  return pipe_log(lp.m, lp.e, tab);
}

template <int K>
__device__ __forceinline__ bool ldl_fast(double (&a)[K * (K + 1) / 2], LogProd &pd) {
  pd.init();
  bool bad = false;   // flagged, not branched on (see ldl_invdiag)
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double dj = a[TRI(j, j)];
    bad |= !(dj > 0.0);
    pd.mul(dj);
    if ((j & 7) == 7) pd.renorm();
    const double r = pivot_rcp(dj);
    a[TRI(j, j)] = r;
#pragma unroll
    for (int i = K - 1; i > j; --i) {
      const double lij = a[TRI(i, j)] * r;
#pragma unroll
      for (int m = j + 1; m <= i; ++m) a[TRI(i, m)] = fma(-lij, a[TRI(m, j)], a[TRI(i, m)]);
      a[TRI(i, j)] = lij;
    }
  }
  pd.renorm();
  return !bad;
}

// U = L^-1 in place, then lam = log prod_j (M^-1)_jj, (M^-1)_jj = sum_i U_ij^2 / d_i
template <int K>
__device__ __forceinline__ LogProd inv_diag_logprod(double (&a)[K * (K + 1) / 2]) {
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
    double sacc = a[TRI(j, j)];
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      const double u = a[TRI(i, j)];
      sacc = fma(u * u, a[TRI(i, i)], sacc);
    }
    pl.mul(sacc);
    if ((j & 7) == 7) pl.renorm();
  }
  pl.renorm();
  return pl;
}

constexpr int kPipeThreads = 128;

template <int K>
__global__ void __launch_bounds__(kPipeThreads, 3) k_eval_pipe(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw) + threadIdx.x;
  __shared__ double2 s_plog[256];
  const int tid = threadIdx.x;
  for (int x = tid; x < 256; x += kPipeThreads) s_plog[x] = c_plog[x];
  __syncthreads();
  const int D = A.D, N = A.N;
  const int64_t t0 = blockIdx.x * (int64_t)kPipeThreads + tid;
  const int64_t step = (int64_t)gridDim.x * kPipeThreads;   // a multiple of D
  const int d = (int)(t0 % D);
  const int64_t db = step / D;
  const double *Rd = A.src + d;
  const int rowN = N * D;

  // element offsets fit in 32 bits (N*N*D < 2^31, checked at launch): one
  // integer add and one wide multiply-add per gathered element
  auto issue = [&](int64_t b) {
    if (b < A.B) {
      const int32_t *ix = A.idx + b * A.idx_stride;
      int col[K], row[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int v = __ldg(ix + i);
        col[i] = v * D;
        row[i] = v * rowN;
      }
#pragma unroll
      for (int i = 1; i < K; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j)
          cp_async8(stage + (TRI(i, j) - i) * kPipeThreads, Rd + (row[i] + col[j]));
    }
    cp_async_commit();
  };

  int64_t b = t0 / D;
  issue(b);
  const int s_dummy[K] = {};
  const double cs_dummy[K] = {};
  for (; b < A.B; b += db) {
    cp_async_wait_all();
    double a[K * (K + 1) / 2];
#pragma unroll
    for (int i = 0; i < K; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) a[TRI(i, j)] = stage[(TRI(i, j) - i) * kPipeThreads];
      a[TRI(i, i)] = 1.0;
    }
    LogProd pd;
    const bool ok = ldl_fast<K>(a, pd);
    // every staged value has been consumed by the factorisation (and the
    // stage is only ever touched by this thread): the next unit's gather
    // streams in behind the rest of this unit's work
    issue(b + db);
    if (!ok) {
      eval_retry<K, true, false>(A, A.src, b, d, K);
      continue;
    }
    const LogProd pl = inv_diag_logprod<K>(a);
    finish_unit<K, true, false>(A, b, d, K, s_dummy, true, logprod_value(pd, s_plog),
                                logprod_value(pl, s_plog), cs_dummy);
  }
}

template <int K>
int launch_pipe(const EvalArgs &A, cudaStream_t s) {
  constexpr int NE = K * (K - 1) / 2;
  const int smem = (int)(NE * kPipeThreads * sizeof(double));
  static thread_local int cap_for = -1, cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cap_for != dev) {
    cudaFuncSetAttribute(k_eval_pipe<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eval_pipe<K>, kPipeThreads, smem);
    cap = sms * (per > 0 ? per : 1);
    cap_for = dev;
  }
  // grid x 128 must be a multiple of D (each thread keeps its dataset)
  int g = 1;
  while ((g * kPipeThreads) % A.D) ++g;
  const int64_t units = A.B * (int64_t)A.D;
  int64_t want = (units + kPipeThreads - 1) / kPipeThreads;
  int64_t grid = want < cap ? want : cap;
  grid = ((grid + g - 1) / g) * g;
  if (grid < 1) grid = g;
  k_eval_pipe<K><<<(int)grid, kPipeThreads, smem, s>>>(A);
  return check_launch("k_eval_pipe");
}

}  // namespace

// -1 when the launch is not this kernel's (see nplet_eval.cu launch_eval):
// fixed orders 4..12, FP64 measures only, index rows, R in global memory.
static void upload_plog() {
  static thread_local int done_for = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_for == dev) return;
  double2 t[256];
  for (int j = 0; j < 256; ++j) {
    const long double c = 1.0L / (1.0L + (long double)j / 256.0L);
    t[j].x = (double)c;
    t[j].y = (double)(-logl((long double)(double)c));
  }
  cudaMemcpyToSymbol(c_plog, t, sizeof(t));
  done_for = dev;
}

int launch_eval_pipe(const EvalArgs &A, int K, cudaStream_t s) {
  if (A.mats || !A.idx || A.fp32 || A.logdet || A.invdiag || A.row_map || !A.out) return -1;
  if ((size_t)A.N * A.N * A.D * sizeof(double) <= (size_t)kEvalSmemMax) return -1;
  if ((int64_t)A.N * A.N * A.D >= (1ll << 31)) return -1;
  if (A.B * (int64_t)A.D < (int64_t)kPipeThreads * 148) return -1;   // small batches: k_eval
  upload_binomials();
  upload_plog();
  switch (K) {
    case 4: return launch_pipe<4>(A, s);
    case 5: return launch_pipe<5>(A, s);
    case 6: return launch_pipe<6>(A, s);
    case 7: return launch_pipe<7>(A, s);
    case 8: return launch_pipe<8>(A, s);
    case 9: return launch_pipe<9>(A, s);
    case 10: return launch_pipe<10>(A, s);
    case 11: return launch_pipe<11>(A, s);
    case 12: return launch_pipe<12>(A, s);
    default: return -1;
  }
}

}  // namespace hoib
