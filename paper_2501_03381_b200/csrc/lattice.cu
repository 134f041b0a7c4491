// Engine 2: subset-lattice engine for exhaustive scans (12 <= N <= 32).
//
// In the correlation form every measure of an n-plet S of order k depends
// on l(S) = log det R_S and on the leave-one-out log-determinants
// l(S \ j), j in S (ref:nplet_engine.py:267-273: logdet(Sigma_-j) =
// logdet Sigma + log (Sigma^-1)_jj):
//   tc  = -l/2                        - k*eta1 + eta_k
//   dtc = ((1-k) l + sum_j l(S\j))/2  + (k-1)*eta_k - k*eta_{k-1}
//   o   = ((k-2) l - sum_j l(S\j))/2  - k*eta1 - (k-2)*eta_k + k*eta_{k-1}
//   s   = tc + dtc
// An exhaustive scan visits every subset, so every leave-one-out term is
// itself the log-determinant of another visited subset.  The engine
// therefore (phase 1) computes the table T[S] = l(S) for all 2^N subsets
// with one Schur-complement elimination tree -- a handful of FMAs and ONE
// log per subset instead of an O(k^3) factorisation -- and (phase 2)
// streams the table through a hypercube stencil that sums the k
// neighbours T[S \ j] and writes the four measures straight into the
// order-major lexicographic output position.
//
// Table layout: variables 0..N-CB-1 form the block index ("prefix"
// variables, bit j = variable j) and the last CB = 10 variables F form the
// 1024-entry block (bit t = variable N-CB+t).  For a fixed prefix set P and
// |Q| = q, the subsets P u Q (Q a q-subset of F) are CONTIGUOUS in the
// reference's lexicographic order, so phase 2 writes C(10,q)-long
// coalesced runs.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace hoib {
namespace {

constexpr int CB = 10;            // suffix variables per block
constexpr int BLK = 1 << CB;      // 1024 table entries per block
constexpr int LANE_BITS = 5;      // F0..F4 -> lane, F5..F9 -> register recursion
constexpr int MAXV = 32;          // max variables
constexpr int MAXB = 6;           // prefix variables expanded inside one CTA
// Schur pivots of a correlation matrix lie in (0, 1]; a pivot below this
// means R is (numerically) singular and the table would carry rounding
// noise, so the engine declines and the per-n-plet engine (with the
// reference's per-matrix jitter rule) takes the scan.
constexpr double kMinPivot = 1e-12;
// Stencil configuration: the measured best on B200 (cfg4).
//   full output, pass 2 : 4-slot TMA ring, 4 CTAs/SM, double-buffered
//                         neighbour sums (kRingFull / kCtasFull)
//   low-sum pass 1 and the TopK filter: 6-slot ring, no neighbour-sum buffer
//                         (entries finish from registers), 4 CTAs/SM
//   own block loaded L2 evict_last; neighbour blocks evict_normal
//   full output N >= 24: two passes split by prefix-bit groups; filter:
//                         single pass (bound by per-job latency, not bytes)
//   pass 2 issues the DRAM-sourced pass-1-sum job before the neighbours
// Alternatives measured and dropped (round 1): 5/6-slot full rings, 3 or 2
// CTAs/SM, evict-first far neighbours, claim-ahead L2 prefetch, a chunked
// table/stencil two-stream pipeline and a single fused produce/consume
// kernel -- all equal or slower.
constexpr int kRingLean = 6;

constexpr int kLogBits = 8;                  // fast_log table index bits
constexpr int kLogTab = 1 << kLogBits;
constexpr int kLogRep = 8;                   // bank-private replicas in shared memory
__device__ double2 g_logtab[kLogTab];        // (c_j, L_j) of fast_log (copied to shared per CTA)
__constant__ uint16_t c_lexrank[BLK];        // Q mask -> rank among |Q|-subsets of F
__constant__ uint16_t c_runmask[BLK];        // run q, position t -> Q mask (runs concatenated)
__constant__ uint16_t c_runstart[CB + 2];    // start of run q in c_runmask
// Global copies of the tables that are indexed per lane (constant memory
// serialises divergent indices; these go through L1 with coalescing).
__device__ uint16_t g_runmask[BLK];
__device__ uint32_t g_run[BLK];          // run position p -> e | lexrank << 10 | q << 20
__device__ uint16_t g_lexrank[BLK];      // Q mask -> rank among |Q|-subsets (filter epilogue)
__device__ uint64_t g_binom[kBinomN * kBinomN];

__device__ __forceinline__ uint64_t binom_g(int n, int m) {
  return (m < 0 || n < 0 || m > n) ? 0ull : __ldg(g_binom + n * kBinomN + m);
}

__device__ __forceinline__ void lp_mul(double &m, int &e, double x) {
  m *= x;
  double a = fabs(m);
  if (a < 1e-150 || a > 1e150) {
    int ex;
    m = frexp(m, &ex);
    e += ex;
  }
}

// Table-driven FP64 natural log of m * 2^e_extra (m > 0 normal): with
// x = 2^e * f, f in [1,2), j = top 8 bits of f, c_j = RN(1/(1+j/256)) and
// L_j = -log(c_j) (host-evaluated in 80-bit precision), r = f*c_j - 1 lies in
// (-2^-52, 2^-8) and log x = e*ln2 + L_j + log1p(r) with a degree-7
// polynomial (truncation < 2^-67).  ~10 FP64 instructions; exact 0 for
// x = 1 (c_0 = 1, L_0 = 0), so identity blocks keep exact zeros.
// The (c_j, L_j) pairs are random per lane, so one shared table costs ~10
// wavefronts per warp load (bank conflicts; 81% L1 throughput, the table
// kernel's top stall in round-2 ncu).  The table is replicated 8 times,
// entry j of replica q at 16 B x (8 j + q): lane l reads replica l & 7, so
// the 8 lanes of each quarter-warp phase hit 8 distinct 16-byte bank groups
// and a warp load is the minimum 4 wavefronts.
__device__ __forceinline__ double fast_log(double m, int e_extra, const double2 *__restrict__ tab,
                                           int q) {
  const long long b = __double_as_longlong(m);
  const int e = (int)((b >> 52) & 0x7FF) - 1023 + e_extra;
  const int j = (int)((b >> (52 - kLogBits)) & (kLogTab - 1));
  const double f = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  const double2 t = tab[j * kLogRep + q];
  const double r = fma(f, t.x, -1.0);
  double p = fma(r, 0.14285714285714285, -0.16666666666666666);
  p = fma(r, p, 0.2);
  p = fma(r, p, -0.25);
  p = fma(r, p, 0.33333333333333331);
  p = fma(r, p, -0.5);
  p = fma(r, p, 1.0);
  const double ed = (double)e;
  return fma(ed, 6.93147180369123816490e-01, fma(ed, 1.90821492927058770002e-10, fma(r, p, t.y)));
}

// 1/x for x > 0 normal: hardware approximation + one cubic Newton step
// (e = 1 - x r; r' = r (1 + e + e^2)); the ~2^-22 error of the
// approximation cubes to below double precision (the Schur pivots lie in
// (1e-12, 1]).  3 DFMA against __drcp_rn's longer correctly rounded
// sequence with its special-case branch.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Shared-memory swizzle of a block's 1024 entries: the output pass reads
// them in lexicographic-run order, which in mask order is a scatter with a
// ~14-wavefront bank-conflict degree; XOR-ing the low 5 index bits with
// the high 5 brings it to ~3.6 while neighbour/stencil and linear accesses
// stay conflict-free (2 wavefronts per 8-byte warp access).
__device__ __forceinline__ int swz(int e) { return (e & ~31) | ((e ^ (e >> 5)) & 31); }

// Leaf recursion over the last R suffix variables held in registers as a
// packed lower triangle.  Include/exclude variable 0 of the remainder; the
// include branch takes the Schur complement.  2^R leaves, one log each.
// The running pivot product m enters normalised to [0.5, 1) and picks up at
// most R factors in [1e-12, 1], so it cannot underflow inside the recursion.
template <int R, bool SW>
struct Leaf {
  static __device__ __forceinline__ void run(const double (&a)[R * (R + 1) / 2], double m, int e,
                                             int bits, double *__restrict__ out, int lane,
                                             int &bad, const double2 *__restrict__ tab) {
    constexpr int R1 = R - 1;
    double ex[R1 * (R1 + 1) / 2 > 0 ? R1 * (R1 + 1) / 2 : 1];
    // exclude variable (CB - R): remainder unchanged
#pragma unroll
    for (int i = 1; i < R; ++i)
#pragma unroll
      for (int l = 1; l <= i; ++l) ex[(i - 1) * i / 2 + (l - 1)] = a[i * (i + 1) / 2 + l];
    Leaf<R1, SW>::run(ex, m, e, bits, out, lane, bad, tab);
    // include: pivot a00, Schur complement of the rest
    const double p = a[0];
    bad |= !(p > kMinPivot);
    const double rp = fast_rcp(p);
    double in[R1 * (R1 + 1) / 2 > 0 ? R1 * (R1 + 1) / 2 : 1];
#pragma unroll
    for (int i = 1; i < R; ++i) {
      const double ai = a[i * (i + 1) / 2] * rp;
#pragma unroll
      for (int l = 1; l <= i; ++l)
        in[(i - 1) * i / 2 + (l - 1)] = fma(-ai, a[l * (l + 1) / 2], a[i * (i + 1) / 2 + l]);
    }
    Leaf<R1, SW>::run(in, m * p, e, bits | (1 << (CB - R)), out, lane, bad, tab);
  }
};

template <bool SW>
struct Leaf<0, SW> {
  static __device__ __forceinline__ void run(const double (&)[1], double m, int e, int bits,
                                             double *__restrict__ out, int lane, int &,
                                             const double2 *__restrict__ tab) {
    // bits holds the F5..F9 pattern at bit positions 5..9
    out[SW ? swz(bits + lane) : bits + lane] = fast_log(m, e, tab, lane & (kLogRep - 1));
  }
};

// One Schur step on a symmetric matrix kept as its lower triangle (row
// stride ld): eliminate pivot j, D[i][l] = S[i][l] - S[i][j] (S[l][j] / S[j][j])
// for j < l <= i < n (S == D in place, or S -> D for a step that also
// copies).  The trailing triangle is flattened: entry e (row-major lower
// triangle of the (n-1-j)-square trailing block) goes to thread e mod nt, so
// every thread updates at most SLOTS independent entries -- the row-major
// enumeration of a smaller trailing block is a prefix of the larger one's,
// so a thread's (row, column) offsets are fixed for the whole elimination.
// (Round 2 first form: thread = column, loop over its rows -- a triangle of
// serial loads, the table kernel's top stall source in ncu.)  Same
// arithmetic per entry as before (__drcp_rn pivot, alj = S[l][j] * rp, one
// fma), so the table is bit-identical.
// slot = e | ti << 10 | tl << 16 (e < 1024, ti, tl < 32): one register
__device__ __forceinline__ int tri_slot(int e) {
  int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= e) ++i;
  while (i * (i + 1) / 2 > e) --i;
  return e | (i << 10) | ((e - i * (i + 1) / 2) << 16);
}
template <int SLOTS>
__device__ __forceinline__ void schur_flat(const double *S, double *Dst, int ld, int n, int j,
                                           const int (&sl)[SLOTS]) {
  const double rp = __drcp_rn(S[j * ld + j]);
  const int sz = n - 1 - j, T = sz * (sz + 1) / 2;
  double v[SLOTS];
#pragma unroll
  for (int k = 0; k < SLOTS; ++k) {
    if ((sl[k] & 1023) < T) {
      const int i = j + 1 + ((sl[k] >> 10) & 31), l = j + 1 + (sl[k] >> 16);
      const double alj = S[l * ld + j] * rp;
      v[k] = fma(-S[i * ld + j], alj, S[i * ld + l]);
    }
  }
#pragma unroll
  for (int k = 0; k < SLOTS; ++k) {
    if ((sl[k] & 1023) < T)
      Dst[(j + 1 + ((sl[k] >> 10) & 31)) * ld + (j + 1 + (sl[k] >> 16))] = v[k];
  }
}

// Phase 1: one CTA per pattern of the "fixed" prefix variables b..N-CB-1
// (b = 6).  The CTA eliminates its fixed variables once; warp w eliminates
// the set bits of w among prefix variables 0..2 once (shared by its 8
// patterns), then each of its 8 patterns of variables 3..5 from that state
// -- every warp runs the same mix of patterns, so the CTA tail is short.
// Each lane of a warp owns one pattern of F0..F4 and recurses over F5..F9
// in registers.
template <int NW>
__global__ void __launch_bounds__(32 * NW, 16 / NW)
k_lattice_table(const double *__restrict__ corr, int N, int D, int d, int b,
                double *__restrict__ table, int *__restrict__ flag, unsigned cta_off) {
  constexpr int NT = 32 * NW;
  const unsigned cta = blockIdx.x + cta_off;
  // blockIdx.y > 0: a batch of datasets d, d+1, ... with their tables
  // stacked 2^N doubles apart (scan_full_lattice's multi-dataset batches)
  const int dd = d + (int)blockIdx.y;
  table += (int64_t)blockIdx.y << N;
  extern __shared__ double2 s_logtab[];            // kLogTab x kLogRep entries (dynamic: 32 KB)
  constexpr int MS = MAXV + 1;
  // per-warp matrix row stride, odd: the Schur steps' lanes read column j of
  // consecutive rows (A[i][j]), which at the even stride 16 was a 16-way
  // bank conflict (87M excess wavefronts in round-2 ncu)
  constexpr int WS = MAXB + CB + 1;
  __shared__ double M[MAXV * MS];                  // gathered matrix, row stride MS
  __shared__ double W[NW][2][WS * WS];             // per-warp base / work (lower triangles)
  __shared__ int vars[MAXV];
  __shared__ int s_nfix;
  __shared__ double s_m0;
  __shared__ int s_e0;
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nP = N - CB;
  for (int x = tid; x < kLogTab * kLogRep; x += NT) s_logtab[x] = __ldg(&g_logtab[x / kLogRep]);
  if (tid == 0) {
    int nf = 0;
    for (int j = b; j < nP; ++j)
      if ((cta >> (j - b)) & 1) vars[nf++] = j;
    s_nfix = nf;
    for (int j = 0; j < b; ++j) vars[nf + j] = j;
    for (int t = 0; t < CB; ++t) vars[nf + b + t] = nP + t;
    s_bad = 0;
  }
  __syncthreads();
  const int nfix = s_nfix, m = nfix + b + CB;
  for (int i = tid >> 5; i < m; i += NW)
    if (lane <= i) M[i * MS + lane] = corr[((int64_t)vars[i] * N + vars[lane]) * D + dd];
  __syncthreads();
  // eliminate the fixed prefix variables (right-looking, lower triangle)
  constexpr int CS = (MAXV * (MAXV - 1) / 2 + NT - 1) / NT;   // CTA slots per thread
  int csl[CS];
#pragma unroll
  for (int k = 0; k < CS; ++k) csl[k] = tri_slot(tid + NT * k);
  double m0 = 1.0;
  int e0 = 0;
  for (int j = 0; j < nfix; ++j) {
    const double p = M[j * MS + j];
    if (tid == 0) {
      if (!(p > kMinPivot)) s_bad = 1;
      lp_mul(m0, e0, p);
    }
    schur_flat<CS>(M, M, MS, m, j, csl);
    __syncthreads();
  }
  if (tid == 0) {
    s_m0 = m0;
    s_e0 = e0;
  }
  __syncthreads();
  const int w = b + CB;                            // expansion size
  constexpr int LW = NW == 8 ? 3 : NW == 4 ? 2 : NW == 2 ? 1 : 0;
  const int blo = b < LW ? b : LW;                 // prefix bits fixed per warp
  const double *S0 = M + nfix * MS + nfix;
  double *Wb = W[warp][0], *Wm = W[warp][1];
  __shared__ double s_mb[NW];
  __shared__ int s_eb[NW];
  // warp slots per lane (recomputed where used: kept live across the leaf
  // recursion they spilled)
  constexpr int WSL = ((MAXB + CB) * (MAXB + CB - 1) / 2 + 31) / 32;
  const int ulo = warp & ((1 << blo) - 1);
  if (warp < (1 << blo)) {
    double mb = s_m0;
    int ebase = s_e0;
    for (int i = 0; i < w; ++i)
      if (lane <= i) Wb[i * WS + lane] = S0[i * MS + lane];
    __syncwarp();
    int wsl[WSL];
#pragma unroll
    for (int k = 0; k < WSL; ++k) wsl[k] = tri_slot(lane + 32 * k);
    for (int j = 0; j < blo; ++j) {
      if (!((ulo >> j) & 1)) continue;             // warp-uniform
      const double p = Wb[j * WS + j];
      if (!(p > kMinPivot)) s_bad = 1;
      lp_mul(mb, ebase, p);
      schur_flat<WSL>(Wb, Wb, WS, w, j, wsl);
      __syncwarp();
    }
    if (lane == 0) {
      s_mb[warp] = mb;
      s_eb[warp] = ebase;
    }
    __syncwarp();
  }
  for (int uh = 0; uh < (1 << (b - blo)); ++uh) {
    if (warp >= (1 << blo)) break;
    const int u = ulo | (uh << blo);
    double mu = s_mb[warp];
    int eu = s_eb[warp];
    // the pattern's first step reads the warp's base and writes the work
    // matrix's trailing triangle (every entry later steps and the suffix
    // read), so no copy of the base is made; a pattern without set bits
    // here reads the base directly
    const double *Sw = Wb;
    int wsl[WSL];
#pragma unroll
    for (int k = 0; k < WSL; ++k) wsl[k] = tri_slot(lane + 32 * k);
    for (int j = blo; j < b; ++j) {
      if (!((u >> j) & 1)) continue;               // warp-uniform
      const double p = Sw[j * WS + j];
      if (!(p > kMinPivot)) s_bad = 1;
      lp_mul(mu, eu, p);
      schur_flat<WSL>(Sw, Wm, WS, w, j, wsl);
      __syncwarp();
      Sw = Wm;
    }
    // suffix Schur complement C = Sw[b.., b..] (CB x CB); each lane takes
    // the lower triangle into registers and eliminates its F0..F4 pattern
    double c[CB * (CB + 1) / 2];
#pragma unroll
    for (int i = 0; i < CB; ++i)
#pragma unroll
      for (int l = 0; l <= i; ++l) c[i * (i + 1) / 2 + l] = Sw[(b + i) * WS + (b + l)];
    __syncwarp();
    double ml = mu;
    int el = eu;
    int bad = 0;
#pragma unroll
    for (int j = 0; j < LANE_BITS; ++j) {
      const bool inc = (lane >> j) & 1;
      const double p = c[j * (j + 1) / 2 + j];
      if (inc && !(p > kMinPivot)) bad = 1;
      const double f = inc ? fast_rcp(p) : 0.0;
      if (inc) lp_mul(ml, el, p);
#pragma unroll
      for (int i = j + 1; i < CB; ++i) {
        const double ci = c[i * (i + 1) / 2 + j] * f;
#pragma unroll
        for (int l = j + 1; l <= i; ++l)
          c[i * (i + 1) / 2 + l] = fma(-ci, c[l * (l + 1) / 2 + j], c[i * (i + 1) / 2 + l]);
      }
    }
    constexpr int R = CB - LANE_BITS;
    double a[R * (R + 1) / 2];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int l = 0; l <= i; ++l)
        a[i * (i + 1) / 2 + l] = c[(i + LANE_BITS) * (i + LANE_BITS + 1) / 2 + (l + LANE_BITS)];
    const int64_t blk = ((int64_t)cta << b) | u;
    {
      int ex;
      ml = frexp(ml, &ex);
      el += ex;
    }
    Leaf<R, true>::run(a, ml, el, 0, table + blk * BLK, lane, bad, s_logtab);   // swizzled
    if (bad) s_bad = 1;
  }
  __syncthreads();
  if (tid == 0 && s_bad) atomicExch(flag, 1);
}

// Table-kernel launch: its replicated fast_log table is 32 KB of dynamic
// shared memory on top of ~42 KB static (over the 48 KB default).
template <int NW>
static void launch_table(dim3 grid, cudaStream_t s, const double *corr, int N, int D, int d, int b,
                         double *table, int *flag, unsigned cta_off) {
  constexpr int kDyn = kLogTab * kLogRep * (int)sizeof(double2);
  static thread_local int set_for = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_for != dev) {
    cudaFuncSetAttribute(k_lattice_table<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDyn);
    set_for = dev;
  }
  k_lattice_table<NW><<<grid, 32 * NW, kDyn, s>>>(corr, N, D, d, b, table, flag, cta_off);
}

// TMA bulk-copy / mbarrier helpers (the sm_90+/sm_100 bulk copy engine).
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr uint32_t kSuspendHintNs = 20000;   // upper bound on one suspension

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing the probe.  Without
// it the probe loops were ~1/3 of the instructions the filtered stencil
// issued (ncu source view); with it they are gone from the top lines, but
// the kernel time did not move (10.18 ms either way): the waits are real
// data waits, the probes only filled idle issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase), "r"(kSuspendHintNs)
        : "memory");
  }
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy(bool evict_first) {
  uint64_t p;
  if (evict_first)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

constexpr int kConsumerWarps = 8;
constexpr int kStencilThreads = 32 * kConsumerWarps;   // consumers; + 1 producer warp
constexpr int PER = BLK / kStencilThreads;

// Dynamic shared memory of the stencil kernel (kRing 8 KB table blocks in
// flight per CTA).
// kNbs = 1: one neighbour-sum buffer (a second consumer barrier per block,
// 12 KB less shared memory per CTA -> one more ring slot at 4 CTAs/SM; the
// run table is then read from the global copy g_run through L1).
// kNbs = 0 (filter mode only): entries finish from registers, no buffer.
template <int kRing, int kNbs = 2>
struct StencilSmem {
  double ring[kRing][BLK];           // TMA destination ring
  double nbs[kNbs > 0 ? kNbs : 1][kNbs > 0 ? BLK : 1];   // leave-one-out log-det sums per entry
  uint32_t run[kNbs == 2 ? BLK : 1]; // run position p -> e | lexrank << 10 | q << 20
  uint64_t full[kRing];              // TMA landed
  uint64_t empty[kRing];             // every consumer warp is done with the slot
  int64_t base[2][CB + 1];           // output row of the first n-plet of run q
};

// Lexicographic rank contributions that depend only on the run length q:
// the n-plet P u {first q suffix variables} has rank
//   C(N,k) - 1 - sum_i C(N-1-p_i, k-i) - sum_{t<q} C(CB-1-t, q-t)
// (unranking identity of ref nplet_engine.py:128-136's lexicographic order).
__constant__ uint64_t c_suffix_term[CB + 1];

constexpr int64_t kNoRun = INT64_MIN;

// Output row (relative to g_begin) of P u {first q suffix variables}, or
// kNoRun when its order is outside [kmin, kmax].  Every binomial load is
// independent (fixed unrolled loop, predicated), so one L1 latency.
__device__ __forceinline__ int64_t run_base(unsigned P, int q, int N, int kmin, int kmax,
                                            const int64_t *__restrict__ order_off,
                                            int64_t g_begin) {
  const int nP = N - CB;
  const int k = __popc(P) + q;
  if (k < kmin || k > kmax || k < 1) return kNoRun;
  uint64_t a = 0;
#pragma unroll
  for (int j = 0; j < MAXV - CB; ++j) {
    const bool on = j < nP && ((P >> j) & 1u);
    const int i = __popc(P & ((1u << j) - 1u));
    a += on ? binom_g(N - 1 - j, k - i) : 0ull;
  }
  const uint64_t r = binom_g(N, k) - 1ull - a - c_suffix_term[q];
  return order_off[k - kmin] + (int64_t)r - g_begin;
}

// A pseudo-random 1/every of the table blocks (the sampled pass of a
// filtered TopK scan): a Fibonacci hash of P, high bits.  (P % every == 0
// would keep only subsets that avoid the low prefix variables: a biased
// sample, whose k-th key bounds the global one far more loosely.)
__global__ void k_block_sample(unsigned nblocks, unsigned every, uint8_t *__restrict__ active) {
  const unsigned P = blockIdx.x * blockDim.x + threadIdx.x;
  if (P < nblocks) {
    const unsigned h = P * 2654435761u;
    active[P] = (((uint64_t)h * every) >> 32) == 0 ? 1 : 0;
  }
}

// Block shards `mask` of 2^sb: the table blocks whose top sb prefix bits
// name a shard in the mask (optionally intersected with a hash sample,
// every > 1).
__global__ void k_block_shard(unsigned nblocks, int nP, int sb, unsigned long long mask,
                              unsigned every, uint8_t *__restrict__ active) {
  const unsigned P = blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= nblocks) return;
  bool on = sb == 0 || ((mask >> (P >> (nP - sb))) & 1ull);
  if (every > 1) on = on && (((uint64_t)(P * 2654435761u) * every) >> 32) == 0;
  active[P] = on ? 1 : 0;
}

// 1 if table block P has at least one output row in [g_begin, g_end).
__global__ void k_block_active(int N, int kmin, int kmax, const int64_t *__restrict__ order_off,
                               int64_t g_begin, int64_t g_end, unsigned nblocks,
                               uint8_t *__restrict__ active) {
  const unsigned P = blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= nblocks) return;
  bool any = false;
  for (int q = 0; q <= CB; ++q) {
    const int64_t b0 = run_base(P, q, N, kmin, kmax, order_off, g_begin);
    if (b0 == kNoRun) continue;
    const int64_t len = (int64_t)binom(CB, q);
    if (b0 + len > 0 && b0 < g_end - g_begin) any = true;
  }
  active[P] = any ? 1 : 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// A consumer thread's shared-memory reads of a ring slot must be complete
// before the slot is handed back to the producer, whose next TMA write
// (async proxy) would otherwise overtake loads still in flight -- observed
// on B200 as the first entries of a neighbour slot holding the NEXT job's
// data once consumers fell behind (multi-dataset scans, slow strided output
// stores).  Every consumer thread orders its generic-proxy accesses before
// the async proxy, then the warp releases the slot.  Cost on cfg4: pass 1
// 3.44 -> 3.62 ms, pass 2 11.42 -> 11.86 ms; making the release wait on a
// warp vote over the loaded values instead measured the same (3.61 / 11.98
// ms), i.e. the cost is holding the slot until its reads are done.
__device__ __forceinline__ void release_slot(uint64_t *empty_bar, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_bar);
}

constexpr unsigned kEndBlock = 0xFFFFFFFFu;
constexpr int kBlkQ = 16;              // > blocks the producer can run ahead (kRing + 1)

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Phase 2 (persistent, warp-specialised).  Warp 8 is the producer: one lane
// claims table blocks from a global counter in increasing order (dynamic
// claiming keeps the processing front a few hundred blocks wide, so a
// neighbour block T[P ^ 2^j] below the L2 window is still L2-resident when
// read; static strided assignment lets CTAs drift apart by thousands of
// blocks and doubled DRAM reads) and streams, per block, the neighbour
// blocks T[P \ j] (far bits first, evict-first beyond the L2 window) and
// then the own block T[P] as 8 KB TMA bulk copies into a kRing-deep ring
// guarded by full/empty mbarriers.  The ring never drains between blocks, so
// the next block's neighbours stream in while this block's stencil and
// epilogue run.  Warps 0-7 consume: each thread accumulates its 4 entries
// from every neighbour slot and releases it (one arrival per warp, no
// CTA-wide barrier), adds the in-block neighbours from the own block, and --
// after the only per-block barrier (named, consumers only; nbs/base are
// double-buffered) -- writes the four measures of each run (P, q) as one
// coalesced, contiguous span of the order-major lexicographic output.
// Filter mode (scan with a TopK reducer): instead of the 32 B/n-plet output,
// emit only the n-plets whose key sign * measure[m_idx] is <= *key_max, as
// 40-byte records (global rank as int64 bits, tc, dtc, o, s), appended with
// one atomic per warp.  `count` keeps counting past `cap` (overflow check).
struct StencilFilter {
  int m_idx;
  double sign;
  const uint64_t *key_max;
  double *cand;
  unsigned long long *count;
  int64_t cap;
};

// Pass configuration of the stencil (see the two-pass split in DESIGN.md):
//   nbmask  prefix bits whose neighbour blocks T[P ^ 2^j] are streamed;
//   extra   if set, block P of this array (the partial sums of the low
//           pass) is streamed and added like a neighbour;
//   sums    MODE_LOWSUM: where the neighbour sums are written (T layout);
//   perm_lb claim order: 0 = natural, else the high nP-perm_lb bits vary
//           fastest (so the streamed high-bit neighbours are recent).
//   list    if set, the blocks to process in claim order (*nlist of them):
//           the compacted active blocks of a partial or sampled scan.
struct StencilPass {
  unsigned nbmask;
  const double *extra;
  double *sums;
  int perm_lb;
  const unsigned *list;
  const unsigned *nlist;
  unsigned nstack;    // > 0: a stack of that many datasets' tables (see claim())
  int local;          // MODE_FULL: write block-major local rows (claim index c:
                      // rows c*1024 + run position) instead of global rows
};

// Compact the flagged blocks into a list in claim order (natural, or
// high-bits-fastest when perm_lb > 0).  Skipping inactive blocks one atomic
// claim at a time would cost every producer ~nblocks/active serialized
// atomics per block it keeps.  Two launches over tiles of kCompactTile claim
// positions, 256 threads per tile, position c = tile * 4096 + i * 256 + tid:
// k_count_blocks counts each tile's flags, k_write_blocks sums the counts of
// the tiles before its own (<= 1024 of them) and writes its flagged blocks
// warp-ballot by warp-ballot, preserving claim order.  (One 1024-thread CTA
// scanning contiguous slices took 1.1 ms for 2^20 blocks: strided byte loads.)
constexpr unsigned kCompactTile = 4096;

__device__ __forceinline__ unsigned claim_perm(unsigned c, int nP, int perm_lb) {
  const int hb = nP - perm_lb;
  return perm_lb ? (((c & ((1u << hb) - 1u)) << perm_lb) | (c >> hb)) : c;
}

__global__ void __launch_bounds__(256)
k_count_blocks(const uint8_t *__restrict__ active, int nP, int perm_lb, unsigned *__restrict__ tile_cnt) {
  const unsigned n = 1u << nP, c0 = blockIdx.x * kCompactTile;
  int cnt = 0;
  for (unsigned i = 0; i < kCompactTile / 256; ++i) {
    const unsigned c = c0 + i * 256 + threadIdx.x;
    cnt += (c < n && active[claim_perm(c, nP, perm_lb)]) ? 1 : 0;
  }
  __shared__ int red[8];
  #pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    tile_cnt[blockIdx.x] = (unsigned)t;
  }
}

__global__ void __launch_bounds__(256)
k_write_blocks(const uint8_t *__restrict__ active, int nP, int perm_lb,
               const unsigned *__restrict__ tile_cnt, unsigned *__restrict__ list,
               unsigned *__restrict__ count) {
  __shared__ unsigned wsum[8];
  __shared__ unsigned base_s;
  const unsigned n = 1u << nP, c0 = blockIdx.x * kCompactTile;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned pre = 0;
  for (unsigned t = threadIdx.x; t < blockIdx.x; t += 256) pre += tile_cnt[t];
  #pragma unroll
  for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) wsum[warp] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < 8; ++w) t += wsum[w];
    base_s = t;
  }
  __syncthreads();
  unsigned base = base_s;
  for (unsigned i = 0; i < kCompactTile / 256; ++i) {
    const unsigned c = c0 + i * 256 + threadIdx.x;
    const unsigned q = c < n ? claim_perm(c, nP, perm_lb) : 0u;
    const bool on = c < n && active[q];
    const unsigned m = __ballot_sync(0xffffffffu, on);
    __syncthreads();                       // previous round's wsum reads done
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    unsigned before = 0, total = 0;
    #pragma unroll
    for (int w = 0; w < 8; ++w) {
      const unsigned v = wsum[w];
      before += (unsigned)w < warp ? v : 0u;
      total += v;
    }
    if (on) list[base + before + __popc(m & ((1u << lane) - 1u))] = q;
    base += total;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count = base;
}

__global__ void k_count_to_i64(const unsigned *__restrict__ c, int64_t *__restrict__ out) {
  *out = (int64_t)*c;
}

enum { MODE_FULL = 0, MODE_FILTER = 1, MODE_LOWSUM = 2 };

template <int kRing, int kMinCtas, int MODE, int NB = 2>
__global__ void __launch_bounds__(kStencilThreads + 32, kMinCtas)
k_lattice_measures(const double *__restrict__ table, int N, int D, int d, int kmin, int kmax,
                   const double *__restrict__ eta, int kstride, const int64_t *__restrict__ order_off,
                   int64_t g_begin, int64_t g_end, double *__restrict__ out, int64_t plane,
                   unsigned blk_begin, unsigned blk_end, const uint8_t *__restrict__ active,
                   unsigned *__restrict__ counter, StencilFilter flt, StencilPass ps) {
  constexpr bool FILTER = MODE == MODE_FILTER;
  constexpr bool OWN = MODE != MODE_LOWSUM;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StencilSmem<kRing, NB> &sm = *reinterpret_cast<StencilSmem<kRing, NB> *>(smem_raw);
  __shared__ unsigned blkq[kBlkQ];
  __shared__ unsigned blkc[kBlkQ];                 // claim index of blkq's block (local rows)
  constexpr uint32_t kBlkBytes = BLK * sizeof(double);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (OWN && NB == 2) {
    for (int p = tid; p < BLK; p += blockDim.x) {
      const int e = __ldg(g_runmask + p);
      const int q = __popc(e);
      sm.run[p] = (uint32_t)e | ((uint32_t)(p - c_runstart[q]) << 10) | ((uint32_t)q << 20);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned nbmask = ps.nbmask;
  const int nP = N - CB;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------ producer ----
    if (lane != 0) return;
    const uint64_t pol_near = l2_policy(false), pol_own = l2_policy_last();
    const int hb = nP - ps.perm_lb;
    unsigned c = 0;                                // claim index of the last claim
    auto claim = [&]() -> unsigned {
      if (ps.list) {
        c = atomicAdd(counter, 1u);
        return c < *ps.nlist ? ps.list[c] : kEndBlock;
      }
      for (;;) {
        c = atomicAdd(counter, 1u);
        if (c >= blk_end - blk_begin) return kEndBlock;
        if (ps.nstack > 0) {
          // stacked datasets, claimed 4 datasets per block: output rows are
          // (rows, D) with datasets adjacent, so the 4 writes that fill a
          // 32 B sector arrive together and merge in L2 (measured at N = 20,
          // D = 52: 7.1 ms per stack vs 9.2 ms dataset-major).  Returns
          // (dataset << nP) | block.
          const unsigned dl = ((c >> (2 + nP)) << 2) | (c & 3u);
          if (dl >= ps.nstack) continue;
          return (dl << nP) | ((c >> 2) & ((1u << nP) - 1u));
        }
        const unsigned q = ps.perm_lb ? (((c & ((1u << hb) - 1u)) << ps.perm_lb) | (c >> hb)) : c;
        if (!active || active[blk_begin + q]) return blk_begin + q;
      }
    };
    uint32_t pJ = 0;
    for (uint32_t seq = 0;; ++seq) {
      const unsigned P = claim();
      unsigned prem = P == kEndBlock ? 0u : (P & nbmask);
      // jobs of P: [the partial-sum block,] neighbours (far bits first), the
      // own block.  The DRAM-sourced partial sums go first so their load can
      // start in a slot freed during the previous block's epilogue.
      int stage = ps.extra ? 1 : (prem ? 0 : (OWN ? 2 : 3));
      for (bool first = true;; first = false) {
        const int slot = pJ % kRing;
        if (pJ >= kRing) mbar_wait(&sm.empty[slot], ((pJ / kRing) - 1) & 1u);
        if (first) {                               // published by the arrive below
          blkq[seq % kBlkQ] = P;
          blkc[seq % kBlkQ] = c;
        }
        if (P == kEndBlock) {
          mbar_arrive(&sm.full[slot]);             // tx-free arrival: the end marker
          return;
        }
        const double *srcp;
        uint64_t pol = pol_near;
        if (stage == 0) {
          const int j = 31 - __clz(prem);
          prem &= ~(1u << j);
          srcp = table + (int64_t)(P ^ (1u << j)) * BLK;
          if (!prem) stage = OWN ? 2 : 4;
        } else if (stage == 1) {
          srcp = ps.extra + (int64_t)P * BLK;
          stage = prem ? 0 : (OWN ? 2 : 4);
        } else if (stage == 2) {
          srcp = table + (int64_t)P * BLK;
          pol = pol_own;
          stage = 4;
        } else {                                   // stage 3: a block with no job at all
          mbar_arrive(&sm.full[slot]);
          ++pJ;
          break;
        }
        mbar_expect_tx(&sm.full[slot], kBlkBytes);
        tma_load_1d(sm.ring[slot], srcp, kBlkBytes, &sm.full[slot], pol);
        ++pJ;
        if (stage == 4) break;                     // block complete
      }
    }
  }

  // -------------------------------------------------------- consumers ----
  const int64_t rows = g_end - g_begin;
  const uint64_t key_max = FILTER ? *flt.key_max : 0ull;
  // Each thread owns PAIRS entry pairs (e, e+1), e = 2*pi, pi = tid + 256 r.
  // swz(e+1) == swz(e) ^ 1, so a pair is one aligned 16-byte word whose
  // halves are swapped when bit 5 of e is set (flip): every neighbour block
  // is consumed with 128-bit loads and summed in memory order.
  constexpr int PAIRS = PER / 2;
  int pw[PAIRS];
  bool flip[PAIRS];
#pragma unroll
  for (int r = 0; r < PAIRS; ++r) {
    const int e = 2 * (tid + kStencilThreads * r);
    pw[r] = swz(e) & ~1;
    flip[r] = (e >> 5) & 1;
  }
  uint32_t J = 0;
  for (uint32_t seq = 0;; ++seq) {
    const int buf = seq & 1;
    mbar_wait(&sm.full[J % kRing], (J / kRing) & 1u);   // first job of the block (or the end)
    const unsigned Pg = *(volatile unsigned *)&blkq[seq % kBlkQ];
    if (Pg == kEndBlock) break;
    const int64_t lrow0 = (int64_t)(*(volatile unsigned *)&blkc[seq % kBlkQ]) * BLK;
    // stacked multi-dataset launch: block Pg of the stack is block P of
    // dataset d + (Pg >> nP) (one dataset: Pg = P)
    const unsigned P = Pg & ((1u << nP) - 1u);
    const int dd = d + (int)(Pg >> nP);
    const double *et = eta ? eta + (int64_t)dd * kstride : nullptr;
    const double e1 = et ? et[1] : 0.0;
    const int kP = __popc(P);
    const int nj = __popc(P & nbmask) + (ps.extra ? 1 : 0);
    if (OWN && tid <= CB) sm.base[buf][tid] = run_base(P, tid, N, kmin, kmax, order_off, g_begin);
    double2 acc[PAIRS];
#pragma unroll
    for (int r = 0; r < PAIRS; ++r) acc[r] = make_double2(0.0, 0.0);
    for (int m = 0; m < nj; ++m, ++J) {
      const int slot = J % kRing;
      mbar_wait(&sm.full[slot], (J / kRing) & 1u);
      const double *src = sm.ring[slot];
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) {
        const double2 v = *reinterpret_cast<const double2 *>(src + pw[r]);
        acc[r].x += v.x;
        acc[r].y += v.y;
      }
      release_slot(&sm.empty[slot], lane);
    }
    if (!OWN) {
      // low pass: the neighbour sums of P, in the table's (swizzled) layout
      if (nj == 0) {                               // the zero job that carried P
        release_slot(&sm.empty[J % kRing], lane);
        ++J;
      }
      double *dst = ps.sums + (int64_t)Pg * BLK;
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) __stcg(reinterpret_cast<double2 *>(dst + pw[r]), acc[r]);
      continue;
    }
    const int slot = J % kRing;
    mbar_wait(&sm.full[slot], (J / kRing) & 1u);
    const double *own = sm.ring[slot];
    if (FILTER) {
      // Filter mode writes no ordered output, so each thread finishes its own
      // entry pairs from registers and the own slot goes back to the producer
      // BEFORE the epilogue: the ring (4 slots, ~7 jobs per block) can then
      // hold the next block's loads while this block's measures are filtered,
      // instead of exposing their latency after it.  Rows: base[q] + lexrank.
      double lv[PAIRS][2], nv[PAIRS][2];
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) {
        const int e0 = 2 * (tid + kStencilThreads * r);
        const double2 ov = *reinterpret_cast<const double2 *>(own + pw[r]);
        const double o0 = flip[r] ? ov.y : ov.x, o1 = flip[r] ? ov.x : ov.y;
        double s0 = flip[r] ? acc[r].y : acc[r].x;
        double s1 = (flip[r] ? acc[r].x : acc[r].y) + o0;   // bit-0 neighbour of e0+1 is e0
#pragma unroll
        for (int t = 1; t < CB; ++t) {
          if ((e0 >> t) & 1) {
            const int n0 = e0 ^ (1 << t);
            const double2 v = *reinterpret_cast<const double2 *>(own + (swz(n0) & ~1));
            const bool f = (n0 >> 5) & 1;
            s0 += f ? v.y : v.x;
            s1 += f ? v.x : v.y;
          }
        }
        lv[r][0] = o0;
        lv[r][1] = o1;
        nv[r][0] = s0;
        nv[r][1] = s1;
      }
      release_slot(&sm.empty[slot], lane);          // own slot free before the epilogue
      named_bar_sync(1, kStencilThreads);           // base[buf] complete
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * (tid + kStencilThreads * r) + h;
          const int q = __popc(e);
          const int64_t b0 = sm.base[buf][q];
          const int k = kP + q;
          const int64_t row = b0 + (int64_t)__ldg(g_lexrank + e);
          const bool valid = b0 != kNoRun && row >= 0 && row < rows;
          double tc = 0.0, dtc = 0.0, o = 0.0;
          if (valid) {
            const double l = lv[r][h], nb = nv[r][h];
            const double kd = (double)k;
            if (et) {
              const double ek = et[k], ek1 = et[k - 1];
              tc = -0.5 * l - kd * e1 + ek;
              dtc = 0.5 * ((1.0 - kd) * l + nb) + (kd - 1.0) * ek - kd * ek1;
              o = 0.5 * ((kd - 2.0) * l - nb) - kd * e1 - (kd - 2.0) * ek + kd * ek1;
            } else {
              tc = -0.5 * l;
              dtc = 0.5 * ((1.0 - kd) * l + nb);
              o = 0.5 * ((kd - 2.0) * l - nb);
            }
          }
          const double sv = tc + dtc;
          const double v = flt.m_idx == 0 ? tc : flt.m_idx == 1 ? dtc : flt.m_idx == 2 ? o : sv;
          const bool keep = valid && orderable_key(flt.sign * v) <= key_max;
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (bal) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(flt.count, (unsigned long long)__popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (keep) {
              const unsigned long long slot2 = base + __popc(bal & ((1u << lane) - 1u));
              if ((int64_t)slot2 < flt.cap) {
                double *rec = flt.cand + 5 * slot2;
                rec[0] = __longlong_as_double(row + g_begin);
                rec[1] = tc;
                rec[2] = dtc;
                rec[3] = o;
                rec[4] = sv;
              }
            }
          }
        }
      }
      ++J;
      continue;
    }
    double *nbs = sm.nbs[NB == 2 ? buf : 0];
#pragma unroll
    for (int r = 0; r < PAIRS; ++r) {
      const int e0 = 2 * (tid + kStencilThreads * r);
      const double2 ov = *reinterpret_cast<const double2 *>(own + pw[r]);
      const double o0 = flip[r] ? ov.y : ov.x;
      double s0 = flip[r] ? acc[r].y : acc[r].x;
      double s1 = (flip[r] ? acc[r].x : acc[r].y) + o0;   // bit-0 neighbour of e0+1 is e0
#pragma unroll
      for (int t = 1; t < CB; ++t) {
        if ((e0 >> t) & 1) {
          const int n0 = e0 ^ (1 << t);
          const double2 v = *reinterpret_cast<const double2 *>(own + (swz(n0) & ~1));
          const bool f = (n0 >> 5) & 1;
          s0 += f ? v.y : v.x;
          s1 += f ? v.x : v.y;
        }
      }
      *reinterpret_cast<double2 *>(nbs + pw[r]) = flip[r] ? make_double2(s1, s0) : make_double2(s0, s1);
    }
    named_bar_sync(1, kStencilThreads);           // nbs[buf] and base[buf] complete
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t w = NB == 2 ? sm.run[tid + kStencilThreads * r]
                                 : __ldg(g_run + tid + kStencilThreads * r);
      const int e = w & 1023, t = (w >> 10) & 1023, q = w >> 20;
      const int64_t b0 = sm.base[buf][q];
      const int k = kP + q;
      const int64_t row = ps.local ? lrow0 + tid + kStencilThreads * r : b0 + t;
      const bool valid = b0 != kNoRun && (ps.local || (row >= 0 && row < rows));
      double tc = 0.0, dtc = 0.0, o = 0.0;
      if (valid) {
        const double l = own[swz(e)], nb = nbs[swz(e)];
        const double kd = (double)k;
        if (et) {
          const double ek = et[k], ek1 = et[k - 1];
          tc = -0.5 * l - kd * e1 + ek;
          dtc = 0.5 * ((1.0 - kd) * l + nb) + (kd - 1.0) * ek - kd * ek1;
          o = 0.5 * ((kd - 2.0) * l - nb) - kd * e1 - (kd - 2.0) * ek + kd * ek1;
        } else {
          tc = -0.5 * l;
          dtc = 0.5 * ((1.0 - kd) * l + nb);
          o = 0.5 * ((kd - 2.0) * l - nb);
        }
      }
      const double sv = tc + dtc;
      if (!FILTER) {
        if (valid) {
          // streaming (evict-first) stores: the 32 B/n-plet output must not
          // push the log-det table's neighbour blocks out of L2
          const int64_t oi = row * D + dd;
          __stcs(out + oi, tc);
          __stcs(out + plane + oi, dtc);
          __stcs(out + 2 * plane + oi, o);
          __stcs(out + 3 * plane + oi, sv);
        }
      } else {
        const double v = flt.m_idx == 0 ? tc : flt.m_idx == 1 ? dtc : flt.m_idx == 2 ? o : sv;
        const bool keep = valid && orderable_key(flt.sign * v) <= key_max;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (bal) {
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(flt.count, (unsigned long long)__popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (keep) {
            const unsigned long long slot2 = base + __popc(bal & ((1u << lane) - 1u));
            if ((int64_t)slot2 < flt.cap) {
              double *rec = flt.cand + 5 * slot2;
              rec[0] = __longlong_as_double(row + g_begin);
              rec[1] = tc;
              rec[2] = dtc;
              rec[3] = o;
              rec[4] = sv;
            }
          }
        }
      }
    }
    release_slot(&sm.empty[slot], lane);          // own slot free
    if (NB == 1) named_bar_sync(1, kStencilThreads);   // nbs free for the next block
    ++J;
  }
}

// Full-output stencil with the own block OUTSIDE the ring (the round-2
// pass-2 kernel).  In k_lattice_measures<MODE_FULL> the own block is the
// last job of a block's in-order ring and stays in its slot through the
// run-ordered epilogue, so the next block's later jobs cannot be issued
// until the epilogue ends and their L2/DRAM latency is exposed once per
// block (ncu, round 1: consumer warps spent ~30% of their issue slots
// polling ring barriers).  Here the producer loads each block's own T[P]
// FIRST, into a double-buffered own area with its own full/empty
// mbarriers (released after the epilogue), and the ring carries only the
// partial-sum and neighbour jobs, which are released as soon as they are
// accumulated.  One neighbour-sum buffer (a second named barrier keeps the
// next block's nbs writes behind this block's epilogue reads) keeps the
// CTA at 53 KB of shared memory: 4 CTAs per SM.
constexpr int kRingOwn = 3;

template <int RING, bool NBS>
struct FullSmemT {
  double ring[RING][BLK];
  double own[2][BLK];
  double nbs[NBS ? BLK : 1];
  uint32_t run[BLK];
  uint64_t full[RING];
  uint64_t empty[RING];
  uint64_t own_full[2];
  uint64_t own_empty[2];
  int64_t base[2][CB + 1];
};
// HOLD (the FAST instantiation, whose blocks always carry the pass-1-sum
// job): no separate neighbour-sum buffer; a block's last ring job is not
// released after it is accumulated, the block's neighbour sums are written
// over it (each thread over the very pairs it read) and the slot is freed
// after the epilogue.  The 8 KB buy a 4th ring slot at the same 4 CTAs/SM.
template <bool HOLD>
using FullSmem = FullSmemT<HOLD ? 4 : kRingOwn, !HOLD>;

// FAST: one dataset, no bias, the whole rank range, global rows -- the
// headline configuration -- with every branch of the general epilogue
// (bias terms, partial-range and local-row checks, the dataset column)
// resolved at compile time.
template <bool FAST>
__global__ void __launch_bounds__(kStencilThreads + 32, 4)
k_lattice_full(const double *__restrict__ table, int N, int D, int d, int kmin, int kmax,
               const double *__restrict__ eta, int kstride, const int64_t *__restrict__ order_off,
               int64_t g_begin, int64_t g_end, double *__restrict__ out, int64_t plane,
               unsigned blk_begin, unsigned blk_end, const uint8_t *__restrict__ active,
               unsigned *__restrict__ counter, StencilPass ps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr bool HOLD = FAST;
  constexpr int RING = HOLD ? 4 : kRingOwn;
  FullSmem<HOLD> &sm = *reinterpret_cast<FullSmem<HOLD> *>(smem_raw);
  __shared__ unsigned blkq[kBlkQ];
  __shared__ unsigned blkc[kBlkQ];
  constexpr uint32_t kBlkBytes = BLK * sizeof(double);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int p = tid; p < BLK; p += blockDim.x) {
    const int e = __ldg(g_runmask + p);
    const int q = __popc(e);
    sm.run[p] = (uint32_t)e | ((uint32_t)(p - c_runstart[q]) << 10) | ((uint32_t)q << 20);
  }
  if (tid == 0) {
    for (int s = 0; s < RING; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.own_full[b], 1);
      mbar_init(&sm.own_empty[b], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned nbmask = ps.nbmask;
  const int nP = N - CB;
  // FAST block pairs: a CTA claims two consecutive claim indices, i.e. the
  // blocks P and P | pbit (pbit = the lowest high prefix bit, the claim
  // order varies it fastest).  P is the pair's second block's neighbour
  // over pbit, and it is already on chip as the first block's own block, so
  // that neighbour job is not streamed: the second block adds it from the
  // other own buffer (last, where far-bits-first order puts pbit), and the
  // first block's own buffer is freed after that instead of after its own
  // epilogue.  One ring job per pair fewer.
  const bool pair = FAST && ps.perm_lb > 0 && ((nbmask >> ps.perm_lb) & 1u) &&
                    (((blk_end - blk_begin) & 1u) == 0) && !active && !ps.list && ps.nstack == 0;
  const unsigned pbit = pair ? (1u << ps.perm_lb) : 0u;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------ producer ----
    if (lane != 0) return;
    const uint64_t pol_near = l2_policy(false), pol_own = l2_policy_last();
    const int hb = nP - ps.perm_lb;
    unsigned c = 0;
    auto claim = [&]() -> unsigned {
      if (ps.list) {
        c = atomicAdd(counter, 1u);
        return c < *ps.nlist ? ps.list[c] : kEndBlock;
      }
      for (;;) {
        c = atomicAdd(counter, 1u);
        if (c >= blk_end - blk_begin) return kEndBlock;
        if (ps.nstack > 0) {                       // see k_lattice_measures
          const unsigned dl = ((c >> (2 + nP)) << 2) | (c & 3u);
          if (dl >= ps.nstack) continue;
          return (dl << nP) | ((c >> 2) & ((1u << nP) - 1u));
        }
        const unsigned q = ps.perm_lb ? (((c & ((1u << hb) - 1u)) << ps.perm_lb) | (c >> hb)) : c;
        if (!active || active[blk_begin + q]) return blk_begin + q;
      }
    };
    uint32_t pJ = 0;
    unsigned Pnext = kEndBlock, cnext = 0;
    for (uint32_t seq = 0;; ++seq) {
      unsigned Pg, cg;
      if (pair) {
        if ((seq & 1) == 0) {
          c = atomicAdd(counter, 2u);
          if (c >= blk_end - blk_begin) {
            Pg = kEndBlock;
          } else {
            Pg = blk_begin + (((c & ((1u << hb) - 1u)) << ps.perm_lb) | (c >> hb));
            Pnext = Pg | pbit;
            cnext = c + 1;
          }
          cg = c;
        } else {
          Pg = Pnext;
          cg = cnext;
        }
      } else {
        Pg = claim();
        cg = c;
      }
      const int ob = seq & 1;
      if (seq >= 2) mbar_wait(&sm.own_empty[ob], ((seq >> 1) - 1) & 1u);
      blkq[seq % kBlkQ] = Pg;                      // published by the own-block arrival
      blkc[seq % kBlkQ] = cg;
      if (Pg == kEndBlock) {
        mbar_arrive(&sm.own_full[ob]);             // tx-free arrival: the end marker
        return;
      }
      const unsigned dl = Pg >> nP, P = Pg & ((1u << nP) - 1u);
      const double *tab = table + ((int64_t)dl << N);
      mbar_expect_tx(&sm.own_full[ob], kBlkBytes);
      tma_load_1d(sm.own[ob], tab + (int64_t)P * BLK, kBlkBytes, &sm.own_full[ob], pol_own);
      unsigned prem = P & nbmask;
      if (pair && (seq & 1)) prem &= ~pbit;         // the pair's first block, on chip
      bool extra = ps.extra != nullptr;
      while (extra || prem) {
        const int slot = pJ % RING;
        if (pJ >= RING) mbar_wait(&sm.empty[slot], ((pJ / RING) - 1) & 1u);
        const double *srcp;
        if (extra) {                               // DRAM-sourced: first
          srcp = ps.extra + (int64_t)P * BLK;
          extra = false;
        } else {
          const int j = 31 - __clz(prem);          // far bits first
          prem &= ~(1u << j);
          srcp = tab + (int64_t)(P ^ (1u << j)) * BLK;
        }
        mbar_expect_tx(&sm.full[slot], kBlkBytes);
        tma_load_1d(sm.ring[slot], srcp, kBlkBytes, &sm.full[slot], pol_near);
        ++pJ;
      }
    }
  }

  // -------------------------------------------------------- consumers ----
  const int64_t rows = g_end - g_begin;
  constexpr int PAIRS = PER / 2;
  int pw[PAIRS];
  bool flip[PAIRS];
#pragma unroll
  for (int r = 0; r < PAIRS; ++r) {
    const int e = 2 * (tid + kStencilThreads * r);
    pw[r] = swz(e) & ~1;
    flip[r] = (e >> 5) & 1;
  }
  uint32_t J = 0;
  for (uint32_t seq = 0;; ++seq) {
    const int buf = seq & 1;
    mbar_wait(&sm.own_full[buf], (seq >> 1) & 1u);
    const unsigned Pg = *(volatile unsigned *)&blkq[seq % kBlkQ];
    if (Pg == kEndBlock) break;
    const int64_t lrow0 = (int64_t)(*(volatile unsigned *)&blkc[seq % kBlkQ]) * BLK;
    const unsigned P = Pg & ((1u << nP) - 1u);
    const int dd = d + (int)(Pg >> nP);
    const double *et = eta ? eta + (int64_t)dd * kstride : nullptr;
    const double e1 = et ? et[1] : 0.0;
    const int kP = __popc(P);
    const bool second = pair && (seq & 1);
    const int nj = __popc(P & nbmask) + (ps.extra ? 1 : 0) - (second ? 1 : 0);
    if (tid <= CB) sm.base[buf][tid] = run_base(P, tid, N, kmin, kmax, order_off, g_begin);
    double2 acc[PAIRS];
#pragma unroll
    for (int r = 0; r < PAIRS; ++r) acc[r] = make_double2(0.0, 0.0);
    int hslot = 0;
    for (int m = 0; m < nj; ++m, ++J) {
      const int slot = J % RING;
      mbar_wait(&sm.full[slot], (J / RING) & 1u);
      const double *src = sm.ring[slot];
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) {
        const double2 v = *reinterpret_cast<const double2 *>(src + pw[r]);
        acc[r].x += v.x;
        acc[r].y += v.y;
      }
      if (HOLD && m == nj - 1)
        hslot = slot;                              // kept: becomes this block's nbs
      else
        release_slot(&sm.empty[slot], lane);
    }
    if (second) {                                  // neighbour over pbit: the first block
      const double *po = sm.own[buf ^ 1];
#pragma unroll
      for (int r = 0; r < PAIRS; ++r) {
        const double2 v = *reinterpret_cast<const double2 *>(po + pw[r]);
        acc[r].x += v.x;
        acc[r].y += v.y;
      }
      release_slot(&sm.own_empty[buf ^ 1], lane);
    }
    const double *own = sm.own[buf];
    double *nbs = HOLD ? sm.ring[hslot] : sm.nbs;
    if (!HOLD && seq > 0) named_bar_sync(2, kStencilThreads);   // previous epilogue done with nbs
#pragma unroll
    for (int r = 0; r < PAIRS; ++r) {
      const int e0 = 2 * (tid + kStencilThreads * r);
      const double2 ov = *reinterpret_cast<const double2 *>(own + pw[r]);
      const double o0 = flip[r] ? ov.y : ov.x;
      double s0 = flip[r] ? acc[r].y : acc[r].x;
      double s1 = (flip[r] ? acc[r].x : acc[r].y) + o0;   // bit-0 neighbour of e0+1 is e0
#pragma unroll
      for (int t = 1; t < CB; ++t) {
        if ((e0 >> t) & 1) {
          const int n0 = e0 ^ (1 << t);
          const double2 v = *reinterpret_cast<const double2 *>(own + (swz(n0) & ~1));
          const bool f = (n0 >> 5) & 1;
          s0 += f ? v.y : v.x;
          s1 += f ? v.x : v.y;
        }
      }
      *reinterpret_cast<double2 *>(nbs + pw[r]) = flip[r] ? make_double2(s1, s0) : make_double2(s0, s1);
    }
    named_bar_sync(1, kStencilThreads);           // nbs and base[buf] complete
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t w = sm.run[tid + kStencilThreads * r];
      const int e = w & 1023, t = (w >> 10) & 1023, q = w >> 20;
      const int64_t b0 = sm.base[buf][q];
      const int k = kP + q;
      const int64_t row = (!FAST && ps.local) ? lrow0 + tid + kStencilThreads * r : b0 + t;
      const bool valid = b0 != kNoRun && (FAST || ps.local || (row >= 0 && row < rows));
      if (!valid) continue;
      const double l = own[swz(e)], nb = nbs[swz(e)];
      const double kd = (double)k;
      double tc, dtc, o;
      if (!FAST && et) {
        const double ek = et[k], ek1 = et[k - 1];
        tc = -0.5 * l - kd * e1 + ek;
        dtc = 0.5 * ((1.0 - kd) * l + nb) + (kd - 1.0) * ek - kd * ek1;
        o = 0.5 * ((kd - 2.0) * l - nb) - kd * e1 - (kd - 2.0) * ek + kd * ek1;
      } else {
        tc = -0.5 * l;
        dtc = 0.5 * ((1.0 - kd) * l + nb);
        o = 0.5 * ((kd - 2.0) * l - nb);
      }
      // streaming (evict-first) stores: the 32 B/n-plet output must not
      // push the log-det table's neighbour blocks out of L2
      const int64_t oi = FAST ? row : row * D + dd;
      __stcs(out + oi, tc);
      __stcs(out + plane + oi, dtc);
      __stcs(out + 2 * plane + oi, o);
      __stcs(out + 3 * plane + oi, tc + dtc);
    }
    if (HOLD) release_slot(&sm.empty[hslot], lane);   // the held job slot
    if (!pair || (seq & 1))                       // a pair's first block: freed by the second
      release_slot(&sm.own_empty[buf], lane);     // own block free for block seq + 2
  }
}

void upload_tables() {
  static thread_local int uploaded_for = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (uploaded_for == dev) return;
  std::vector<uint16_t> lr(BLK), rm(BLK), rs(CB + 2);
  std::vector<std::vector<int>> runs(CB + 1);
  // lexicographic order of the q-subsets of {0..CB-1}: enumerate masks in
  // tuple order by sorting
  for (int q = 0; q <= CB; ++q) {
    std::vector<std::vector<int>> tuples;
    for (int mask = 0; mask < BLK; ++mask) {
      if (__builtin_popcount(mask) != q) continue;
      std::vector<int> t;
      for (int b = 0; b < CB; ++b)
        if ((mask >> b) & 1) t.push_back(b);
      tuples.push_back(t);
    }
    std::sort(tuples.begin(), tuples.end());
    for (size_t r = 0; r < tuples.size(); ++r) {
      int mask = 0;
      for (int b : tuples[r]) mask |= 1 << b;
      lr[mask] = (uint16_t)r;
      runs[q].push_back(mask);
    }
  }
  int at = 0;
  for (int q = 0; q <= CB; ++q) {
    rs[q] = (uint16_t)at;
    for (int mask : runs[q]) rm[at++] = (uint16_t)mask;
  }
  rs[CB + 1] = (uint16_t)at;
  std::vector<double2> lt(kLogTab);
  for (int j = 0; j < kLogTab; ++j) {
    long double c = 1.0L / (1.0L + (long double)j / (long double)kLogTab);
    double cd = (double)c;
    lt[j].x = cd;
    lt[j].y = (double)(-logl((long double)cd));
  }
  cudaMemcpyToSymbol(g_logtab, lt.data(), sizeof(double2) * kLogTab);
  cudaMemcpyToSymbol(g_runmask, rm.data(), sizeof(uint16_t) * BLK);
  {
    std::vector<uint32_t> gr(BLK);
    for (int p = 0; p < BLK; ++p) {
      const int e = rm[p], q = __builtin_popcount(e);
      gr[p] = (uint32_t)e | ((uint32_t)(p - rs[q]) << 10) | ((uint32_t)q << 20);
    }
    cudaMemcpyToSymbol(g_run, gr.data(), sizeof(uint32_t) * BLK);
  }
  {
    std::vector<uint64_t> hb(kBinomN * kBinomN);
    fill_binomials(hb.data());
    cudaMemcpyToSymbol(g_binom, hb.data(), sizeof(uint64_t) * hb.size());
  }
  cudaMemcpyToSymbol(c_lexrank, lr.data(), sizeof(uint16_t) * BLK);
  cudaMemcpyToSymbol(g_lexrank, lr.data(), sizeof(uint16_t) * BLK);
  cudaMemcpyToSymbol(c_runmask, rm.data(), sizeof(uint16_t) * BLK);
  cudaMemcpyToSymbol(c_runstart, rs.data(), sizeof(uint16_t) * (CB + 2));
  {
    uint64_t st[CB + 1];
    for (int q = 0; q <= CB; ++q) {
      st[q] = 0;
      for (int t = 0; t < q; ++t) st[q] += host_binom(CB - 1 - t, q - t);
    }
    cudaMemcpyToSymbol(c_suffix_term, st, sizeof(st));
  }
  uploaded_for = dev;
}

}  // namespace

bool lattice_available() { return true; }

bool lattice_supports(int N) { return N >= CB + 2 && N <= MAXV; }

int batch_slots(int N, int D);

int lattice_ws_bytes(int N, int D, size_t *bytes) {
  if (!lattice_supports(N)) return fail(HOI_INVALID_ARG, "lattice engine needs 12 <= N <= 32");
  // table 2^N f64 | misc (flag, err, counter, order offsets) 4 KB | flags
  // 2^(N-10) u32 | pad to 256 B | low-pass neighbour sums 2^N f64 (N >= 24)
  *bytes = (sizeof(double) << N) + 4096 + (sizeof(unsigned) << (N - CB));
  if (N - CB >= 14) *bytes = ((*bytes + 255) & ~(size_t)255) + (sizeof(double) << N);
  // | compacted block lists 2 x 2^(N-10) u32 | 2 counts (64 B) | 2 x 1024
  // per-tile counts of the compaction
  *bytes = ((*bytes + 255) & ~(size_t)255) + (sizeof(unsigned) << (N - CB + 1)) + 64 + 8192;
  // | multi-dataset batch: batch_slots(N, D) tables stacked (D > 1, N < 24)
  const int slots = batch_slots(N, D);
  if (slots > 1) *bytes = ((*bytes + 255) & ~(size_t)255) + ((size_t)slots << N) * sizeof(double);
  return HOI_OK;
}

// Datasets per stacked launch (scan_full_lattice): below N = 24 one
// dataset's table is small (<= 64 MB) and its stencil (2^(N-10) <= 8,192
// blocks) cannot fill the GPU's persistent CTAs, so several datasets' tables
// are built and streamed by one launch each (up to 512 MB of tables).
int batch_slots(int N, int D) {
  if (D <= 1 || N - CB >= 14) return 1;
  const size_t per = sizeof(double) << N;
  size_t cap = (size_t)512 << 20;
  int slots = (int)(cap / per);
  return slots < D ? (slots > 1 ? slots : 1) : D;
}

// The batch tables: after the single-dataset layout (whose offsets, and so
// hoi_lattice_status, do not depend on D).
static double *batch_tables(void *ws, int N) {
  size_t off = (sizeof(double) << N) + 4096 + (sizeof(unsigned) << (N - CB));
  off = (off + 255) & ~(size_t)255;
  if (N - CB >= 14) off = ((off + (sizeof(double) << N)) + 255) & ~(size_t)255;
  off += (sizeof(unsigned) << (N - CB + 1)) + 64 + 8192;
  off = (off + 255) & ~(size_t)255;
  return reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + off);
}

// Workspace: [table 2^N doubles][flag int x16][order offsets int64 x33]
struct LatticeWs {
  double *table;
  int *flag;          // phase-1 not-PD flag
  int *err;           // fused pass: 1 not PD, 2 spin timeout
  unsigned *counter;  // fused pass: block claim counter
  int64_t *offs;      // order offsets
  unsigned *ready;    // fused pass: per-block publish flags
  double *lowsum;     // two-pass stencil: low-bit neighbour sums (or nullptr)
  unsigned *list;     // compacted block lists (2 x 2^(N-10)) + 2 counts + tile counts
};

static LatticeWs ws_view(void *ws, int N) {
  LatticeWs w;
  char *base = reinterpret_cast<char *>(ws) + (sizeof(double) << N);
  w.table = reinterpret_cast<double *>(ws);
  w.flag = reinterpret_cast<int *>(base);
  w.err = w.flag + 4;
  w.counter = reinterpret_cast<unsigned *>(w.flag + 8);
  w.offs = reinterpret_cast<int64_t *>(base + 64);
  w.ready = reinterpret_cast<unsigned *>(base + 4096);
  w.lowsum = nullptr;
  size_t off = (sizeof(double) << N) + 4096 + (sizeof(unsigned) << (N - CB));
  off = (off + 255) & ~(size_t)255;
  if (N - CB >= 14) {
    w.lowsum = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + off);
    off = (off + (sizeof(double) << N) + 255) & ~(size_t)255;
  }
  w.list = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(ws) + off);
  return w;
}

int lattice_table(const double *corr, int N, int D, int d, void *ws, size_t ws_bytes,
                  cudaStream_t s, bool reset_flag = true) {
  size_t need = 0;
  int st = lattice_ws_bytes(N, D, &need);
  if (st) return st;
  if (ws_bytes < need) return fail(HOI_CAPACITY, "lattice: workspace too small");
  upload_tables();
  LatticeWs w = ws_view(ws, N);
  if (reset_flag) cudaMemsetAsync(w.flag, 0, sizeof(int), s);
  const int nP = N - CB;
  const int b = nP < MAXB ? nP : MAXB;
  launch_table<8>(dim3(1u << (nP - b)), s, corr, N, D, d, b, w.table, w.flag, 0u);
  return check_launch("k_lattice_table");
}

static int64_t total_rows(int N, int kmin, int kmax, int64_t *h_off) {
  int64_t acc = 0;
  for (int k = kmin; k <= kmax; ++k) {
    h_off[k - kmin] = acc;
    acc += (int64_t)host_binom(N, k);
  }
  return acc;
}

// Pass 1 of the two-pass full-output stencil as a column pass: the low-bit
// neighbour sum S[P] = sum_{j in P_low} T[P ^ 2^j] only couples blocks that
// share their high prefix bits and only entries at the same position, so a
// CTA takes one high-bit pattern Ph and a column of E adjacent storage
// positions, stages that column of all 2^LB low-bit blocks in shared memory
// (2^LB segments of 8E bytes, cp.async), and writes the column of S with
// every neighbour read from shared memory.  Each table entry crosses HBM
// once and each sum once: no neighbour block is re-read through L2 (the
// TMA-ring pass it replaces re-read ~5 neighbour blocks per block from L2
// and ran at 4.9 TB/s; this one runs at ~6.2 TB/s, 0.93 of the measured copy
// rate).  Persistent 256-thread CTAs (one per SM at LB = 10), the next
// column's loads in flight while the current one is summed (two stages).  Positions
// are storage positions, so S keeps T's swizzled layout; neighbours are
// added far bits first, as the TMA-ring pass adds them (compacted partial
// scans and block shards still run that pass, and their rows must stay
// bit-identical to the whole-range scan's).  Measured alternatives (cfg4, ncu): one
// stage of 16-entry columns 3.05 ms, three CTAs/SM of 8-entry columns 3.32,
// 512 threads 2.90, a loop over the set bits only 4.6 (divergent) -- this
// form 2.76 ms.
constexpr int kColThreads = 256;

template <int LB, int E>
__device__ __forceinline__ void col_load(const double *__restrict__ T, double *buf, unsigned job) {
  constexpr int NB = 1 << LB, H = E / 2;
  constexpr unsigned kCols = BLK / E;
  const unsigned ph = job / kCols, col = job % kCols;
  const int64_t base = ((int64_t)ph << LB) * BLK + (int64_t)col * E;
#pragma unroll 4
  for (int x = threadIdx.x; x < NB * H; x += kColThreads) {
    const int pl = x / H, q = x % H;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(buf + pl * E + 2 * q)),
                 "l"(T + base + (int64_t)pl * BLK + 2 * q)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int LB, int E>
__device__ __forceinline__ void col_sum(const double *buf, double *__restrict__ S, unsigned job) {
  constexpr int NB = 1 << LB, H = E / 2;
  constexpr unsigned kCols = BLK / E;
  const unsigned ph = job / kCols, col = job % kCols;
  const int64_t base = ((int64_t)ph << LB) * BLK + (int64_t)col * E;
  const double2 *b2 = reinterpret_cast<const double2 *>(buf);
#pragma unroll 2
  for (int x = threadIdx.x; x < NB * H; x += kColThreads) {
    const int pl = x / H, q = x % H;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = LB - 1; j >= 0; --j)    // far bits first: the TMA-ring pass's order
      if ((pl >> j) & 1) {
        const double2 v = b2[(pl ^ (1 << j)) * H + q];
        acc.x += v.x;
        acc.y += v.y;
      }
    *reinterpret_cast<double2 *>(S + base + (int64_t)pl * BLK + 2 * q) = acc;
  }
}

template <int LB, int E>
__global__ void __launch_bounds__(kColThreads, 1)
k_lattice_lowsum(const double *__restrict__ T, double *__restrict__ S, unsigned njobs) {
  extern __shared__ __align__(16) double sv[];   // [2][2^LB][E]
  constexpr int STAGE = (1 << LB) * E;
  unsigned job = blockIdx.x;
  int cur = 0;
  if (job < njobs) col_load<LB, E>(T, sv, job);
  for (; job < njobs; job += gridDim.x) {
    const unsigned nxt = job + gridDim.x;
    if (nxt < njobs) {
      col_load<LB, E>(T, sv + (cur ^ 1) * STAGE, nxt);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    col_sum<LB, E>(sv + cur * STAGE, S, job);
    __syncthreads();   // the stage is refilled by the next iteration's loads
    cur ^= 1;
  }
}

template <int LB>
static int launch_lowsum_t(const double *T, double *S, int nP, cudaStream_t s) {
  // two stages <= 128 KB; 16-entry columns measured slower at LB = 9 (3.30
  // vs 2.74 ms at LB = 10 with 8), and a 9/11 split of cfg4's prefix bits
  // slower than 10/10 either way (pass 2 +0.5 ms / column pass +1.9 ms)
  constexpr int E = LB >= 11 ? 4 : 8;
  constexpr int kSmem = 2 * (1 << LB) * E * (int)sizeof(double);
  constexpr int kPerSm = kSmem <= 64 * 1024 ? 3 : 1;
  static thread_local int set_for = -1, sms = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_for != dev) {
    cudaFuncSetAttribute(k_lattice_lowsum<LB, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    set_for = dev;
  }
  const unsigned njobs = (1u << (nP - LB)) * (unsigned)(BLK / E);
  const unsigned grid = std::min<unsigned>(njobs, (unsigned)sms * kPerSm);
  k_lattice_lowsum<LB, E><<<grid, kColThreads, kSmem, s>>>(T, S, njobs);
  return check_launch("k_lattice_lowsum");
}

// -1: no column kernel for this split (the caller runs the TMA-ring pass)
static int launch_lowsum(const double *T, double *S, int nP, int lb, cudaStream_t s) {
  switch (lb) {
    case 7: return launch_lowsum_t<7>(T, S, nP, s);
    case 8: return launch_lowsum_t<8>(T, S, nP, s);
    case 9: return launch_lowsum_t<9>(T, S, nP, s);
    case 10: return launch_lowsum_t<10>(T, S, nP, s);
    case 11: return launch_lowsum_t<11>(T, S, nP, s);
    default: return -1;
  }
}

template <int R, int C, int F, int NB = 2>
static int run_stencil(const LatticeWs &w, int N, int D, int d, const double *eta, int kstride,
                       int kmin, int kmax, int64_t g_begin, int64_t g_end, double *out,
                       int64_t plane, unsigned blk_begin, unsigned blk_end, const uint8_t *active,
                       const StencilFilter &flt, const StencilPass &ps, cudaStream_t s) {
  static thread_local int set_for = -1;
  static thread_local int grid_cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = (int)sizeof(StencilSmem<R, NB>);
  if (set_for != dev) {
    cudaFuncSetAttribute(k_lattice_measures<R, C, F, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lattice_measures<R, C, F, NB>,
                                                  kStencilThreads + 32, smem);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
    set_for = dev;
  }
  const unsigned n = blk_end - blk_begin;
  const unsigned grid = n < (unsigned)grid_cap ? n : (unsigned)grid_cap;
  if (grid == 0) return HOI_OK;
  k_lattice_measures<R, C, F, NB><<<grid, kStencilThreads + 32, smem, s>>>(
      w.table, N, D, d, kmin, kmax, eta, kstride, w.offs, g_begin, g_end, out, plane, blk_begin,
      blk_end, active, w.counter, flt, ps);
  return check_launch("k_lattice_measures");
}

template <bool FAST>
static int run_full_t(const LatticeWs &w, int N, int D, int d, const double *eta, int kstride,
                      int kmin, int kmax, int64_t g_begin, int64_t g_end, double *out,
                      int64_t plane, unsigned blk_begin, unsigned blk_end, const uint8_t *active,
                      const StencilPass &ps, cudaStream_t s) {
  static thread_local int set_for = -1;
  static thread_local int grid_cap = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = (int)sizeof(FullSmem<FAST>);
  if (set_for != dev) {
    cudaFuncSetAttribute(k_lattice_full<FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lattice_full<FAST>,
                                                  kStencilThreads + 32, smem);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
    set_for = dev;
  }
  const unsigned n = blk_end - blk_begin;
  const unsigned grid = n < (unsigned)grid_cap ? n : (unsigned)grid_cap;
  if (grid == 0) return HOI_OK;
  k_lattice_full<FAST><<<grid, kStencilThreads + 32, smem, s>>>(w.table, N, D, d, kmin, kmax, eta,
                                                                kstride, w.offs, g_begin, g_end,
                                                                out, plane, blk_begin, blk_end,
                                                                active, w.counter, ps);
  return check_launch("k_lattice_full");
}

static int run_full(const LatticeWs &w, int N, int D, int d, const double *eta, int kstride,
                    int kmin, int kmax, int64_t g_begin, int64_t g_end, double *out, int64_t plane,
                    unsigned blk_begin, unsigned blk_end, const uint8_t *active,
                    const StencilPass &ps, cudaStream_t s) {
  int64_t h_off[MAXV + 1];
  const bool whole = g_begin == 0 && g_end == total_rows(N, kmin, kmax, h_off);
  // FAST holds each block's last ring job (its pass-1-sum job at least: the
  // two-pass split) as the neighbour-sum buffer, so it needs ps.extra
  if (D == 1 && !eta && whole && !ps.local && ps.nstack == 0 && ps.extra)
    return run_full_t<true>(w, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out, plane,
                            blk_begin, blk_end, active, ps, s);
  return run_full_t<false>(w, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out, plane,
                           blk_begin, blk_end, active, ps, s);
}

// Persistent stencil launch over table blocks [blk_begin, blk_end): one
// CTA per resident slot (SMs x occupancy).  For a partial rank range the
// blocks without output are flagged first (one thread per block) and
// skipped without streaming them.  local: write block-major local rows
// (the compacted list's claim order; see StencilPass::local).
static int launch_stencil(const LatticeWs &w, int N, int D, int d, const double *eta, int kstride,
                          int kmin, int kmax, int64_t g_begin, int64_t g_end, double *out,
                          unsigned blk_begin, unsigned blk_end, bool partial, bool flags_ready,
                          cudaStream_t s, const StencilFilter *flt = nullptr,
                          int64_t local_rows = 0) {
  const unsigned nblocks = 1u << (N - CB);
  uint8_t *active = partial ? reinterpret_cast<uint8_t *>(w.ready) : nullptr;
  if (partial && !flags_ready) {
    k_block_active<<<(nblocks + 255) / 256, 256, 0, s>>>(N, kmin, kmax, w.offs, g_begin, g_end,
                                                          nblocks, active);
    int st = check_launch("k_block_active");
    if (st) return st;
  }
  const int64_t plane = (local_rows ? local_rows : g_end - g_begin) * (int64_t)D;
  const int nP = N - CB;
  const unsigned all = (1u << nP) - 1u;
  // Two-pass split over the whole block space (nP >= 14): pass 1 writes the
  // sums over the low LB = nP/2 prefix bits' neighbours (natural order: they
  // lie within 2^LB blocks); pass 2 claims blocks high-bits-fastest and
  // streams only the high-bit neighbours (within 2^(nP-LB) blocks) plus the
  // pass-1 sums and the own block.  Both windows are a few MB, so neighbour
  // reads hit L2 instead of costing ~(nP - log2 L2-blocks)/2 DRAM re-reads per
  // block; the price is one extra write + read of the table size.
  // Measured on B200, cfg4: full output 19.25 ms two-pass vs 20.41 single
  // (DRAM 68.8 vs 84.2 GB); the filtered (TopK) pass writes nothing and is
  // bound by per-job TMA latency rather than bytes, so there the single pass
  // wins (11.4 ms vs 3.4 + 9.6 ms).
  const bool two = !flt && nP >= 14 && blk_begin == 0 && blk_end == (1u << nP) && w.lowsum;
  const int lb = nP / 2;
  const StencilFilter none{};
  StencilPass ps{all, nullptr, nullptr, 0, nullptr, nullptr, 0u, local_rows ? 1 : 0};
  // partial / sampled scans over the whole block space: compacted block
  // lists (natural order for a single pass or pass 1, high-bits-fastest for
  // pass 2) in the workspace after the flags
  const bool listed = active && blk_begin == 0 && blk_end == (1u << nP);
  if (local_rows && !listed) return fail(HOI_INVALID_ARG, "lattice: local rows need a block list");
  unsigned *list1 = w.list, *list2 = w.list + (1u << nP), *cnts = w.list + 2 * (1u << nP);
  if (listed) {
    const unsigned ntiles = ((1u << nP) + kCompactTile - 1) / kCompactTile;
    unsigned *tiles = cnts + 16;
    k_count_blocks<<<ntiles, 256, 0, s>>>(active, nP, 0, tiles);
    k_write_blocks<<<ntiles, 256, 0, s>>>(active, nP, 0, tiles, list1, cnts);
    if (two) {
      k_count_blocks<<<ntiles, 256, 0, s>>>(active, nP, lb, tiles + 1024);
      k_write_blocks<<<ntiles, 256, 0, s>>>(active, nP, lb, tiles + 1024, list2, cnts + 1);
    }
    int st = check_launch("k_count_blocks/k_write_blocks");
    if (st) return st;
    ps.list = list1;
    ps.nlist = cnts;
  }
  if (two) {
    // the low pass stores its sums straight from registers: no neighbour-sum
    // buffer or run table, so 6 ring slots fit at 4 CTAs/SM
    // (whole-range scans: the column pass; compacted partial scans keep the
    // TMA-ring pass over their active blocks)
    int st = listed ? -1 : launch_lowsum(w.table, w.lowsum, nP, lb, s);
    if (st < 0) {
      const StencilPass p1{(1u << lb) - 1u, nullptr, w.lowsum, 0, ps.list, ps.nlist, 0u, 0};
      cudaMemsetAsync(w.counter, 0, sizeof(unsigned), s);
      st = run_stencil<kRingLean, 4, MODE_LOWSUM, 0>(w, N, D, d, eta, kstride, kmin, kmax,
                                                     g_begin, g_end, out, plane, blk_begin,
                                                     blk_end, active, none, p1, s);
    }
    if (st) return st;
    ps = StencilPass{all & ~((1u << lb) - 1u), w.lowsum, nullptr, lb, listed ? list2 : nullptr,
                     listed ? cnts + 1 : nullptr, 0u, local_rows ? 1 : 0};
  }
  cudaMemsetAsync(w.counter, 0, sizeof(unsigned), s);
  // Filter mode finishes entries from registers (no neighbour-sum buffer),
  // so 6 ring slots fit at 4 CTAs/SM: 24 TMA jobs in flight per SM, not 16.
  if (flt)
    return run_stencil<kRingLean, 4, MODE_FILTER, 0>(w, N, D, d, eta, kstride, kmin, kmax,
                                                     g_begin, g_end, out, plane, blk_begin,
                                                     blk_end, active, *flt, ps, s);
  return run_full(w, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out, plane, blk_begin,
                  blk_end, active, ps, s);
}

int lattice_measures(void *ws, int N, int D, int d, const double *eta, int kstride, int kmin,
                     int kmax, int64_t g_begin, int64_t g_end, double *out, cudaStream_t s) {
  upload_binomials();
  upload_tables();
  LatticeWs w = ws_view(ws, N);
  int64_t h_off[MAXV + 1];
  const int64_t total = total_rows(N, kmin, kmax, h_off);
  cudaMemcpyAsync(w.offs, h_off, sizeof(int64_t) * (kmax - kmin + 1), cudaMemcpyHostToDevice, s);
  const bool partial = g_begin > 0 || g_end < total;
  return launch_stencil(w, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out, 0u,
                        1u << (N - CB), partial, false, s);
}

// Filtered stencil over the whole rank space of [kmin, kmax] (or every
// `every`-th table block): candidates with key <= *key_max (see
// StencilFilter).  The table must be complete (lattice_table + status).
int lattice_filter(void *ws, int N, int D, int d, const double *eta, int kstride, int kmin,
                   int kmax, int m_idx, double sign, unsigned every, const uint64_t *key_max,
                   double *cand, int64_t cand_cap, unsigned long long *count, cudaStream_t s) {
  upload_binomials();
  upload_tables();
  LatticeWs w = ws_view(ws, N);
  int64_t h_off[MAXV + 1];
  const int64_t total = total_rows(N, kmin, kmax, h_off);
  cudaMemcpyAsync(w.offs, h_off, sizeof(int64_t) * (kmax - kmin + 1), cudaMemcpyHostToDevice, s);
  const unsigned nblocks = 1u << (N - CB);
  bool sampled = every > 1;
  if (sampled) {
    k_block_sample<<<(nblocks + 255) / 256, 256, 0, s>>>(nblocks, every,
                                                         reinterpret_cast<uint8_t *>(w.ready));
    int st = check_launch("k_block_sample");
    if (st) return st;
  }
  StencilFilter f{m_idx, sign, key_max, cand, count, cand_cap};
  return launch_stencil(w, N, D, d, eta, kstride, kmin, kmax, 0, total, nullptr, 0u, nblocks,
                        sampled, sampled, s, &f);
}

// Block-sharded scan (multi-GPU): shard `shard` of 2^sb owns the table
// blocks whose top sb prefix bits equal shard and computes every n-plet of
// those blocks, written at its GLOBAL row in `out` (full-size, rows
// [0, total)); the union over shards is the whole scan and no row is
// written twice.  It rebuilds only the table chunks its stencil reads: its
// own and, for every set bit t of shard, the chunk shard with t cleared
// (neighbours only ever remove a variable).  With filter != nullptr the
// shard's n-plets go through the TopK filter instead (every > 1: a hash
// sample of the shard's blocks).
int lattice_status(void *ws, int N, cudaStream_t s);

// Block shards `mask` (bit c = shard c of 2^sb owned by this GPU): build the
// table chunks their stencil reads -- each owned chunk and every chunk that
// differs from one by a single cleared bit, each once -- then stream the
// owned blocks.  Owning complementary chunks (c and 2^sb - 1 - c) evens out
// the rebuild work across GPUs (sharding.block_shard_plan).
int lattice_shard(const double *corr, int N, int D, int d, const double *eta, int kstride,
                  int kmin, int kmax, unsigned long long mask, int sb, unsigned every,
                  double *out, const StencilFilter *flt, bool build, void *ws, size_t ws_bytes,
                  cudaStream_t s, int64_t local_rows = 0) {
  size_t need = 0;
  int st = lattice_ws_bytes(N, D, &need);
  if (st) return st;
  if (ws_bytes < need) return fail(HOI_CAPACITY, "lattice: workspace too small");
  const int nP = N - CB;
  const int bexp = nP < MAXB ? nP : MAXB;        // prefix variables a table CTA expands
  if (sb < 0 || sb > nP / 2 || sb > 6 || sb > nP - bexp || mask == 0 ||
      (sb < 6 && (mask >> (1 << sb)) != 0))
    return fail(HOI_INVALID_ARG, "lattice_shard: need a non-empty shard mask below 2^(2^sb), "
                                 "sb <= min(6, (N-10)/2, N-16)");
  upload_binomials();
  upload_tables();
  LatticeWs w = ws_view(ws, N);
  int64_t h_off[MAXV + 1];
  const int64_t total = total_rows(N, kmin, kmax, h_off);
  cudaMemcpyAsync(w.offs, h_off, sizeof(int64_t) * (kmax - kmin + 1), cudaMemcpyHostToDevice, s);
  const int b = nP < MAXB ? nP : MAXB;
  const unsigned chunk_ctas = 1u << (nP - b - sb);     // table CTAs of one shard chunk
  if (build) cudaMemsetAsync(w.flag, 0, sizeof(int), s);
  for (unsigned c = 0; build && c < (1u << sb); ++c) {
    bool need = false;                                 // c owned, or an owned shard minus one bit
    for (unsigned o = 0; o < (1u << sb) && !need; ++o)
      need = ((mask >> o) & 1ull) && (c & ~o) == 0 && __builtin_popcount(o ^ c) <= 1;
    if (!need) continue;
    launch_table<8>(dim3(chunk_ctas), s, corr, N, D, d, b, w.table, w.flag,
                                                  c * chunk_ctas);
    if ((st = check_launch("k_lattice_table"))) return st;
  }
  if (build && (st = lattice_status(ws, N, s))) return st;
  const unsigned nblocks = 1u << nP;
  k_block_shard<<<(nblocks + 255) / 256, 256, 0, s>>>(nblocks, nP, sb, mask, every,
                                                      reinterpret_cast<uint8_t *>(w.ready));
  if ((st = check_launch("k_block_shard"))) return st;
  return launch_stencil(w, N, D, d, eta, kstride, kmin, kmax, 0, total, out, 0u, nblocks, true,
                        true, s, flt, local_rows);
}

// The block list the last local-rows stencil claimed from (local block c =
// list[c]): pass 2's high-bits-fastest list when the scan ran two passes.
static void copy_local_list(const LatticeWs &w, int N, unsigned *blocks, int64_t *count,
                            cudaStream_t s) {
  const int nP = N - CB;
  const bool two = nP >= 14 && w.lowsum;
  const unsigned *list = w.list + (two ? (1u << nP) : 0u);
  const unsigned *cnt = w.list + 2 * (1u << nP) + (two ? 1 : 0);
  cudaMemcpyAsync(blocks, list, sizeof(unsigned) << nP, cudaMemcpyDeviceToDevice, s);
  k_count_to_i64<<<1, 1, 0, s>>>(cnt, count);
}

// Local rows -> global rows: local block c (table block P = blocks[c]) holds
// 1024 rows in run order; row p of it is the n-plet P u Q(p) at global rank
// run_base(P, q) + t.  Rows in [g_begin, g_end) are copied to
// out[row - g_begin] (the 4 planes of a (rows, D) output); rows of orders
// outside [kmin, kmax] are holes and are skipped.
__global__ void k_local_scatter(const double *__restrict__ local, int64_t lplane,
                                const unsigned *__restrict__ blocks, const int64_t *__restrict__ nb,
                                int N, int D, int kmin, int kmax,
                                const int64_t *__restrict__ order_off, int64_t g_begin,
                                int64_t g_end, double *__restrict__ out, int64_t oplane) {
  __shared__ int64_t base[CB + 1];
  const int64_t n = *nb;
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
    const unsigned P = blocks[c];
    __syncthreads();
    if (threadIdx.x <= CB) base[threadIdx.x] = run_base(P, threadIdx.x, N, kmin, kmax, order_off, g_begin);
    __syncthreads();
    for (int p = threadIdx.x; p < BLK; p += blockDim.x) {
      const uint32_t wv = __ldg(g_run + p);
      const int t = (wv >> 10) & 1023, q = wv >> 20;
      const int64_t b0 = base[q];
      if (b0 == kNoRun) continue;
      const int64_t row = b0 + t;
      if (row < 0 || row >= g_end - g_begin) continue;
      for (int dd = 0; dd < D; ++dd) {
        const int64_t li = (c * BLK + p) * D + dd, oi = row * D + dd;
#pragma unroll
        for (int m = 0; m < 4; ++m) out[m * oplane + oi] = local[m * lplane + li];
      }
    }
  }
}

int lattice_status(void *ws, int N, cudaStream_t s) {
  LatticeWs w = ws_view(ws, N);
  int h_flag = 0;
  cudaMemcpyAsync(&h_flag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (h_flag) return fail(HOI_FALLBACK, "lattice: correlation matrix not numerically positive "
                                        "definite; rerun with the per-n-plet engine");
  return HOI_OK;
}

int scan_full_lattice(const double *corr, const double *eta, int kstride, int N, int D, int kmin,
                      int kmax, int64_t g_begin, int64_t g_end, double *out, int32_t *err_count,
                      void *ws, size_t ws_bytes, cudaStream_t s) {
  (void)err_count;
  // Sequential table -> stencil per dataset (the chunked two-stream
  // pipeline measured no gain).  The not-PD flag is checked
  // once after every dataset (one host sync per scan, not per dataset): a
  // failing table leaves garbage rows, and HOI_FALLBACK makes the host rerun
  // the whole scan on the per-n-plet engine with the reference's jitter rule.
  int64_t h_off[MAXV + 1];
  const int64_t total = total_rows(N, kmin, kmax, h_off);
  const int slots = batch_slots(N, D);
  if (slots > 1 && g_begin == 0 && g_end == total) {
    // stacked: tables of `slots` datasets in one table launch (grid.y) and
    // one stencil launch over their 2^(N-10) x slots blocks
    upload_binomials();
    upload_tables();
    LatticeWs w = ws_view(ws, N);
    cudaMemsetAsync(w.flag, 0, sizeof(int), s);
    cudaMemcpyAsync(w.offs, h_off, sizeof(int64_t) * (kmax - kmin + 1), cudaMemcpyHostToDevice, s);
    LatticeWs wb = w;
    wb.table = batch_tables(ws, N);
    const int nP = N - CB;
    const int b = nP < MAXB ? nP : MAXB;
    for (int d0 = 0; d0 < D; d0 += slots) {
      const int n = D - d0 < slots ? D - d0 : slots;
      launch_table<8>(dim3(1u << (nP - b), (unsigned)n), s, corr, N, D, d0, b,
                                                                           wb.table, w.flag, 0u);
      int st = check_launch("k_lattice_table");
      if (st) return st;
      const StencilPass ps{(1u << nP) - 1u, nullptr, nullptr, 0, nullptr, nullptr, (unsigned)n, 0};
      cudaMemsetAsync(w.counter, 0, sizeof(unsigned), s);
      const unsigned claims = (unsigned)((n + 3) & ~3) << nP;   // 4-dataset groups
      st = run_full(wb, N, D, d0, eta, kstride, kmin, kmax, 0, total, out, total * (int64_t)D, 0u,
                    claims, nullptr, ps, s);
      if (st) return st;
    }
    return lattice_status(ws, N, s);
  }
  LatticeWs w = ws_view(ws, N);
  cudaMemsetAsync(w.flag, 0, sizeof(int), s);
  for (int d = 0; d < D; ++d) {
    int st = lattice_table(corr, N, D, d, ws, ws_bytes, s, false);
    if (st) return st;
    st = lattice_measures(ws, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out, s);
    if (st) return st;
  }
  return lattice_status(ws, N, s);
}

}  // namespace hoib

using namespace hoib;

extern "C" int hoi_lattice_table(const double *corr, int32_t N, int32_t D, int32_t d, void *ws,
                                 size_t ws_bytes, void *stream) {
  HOI_CHECK_ARG(corr && ws && d >= 0 && d < D, "hoi_lattice_table: bad args");
  return lattice_table(corr, N, D, d, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int hoi_lattice_measures(void *ws, int32_t N, int32_t D, int32_t d, const double *eta,
                                    int32_t kstride, int32_t kmin, int32_t kmax, int64_t g_begin,
                                    int64_t g_end, double *out, void *stream) {
  HOI_CHECK_ARG(ws && out && lattice_supports(N) && d >= 0 && d < D && kmin >= 1 &&
                    kmin <= kmax && kmax <= N && g_begin >= 0 && g_begin <= g_end,
                "hoi_lattice_measures: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_measures: bias table too short");
  return lattice_measures(ws, N, D, d, eta, kstride, kmin, kmax, g_begin, g_end, out,
                          (cudaStream_t)stream);
}

extern "C" int hoi_lattice_filter(void *ws, int32_t N, int32_t D, int32_t d, const double *eta,
                                  int32_t kstride, int32_t kmin, int32_t kmax, int32_t m_idx,
                                  double sign, int32_t every, const uint64_t *key_max,
                                  double *cand, int64_t cand_cap, uint64_t *count, void *stream) {
  HOI_CHECK_ARG(ws && key_max && cand && count && lattice_supports(N) && d >= 0 && d < D &&
                    kmin >= 1 && kmin <= kmax && kmax <= N && m_idx >= 0 && m_idx < 4 &&
                    every >= 1 && cand_cap >= 0,
                "hoi_lattice_filter: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_filter: bias table too short");
  return lattice_filter(ws, N, D, d, eta, kstride, kmin, kmax, m_idx, sign, (unsigned)every,
                        key_max, cand, cand_cap, reinterpret_cast<unsigned long long *>(count),
                        (cudaStream_t)stream);
}

extern "C" int hoi_lattice_shard(const double *corr, int32_t N, int32_t D, int32_t d,
                                 const double *eta, int32_t kstride, int32_t kmin, int32_t kmax,
                                 int32_t shard, int32_t shard_bits, double *out, void *ws,
                                 size_t ws_bytes, void *stream) {
  HOI_CHECK_ARG(corr && ws && out && lattice_supports(N) && d >= 0 && d < D && kmin >= 1 &&
                    kmin <= kmax && kmax <= N,
                "hoi_lattice_shard: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_shard: bias table too short");
  HOI_CHECK_ARG(shard_bits >= 0 && shard_bits <= 6 && shard >= 0 && shard < (1 << shard_bits),
                "hoi_lattice_shard: need 0 <= shard < 2^shard_bits <= 64");
  return lattice_shard(corr, N, D, d, eta, kstride, kmin, kmax, 1ull << shard, shard_bits, 1u,
                       out, nullptr, true, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int hoi_lattice_shard_set(const double *corr, int32_t N, int32_t D, int32_t d,
                                     const double *eta, int32_t kstride, int32_t kmin,
                                     int32_t kmax, uint64_t shard_mask, int32_t shard_bits,
                                     double *out, void *ws, size_t ws_bytes, void *stream) {
  HOI_CHECK_ARG(corr && ws && out && lattice_supports(N) && d >= 0 && d < D && kmin >= 1 &&
                    kmin <= kmax && kmax <= N,
                "hoi_lattice_shard_set: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_shard_set: bias table too short");
  return lattice_shard(corr, N, D, d, eta, kstride, kmin, kmax, shard_mask, shard_bits, 1u, out,
                       nullptr, true, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int hoi_lattice_shard_local(const double *corr, int32_t N, int32_t D, int32_t d,
                                       const double *eta, int32_t kstride, int32_t kmin,
                                       int32_t kmax, uint64_t shard_mask, int32_t shard_bits,
                                       double *out, int64_t local_rows, uint32_t *blocks,
                                       int64_t *nblocks, void *ws, size_t ws_bytes, void *stream) {
  HOI_CHECK_ARG(corr && ws && out && blocks && nblocks && lattice_supports(N) && d >= 0 &&
                    d < D && kmin >= 1 && kmin <= kmax && kmax <= N && local_rows > 0,
                "hoi_lattice_shard_local: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_shard_local: bias table too short");
  const int sb = shard_bits;
  HOI_CHECK_ARG(sb >= 0 && sb <= 6 && shard_mask != 0, "hoi_lattice_shard_local: bad shards");
  const int64_t need = (int64_t)__builtin_popcountll(shard_mask) << (N - sb);
  HOI_CHECK_ARG(local_rows >= need, "hoi_lattice_shard_local: local_rows < shard blocks x 1024");
  cudaStream_t s = (cudaStream_t)stream;
  int st = lattice_shard(corr, N, D, d, eta, kstride, kmin, kmax, shard_mask, shard_bits, 1u,
                         out, nullptr, true, ws, ws_bytes, s, local_rows);
  if (st) return st;
  copy_local_list(ws_view(ws, N), N, blocks, nblocks, s);
  return check_launch("k_count_to_i64");
}

extern "C" int hoi_lattice_local_scatter(const double *local, int64_t local_rows,
                                         const uint32_t *blocks, const int64_t *nblocks,
                                         int32_t N, int32_t D, int32_t kmin, int32_t kmax,
                                         int64_t g_begin, int64_t g_end, double *out,
                                         void *stream) {
  HOI_CHECK_ARG(local && blocks && nblocks && out && lattice_supports(N) && D >= 1 &&
                    kmin >= 1 && kmin <= kmax && kmax <= N && g_begin >= 0 && g_begin <= g_end,
                "hoi_lattice_local_scatter: bad args");
  upload_binomials();
  upload_tables();
  int64_t h_off[MAXV + 1];
  total_rows(N, kmin, kmax, h_off);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *offs = nullptr;
  if (stream_alloc((void **)&offs, sizeof(h_off), s) != cudaSuccess)
    return fail(HOI_CUDA_ERROR, "hoi_lattice_local_scatter: allocation failed");
  cudaMemcpyAsync(offs, h_off, sizeof(int64_t) * (kmax - kmin + 1), cudaMemcpyHostToDevice, s);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_local_scatter<<<8 * sms, 256, 0, s>>>(local, local_rows * (int64_t)D, blocks, nblocks,
                                                  N, D, kmin, kmax, offs, g_begin, g_end, out,
                                                  (g_end - g_begin) * (int64_t)D);
  const int st = check_launch("k_local_scatter");
  cudaFreeAsync(offs, s);
  return st;
}

extern "C" int hoi_lattice_shard_filter(const double *corr, int32_t N, int32_t D, int32_t d,
                                        const double *eta, int32_t kstride, int32_t kmin,
                                        int32_t kmax, int32_t shard, int32_t shard_bits,
                                        int32_t every, int32_t m_idx, double sign,
                                        const uint64_t *key_max, double *cand, int64_t cand_cap,
                                        uint64_t *count, int32_t build_table, void *ws,
                                        size_t ws_bytes, void *stream) {
  HOI_CHECK_ARG(corr && ws && key_max && cand && count && lattice_supports(N) && d >= 0 &&
                    d < D && kmin >= 1 && kmin <= kmax && kmax <= N && m_idx >= 0 && m_idx < 4 &&
                    every >= 1,
                "hoi_lattice_shard_filter: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_shard_filter: bias table too short");
  HOI_CHECK_ARG(shard_bits >= 0 && shard_bits <= 6 && shard >= 0 && shard < (1 << shard_bits),
                "hoi_lattice_shard_filter: need 0 <= shard < 2^shard_bits <= 64");
  StencilFilter f{m_idx, sign, key_max, cand, reinterpret_cast<unsigned long long *>(count),
                  cand_cap};
  return lattice_shard(corr, N, D, d, eta, kstride, kmin, kmax, 1ull << shard, shard_bits,
                       (unsigned)every, nullptr, &f, build_table != 0, ws, ws_bytes,
                       (cudaStream_t)stream);
}

extern "C" int hoi_lattice_shard_set_filter(const double *corr, int32_t N, int32_t D, int32_t d,
                                            const double *eta, int32_t kstride, int32_t kmin,
                                            int32_t kmax, uint64_t shard_mask,
                                            int32_t shard_bits, int32_t every, int32_t m_idx,
                                            double sign, const uint64_t *key_max, double *cand,
                                            int64_t cand_cap, uint64_t *count,
                                            int32_t build_table, void *ws, size_t ws_bytes,
                                            void *stream) {
  HOI_CHECK_ARG(corr && ws && key_max && cand && count && lattice_supports(N) && d >= 0 &&
                    d < D && kmin >= 1 && kmin <= kmax && kmax <= N && m_idx >= 0 && m_idx < 4 &&
                    every >= 1,
                "hoi_lattice_shard_set_filter: bad args");
  HOI_CHECK_ARG(!eta || kstride > kmax, "hoi_lattice_shard_set_filter: bias table too short");
  StencilFilter f{m_idx, sign, key_max, cand, reinterpret_cast<unsigned long long *>(count),
                  cand_cap};
  return lattice_shard(corr, N, D, d, eta, kstride, kmin, kmax, shard_mask, shard_bits,
                       (unsigned)every, nullptr, &f, build_table != 0, ws, ws_bytes,
                       (cudaStream_t)stream);
}

extern "C" int hoi_lattice_status(void *ws, int32_t N, void *stream) {
  HOI_CHECK_ARG(ws && lattice_supports(N), "hoi_lattice_status: bad args");
  return lattice_status(ws, N, (cudaStream_t)stream);
}
