/*
 * hoi_b200.h -- C ABI of libhoib200.so, the B200 (sm_100a) engine behind the
 * n-plet higher-order-interaction hot path.
 *
 * The reference (/root/reference/pkg/src/hoi) is a pure-Python package and
 * has no FFI of its own.  Each entry point below replaces one numeric stage
 * of its hot path; the citation names the reference function whose
 * behaviour it carries (ref:<file>:<line>).  The Python host layer
 * (paper_2501_03381_b200/) keeps the reference's Python signatures and calls
 * these through ctypes (see INTEGRATION.md for the binding).
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless named h_*;
 *     buffers are caller-allocated, the library never allocates in a hot
 *     call except inside an explicit workspace argument;
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     asynchronous on that stream unless documented otherwise;
 *   - calls on different streams/devices are reentrant; the only global
 *     state is a thread-local last-error string;
 *   - return value is an HOI_* status code.
 *
 * Layouts
 *   corr    (N, N, D) float64, dataset index fastest: corr[(i*N + j)*D + d]
 *           is the correlation form R = D^-1/2 Sigma D^-1/2 of dataset d
 *           (unit diagonal, exactly symmetric);
 *   sdiag   (D, N) float64, the covariance diagonal Sigma_jj (jitter scale);
 *   eta     (D, kstride) float64 finite-sample bias table eta(k, T_d) or NULL
 *           (ref:copula_core.py:234-244);
 *   out     4 planes of (B, D) float64: tc, dtc, o, s, plane stride B*D
 *           (the HoiBatch layout, ref:measures.py:18-27).
 */
#ifndef HOI_B200_H
#define HOI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HOI_OK = 0,
  HOI_INVALID_ARG = 1,          /* -> InvalidData / InvalidNplet            */
  HOI_INSUFFICIENT_SAMPLES = 2, /* -> InsufficientSamples                   */
  HOI_NOT_PD = 3,               /* -> NotPositiveDefinite (see err buffers) */
  HOI_CUDA_ERROR = 4,
  HOI_CAPACITY = 5,             /* workspace / output too small             */
  HOI_FALLBACK = 6              /* lattice engine declined (matrix not PD):
                                   rerun with engine 1, whose per-n-plet
                                   jitter retry matches the reference      */
};

/* Library version (major*10000 + minor*100 + patch). */
int hoi_version(void);

/* Last error message of the calling thread ("" if none). */
const char *hoi_last_error(void);

/* Number of kernels this library launched from the calling process
 * (monotone counter; used by bench.py's gpu_launches and by tests). */
int64_t hoi_launch_count(void);

/* ---------------------------------------------------------------------------
 * (1) Gaussian copula + covariance.
 * ------------------------------------------------------------------------- */

/* Ordinal per-column ranks with ties broken by row (stable) and the copula
 * values z = qgrid[rank-1].  Replaces rank_columns + copula_transform
 * (ref:copula_core.py:155-174).
 *   x      (D, T, N) float64 row-major data (already validated/finite);
 *   qgrid  (T,) float64 = ndtri((1..T)/(T+1)) computed on the host with the
 *          reference's scipy routine, so z is bit-identical to the reference;
 *   ranks  (D, T, N) int64 output, 1-based, or NULL;
 *   z      (D, T, N) float64 output;
 *   ws     device workspace of ws_bytes (query with ws == NULL: the required
 *          size is written to *ws_bytes and HOI_OK returned). */
int hoi_rank_copula(const double *x, int64_t T, int32_t N, int32_t D,
                    const double *qgrid, int64_t *ranks, double *z,
                    void *ws, size_t *ws_bytes, void *stream);

/* hoi_rank_copula with column-major outputs: ranks_t and z_t are (D, N, T)
 * (a variable's T values contiguous), the layout the rank sort and the
 * covariance panels stream; the (T, N) outputs of hoi_rank_copula are one
 * more transpose of these.  ws: query with ws == NULL as above. */
int hoi_rank_copula_cols(const double *x, int64_t T, int32_t N, int32_t D,
                         const double *qgrid, int64_t *ranks_t, double *z_t, void *ws,
                         size_t *ws_bytes, void *stream);

/* Unbiased covariance (divisor T-1) of centred columns, upper triangle
 * computed once and mirrored so cov == cov^T exactly.  Replaces
 * estimate_covariance (ref:copula_core.py:177-189).
 *   z (D, T, N) float64 -> cov (D, N, N) float64. */
int hoi_covariance(const double *z, int64_t T, int32_t N, int32_t D,
                   double *cov, void *stream);
/* hoi_covariance of a column-major (D, N, T) z_t (hoi_rank_copula_cols). */
int hoi_covariance_cols(const double *z_t, int64_t T, int32_t N, int32_t D, double *cov,
                        void *stream);

/* Correlation form used by every measure kernel: corr (N,N,D) and sdiag (D,N)
 * from cov (D,N,N).  The measures only depend on log det R_S and the
 * inverse diagonal of R_S (the per-variable log Sigma_jj terms cancel in
 * tc/dtc/o/s, ref:measures.py:41-69). */
int hoi_correlation(const double *cov, int32_t N, int32_t D, double *corr,
                    double *sdiag, void *stream);

/* ---------------------------------------------------------------------------
 * (2) Batched n-plet evaluation (gather + Cholesky + inverse diagonal +
 *     bias + TC/DTC/O/S epilogue).  Replaces extract_subcov_batch +
 *     _batched_logdet_invdiag + entropy_terms + compute_hoi_batch for
 *     fixed-order batches (ref:nplet_engine.py:185-201,227-330;
 *     ref:measures.py:72-81).
 *
 *   idx        (B, K) int32 strictly increasing rows;
 *   out        4 x (B, D) measures or NULL;
 *   logdet     (B, D) log det Sigma_S or NULL         } entropy_terms compat
 *   invdiag    (B, D, K) (Sigma_S^-1)_jj or NULL      } (ref:nplet_engine.py:312-330)
 *   err_count  device int32 counter (caller zeroes it);
 *   err_coords device int64 pairs (b, d) of matrices that stayed non-PD
 *              after the reference's single jitter retry
 *              eps = 1e-10 * trace(Sigma_S) / K (ref:nplet_engine.py:237-264);
 *              at most err_cap pairs are stored, the counter keeps counting.
 * ------------------------------------------------------------------------- */
int hoi_eval_indices(const double *corr, const double *sdiag, const double *eta,
                     int32_t kstride, int32_t N, int32_t D, const int32_t *idx,
                     int64_t B, int32_t K, double *out, double *logdet,
                     double *invdiag, int32_t *err_count, int64_t *err_coords,
                     int32_t err_cap, void *stream);

/* hoi_eval_indices (measures only) into rows [0, B) of a larger output
 * whose planes are out_plane elements apart: one chunk of a (4, rows, D)
 * result (pass out + r0 * D).  Lets a large host index batch stream to the
 * device chunk by chunk, each chunk's kernel overlapping the next chunk's
 * upload.  Error rows are chunk-relative. */
int hoi_eval_indices_into(const double *corr, const double *sdiag, const double *eta,
                          int32_t kstride, int32_t N, int32_t D, const int32_t *idx, int64_t B,
                          int32_t K, double *out, int64_t out_plane, int32_t *err_count,
                          int64_t *err_coords, int32_t err_cap, void *stream);

/* Mixed-order (mask) batches: masks (B, W) uint64 words (bit j of word j/64
 * = variable j).  Equivalent to identity padding (ref:nplet_engine.py:204-224,
 * 332-351): each row is compacted to its members and evaluated at its own
 * order.  invdiag, when requested, is (B, D, N) with zeros outside the row
 * and logdet (B, D). */
int hoi_eval_masks(const double *corr, const double *sdiag, const double *eta,
                   int32_t kstride, int32_t N, int32_t D, const uint64_t *masks,
                   int32_t W, int64_t B, double *out, double *logdet,
                   double *invdiag, int32_t *err_count, int64_t *err_coords,
                   int32_t err_cap, void *stream);

/* Raw matrix stack: (logdet, inverse diagonal) of M matrices (M, K, K) with
 * the same jitter rule.  Replaces _batched_logdet_invdiag
 * (ref:nplet_engine.py:267-281); err_coords hold (m, 0). */
/* FP32 fast path of hoi_eval_indices (the north star's optional FP32 path,
 * within 1e-4 nats of the FP64 result): the same units, gathered from corr32
 * (an FP32 copy of corr) and factorised in FP32 for orders K <= 16 (log
 * products, bias and the epilogue stay FP64; a failing pivot reruns that unit
 * on the FP64 path with the reference's jitter rule); orders above 16 run
 * the FP64 kernels.  Measures only (no log det / inverse-diagonal outputs). */
int hoi_eval_indices_fp32(const double *corr, const float *corr32, const double *sdiag,
                          const double *eta, int32_t kstride, int32_t N, int32_t D,
                          const int32_t *idx, int64_t B, int32_t K, double *out,
                          int32_t *err_count, int64_t *err_coords, int32_t err_cap,
                          void *stream);

int hoi_logdet_invdiag(const double *mats, int64_t M, int32_t K,
                       double *logdet, double *invdiag, int32_t *err_count,
                       int64_t *err_coords, int32_t err_cap, void *stream);

/* ---------------------------------------------------------------------------
 * (3) Enumeration: global order-major lexicographic rank -> k-subset
 *     (ref:nplet_engine.py:118-136 chained at ref:scanner.py:345-347).
 *     idx_out (count, kmax) int32 padded with -1; order_out (count,) int32.
 *     Requires N <= 64.
 * ------------------------------------------------------------------------- */
int hoi_unrank(int32_t N, int32_t kmin, int32_t kmax, int64_t g_begin,
               int64_t count, int32_t *idx_out, int32_t *order_out,
               void *stream);

/* Same for an explicit list of global ranks (TopK candidates). */
int hoi_unrank_list(int32_t N, int32_t kmin, int32_t kmax, const int64_t *ranks,
                    int64_t count, int32_t *idx_out, int32_t *order_out, void *stream);

/* ---------------------------------------------------------------------------
 * (4) Exhaustive scan over the global rank range [g_begin, g_end) of orders
 *     kmin..kmax, full output: out is 4 planes of ((g_end-g_begin), D)
 *     measures in enumeration order (the concatenation of every batch the
 *     reference's scan would hand to its reducer, ref:scanner.py:308-365).
 *
 *     engine: 0 = auto, 1 = per-n-plet Cholesky (unrank + K-templated
 *     register kernels, any N <= 64), 2 = subset-lattice engine (N <= 34:
 *     log-det table over all 2^N subsets + leave-one-out stencil; needs the
 *     workspace, query its size with ws == NULL).
 * ------------------------------------------------------------------------- */
int hoi_scan_full(const double *corr, const double *sdiag, const double *eta,
                  int32_t kstride, int32_t N, int32_t D, int32_t kmin,
                  int32_t kmax, int64_t g_begin, int64_t g_end, int32_t engine,
                  double *out, int32_t *err_count, int64_t *err_coords,
                  int32_t err_cap, void *ws, size_t *ws_bytes, void *stream);

/* The two phases of engine 2, exposed separately so a caller can time them
 * or reuse one table across several rank ranges.  ws is the engine-2
 * workspace of hoi_scan_full (query its size there).
 *   hoi_lattice_table:    T[S] = log det R_S for all 2^N subsets of dataset d;
 *   hoi_lattice_status:   synchronous; HOI_FALLBACK if a pivot was <= 0;
 *   hoi_lattice_measures: stencil + measures for ranks [g_begin, g_end) of
 *                         orders kmin..kmax into out (layout of hoi_scan_full). */
int hoi_lattice_table(const double *corr, int32_t N, int32_t D, int32_t d, void *ws,
                      size_t ws_bytes, void *stream);
int hoi_lattice_status(void *ws, int32_t N, void *stream);
int hoi_lattice_measures(void *ws, int32_t N, int32_t D, int32_t d, const double *eta,
                         int32_t kstride, int32_t kmin, int32_t kmax, int64_t g_begin,
                         int64_t g_end, double *out, void *stream);

/* Filtered stencil (scan with a TopK reducer, ref:scanner.py:50-105):
 * the engine-2 stencil over every n-plet of orders kmin..kmax of dataset d
 * (or over every `every`-th table block, a sample) that writes, instead of
 * the full output, the n-plets whose key sign * measure[m_idx] (m_idx:
 * 0 tc, 1 dtc, 2 o, 3 s) has an order-preserving 64-bit form <= *key_max
 * (device), as 40-byte records {global rank (int64 bits), tc, dtc, o, s}
 * appended to cand.  *count (device uint64, caller zeroes) counts every
 * match even past cand_cap.  The table of dataset d must be built
 * (hoi_lattice_table + hoi_lattice_status).  Asynchronous. */
int hoi_lattice_filter(void *ws, int32_t N, int32_t D, int32_t d, const double *eta,
                       int32_t kstride, int32_t kmin, int32_t kmax, int32_t m_idx,
                       double sign, int32_t every, const uint64_t *key_max, double *cand,
                       int64_t cand_cap, uint64_t *count, void *stream);

/* Block-sharded engine-2 scan (one process per GPU, no data-path
 * collective; replaces the reference's in-process thread pool over batches,
 * ref:scanner.py:290-305, across GPUs, with scan's output semantics,
 * ref:scanner.py:308-365): shard `shard` of 2^shard_bits (shard_bits <= (N-10)/2) owns
 * the log-det table blocks whose top shard_bits prefix-variable bits equal
 * `shard`, i.e. every n-plet whose intersection with variables
 * N-10-shard_bits..N-11 is that pattern.  It rebuilds only the table
 * chunks its stencil reads (its own and the chunks with one of its bits
 * cleared) and writes each of its n-plets at its GLOBAL row of `out`
 * (full-size layout of hoi_scan_full over [0, total)); the shards' row sets
 * partition the scan.  Synchronous on a non-PD table (HOI_FALLBACK).
 * hoi_lattice_shard_filter: the same shard through the TopK filter of
 * hoi_lattice_filter (every > 1: a hash sample of the shard's blocks;
 * build_table = 0 reuses the chunks built by a previous call). */
int hoi_lattice_shard(const double *corr, int32_t N, int32_t D, int32_t d, const double *eta,
                      int32_t kstride, int32_t kmin, int32_t kmax, int32_t shard,
                      int32_t shard_bits, double *out, void *ws, size_t ws_bytes, void *stream);
int hoi_lattice_shard_filter(const double *corr, int32_t N, int32_t D, int32_t d,
                             const double *eta, int32_t kstride, int32_t kmin, int32_t kmax,
                             int32_t shard, int32_t shard_bits, int32_t every, int32_t m_idx,
                             double sign, const uint64_t *key_max, double *cand,
                             int64_t cand_cap, uint64_t *count, int32_t build_table, void *ws,
                             size_t ws_bytes, void *stream);
/* hoi_lattice_shard_set / _set_filter: several shards on one GPU, bit c of
 * shard_mask = shard c of 2^shard_bits (shard_bits <= 6); each needed table
 * chunk is built once.  Owning complementary shards (c and 2^shard_bits-1-c)
 * balances the rebuild work across GPUs (sharding.block_shard_plan). */
int hoi_lattice_shard_set(const double *corr, int32_t N, int32_t D, int32_t d, const double *eta,
                          int32_t kstride, int32_t kmin, int32_t kmax, uint64_t shard_mask,
                          int32_t shard_bits, double *out, void *ws, size_t ws_bytes,
                          void *stream);
int hoi_lattice_shard_set_filter(const double *corr, int32_t N, int32_t D, int32_t d,
                                 const double *eta, int32_t kstride, int32_t kmin, int32_t kmax,
                                 uint64_t shard_mask, int32_t shard_bits, int32_t every,
                                 int32_t m_idx, double sign, const uint64_t *key_max,
                                 double *cand, int64_t cand_cap, uint64_t *count,
                                 int32_t build_table, void *ws, size_t ws_bytes, void *stream);

/* Multi-GPU FULL output with compact shards (ref:scanner.py:290-305's
 * ordered merge, done by the caller): hoi_lattice_shard_set's n-plets
 * written block-major to a LOCAL output -- local block c holds the 1024
 * n-plets P u Q of table block P = blocks[c] in run order at rows
 * c*1024 .. c*1024+1023 (rows of orders outside [kmin, kmax] are holes) --
 * instead of at their global rows.  local_rows >= popcount(shard_mask) *
 * 2^(N - shard_bits); out is 4 planes of (local_rows, D).  blocks (device,
 * 2^(N-10) u32) and *nblocks (device int64) receive the block list.
 * Asynchronous after the table's not-PD check. */
int hoi_lattice_shard_local(const double *corr, int32_t N, int32_t D, int32_t d,
                            const double *eta, int32_t kstride, int32_t kmin, int32_t kmax,
                            uint64_t shard_mask, int32_t shard_bits, double *out,
                            int64_t local_rows, uint32_t *blocks, int64_t *nblocks, void *ws,
                            size_t ws_bytes, void *stream);
/* Local rows -> global rows: every row of a hoi_lattice_shard_local output
 * whose global rank lies in [g_begin, g_end) is copied to
 * out[rank - g_begin] (4 planes of (g_end - g_begin, D)).  The receive side
 * of the rank-ordered gather: the shards of all ranks, scattered into one
 * output, equal the single-GPU scan bit for bit. */
int hoi_lattice_local_scatter(const double *local, int64_t local_rows, const uint32_t *blocks,
                              const int64_t *nblocks, int32_t N, int32_t D, int32_t kmin,
                              int32_t kmax, int64_t g_begin, int64_t g_end, double *out,
                              void *stream);

/* ---------------------------------------------------------------------------
 * (5) Device reducers over a full-output plane (ref:scanner.py:50-137).
 * ------------------------------------------------------------------------- */

/* Exact TopK candidates (ref:scanner.py:75-100): positions p of plane
 * `vals` (stride D, dataset d) whose key sign*vals[p*D+d] is among the k
 * smallest, plus the remainder of the k-th key's final 12-bit radix bucket
 * (at most bucket_cap extra), so every tie at the k-th value is included.
 * Radix select over the order-preserving 64-bit key, then one filter pass.
 * Synchronous; *h_count (HOST) receives the candidate count (may exceed
 * cand_cap when a tie is wider than the buffer; then only cand_cap stored).
 * ws: device workspace of at least 4097 uint64. */
int hoi_topk_select(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                    int64_t k, int64_t bucket_cap, int64_t *cand, int64_t cand_cap,
                    int64_t *h_count, void *ws, void *stream);

/* TopK.update for every dataset of a batch (ref:scanner.py:75-100):
 * hoi_topk_select for all D datasets of a (n, D) plane at once (D <= 64;
 * 8-bit radix digits, per-dataset histograms): dataset d's candidate
 * positions go to cand[d * cand_cap ...] and their count to h_counts[d]
 * (HOST array of D).  ws: device workspace of >= D*256 + 5*D + 32 uint64.
 * The radix rounds run without host round trips; one sync at the end. */
int hoi_topk_select_multi(const double *vals, int64_t n, int32_t D, double sign, int64_t k,
                          int64_t bucket_cap, int64_t *cand, int64_t cand_cap,
                          int64_t *h_counts, void *ws, void *stream);

/* Exact TopK order of the candidates (ref:scanner.py:75-100, key
 * (sign*value, index tuple) ascending) for every dataset of a fixed-order
 * batch: CTA d sorts cand[d*cand_cap ...] (counts[d] of them, DEVICE int64
 * array of D; cand_cap <= 8192) by the orderable key of sign*vals[p*D+d],
 * equal keys by the lexicographic tuple idx[p*K .. p*K+K) (int32), equal
 * tuples by p, and writes the first k positions to top_pos[d*k ...] (-1
 * past counts[d]).  Asynchronous. */
int hoi_topk_order(const double *vals, int32_t D, double sign, const int64_t *cand,
                   int64_t cand_cap, const int64_t *counts, const int32_t *idx, int32_t K,
                   int64_t k, int64_t *top_pos, void *stream);

/* Exact k-th smallest key (the threshold step of TopK, ref:scanner.py:75-100):
 * the order-preserving 64-bit key of the k-th
 * smallest sign*vals[p*D+d] over p < n (full radix select), written to
 * device memory *key_out; all-ones when n <= k.  Synchronous.  ws: device
 * workspace of at least 4096 uint64. */
int hoi_topk_threshold(const double *vals, int64_t n, int32_t D, int32_t d, double sign,
                       int64_t k, uint64_t *key_out, void *ws, void *stream);
/* hoi_topk_bound: an upper bound of that key -- the end of its bucket after
 * resolving its top `bits` bits (12 per synchronous radix round); bits >= 64
 * gives the exact key.  The lattice TopK threshold uses 36 bits. */
int hoi_topk_bound(const double *vals, int64_t n, int32_t D, int32_t d, double sign, int64_t k,
                   int32_t bits, uint64_t *key_out, void *ws, void *stream);

/* Candidate filter for TopK: writes the positions p in [0, n) of plane
 * `vals` (stride D, dataset d) whose key sign*vals[p*D+d] <= *thresh into
 * cand (int64), counting into *cand_count (device int64, caller zeroes).
 * Stores at most cand_cap positions. */
int hoi_topk_filter(const double *vals, int64_t n, int32_t D, int32_t d,
                    double sign, const double *thresh, int64_t *cand,
                    int64_t *cand_count, int64_t cand_cap, void *stream);

/* Optimiser objective (ref:optimizers.py:74-102): energy[b] = sign *
 * aggregate of row b of a (B, D) plane over the D datasets -- mode 0 the
 * mean, mode 1 the paired Cohen's d mean(v_a - v_b) / std(v_a - v_b, ddof 1)
 * over the npairs (cond_a[i], cond_b[i]) (device int32 arrays).  A zero or
 * non-finite pair deviation sets *degenerate (device int32, caller zeroes). */
int hoi_objective(const double *vals, int64_t B, int32_t D, int32_t mode, const int32_t *cond_a,
                  const int32_t *cond_b, int32_t npairs, double sign, double *energy,
                  int32_t *degenerate, void *stream);

/* 21-feature accumulator partials (ref:scanner.py:205-287) of one
 * full-output chunk: 4 planes of (rows, D) at global ranks g0 .. g0+rows-1;
 * ranks in [pair_begin, pair_end) are the order-2 rows.  feat (device,
 * D x 19 doubles): pair count, pair sum tc, pair sum tc^2, count (order >=
 * 3), sums (tc dtc o s), maxima, minima, first global rank attaining the o
 * maximum / minimum, count o < 0.  Deterministic (fixed reduction order).
 * ws: device workspace of >= 8 * 148 * 256 * 19 doubles (ws_doubles). */
int hoi_features(const double *out, int64_t rows, int32_t D, int64_t g0, int64_t pair_begin,
                 int64_t pair_end, double *feat, void *ws, int64_t ws_doubles, void *stream);

/* Histogram with numpy.histogram semantics after clipping to [lo, hi]
 * (ref:scanner.py:126-134): counts (D, bins) int64 accumulated. */
int hoi_histogram(const double *vals, int64_t n, int32_t D, int32_t bins,
                  double lo, double hi, const double *edges, int64_t *counts,
                  void *stream);

/* ---------------------------------------------------------------------------
 * Diagnostics: FP64 pipe peak probe (the roofline denominator for the FP64
 * kernels; MEASURED_PEAKS.json has no FP64 entry).  flops per launch =
 * blocks * 256 * iters * 128.  out needs `blocks` doubles.
 * ------------------------------------------------------------------------- */
int hoi_fp64_probe(double *out, int64_t iters, int32_t blocks, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HOI_B200_H */
