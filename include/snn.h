/*
 * snn.h -- C ABI of the B200-native SNN hot path (arXiv 2212.07679, "sorting-based
 * exact fixed-radius near-neighbour search").  Plain C: no CUDA or torch types.
 *
 * Problem (§3, §3.2): given data p_1..p_n in R^d and query
 * points q (in- or out-of-sample) and a radius R, return every i with ||p_i - q|| <= R
 * (inclusive), with its Euclidean distance ("can also return the corresponding distances
 * if needed").  The result is EXACT: it equals fp64 brute force computed as
 * s = sum_k (p_ik - q_k)^2 left to right without FMA, hit iff s <= R*R (DESIGN.md
 * readings C1, C3, C5).
 *
 * Conventions for every entry point
 *  - Array arguments are row-major with row stride d (contiguous).  They may be DEVICE
 *    pointers (current CUDA device) or HOST pointers (pageable or pinned); host inputs
 *    are staged to the device inside the call (this is the end-to-end path).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    device work is ordered on it.  Every call is synchronous with respect to its
 *    results: on return the outputs are valid (a query reads its output size from the
 *    device once).
 *  - Errors: a non-OK status is returned and snn_last_error() gives a thread-local
 *    message.  Output handles are left NULL on error.  Nothing is leaked on error.
 *  - Index ids are 0-based original row numbers of X; n must be < 2^30.
 *  - Thread safety: an index is immutable after snn_build; concurrent queries and DBSCAN
 *    runs on one index (different streams / threads) are allowed, each
 *    with its own workspace; snn_append / snn_free must not race a query.  Options
 *    (snn_set_option) and the last-query diagnostics are per thread; the profiler
 *    (snn_profile_*) is process-wide.
 */
#ifndef SNN_H
#define SNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SNN_F32 = 0, SNN_F64 = 1 } snn_dtype;

/* Distance of an index (§3 "other distances"):
 *  EUCLIDEAN  ||p - q||, radius R.
 *  COSINE     cdist(u, v) = 1 - u.v on unit vectors; 2 cdist = ||u - v||^2,
 *             so a cosine radius r is the Euclidean radius sqrt(2 r) on normalized rows.
 *  ANGULAR    theta(u, v) <= alpha  iff  ||u - v||^2 <= 2 - 2 cos(alpha);
 *             radius alpha in radians.
 * For COSINE / ANGULAR the rows of X and Q are normalized on the device with the exact
 * rule u_k = x_k / sqrt(sum_k x_k^2) (fp64, left-to-right sum, correctly rounded sqrt and
 * division, then rounded to the input dtype); the search itself is the exact Euclidean
 * search on the normalized rows with the mapped radius (computed in fp64), and returned
 * distances are converted back to the metric (r = d^2 / 2, alpha = 2 asin(d / 2)).
 *  MANHATTAN  ||p - q||_1 <= R.  Since ||.||_2 <= ||.||_1 the Euclidean search with the same
 *             R returns a superset; an exact fp64 post-filter (sum of
 *             |p_k - q_k| left to right) keeps the hits; distance = float(L1).
 *  MIPS       inner-product similarity p^T q >= tau (the radius argument is tau, any finite
 *             value): the index holds p~ = [sqrt(xi^2 - |p|^2), p],
 *             xi = max |p|, queries q~ = [0, q], so |p~ - q~|^2 = xi^2 + |q|^2 - 2 p^T q; the
 *             Euclidean search with radius^2 = (xi^2 + max|q|^2)(1 + 4e-6) - 2 tau (+ slack)
 *             returns a superset, an exact fp64 post-filter (sum of p_k q_k left to right)
 *             keeps p^T q >= tau; "distance" = float(p^T q).  snn_index_info.d is d + 1.
 *  MANHATTAN / MIPS keep a copy of the input rows for the filter; snn_dbscan rejects them
 *  (SNN_ERR_UNSUPPORTED). */
typedef enum { SNN_METRIC_EUCLIDEAN = 0, SNN_METRIC_COSINE = 1, SNN_METRIC_ANGULAR = 2,
               SNN_METRIC_MANHATTAN = 3, SNN_METRIC_MIPS = 4 } snn_metric;

typedef enum {
    SNN_OK = 0,
    SNN_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, d < 1, m < 0, R < 0 or non-finite, ... */
    SNN_ERR_EMPTY = 2,            /* n == 0 ("empty dataset", Alg. 1 needs >= 1 point)   */
    SNN_ERR_NONFINITE = 3,        /* NaN / Inf in X or Q                                 */
    SNN_ERR_DIM_MISMATCH = 4,     /* query d or dtype differs from the index             */
    SNN_ERR_OUT_OF_MEMORY = 5,
    SNN_ERR_CUDA = 6,             /* any other CUDA runtime error                        */
    SNN_ERR_UNSUPPORTED = 7       /* n >= 2^30, or device is not sm_100                  */
} snn_status;

typedef struct snn_index_s *snn_index;   /* opaque; immutable after build  */
typedef struct snn_result_s *snn_result; /* opaque; owns CSR device buffers */

/* CSR view of a query result.  Row j = query j in the caller's query order.  All three
 * arrays are DEVICE pointers owned by the snn_result.  Within a row, hits are in
 * ascending order of the index's sort key (deterministic); graded as sets. */
typedef struct {
    int64_t m;                 /* number of queries (rows)                        */
    int64_t nnz;               /* number of (query, point) hits                   */
    const int64_t *offsets;    /* m + 1, offsets[0] = 0, offsets[m] = nnz         */
    const int32_t *indices;    /* nnz original row ids of X                       */
    const float *distances;    /* nnz Euclidean distances, = (float)sqrt(s_fp64)  */
} snn_csr;

/* Spectrum diagnostic (eq:svd; sigma_2 enters the analysis of the
 * window, eq:sigma2): sigma[0..k) = the k largest singular values of the centred data the
 * index was BUILT from (appended rows are not included), by power iteration with
 * deflation on the kept Gram matrix (fp64, one CTA on the device; k <= min(d, 16); MIPS
 * indexes: of the d + 1 transformed rows).  A large tensor-core build (n*d >= 2^27,
 * option "gram_rows") keeps only the Gram matrix of a strided row sample -- v1 only steers
 * the pruning -- and then this call first recomputes the full Gram matrix from the rows
 * currently indexed (appended rows included, centred at the build mean).  sigma: host array
 * of k doubles.  Diagnostic only -- the search uses v1 from the build.  Synchronizes the
 * stream. */
snn_status snn_index_sigma(snn_index idx, int32_t k, double *sigma, void *stream);

/* Diagnostics of a built index (Algorithm 1 outputs). */
typedef struct {
    int64_t n;
    int32_t d;
    int32_t dtype;             /* snn_dtype                                        */
    int32_t ld;                /* row stride (elements) of the sorted copy; 0 = AoSoA4:
                                  element (i, k) at xs[(i/4)*4*d + k*4 + i%4] (d <= 8) */
    int32_t power_iters;       /* power iterations used for v1                     */
    double sigma1;             /* top singular value of the centered data          */
    double key_err;            /* rigorous bound E_x on |computed key - exact key|  */
    double v1_norm;            /* ||v1 as stored in fp32||_2                        */
    const double *mu;          /* device, d: column mean (fp64)                     */
    const float *v1;           /* device, d: top principal direction (fp32, unit)   */
    const float *keys;         /* device, n: sorted projection keys alpha (fp32)    */
    const int32_t *perm;       /* device, n: pi[sorted position] = original id      */
    const float *xbar;         /* device, n: half squared norms of centered sorted rows */
    const void *xs;            /* device, n x ld: original coordinates in key order */
    int32_t tc_operand;        /* tensor-core filter operands: 0 none (FFMA / SIMT path),
                                  1 FP16 (kind::f16, scaled by 2^tc_exp), 2 TF32         */
    int32_t tc_kpad;           /* K of the tensor-core operand copy (padded d)          */
    int32_t tc_exp;            /* FP16 operand scale exponent of the index copy         */
    int32_t metric;            /* snn_metric                                            */
} snn_index_info_t;

/*
 * snn_build -- Algorithm 1 "SNN Index":
 *   mu = mean(p_j) (l.2), X = P - mu (l.3), v1 = top right singular vector of X (l.4,
 *   eq:svd PAPER.md:94-102; computed by power iteration on X^T X), alpha_i = x_i^T v1
 *   (l.5), sort by alpha (l.6; stable, ties by original id), xbar_i = x_i^T x_i / 2 (l.7).
 * X: n x d, dtype dt (SNN_F32 or SNN_F64), host or device.  X may be freed after return
 * (the index keeps its own sorted copy).  Errors: n == 0 -> SNN_ERR_EMPTY; d < 1, NULL X
 * or out -> SNN_ERR_INVALID_ARGUMENT; NaN/Inf -> SNN_ERR_NONFINITE; n >= 2^30 ->
 * SNN_ERR_UNSUPPORTED.
 */
snn_status snn_build(const void *X, int64_t n, int32_t d, snn_dtype dt, void *stream,
                     snn_index *out);

/* Streaming append ("applicable in an online streaming setting"): adds k rows Y
 * (k x d row-major, device or host pointer, the index's dtype; the index's metric applies,
 * COSINE / ANGULAR rows are normalized) with ids n .. n+k-1.  mu and v1 stay frozen: the
 * window bound of eq:lower holds for any fixed unit vector and centring,
 * so results stay exact; only pruning may degrade if the new rows drift.  Keys of the new
 * rows under (mu, v1), one stable re-sort (ties by original id), key error bounds and the
 * tensor-core operand copy recomputed.  Errors: DIM_MISMATCH; NONFINITE (index unchanged);
 * UNSUPPORTED for MIPS (xi would change) or n + k >= 2^30.  k = 0 is a no-op.
 * Synchronizes the stream. */
snn_status snn_append(snn_index idx, const void *Y, int64_t k, int32_t d, snn_dtype dt, void *stream);

/* Save / load the built index (all device arrays incl. the kept Gram; no rebuild on load).  File: "SNNG",
 * u32 version 1, 23 int64 header words, then the arrays in a fixed order, little endian.
 * snn_load validates the magic ("bad magic"), version ("unsupported version"), header
 * ("invalid header"), length ("truncated" / "trailing bytes") and the index invariants
 * (keys sorted and finite, perm a permutation) before touching the device; all of these
 * return SNN_ERR_INVALID_ARGUMENT.  A loaded index answers queries bit-identically, and
 * save -> load -> save writes identical bytes.  Both synchronize the stream. */
snn_status snn_save(snn_index idx, const char *path, void *stream);
snn_status snn_load(const char *path, void *stream, snn_index *out);

/* snn_build for a metric (snn_metric).  EUCLIDEAN == snn_build.  COSINE / ANGULAR: rows
 * are normalized first (see snn_metric); a zero row -> SNN_ERR_INVALID_ARGUMENT.  Radii
 * of snn_query_radius / snn_query_self / snn_dbscan on this index are in the metric's
 * units (cosine distance in [0, 2], angle in radians), and so are returned distances. */
snn_status snn_build_metric(const void *X, int64_t n, int32_t d, snn_dtype dt, int32_t metric,
                            void *stream, snn_index *out);

/*
 * snn_query_radius -- Algorithm 2 "SNN Query" for a batch of m
 * queries (batched as in PAPER.md:218-219, per block of consecutive key-sorted queries):
 *   x_q = q - mu (l.2), alpha_q = x_q^T v1 (l.3), candidate range J from the sorted keys
 *   by binary search (l.4, eq:lower PAPER.md:142-153, padded by rigorous rounding bounds),
 *   exact radius test over X(J,:) (l.5-6, eq:ip1/eq:ip2 PAPER.md:205-216).
 * Q: m x d, same dtype as the index (dt), host or device.  m == 0 is valid (offsets =
 * {0}).  R >= 0 and finite (R == 0 returns exact coincidences).  Errors: d or dt differ
 * from the index -> SNN_ERR_DIM_MISMATCH; R < 0 / NaN, m < 0, NULL -> INVALID_ARGUMENT;
 * NaN/Inf in Q -> SNN_ERR_NONFINITE.  *out owns the CSR buffers (snn_result_free).
 */
snn_status snn_query_radius(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt,
                            double R, void *stream, snn_result *out);

/* Self-query: identical to snn_query_radius(idx, X, n, d, dt, R, ...) with the X the
 * index was built from (every point is its own neighbour), without re-projecting X. */
snn_status snn_query_self(snn_index idx, double R, void *stream, snn_result *out);

/* Query sharding across GPUs (queries are independent,
 * batching only forms a union of windows).  Every GPU holds a replicated index (built from
 * the same X) and calls the _part variant with its rank: the key-sorted query blocks are
 * split into `nparts` contiguous ranges balanced by window length (the work), and part
 * `part` computes only its blocks.  The result is a CSR over ALL m queries in which rows
 * of other parts are empty, so the parts' results are disjoint and their union (per row)
 * is exactly the unpartitioned result; no data-path collective is needed (results stay
 * sharded; an all-gather of per-part nnz rebases offsets if a global CSR is wanted).
 * Self-queries stay symmetric (each unordered pair evaluated once): the part owns the
 * rows of its blocks, and the blocks before it whose windows reach its first position run
 * as ghost blocks clipped to its candidates, supplying its rows' mirrored entries (the
 * pairs crossing a part boundary are evaluated by both parts; nothing is exchanged).
 * Errors as snn_query_radius / snn_query_self, plus INVALID_ARGUMENT unless
 * 0 <= part < nparts. */
snn_status snn_query_radius_part(snn_index idx, const void *Q, int64_t m, int32_t d, snn_dtype dt, double R,
                                 int32_t part, int32_t nparts, void *stream, snn_result *out);
snn_status snn_query_self_part(snn_index idx, double R, int32_t part, int32_t nparts, void *stream,
                               snn_result *out);

/* Asynchronous copy of the CSR to caller-owned buffers (as snn_result_copy): the copies
 * are enqueued on `stream` and the call returns at once; the buffers are valid after the
 * stream synchronizes.  A later snn_result_free(r) is ordered after these copies (the
 * device buffers are released on `stream`).  With pinned host buffers the device-to-host
 * transfer overlaps whatever the caller runs next on other streams (bench.py's pipelined
 * end-to-end mode: step k's copy-out runs under step k+1's build and query). */
snn_status snn_result_copy_async(snn_result r, int64_t *offsets, int32_t *indices, float *distances,
                                 void *stream);

/* CSR view (device pointers, valid until snn_result_free). */
snn_status snn_result_csr(snn_result r, snn_csr *view);

/* Copy the CSR to caller-owned buffers, HOST or DEVICE (offsets m+1, indices nnz,
 * distances nnz; indices / distances may be NULL to skip).  Synchronous. */
snn_status snn_result_copy(snn_result r, int64_t *offsets, int32_t *indices,
                           float *distances, void *stream);

void snn_result_free(snn_result r); /* NULL ok */
/* As snn_result_free, with the device buffers released in `stream`'s order (after any
 * snn_result_copy_async copy): memory freed on the stream that allocates next is reused
 * without cross-stream pool dependencies (a compute stream running step after step). */
void snn_result_free_async(snn_result r, void *stream); /* NULL ok */

/*
 * snn_dbscan -- DBSCAN with SNN as the neighbourhood backend, exact
 * readings of DESIGN.md C18: eps-neighbourhoods are closed balls incl. the point itself;
 * core iff |N_eps| >= min_pts; clusters = connected components of core points under
 * eps-adjacency; a non-core point with a core neighbour takes the cluster of its
 * smallest-id core neighbour; others are noise (-1); clusters are numbered 0..K-1 by
 * increasing smallest core id.  labels: n int32, host or device, ORIGINAL order.
 * *n_clusters (host) receives K.  d <= 8: fused count / union / border passes over the
 * candidate windows (neighbour lists are never materialised); larger d: the exact
 * self-query CSR (snn_query_self) feeds the same count / union / border steps.
 * Errors: NULL arguments, eps < 0 or non-finite, min_pts < 1 -> SNN_ERR_INVALID_ARGUMENT.
 */
snn_status snn_dbscan(snn_index idx, double eps, int32_t min_pts, int32_t *labels,
                      int32_t *n_clusters, void *stream);

void snn_free(snn_index idx); /* NULL ok */
/* Grow the device's stream-ordered memory pool (which every call allocates from and which
 * keeps freed memory) by `bytes` up front, so that later calls do not map new memory
 * while other streams are busy.  Synchronizes the stream. */
snn_status snn_pool_reserve(uint64_t bytes, void *stream);

/* As snn_free, with the index's device buffers released in `stream`'s order. */
void snn_free_async(snn_index idx, void *stream); /* NULL ok */

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char *snn_last_error(void);

snn_status snn_index_info(snn_index idx, snn_index_info_t *info);

/* Number of kernels this library has launched in this process (monotone counter). */
uint64_t snn_launch_count(void);

/* Kernel-time profiling (diagnostics; process-global; off by default).  While enabled,
 * the library brackets each kernel family with CUDA events on the launching stream and
 * accumulates device time.  snn_profile_enable(1) also resets the counters.
 * snn_profile_read synchronises the recorded events and returns, for `family`:
 *   ms        summed device milliseconds,      launches  number of bracketed launches,
 *   units     work units processed (window passes: candidate pairs evaluated; build:
 *             points indexed), summed.
 * Families: "build"; "window_count" (low d: the scan pass that counts and records hits;
 * generic d: the count pass; tensor-core path: the tcgen05 filter; DBSCAN: the count
 * pass); "window_write" (low d: CSR compaction + overflow fix,
 * units = hits; generic d: the recomputing write pass); "query" (whole query call);
 * "dbscan" (whole snn_dbscan call, units = points);
 * "overflow" (units = hit records that went to the overflow list in the last low-d query);
 * "lost" (units = work items re-run by the fix pass in the last low-d query).
 * Unknown family -> SNN_ERR_INVALID_ARGUMENT. */
snn_status snn_profile_enable(int on);
snn_status snn_profile_read(const char *family, double *ms, uint64_t *launches, double *units);

/* Test / tuning hooks.  Options are PER CALLING THREAD: snn_set_option changes the options
 * of the calls this thread makes (every thread starts from the defaults), so concurrent
 * callers never switch each other's paths.  0 restores the default:
 *   "force_generic"  1 = use the generic-d FFMA tile kernel even for d <= 16
 *   "query_block"    queries per block for the low-d kernel (32..256, multiple of 32)
 *   "chunk"          candidates per work item (multiple of 64)
 *   "power_iters"    cap on power iterations (>= 1)
 *   "cap"            hit-record slots per (work item, query) in the low-d scan pass
 *                    (1..1024); further records go to a global overflow list
 *   "ovf_records"    capacity of that overflow list (entries that do not fit are
 *                    recomputed by a fix pass)
 *   "variant"        low-d scan loop: 1 = deferred-hit 2-group loop (default), 2 = 8-pair
 *                    direct loop
 *   "symmetric"      -1 = evaluate every pair twice in low-d self-queries (default: once)
 *   "scan2q"         fp32 low-d scan with two queries per thread (128-thread CTAs, each staged
 *                    filter row feeds two queries): 0 = auto (default: on for 2 <= d <= 8),
 *                    1 = on for every d <= 8, -1 = off
 *   "chunk2q"        candidates per work item of that scan (default 640, multiple of 64)
 *   "stage_rows"     1 = the compaction assembles rows in a key-order staging buffer, then
 *                    moves each row whole; default (0 / -1): it writes the final rows directly
 *   "balanced_compact" -1 = per-entry compaction threads (default for symmetric self-queries:
 *                    one slot record per thread after CTA scans)
 *   "window_all"     1 = brute-force ablation: every query scans all n candidates
 *   "gram_rows", "gram_min_elems"   tensor-core Gram of a build with n*d >= gram_min_elems
 *                    (default 2^27) uses every ceil(n / gram_rows)-th row (default 65536;
 *                    -1 = every row)
 *   "finalize_order" -1 = row assembly walks rows in key order (default: original-id order,
 *                    sequential CSR writes)
 *   "count_warp"     -1 = DBSCAN core counts by one CTA per query block over whole chunks
 *                    (default: one warp per point, scanning outward from its position)
 *   "union_load"     DBSCAN union pass: how the parent[j] pre-check is loaded (1 = default
 *                    ld.relaxed.gpu, -1 volatile, 2 ld.global.cg; every value is a valid
 *                    filter; snn_get_option reports 0 volatile / 1 relaxed / 2 cg)
 *                    (applies to the window_lowd union pass, union_snap = -1)
 *   "union_snap"     DBSCAN union pass for fp32, d <= 8: 1 = default, the staged root-snapshot
 *                    kernel (a pair reaches the union path only when its staged root differs
 *                    from the query's); -1 = window_lowd union pass; 2 = the same kernel
 *                    without the register cap; 3, 4 = diagnostics only (no unions, labels
 *                    NOT valid)
 *   "union_behind"   union_snap pass: 1 = default, candidates behind the block (pairs j < i,
 *                    already settled); -1 = candidates ahead (pairs j > i)
 *   "union_chunk"    union_snap pass: candidates per work item (default 512; 64..8192)
 *   "union_seed"     union_snap pass (behind): a seed pass first unites every core point
 *                    with its nearest core neighbour behind it, scanning up to this many
 *                    steps of 32 positions (default 8; -1 = no seed pass)
 *   "union_phased"   union_snap pass: 1 = one launch per chunk index (chunk k of every block);
 *                    default off
 *   "union_stats"    1 = count the union_snap pass's union-path pairs; read back with
 *                    snn_get_option("last_union_path" / "last_union_hits" / "last_union_links")
 *   "dbscan_block"   DBSCAN queries per block (default 256; 32..256, multiple of 32)
 *   "simt_filter"    low-d fp32 expanded-form pre-filter: default on for radius queries and
 *                    off for DBSCAN; 1 = on everywhere, -1 = off everywhere
 *   "lowd_tc", "lowd_tc_tiles", "lowd_tc_group"   low-d tcgen05 path (default off)
 *   "tc", "tc_min_d", "tc_tiles", "tc_f16", "tc_group", "tc_diag", "tc_gram_min_d",
 *   "tc_warp_arrive"  (tc_diag 1..4 = diagnostics, results NOT valid: 1 no epilogue work,
 *                    2 no MMA, 3 no MMA and no hit path, 4 no hit path)
 *                    tensor-core path selection and tiling (tests / sweeps)
 * "force_generic" is read by snn_build (it fixes the sorted copy's layout).
 * Returns SNN_ERR_INVALID_ARGUMENT for an unknown key or bad value. */
snn_status snn_set_option(const char *key, int64_t value);
/* The calling thread's current value of an option (same keys as snn_set_option). */
snn_status snn_get_option(const char *key, int64_t *value);

#ifdef __cplusplus
}
#endif
#endif /* SNN_H */
