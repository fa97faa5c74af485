// query.h -- launchers of the query-side kernels (query.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {
// A hit record beyond the per-entry slot capacity (low-d scan pass).
struct OvfRec {
    int32_t e;        // entry = item * B + thread
    int32_t before;   // hits of this entry recorded before this record
    uint32_t v;       // group << 4 | 4-bit hit mask
};

// K7: per-block union window of B consecutive key-sorted queries (Alg. 2 l.4,
// PAPER.md:296; eq:lower PAPER.md:142-153; batching PAPER.md:218-219).
struct WindowSpec {
    const float *qkeys;     // m sorted query keys
    int64_t m;
    int B;                  // queries per block
    const float *keys;      // n sorted index keys
    int64_t n, n_pad;       // n_pad = round_up(n, 4): rows [n, n_pad) are NaN sentinels (never hits)
    double R;
    const double *wnorm;    // device scalar ||v1|| (as used for the keys)
    const double *ex;       // device scalar E_x (index key error bound)
    const double *eq;       // device scalar E_q (query key error bound)
    int chunk;              // candidates per work item (multiple of 4)
    int align = 4;          // window bounds rounded out to multiples of this (>= 4)
    int all = 0;            // ablation ("brute force 2"): window = every point
    int64_t *blk_lo, *blk_hi, *nitems;   // outputs, nblocks each
    unsigned long long *pairs;           // += sum over blocks of |window| x queries (zeroed)
};
void launch_block_windows(const WindowSpec &w, cudaStream_t s);
// item_block[item] = the query block of every work item (item_start: exclusive scan of the
// per-block item counts, nblocks + 1 entries)
void launch_item_blocks(const int64_t *item_start, int64_t nblocks, int32_t *item_block, cudaStream_t s);
// multi-GPU query sharding: keep only the query blocks of `part` (contiguous key-order
// ranges balanced by window length); other blocks get empty windows.  tmp: 2 nblocks + 1
// int64; scan_tmp: scan_temp_bytes(nblocks).
void launch_restrict_part_sym(int64_t *blk_lo, int64_t *blk_hi, int64_t *nitems, int64_t nblocks, int B, int64_t m,
                              int part, int nparts, int64_t *tmp, void *scan_tmp, int64_t *own, cudaStream_t s);
void launch_restrict_part(int64_t *blk_lo, int64_t *blk_hi, int64_t *nitems, int64_t nblocks, int part, int nparts,
                          int64_t *tmp, void *scan_tmp, cudaStream_t s);

// K8: windowed exact radius test over the work list.
struct PassArgs {
    const void *Xs;         // sorted index rows (original coordinates); layout below
    const void *Qs;         // sorted query rows, same layout
    int ld;                 // row stride (generic path); 0 = AoSoA4 layout (low-d path)
    int d;
    bool f64;
    int64_t m;
    const int32_t *perm;    // sorted index position -> original id
    const int32_t *qperm;   // sorted query position -> original query id
    const int64_t *blk_lo, *blk_hi, *item_start;
    const int32_t *item_block = nullptr;   // work item -> query block (else binary search)
    int64_t nblocks, total_items;
    int B, chunk;
    float T_in, T_out;      // fp32 sure-in / sure-out thresholds on the fp32 d^2
    double R2;              // R*R (fp64), the oracle's threshold
    int32_t *cnt;           // total_items x B hit counts (count / scan pass)
    int32_t *pre;           // total_items x B exclusive per-row prefixes (after row totals)
    uint16_t *slots;        // low-d scan pass: total_items x B x cap chunk-local hit indices
    uint16_t *nrec = nullptr;   // records in the slots per (item, query) entry (balanced compaction)
    int cap;
    OvfRec *ovf_rec;        // low-d: records beyond `cap` (global overflow list)
    int32_t *ovf_rec_count; // device counter for ovf_rec
    int32_t ovf_rec_cap;    // capacity of ovf_rec
    int64_t n_ovf_rec;      // host copy
    int32_t *ovf_items;     // low-d: ids of items with a lost entry (ovf_rec full)
    int32_t *ovf_count;     // device counter for ovf_items
    int64_t n_ovf;          // host copy (fix pass)
    const int64_t *offsets; // m+1 CSR offsets (write / compaction / fix)
    int32_t *out_idx;
    float *out_dist;
    int sm_count;
    int variant;            // low-d inner loop: groups of 4 candidates per iteration (1 or 2)
    int scan2q = 0;         // fp32 expanded-filter scan: two queries per thread (window_lowd_2q)
    // DBSCAN modes (sorted positions)
    const uint8_t *core;    // core flags
    int32_t *parent;        // union-find parents
    int32_t *best;          // M_BORDER: smallest cluster number of a core neighbour (atomicMin)
    const int32_t *blab = nullptr;   // M_BORDER: cluster number of each sorted position (core points)
    int32_t min_pts;        // M_COUNT: counts are only needed up to min_pts (early exit)
    int64_t n_index = 0;    // M_UNION: number of index points (parent array length)
    int uload = 1;          // M_UNION pre-check load of parent[j]: 0 volatile, 1 ld.relaxed.gpu, 2 ld.cg
    int count_warp = 0;     // DBSCAN core counts: one warp per point scanning outward (core_count_warp_kernel)
    // symmetric self-query (each unordered pair evaluated once): the scan keeps only
    // candidates j > i (U rows) and counts the mirrored hits per candidate; the mirrored
    // entries (L rows) are scattered during compaction and sorted per row afterwards
    int sym = 0;
    int32_t *lcnt = nullptr;             // per sorted position: |{j < i : i in U(j)}|
    unsigned long long *lpos = nullptr;  // per sorted position: next L slot (starts at the row start)
    unsigned long long *tmpL = nullptr;  // nnz: (position << 32 | fp32 distance bits) at row start
    // staged rows (low-d path): the compaction writes every row at its key-order start
    // soff[sp] (so concurrent CTAs write neighbouring memory), rows_finalize then moves
    // each row whole to its original-id position offsets[qperm[sp]]
    const int64_t *soff = nullptr;
    unsigned long long *stage = nullptr;   // staged entries: (fp32 distance bits << 32 | id)
    const int32_t *qinv = nullptr;         // inverse of qperm (original id -> key position): rows_finalize order
    // direct rows: the mirrored entries of row sp are collected at loff[sp] (exclusive scan of
    // lcnt in KEY order, nullptr: at the row's CSR start), so the compaction's scattered 8-byte
    // stores land in a window of the buffer that follows its sweep through the blocks
    const int64_t *loff = nullptr;
    int fpipe = 1;                         // symmetric direct rows: rows_finalize_pipe (0: rows_finalize_warp)
    // partitioned symmetric self-query: the rows this part owns (key positions); queries
    // before own_lo are ghost queries (mirrored entries only), mirrors into rows >= own_hi
    // are left to their owning part
    int64_t own_lo = 0, own_hi = INT64_MAX;
    // expanded-form SIMT filter (scan variant 3; nullptr = off): AoSoA4 rows with D+1
    // floats (centred coordinates, xbar c1h), the margin constants and mu_f
    const float *Xf = nullptr;
    double c1h = 1.0, r2h = 0.0;
    const float *mu_f = nullptr;
};
// DBSCAN core counts with early exit: count[sp] = |N_eps| if < min_pts, else some value
// >= min_pts (one CTA per query block, chunks in order, stop when the block is decided)
void launch_core_counts(const PassArgs &a, int32_t *count, unsigned long long *evaluated, cudaStream_t s);
// DBSCAN union seed: every core point united with its nearest core neighbour behind it in
// key order (within its block's window and max_steps x 32 positions; a.core, a.parent,
// a.blk_lo set), before the union pass
void launch_union_seed(const PassArgs &a, int max_steps, cudaStream_t s);
// DBSCAN union pass work list: window of block b clipped to start at its first position
// (pairs, nullable, += candidate pairs of the clipped windows for m queries / n points)
void launch_truncate_windows(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B, int chunk,
                             int64_t *lo2, int64_t *nitems2, int64_t m, int64_t n, unsigned long long *pairs,
                             cudaStream_t s);
// filter rows for the expanded-form scan variant from the AoSoA4 sorted copy
void launch_filter_rows(const float *Xs, int d, int64_t n, int64_t n_pad, const float *mu_f, double c1h, float *Xf,
                        cudaStream_t s);
// margin constants of the expanded-form fp32 filter (reading C20, SIMT form)
void simt_filter_consts(int d, double R, double *c1h, double *r2h);

bool lowd_supported(int d);   // d handled by the register-resident low-d kernels

// Low-d path (AoSoA4, d <= 8): one scan pass records hits, then compaction, then a fix
// pass that recomputes only (item, query) entries whose hits overflowed `cap`.
void launch_lowd_scan(const PassArgs &a, cudaStream_t s);
void launch_lowd_compact(const PassArgs &a, cudaStream_t s);
void launch_lowd_fix(const PassArgs &a, cudaStream_t s);
// DBSCAN passes over the self-query work list: mode 2 = count, 3 = union, 4 = border.
void launch_lowd_mode(int mode, const PassArgs &a, cudaStream_t s);
// DBSCAN union pass with the staged parent-snapshot pre-check (fp32, d <= 8; false: not
// supported for these arguments; variant 2: register cap for 6 CTAs per SM).  phases > 0
// (nit = items per query block): `phases` launches, launch k processing chunk k of every
// block (chunk-major order: near pairs first), else one launch over all items.  ustats (nullable, 3 zeroed counters): pairs sent to
// the union path, exact hits among them, unions that linked two components.
bool launch_union_snap(const PassArgs &a, int variant, const int64_t *nit, int64_t phases, int behind,
                       unsigned long long *ustats, cudaStream_t s);
// DBSCAN union pass, candidates behind (pairs j < i): window of block b clipped to end
// after its last position (rounded up to 4); lo unchanged
void launch_truncate_windows_behind(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int B, int chunk,
                                    int64_t *hi2, int64_t *nitems2, int64_t m, int64_t n, unsigned long long *pairs,
                                    cudaStream_t s);
// *out = max(*out, max_i v[i]) for non-negative v (out zeroed by the caller)
void launch_max_i64(const int64_t *v, int64_t n, unsigned long long *out, cudaStream_t s);

// Generic-d path (row-major, any d): count pass + write pass (write recomputes).
void launch_generic_pass(bool write, const PassArgs &a, cudaStream_t s);

// symmetric self-query: totals = U hits + L hits + self; pre[e] starts after L + self
// srow (nullable): the same totals in key order (staged rows)
void launch_row_totals_sym(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m, int B,
                           const int32_t *qperm, const int32_t *lcnt, int32_t *row_count, int32_t *maxl,
                           int32_t *srow, int64_t own_lo, int64_t own_hi, cudaStream_t s);
// symmetric self-query: L cursors = row starts (lpos[sp] = row base of sp)
void launch_sym_lpos_init(const PassArgs &a, cudaStream_t s);
// rows -> final CSR: symmetric self-query: sort every row's L segment by position, write it
// and the self entry; staged rows: move every row to offsets[qperm[sp]]
void launch_rows_finalize(const PassArgs &a, int32_t max_l, cudaStream_t s);
void launch_invert_perm(const int32_t *perm, int64_t m, int32_t *inv, cudaStream_t s);
// K11 helper: per-row totals over a block's items; pre = exclusive per-item prefixes
// (pre may alias cnt); row_count[qperm[sp]] = total (qperm NULL: row_count[sp]).
void launch_row_totals(const int32_t *cnt, int32_t *pre, const int64_t *item_start, int64_t m,
                       int B, const int32_t *qperm, int32_t *row_count, int32_t *srow, cudaStream_t s);

}  // namespace snn
