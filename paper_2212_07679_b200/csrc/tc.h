// tc.h -- tensor-core (tcgen05, kind::tf32) windowed candidate filter, d >= 32.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {

struct TcArgs {
    const float *xbar;      // index half norms of the TF32-path centred rows (sorted, n_pad)
    const float *qbar;      // query half norms (sorted, m)
    int64_t n, m;
    int kpad, kblocks;      // K padded to 32; kpad / 32
    const int64_t *blk_lo, *blk_hi;
    const int64_t *grp_lo, *grp_start;   // grouped raster: union lo / first item per group
    int64_t nblocks, ngroups, total_items;
    int group;              // query blocks per raster group
    int chunk;              // candidates per work item (multiple of 256)
    float c1h;              // 1 - c1/2   (separable margin, reading C20)
    float sc;               // operand scale product 2^(a+b) (FP16 operands), 1 for TF32
    float r2h;              // (R^2 (1 + 1e-12) + c0) / 2
    int32_t *pair_q, *pair_j;            // candidate pairs (sorted query pos, sorted index pos)
    unsigned long long *pair_count;
    int64_t pair_cap;
    int diag;               // 0; diagnostics: 1 = skip epilogue work, 2 = skip MMAs
    int ares;               // resident query tile per work item when K fits one block
    uint32_t wait_hint;     // mbarrier try_wait suspend-time hint in ns (0: plain probe loop)
    int warp_arrive = 1;    // epilogue releases TMEM / x-bar slots with one arrive per warp (else per thread)
};

int tc_tile_rows();   // queries per tile (128)
int tc_tile_cols();   // candidates per tile (256)
int tc_kpad(int d, bool f16);   // d rounded up to 64 (FP16) or 32 (TF32)
int64_t tc_claim_slack();   // pair-list slots a CTA may leave unused (claimed blocks)

// TF32 centred copy (row-major, kpad columns) + half norms of the centred rows.
void launch_gather_tf32(const void *X, bool f64, int64_t rows, int d, const uint32_t *perm, const float *mu_f,
                        float *out, float *half_norm, cudaStream_t s);
// FP16 centred copy scaled by `scale` (a power of two), zero padded to kpad = tc_kpad(d, true).
// Fused sorted copy + FP16 operand copy + half norms (one read of X; FP16 indexes).
void launch_gather_xs_f16(const void *X, bool f64, int64_t n, int64_t n_pad, int d, int ld, const uint32_t *perm,
                          const float *mu_f, float scale, void *Xs, void *out, float *half_norm, cudaStream_t s);
void launch_gather_f16(const void *X, bool f64, int64_t rows, int d, const uint32_t *perm, const float *mu_f,
                       float scale, void *out, float *half_norm, cudaStream_t s);
// grp_lo / grp_items for ceil(nblocks / group) raster groups
void launch_tc_group_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                           int64_t *grp_lo, int64_t *grp_items, cudaStream_t s);
// false if the TMA tensor maps could not be created.
bool launch_tc_window(const void *Qt, const void *Xt, bool f16, const TcArgs &a, int sm_count, cudaStream_t s);
// K10: exact fp64 recheck of pairs on the original (row-major) coordinates.
void launch_recheck(const void *Xs, const void *Qs, bool f64, int ld, int d, const int32_t *pq, const int32_t *pj,
                    int64_t npairs, double R2, uint32_t *flag, float *dist, cudaStream_t s);

}  // namespace snn

namespace snn {
// CSR assembly for the tensor-core path (hits -> rows in original query order, within a
// row ascending sorted-index position).
void launch_tc_scatter(const uint32_t *flag, const int64_t *pos, const int32_t *pq, const int32_t *pj,
                       const float *dist, const int32_t *qperm, int64_t P, uint32_t *hq, uint32_t *hj, float *hd,
                       int32_t *row_count, cudaStream_t s);
void launch_gather_u32(const uint32_t *src, const uint32_t *idx, int64_t H, uint32_t *dst, cudaStream_t s);
void launch_tc_write(const uint32_t *order, const uint32_t *hj, const float *hd, const int32_t *perm, int64_t H,
                     int32_t *out_idx, float *out_dist, cudaStream_t s);
}  // namespace snn

namespace snn {
// Low-d tensor-core path (tc_lowd.cu): folded split-FP16 filter (K = 3d + 4 in 16 / 32
// columns) fused with the exact decision; per-(item, query) hit records -> CSR.
struct TclArgs {
    int64_t n, m;
    int64_t n_pad, m_pad;               // rows of the AoSoA4 fp32 copies (multiples of 4)
    const int4 *desc;                   // items {block, c0, c1, chunk index in block}
    int64_t total_items;
    const float *Xs, *Qs;               // AoSoA4 fp32 sorted copies (index / queries)
    float T_in, T_out;                  // fp32 sure-in / sure-out thresholds (FFMA path's)
    double R2;
    uint32_t *ecnt;                     // per (item, row): hits (written once)
    unsigned long long *eoff;           // per (item, row): first position in pool, ~0 = not stored
    uint16_t *pool;                     // hit positions within the item, ascending per entry
    unsigned long long *pool_count;     // zeroed
    int64_t pool_cap;
};
struct TclPost {
    int64_t n, m;
    const float *Xs, *Qs;
    const int32_t *perm, *qperm;
    float T_in, T_out;
    double R2;
};
int tcl_kc(int d);              // 16 (d <= 4) or 32 (d <= 8)
bool tcl_supported(int d);
// operand rows from an AoSoA4 fp32 sorted copy; cand: rows_pad x kc, qry: rows x kc (nullable)
void launch_tcl_operands(const float *Xs, int d, int64_t rows, int64_t rows_pad, const float *mu_f, int e, double c1h,
                         double r2h, void *cand, void *qry, cudaStream_t s);
// work list: bcount[b] items of block b; after an exclusive scan (bstart) the descriptors
void launch_tcl_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                      int64_t *bcount, cudaStream_t s);
void launch_tcl_fill_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                           const int64_t *bstart, int4 *desc, int32_t *bitems, cudaStream_t s);
bool launch_tcl_window(const void *qry, const void *cand, int d, int64_t cand_rows, const TclArgs &a, int sm_count,
                       cudaStream_t s);
void launch_tcl_row_totals(const TclPost &p, const int64_t *bstart, const int32_t *bitems, const uint32_t *ecnt,
                           int32_t *pre, int32_t *row_count, cudaStream_t s);
// CSR write; entries the pool could not hold (eoff == ~0) are listed in ovf (novf zeroed)
// and re-decided by a warp-per-entry pass
void launch_tcl_compact(const TclPost &p, int d, int64_t nent, const int4 *desc, const uint32_t *ecnt,
                        const unsigned long long *eoff, const uint16_t *pool, const int32_t *pre,
                        const int64_t *offsets, int32_t *out_idx, float *out_dist, int64_t *ovf,
                        unsigned long long *novf, cudaStream_t s);
}  // namespace snn
