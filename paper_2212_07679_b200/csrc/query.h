// query.h -- launchers of the query-side kernels (query.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {

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
    int64_t *blk_lo, *blk_hi, *nitems;   // outputs, nblocks each
    unsigned long long *pairs;           // += sum over blocks of |window| x queries (zeroed)
};
void launch_block_windows(const WindowSpec &w, cudaStream_t s);

// K8: windowed exact radius test over the work list (count pass / write pass).
struct PassArgs {
    const void *Xs;         // n_pad x ld sorted index rows (original coordinates)
    const void *Qs;         // m x ld sorted query rows
    int ld;
    int d;
    bool f64;
    int64_t m;
    const int32_t *perm;    // sorted index position -> original id
    const int32_t *qperm;   // sorted query position -> original query id
    const int64_t *blk_lo, *blk_hi, *item_start;
    int64_t nblocks, total_items;
    int B, chunk;
    bool generic;           // generic-d FFMA tile kernel (B must be 64)
    float T_in, T_out;      // fp32 sure-in / sure-out thresholds on the fp32 d^2
    double R2;              // R*R (fp64), the oracle's threshold
    int32_t *cnt;           // total_items x B: counts (count pass) -> exclusive prefixes
    const int64_t *offsets; // m+1 CSR offsets (write pass)
    int32_t *out_idx;
    float *out_dist;
    int sm_count;
};
void launch_window_pass(bool write, const PassArgs &a, cudaStream_t s);

// K11 helper: per-row totals over a block's items; cnt -> exclusive per-item prefixes;
// row_count[qperm[sp]] = total.
void launch_row_totals(int32_t *cnt, const int64_t *item_start, int64_t m, int B,
                       const int32_t *qperm, int32_t *row_count, cudaStream_t s);

bool lowd_supported(int d);   // d handled by the register-resident low-d kernel

}  // namespace snn
