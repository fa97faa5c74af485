// csr.cu -- K11 for the pair-list paths: candidate pairs that passed the exact recheck
// -> CSR rows ("retrieve all data points" within R; rows in original query order,
// entries in ascending sorted-index position, i.e. key order; ids via pi, Alg. 1 l.6).
//
//   count   : hits per original query row (atomics), largest row
//   scan    : offsets (int64, m + 1)
//   scatter : each hit to offsets[q] + atomic cursor -> (position << 32 | fp32 dist bits)
//   sort    : every row sorted by sorted-index position (unique within a row, so the result
//             is deterministic): warp rank sort in registers (<= 32), bitonic in shared memory
//             (<= 512), one CTA per row in shared memory (<= 16384); the caller falls
//             back to the global radix path beyond that.
#include <stdint.h>

#include "common.cuh"
#include "csr.h"

namespace snn {
namespace {

constexpr int WCAP = 512;         // entries per warp-sorted row
constexpr int BCAP = 16384;       // entries per CTA-sorted row

__global__ void pairs_row_count_kernel(const uint32_t *flag, const int32_t *pq, const int32_t *qperm, int64_t P,
                                       int32_t *row_count) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x)
        if (flag[k]) atomicAdd(&row_count[qperm[pq[k]]], 1);
}

__global__ void row_max_kernel(const int32_t *row_count, int64_t m, int32_t *maxrow) {
    int32_t mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, row_count[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(maxrow, mx);
}

__global__ void pairs_scatter_kernel(const uint32_t *flag, const int32_t *pq, const int32_t *pj, const float *dist,
                                     const int32_t *qperm, int64_t P, const int64_t *offsets, int32_t *cursor,
                                     uint64_t *tmp) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[k]) continue;
        const int32_t q = qperm[pq[k]];
        const int64_t pos = offsets[q] + atomicAdd(&cursor[q], 1);
        SNN_DASSERT(pos < offsets[q + 1]);
        tmp[pos] = ((uint64_t)(uint32_t)pj[k] << 32) | (uint64_t)__float_as_uint(dist[k]);
    }
}

__device__ __forceinline__ void emit(uint64_t v, const int32_t *perm, int32_t *out_idx, float *out_dist, int64_t pos) {
    out_idx[pos] = perm[(uint32_t)(v >> 32)];
    out_dist[pos] = __uint_as_float((uint32_t)v);
}

// Bitonic stages j = jtop .. 1 of merge size k on a 64-element segment held in registers
// (a = element base + lane, b = element base + 32 + lane): no shared memory, no barrier.
__device__ __forceinline__ void seg_stages(uint64_t &a, uint64_t &b, int base, int k, int jtop, int lane) {
    for (int j = jtop; j > 0; j >>= 1) {
        if (j == 32) {
            const bool up = ((base + lane) & k) == 0;
            if ((a > b) == up) { const uint64_t t = a; a = b; b = t; }
        } else {
            const uint64_t pa = __shfl_xor_sync(0xffffffffu, a, j), pb = __shfl_xor_sync(0xffffffffu, b, j);
            const bool lower = (lane & j) == 0;
            const bool upa = ((base + lane) & k) == 0, upb = ((base + 32 + lane) & k) == 0;
            a = (lower == upa) ? (a < pa ? a : pa) : (a < pa ? pa : a);
            b = (lower == upb) ? (b < pb ? b : pb) : (b < pb ? pb : b);
        }
    }
}

// one warp per row (rows with <= WCAP entries)
__global__ void __launch_bounds__(256) rows_sort_warp_kernel(const int64_t *offsets, int64_t m, const uint64_t *tmp,
                                                             const int32_t *perm, int32_t *out_idx, float *out_dist) {
    __shared__ uint64_t sbuf[8][WCAP];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint64_t *buf = sbuf[w];
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < m;
         r += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t o0 = offsets[r];
        const int cnt = (int)(offsets[r + 1] - o0);
        if (cnt == 0 || cnt > WCAP) continue;
        if (cnt <= 32) {   // rank sort in registers: positions are unique within a row
            const uint64_t v = lane < cnt ? tmp[o0 + lane] : ~0ull;
            const uint32_t key = (uint32_t)(v >> 32);   // lanes >= cnt: ~0, never "<"
            int rank = 0;
            for (int j = 0; j < cnt; j += 4) {
                rank += __shfl_sync(0xffffffffu, key, j) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 1) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 2) < key;
                rank += __shfl_sync(0xffffffffu, key, j + 3) < key;
            }
            if (lane < cnt) emit(v, perm, out_idx, out_dist, o0 + rank);
            continue;
        }
        if (cnt <= 64) {   // two entries per lane
            const uint64_t v0 = tmp[o0 + lane];
            const uint64_t v1 = lane + 32 < cnt ? tmp[o0 + lane + 32] : ~0ull;
            const uint32_t k0 = (uint32_t)(v0 >> 32), k1 = (uint32_t)(v1 >> 32);
            int r0 = 0, r1 = 0;
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const uint32_t kj = __shfl_sync(0xffffffffu, k0, j);
                r0 += kj < k0;
                r1 += kj < k1;
            }
            for (int j = 0; j < cnt - 32; j += 2) {
                const uint32_t kj = __shfl_sync(0xffffffffu, k1, j);
                const uint32_t kk = __shfl_sync(0xffffffffu, k1, j + 1);
                r0 += (kj < k0) + (kk < k0);
                r1 += (kj < k1) + (kk < k1);
            }
            emit(v0, perm, out_idx, out_dist, o0 + r0);
            if (lane + 32 < cnt) emit(v1, perm, out_idx, out_dist, o0 + r1);
            continue;
        }
        int S = 64;
        while (S < cnt) S <<= 1;
        for (int i = lane; i < S; i += 32) buf[i] = i < cnt ? tmp[o0 + i] : ~0ull;
        __syncwarp();
        for (int k = 2; k <= S; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < S / 2; t += 32) {   // one compare-exchange pair per thread
                    const int i = 2 * t - (t & (j - 1)), p = i + j;
                    const uint64_t a = buf[i], b = buf[p];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { buf[i] = b; buf[p] = a; }
                }
                __syncwarp();
            }
        }
        for (int i = lane; i < cnt; i += 32) emit(buf[i], perm, out_idx, out_dist, o0 + i);
        __syncwarp();
    }
}

// one CTA per row with WCAP < entries <= BCAP (dynamic shared memory, S x 8 bytes)
__global__ void __launch_bounds__(1024) rows_sort_block_kernel(const int64_t *offsets, int64_t m, const uint64_t *tmp,
                                                               const int32_t *perm, int32_t *out_idx, float *out_dist) {
    extern __shared__ uint64_t bbuf[];
    __shared__ int64_t s_rows[1024];
    __shared__ int s_nrows;
    // this CTA's rows are blockIdx.x + k * gridDim.x; find the long ones 1024 at a time (one
    // parallel round of offset loads instead of one dependent round trip per row)
    for (int64_t k0 = 0; blockIdx.x + k0 * gridDim.x < m; k0 += blockDim.x) {
        if (threadIdx.x == 0) s_nrows = 0;
        __syncthreads();
        const int64_t rr = blockIdx.x + (k0 + threadIdx.x) * gridDim.x;
        if (rr < m) {
            const int64_t c = offsets[rr + 1] - offsets[rr];
            if (c > WCAP && c <= BCAP) s_rows[atomicAdd(&s_nrows, 1)] = rr;
        }
        __syncthreads();
        const int nr = s_nrows;
    for (int t = 0; t < nr; ++t) {
        const int64_t r = s_rows[t];
        const int64_t o0 = offsets[r];
        const int cnt = (int)(offsets[r + 1] - o0);
        int S = 1024;
        while (S < cnt) S <<= 1;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        // merges up to 64 elements: each warp sorts its 64-element segments in registers
        for (int sg = wid; sg < S / 64; sg += nw) {
            const int base = sg * 64;
            uint64_t a = base + lane < cnt ? tmp[o0 + base + lane] : ~0ull;
            uint64_t b = base + 32 + lane < cnt ? tmp[o0 + base + 32 + lane] : ~0ull;
            for (int k = 2; k <= 64; k <<= 1) seg_stages(a, b, base, k, k >> 1, lane);
            bbuf[base + lane] = a;
            bbuf[base + 32 + lane] = b;
        }
        __syncthreads();
        for (int k = 128; k <= S; k <<= 1) {
            for (int j = k >> 1; j >= 64; j >>= 1) {   // cross-segment stages in shared memory
                for (int pt = threadIdx.x; pt < S / 2; pt += blockDim.x) {   // one compare-exchange pair per thread
                    const int i = 2 * pt - (pt & (j - 1)), p = i + j;
                    const uint64_t x = bbuf[i], y = bbuf[p];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) { bbuf[i] = y; bbuf[p] = x; }
                }
                __syncthreads();
            }
            for (int sg = wid; sg < S / 64; sg += nw) {   // stages j <= 32 in registers
                const int base = sg * 64;
                uint64_t a = bbuf[base + lane], b = bbuf[base + 32 + lane];
                seg_stages(a, b, base, k, 32, lane);
                bbuf[base + lane] = a;
                bbuf[base + 32 + lane] = b;
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) emit(bbuf[i], perm, out_idx, out_dist, o0 + i);
        __syncthreads();
    }
    }
}

int grid_n(int64_t n, int per = 256) {
    int64_t g = ceil_div(n, per);
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

int csr_row_sort_cap() { return BCAP; }

void launch_pairs_row_count(const uint32_t *flag, const int32_t *pq, const int32_t *qperm, int64_t P, int64_t m,
                            int32_t *row_count, int32_t *maxrow, cudaStream_t s) {
    if (P > 0) SNN_LAUNCH(pairs_row_count_kernel, grid_n(P), 256, 0, s, flag, pq, qperm, P, row_count);
    if (m > 0) SNN_LAUNCH(row_max_kernel, grid_n(m), 256, 0, s, row_count, m, maxrow);
}

void launch_pairs_to_rows(const uint32_t *flag, const int32_t *pq, const int32_t *pj, const float *dist,
                          const int32_t *qperm, int64_t P, int64_t m, const int64_t *offsets, int32_t *cursor,
                          uint64_t *tmp, const int32_t *perm, int32_t max_row, int32_t *out_idx, float *out_dist,
                          cudaStream_t s) {
    if (P > 0) SNN_LAUNCH(pairs_scatter_kernel, grid_n(P), 256, 0, s, flag, pq, pj, dist, qperm, P, offsets, cursor, tmp);
    if (m == 0 || max_row == 0) return;
    SNN_LAUNCH(rows_sort_warp_kernel, grid_n(m * 32), 256, 0, s, offsets, m, tmp, perm, out_idx, out_dist);
    if (max_row > WCAP) {
        int S = 1024;
        while (S < max_row && S < BCAP) S <<= 1;
        const size_t smem = (size_t)S * 8;
        cudaFuncSetAttribute(rows_sort_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        SNN_LAUNCH(rows_sort_block_kernel, 148 * 2, 1024, smem, s, offsets, m, tmp, perm, out_idx, out_dist);
    }
}

}  // namespace snn
