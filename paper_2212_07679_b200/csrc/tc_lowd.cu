// tc_lowd.cu -- the windowed candidate filter for LOW d (d <= 8, fp32 data) on the
// tensor cores, and the exact recheck of its pairs on the AoSoA4 sorted copy.
//
// Same test as K9 (eq:ip2, with the rigorous separable margin of
// DESIGN.md reading C20): a pair (q, x) is a CANDIDATE iff
//     x.q - xbar c1h - (qbar c1h - r2h) >= 0,        c1h = 1 - c1/2, r2h = (R^2 + c0)/2,
// with x, q the coordinates centred at mu (fp32).  For low d the whole left side is ONE
// short contraction (K = 3d + 4 <= 16 or 32, kind::f16, FP32 accumulation in TMEM):
//   candidate row  B_j = [ h(x), h(x), l(x), xbar'_h, xbar'_l, 2^15, 2^15, 0 ... ]
//   query row      A_i = [ h(q), l(q), h(q), -2^15,  -2^15,  b'_h,  b'_l, 0 ... ]
// where v = x * 2^e = h + l is split into two FP16 halves (22 significant bits; the
// dropped l.l term is ~2^-22 |x||q|), xbar' = xbar c1h 2^(2e-15) and
// b' = -(qbar c1h - r2h) 2^(2e-15), also split.  A_i . B_j = 2^(2e) * (left side), so the
// epilogue only tests the sign of the accumulator: a 3-way max tree over each run of 32
// candidates and one compare.  The result is a BITMAP with one bit per (query, aligned
// 32-candidate chunk of its window) that may hold a neighbour -- no per-element
// extraction in the epilogue, no divergence.  The flagged chunks are then decided
// exactly (tcl_exact: the FFMA kernel's fp32 direct-form classification with fp64
// fallback, i.e. bit-identical membership with the oracle), and the CSR is written in
// key order straight from the bitmap (tcl_write) -- no sort.  The filter only has to be
// conservative, which the margin guarantees (derivation in api.cu and DESIGN.md; the
// FFMA direct-form kernel stays the fallback whenever the scaled terms do not fit FP16).
// Windows are aligned to 64 candidates so every epilogue thread's two 32-candidate
// chunks of a tile share one 64-bit bitmap word (one atomic OR).
//
// The batched contraction X(J,:) [q_1 .. q_128] of PAPER.md:218-219 is one
// tcgen05.mma (M = 128 queries, N = 256 candidates, K = 16 or 32) per tile: the query
// operand of a work item stays in shared memory for all its tiles, candidate tiles
// stream through an 8-deep TMA ring (32- or 64-byte swizzled rows), accumulators are
// double-buffered in TMEM (2 x 256 columns), 16 epilogue warps drain them.
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"
#include "tc.h"
#include "tcgen05.cuh"

namespace snn {
namespace {
using namespace tc5;

constexpr int TM = 128, TN = 256, LSTAGES = 8;
constexpr int EPI = 512;
constexpr int COLS = TN / (EPI / 128);
constexpr int THREADS = 64 + EPI;

template <int KC> constexpr int row_bytes() { return KC * 2; }
template <int KC> constexpr int smem_bytes() {
    return 1024 + LSTAGES * TN * row_bytes<KC>() + 2 * TM * row_bytes<KC>() + 512;
}
// UMMA K-major descriptor for 32-byte (KC = 16) or 64-byte (KC = 32) swizzled rows:
// 8-row core groups SBO = 8 * row bytes apart; layout type 6 = SWIZZLE_32B, 4 = SWIZZLE_64B.
template <int KC>
__device__ __forceinline__ uint64_t lowd_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((8 * row_bytes<KC>()) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(KC == 16 ? 6 : 4) << 61;
    return d;
}
constexpr uint32_t TCL_IDESC = make_idesc(true, TM, TN);

__device__ __forceinline__ void tcl_locate(const TclArgs &a, int64_t item, int64_t &b, int64_t &c0, int64_t &c1) {
    int64_t lo = 0, hi = a.ngroups;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (a.grp_start[mid] <= item) lo = mid; else hi = mid;
    }
    const int64_t g0 = lo * a.group;
    const int64_t gc = min((int64_t)a.group, a.nblocks - g0);
    const int64_t r = item - a.grp_start[lo];
    const int64_t k = r / gc;
    b = g0 + (r - k * gc);
    const int64_t base = a.grp_lo[lo] + k * a.chunk;
    c0 = max(base, a.blk_lo[b]);
    c1 = min(base + a.chunk, a.blk_hi[b]);
    if (c1 < c0) c1 = c0;
}

template <int KC>
__global__ void __launch_bounds__(THREADS, 1)
tcl_window_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TclArgs a) {
    constexpr int RB = row_bytes<KC>();
    constexpr int B_BYTES = TN * RB, A_BYTES = TM * RB;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    // carve: B ring | A slots [2] | barriers | tmem ptr
    const uint32_t a_base = base + LSTAGES * B_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + LSTAGES * B_BYTES + 2 * A_BYTES);
    uint64_t *full = bars, *empty = bars + LSTAGES, *tfull = bars + 2 * LSTAGES, *tempty = bars + 2 * LSTAGES + 2;
    uint64_t *afull = bars + 2 * LSTAGES + 4, *aempty = bars + 2 * LSTAGES + 6;
    uint32_t *tmem_ptr = reinterpret_cast<uint32_t *>(bars + 2 * LSTAGES + 8);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < LSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI);
            mbar_init(&afull[s], 1); mbar_init(&aempty[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_ptr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_ptr;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            int stage = 0, as = 0;
            uint32_t phase = 0, aph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                int64_t b, c0, c1;
                tcl_locate(a, item, b, c0, c1);
                if (c1 <= c0) continue;
                mbar_wait_u32(smem_u32(&aempty[as]), aph ^ 1);
                mbar_arrive_expect_tx(&afull[as], A_BYTES);
                tma_load_2d(a_base + as * A_BYTES, &tmA, smem_u32(&afull[as]), 0, (int)(b * TM));
                if (++as == 2) { as = 0; aph ^= 1; }
                for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                    mbar_wait_u32(smem_u32(&empty[stage]), phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], B_BYTES);
                    tma_load_2d(base + stage * B_BYTES, &tmB, smem_u32(&full[stage]), 0, (int)t0);
                    if (++stage == LSTAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0, as = 0;
            uint32_t phase = 0, acc = 0, aphase = 0, aph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                int64_t b, c0, c1;
                tcl_locate(a, item, b, c0, c1);
                if (c1 <= c0) continue;
                mbar_wait_u32(smem_u32(&afull[as]), aph);
                tc_fence_after();
                const uint64_t da = lowd_desc<KC>(a_base + as * A_BYTES);
                for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                    mbar_wait_u32(smem_u32(&tempty[acc]), aphase ^ 1);
                    mbar_wait_u32(smem_u32(&full[stage]), phase);
                    tc_fence_after();
                    const uint64_t db = lowd_desc<KC>(base + stage * B_BYTES);
                    const uint32_t dcol = tmem + acc * TN;
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk)   // 16 FP16 (32 bytes) of K per MMA
                        mma_f16(dcol, da + 2 * kk, db + 2 * kk, TCL_IDESC, kk != 0);
                    mma_commit(smem_u32(&empty[stage]));
                    mma_commit(smem_u32(&tfull[acc]));
                    if (++stage == LSTAGES) { stage = 0; phase ^= 1; }
                    acc ^= 1;
                    if (acc == 0) aphase ^= 1;
                }
                mma_commit(smem_u32(&aempty[as]));   // query operand free once its MMAs retire
                if (++as == 2) { as = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (EPI threads)
        // 16 warps: warp w reads TMEM lane quarter (w % 4); the four warps of a quarter
        // take 64-column slices of the 256-column tile.  One thread = one query row.
        const int et = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int slice = et >> 7;
        const int row = quarter * 32 + lane;
        uint32_t acc = 0, aphase = 0;
        for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
            int64_t b, c0, c1;
            tcl_locate(a, item, b, c0, c1);
            if (c1 <= c0) continue;
            const int64_t sp = b * TM + row;
            const bool active = sp < a.m;
            const int64_t lo = a.blk_lo[b];
            const int64_t wpr = ceil_div(a.blk_hi[b] - lo, 64 * 32);   // bitmap words per row
            unsigned long long *bm = a.bitmap + a.bm_off[b] + (int64_t)row * wpr;
            for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                mbar_wait_u32(smem_u32(&tfull[acc]), aphase);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * TN + slice * COLS;
                uint32_t flags = 0;
#pragma unroll
                for (int ch = 0; ch < COLS / 32; ++ch) {
                    float v[32];
                    tmem_ld32(taddr + ch * 32, v);
                    float m[11];
#pragma unroll
                    for (int c = 0; c < 10; ++c) m[c] = fmaxf(fmaxf(v[3 * c], v[3 * c + 1]), v[3 * c + 2]);
                    m[10] = fmaxf(v[30], v[31]);
                    const float m0 = fmaxf(fmaxf(m[0], m[1]), m[2]), m1 = fmaxf(fmaxf(m[3], m[4]), m[5]);
                    const float m2 = fmaxf(fmaxf(m[6], m[7]), m[8]), m3 = fmaxf(m[9], m[10]);
                    const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
                    flags |= (mx >= 0.f ? 1u : 0u) << ch;
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&tempty[acc]));
                const int64_t jb = t0 + slice * COLS;
                if (flags && active && jb < c1) {
                    if (jb + 32 >= c1) flags &= 1u;   // second chunk beyond this item's range
                    const int64_t pos = (jb - lo) >> 5;             // even: windows are 64-aligned
                    atomicOr(bm + (pos >> 6), (unsigned long long)flags << (pos & 63));
                }
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__device__ __forceinline__ void split16(double v, __half &h, __half &l) {
    h = __double2half(v);
    l = __double2half(v - (double)__half2float(h));
}

// Operand rows from the AoSoA4 sorted copy (original coordinates):
//   cand (nullable): n_pad rows, rows >= n get xbar' = 65504 (never candidates)
//   qry  (nullable): rows < m
template <int D, int KC>
__global__ void __launch_bounds__(256) tcl_operands(const float *__restrict__ Xs, int64_t rows, int64_t rows_pad,
                                                    const float *__restrict__ mu_f, float sc, double c1h, double r2h,
                                                    double s2, __half *cand, __half *qry) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows_pad; i += (int64_t)gridDim.x * blockDim.x) {
        __half hv[D], lv[D];
        double hb = 0.0;
        const bool valid = i < rows;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            float v = 0.f;
            if (valid) {
                const float c = (float)((double)Xs[(i >> 2) * 4 * D + 4 * k + (i & 3)] - (double)mu_f[k]);
                hb += (double)c * (double)c;
                v = c * sc;
            }
            hv[k] = __float2half_rn(v);
            lv[k] = __float2half_rn(v - __half2float(hv[k]));
        }
        hb *= 0.5;
        const __half p15 = __float2half_rn(32768.f), n15 = __float2half_rn(-32768.f), z = __float2half_rn(0.f);
        if (cand) {
            __half r[KC];
#pragma unroll
            for (int k = 0; k < KC; ++k) r[k] = z;
#pragma unroll
            for (int k = 0; k < D; ++k) { r[k] = hv[k]; r[D + k] = hv[k]; r[2 * D + k] = lv[k]; }
            if (valid) {
                split16(hb * c1h * s2, r[3 * D], r[3 * D + 1]);
                r[3 * D + 2] = p15;
                r[3 * D + 3] = p15;
            } else {
                r[3 * D] = __float2half_rn(65504.f);
                r[3 * D + 1] = __float2half_rn(65504.f);
            }
            uint4 *dst = reinterpret_cast<uint4 *>(cand + i * KC);
#pragma unroll
            for (int k = 0; k < KC / 8; ++k) dst[k] = *reinterpret_cast<const uint4 *>(&r[8 * k]);
        }
        if (qry && valid) {
            __half r[KC];
#pragma unroll
            for (int k = 0; k < KC; ++k) r[k] = z;
#pragma unroll
            for (int k = 0; k < D; ++k) { r[k] = hv[k]; r[D + k] = lv[k]; r[2 * D + k] = hv[k]; }
            r[3 * D] = n15;
            r[3 * D + 1] = n15;
            split16(-(hb * c1h - r2h) * s2, r[3 * D + 2], r[3 * D + 3]);
            uint4 *dst = reinterpret_cast<uint4 *>(qry + i * KC);
#pragma unroll
            for (int k = 0; k < KC / 8; ++k) dst[k] = *reinterpret_cast<const uint4 *>(&r[8 * k]);
        }
    }
}

// bitmap words per block (128 rows x ceil(chunks / 64))
__global__ void tcl_bm_sizes_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int64_t *words) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nblocks) words[b] = TM * ceil_div(max((int64_t)0, blk_hi[b] - blk_lo[b]), 64 * 32);
}

// flagged chunks per query (sorted position): popcount of its bitmap row
__global__ void tcl_flag_count_kernel(const TclPost p, int64_t *fcnt) {
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sp < p.m;
         sp += (int64_t)gridDim.x * blockDim.x / 32) {
        const int lane = threadIdx.x % 32;
        const int64_t b = sp / TM, row = sp % TM;
        const int64_t wpr = ceil_div(max((int64_t)0, p.blk_hi[b] - p.blk_lo[b]), 64 * 32);
        const unsigned long long *bm = p.bitmap + p.bm_off[b] + row * wpr;
        int64_t c = 0;
        for (int64_t w = lane; w < wpr; w += 32) c += __popcll(bm[w]);
        c = warp_sum(c);
        if (lane == 0) fcnt[sp] = c;
    }
}

// Exact decision of every flagged chunk (one warp per query, lane = candidate): the FFMA
// kernel's classification -- fp32 direct form (eq:ip1) on the original coordinates against
// the rigorous T_in / T_out, oracle-order fp64 sequence in between -- so membership is
// bit-identical to the oracle.  masks[foff[sp] + k] = hit mask of the k-th flagged chunk;
// row_count[qperm[sp]] = hits.
template <int D>
__global__ void __launch_bounds__(256) tcl_exact_kernel(const TclPost p, const int64_t *foff, uint32_t *masks,
                                                        int32_t *row_count) {
    const int lane = threadIdx.x % 32;
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sp < p.m;
         sp += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t b = sp / TM, row = sp % TM;
        const int64_t lo = p.blk_lo[b];
        const int64_t wpr = ceil_div(max((int64_t)0, p.blk_hi[b] - lo), 64 * 32);
        const unsigned long long *bm = p.bitmap + p.bm_off[b] + row * wpr;
        float q[D];
        double qd[D];
#pragma unroll
        for (int k = 0; k < D; ++k) { q[k] = p.Qs[(sp >> 2) * 4 * D + 4 * k + (sp & 3)]; qd[k] = q[k]; }
        int64_t out = foff[sp];
        int32_t hits = 0;
        for (int64_t w = 0; w < wpr; ++w) {
            unsigned long long bits = bm[w];
            while (bits) {
                const int c = __ffsll(bits) - 1;
                bits &= bits - 1;
                const int64_t j = lo + ((w * 64 + c) << 5) + lane;
                bool hit = false;
                if (j < p.n) {
                    float x[D];
                    float d2 = 0.f;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        x[k] = p.Xs[(j >> 2) * 4 * D + 4 * k + (j & 3)];
                        const float t = x[k] - q[k];
                        d2 = fmaf(t, t, d2);
                    }
                    if (d2 <= p.T_out) {
                        hit = d2 <= p.T_in;
                        if (!hit) {
                            double s = 0.0;
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                const double t = __dsub_rn((double)x[k], qd[k]);
                                s = __dadd_rn(s, __dmul_rn(t, t));
                            }
                            hit = s <= p.R2;
                        }
                    }
                }
                const uint32_t msk = __ballot_sync(0xffffffffu, hit);
                if (lane == 0) masks[out] = msk;
                ++out;
                hits += __popc(msk);
            }
        }
        if (lane == 0) row_count[p.qperm[sp]] = hits;
    }
}

// CSR write in key order: for each flagged chunk (bitmap order = ascending candidate
// position) its hits, ids via pi, distance = (float)sqrt of the oracle-order fp64 sum.
template <int D>
__global__ void __launch_bounds__(256) tcl_write_kernel(const TclPost p, const int64_t *foff, const uint32_t *masks,
                                                        const int64_t *offsets, int32_t *out_idx, float *out_dist) {
    const int lane = threadIdx.x % 32;
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sp < p.m;
         sp += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t b = sp / TM, row = sp % TM;
        const int64_t lo = p.blk_lo[b];
        const int64_t wpr = ceil_div(max((int64_t)0, p.blk_hi[b] - lo), 64 * 32);
        const unsigned long long *bm = p.bitmap + p.bm_off[b] + row * wpr;
        double qd[D];
#pragma unroll
        for (int k = 0; k < D; ++k) qd[k] = p.Qs[(sp >> 2) * 4 * D + 4 * k + (sp & 3)];
        int64_t k = foff[sp];
        int64_t pos = offsets[p.qperm[sp]];
        for (int64_t w = 0; w < wpr; ++w) {
            unsigned long long bits = bm[w];
            while (bits) {
                const int c = __ffsll(bits) - 1;
                bits &= bits - 1;
                const uint32_t msk = masks[k++];
                if (!msk) continue;
                if (msk & (1u << lane)) {
                    const int64_t j = lo + ((w * 64 + c) << 5) + lane;
                    double s = 0.0;
#pragma unroll
                    for (int kk = 0; kk < D; ++kk) {
                        const double t = __dsub_rn((double)p.Xs[(j >> 2) * 4 * D + 4 * kk + (j & 3)], qd[kk]);
                        s = __dadd_rn(s, __dmul_rn(t, t));
                    }
                    const int64_t o = pos + __popc(msk & lanemask_lt());
                    out_idx[o] = p.perm[j];
                    out_dist[o] = (float)sqrt(s);
                }
                pos += __popc(msk);
            }
        }
    }
}

bool make_map_lowd(CUtensorMap *m, const void *ptr, int64_t rows, int kc, int box_rows) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kc, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kc * 2};
    cuuint32_t box[2] = {(cuuint32_t)kc, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, kc == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int gridn(int64_t n) {
    int64_t g = ceil_div(n, 256);
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

int tcl_kc(int d) { return 3 * d + 4 <= 16 ? 16 : 32; }
bool tcl_supported(int d) { return d >= 1 && 3 * d + 4 <= 32; }

void launch_tcl_operands(const float *Xs, int d, int64_t rows, int64_t rows_pad, const float *mu_f, int e, double c1h,
                         double r2h, void *cand, void *qry, cudaStream_t s) {
    const float sc = ldexpf(1.0f, e);
    const double s2 = ldexp(1.0, 2 * e - 15);
    __half *c = static_cast<__half *>(cand), *q = static_cast<__half *>(qry);
    const int g = gridn(rows_pad);
#define CASE(D)                                                                                          \
    case D:                                                                                              \
        if (tcl_kc(D) == 16) SNN_LAUNCH((tcl_operands<D, 16>), g, 256, 0, s, Xs, rows, rows_pad, mu_f, sc, c1h, r2h, s2, c, q); \
        else SNN_LAUNCH((tcl_operands<D, 32>), g, 256, 0, s, Xs, rows, rows_pad, mu_f, sc, c1h, r2h, s2, c, q); \
        break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

bool launch_tcl_window(const void *qry, const void *cand, int kc, int64_t cand_rows, const TclArgs &a, int sm_count,
                       cudaStream_t s) {
    if (a.total_items == 0) return true;
    CUtensorMap ma, mb;
    if (!make_map_lowd(&ma, qry, a.m, kc, TM) || !make_map_lowd(&mb, cand, cand_rows, kc, TN)) return false;
    const int g = (int)(a.total_items < sm_count ? a.total_items : sm_count);
    if (kc == 16) {
        cudaFuncSetAttribute(tcl_window_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<16>());
        SNN_LAUNCH(tcl_window_kernel<16>, g, THREADS, smem_bytes<16>(), s, ma, mb, a);
    } else {
        cudaFuncSetAttribute(tcl_window_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<32>());
        SNN_LAUNCH(tcl_window_kernel<32>, g, THREADS, smem_bytes<32>(), s, ma, mb, a);
    }
    return true;
}

void launch_tcl_bm_sizes(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int64_t *words,
                         cudaStream_t s) {
    if (nblocks == 0) return;
    SNN_LAUNCH(tcl_bm_sizes_kernel, (int)ceil_div(nblocks, 256), 256, 0, s, blk_lo, blk_hi, nblocks, words);
}

void launch_tcl_flag_count(const TclPost &p, int64_t *fcnt, cudaStream_t s) {
    if (p.m == 0) return;
    SNN_LAUNCH(tcl_flag_count_kernel, gridn(p.m * 32), 256, 0, s, p, fcnt);
}

void launch_tcl_exact(const TclPost &p, int d, const int64_t *foff, uint32_t *masks, int32_t *row_count,
                      cudaStream_t s) {
    if (p.m == 0) return;
    const int g = gridn(p.m * 32);
#define CASE(D) case D: SNN_LAUNCH(tcl_exact_kernel<D>, g, 256, 0, s, p, foff, masks, row_count); break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

void launch_tcl_write(const TclPost &p, int d, const int64_t *foff, const uint32_t *masks, const int64_t *offsets,
                      int32_t *out_idx, float *out_dist, cudaStream_t s) {
    if (p.m == 0) return;
    const int g = gridn(p.m * 32);
#define CASE(D) case D: SNN_LAUNCH(tcl_write_kernel<D>, g, 256, 0, s, p, foff, masks, offsets, out_idx, out_dist); break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

}  // namespace snn
