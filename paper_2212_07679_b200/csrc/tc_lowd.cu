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
// epilogue only tests the sign of the accumulator: a 3-way max tree over 32 columns and
// one compare, with the rare candidate lanes emitting (query, index) pairs.  The pair
// list is then decided exactly by the oracle's fp64 sequence (tcl_recheck) -- the filter
// only has to be conservative, which the margin guarantees (derivation in api.cu and
// DESIGN.md; the FFMA direct-form kernel stays the fallback whenever the scaled terms do
// not fit FP16).
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
constexpr int STAGE_CAP = 8;
constexpr unsigned long long CLAIM = 256;
constexpr int EPI = 512;
constexpr int COLS = TN / (EPI / 128);
constexpr int THREADS = 64 + EPI;

template <int KC> constexpr int row_bytes() { return KC * 2; }
template <int KC> constexpr int smem_bytes() {
    return 1024 + LSTAGES * TN * row_bytes<KC>() + 2 * TM * row_bytes<KC>() + EPI * STAGE_CAP * 4 + 512;
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
    // carve: B ring | A slots [2] | staged hits | barriers | tmem ptr
    const uint32_t a_base = base + LSTAGES * B_BYTES;
    int32_t *s_hits = reinterpret_cast<int32_t *>(gbase + LSTAGES * B_BYTES + 2 * A_BYTES);
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + LSTAGES * B_BYTES + 2 * A_BYTES + EPI * STAGE_CAP * 4);
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
        const int et = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int slice = et >> 7;
        const int row = quarter * 32 + lane;
        int32_t *my_hits = s_hits + et * STAGE_CAP;
        uint32_t acc = 0, aphase = 0;
        unsigned long long wcur = 0, wend = 0;
        for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
            int64_t b, c0, c1;
            tcl_locate(a, item, b, c0, c1);
            if (c1 <= c0) continue;
            const int64_t sp = b * TM + row;
            const bool active = sp < a.m;
            for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                mbar_wait_u32(smem_u32(&tfull[acc]), aphase);
                tc_fence_after();
                int nh = 0;
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * TN + slice * COLS;
#pragma unroll 1
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
                    if (mx >= 0.f && active) {
                        uint32_t mask = 0;
#pragma unroll
                        for (int c = 0; c < 32; ++c) mask |= (v[c] >= 0.f ? 1u : 0u) << c;
                        const int64_t jb = t0 + slice * COLS + ch * 32;
                        while (mask) {
                            const int c = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const int64_t jj = jb + c;
                            if (jj >= c1) break;
                            if (nh < STAGE_CAP) {
                                my_hits[nh++] = (int32_t)jj;
                            } else {
                                const unsigned long long k = atomicAdd(a.pair_count, 1ull);
                                if (k < (unsigned long long)a.pair_cap) {
                                    a.pair_q[k] = (int32_t)sp;
                                    a.pair_j[k] = (int32_t)jj;
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&tempty[acc]));
                if (__any_sync(0xffffffffu, nh > 0)) {
                    int incl = nh;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int total = __shfl_sync(0xffffffffu, incl, 31);
                    if (wcur + (unsigned long long)total > wend) {
                        for (unsigned long long k = wcur + lane; k < wend; k += 32)
                            if (k < (unsigned long long)a.pair_cap) a.pair_q[k] = -1;
                        const unsigned long long want = total > CLAIM ? (unsigned long long)total : CLAIM;
                        unsigned long long wb = 0;
                        if (lane == 0) wb = atomicAdd(a.pair_count, want);
                        wcur = __shfl_sync(0xffffffffu, wb, 0);
                        wend = wcur + want;
                    }
                    const unsigned long long my0 = wcur + (unsigned long long)(incl - nh);
                    for (int h = 0; h < nh; ++h) {
                        const unsigned long long k = my0 + h;
                        if (k < (unsigned long long)a.pair_cap) {
                            a.pair_q[k] = (int32_t)sp;
                            a.pair_j[k] = my_hits[h];
                        }
                    }
                    wcur += (unsigned long long)total;
                }
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
        for (unsigned long long k = wcur + lane; k < wend; k += 32)
            if (k < (unsigned long long)a.pair_cap) a.pair_q[k] = -1;
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

// exact recheck (oracle sequence, eq:ip1 in fp64) of pairs on the AoSoA4 copies
template <int D>
__global__ void __launch_bounds__(256) tcl_recheck(const float *__restrict__ Xs, const float *__restrict__ Qs,
                                                   const int32_t *__restrict__ pq, const int32_t *__restrict__ pj,
                                                   int64_t npairs, double R2, uint32_t *flag, float *dist) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t q = pq[k];
        if (q < 0) { flag[k] = 0; dist[k] = 0.f; continue; }
        const int32_t j = pj[k];
        double s = 0.0;
#pragma unroll
        for (int kk = 0; kk < D; ++kk) {
            const double t = __dsub_rn((double)Xs[(j >> 2) * 4 * D + 4 * kk + (j & 3)],
                                       (double)Qs[(q >> 2) * 4 * D + 4 * kk + (q & 3)]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        flag[k] = s <= R2;
        dist[k] = (float)sqrt(s);
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
int64_t tcl_claim_slack() { return (int64_t)(EPI / 32) * (int64_t)CLAIM; }

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

void launch_tcl_recheck(const float *Xs, const float *Qs, int d, const int32_t *pq, const int32_t *pj, int64_t np,
                        double R2, uint32_t *flag, float *dist, cudaStream_t s) {
    if (np == 0) return;
    const int g = gridn(np);
#define CASE(D) case D: SNN_LAUNCH(tcl_recheck<D>, g, 256, 0, s, Xs, Qs, pq, pj, np, R2, flag, dist); break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

}  // namespace snn
