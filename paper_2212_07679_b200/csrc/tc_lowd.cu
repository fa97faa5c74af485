// tc_lowd.cu -- radius queries for LOW d (d <= 8, fp32 data) on the tensor cores: a
// tcgen05 candidate filter fused with the exact decision, writing per-(work item, query)
// hit records that a compaction pass turns into the CSR in key order.
//
// Filter (eq:ip2, with the rigorous separable margin of DESIGN.md
// reading C20): a pair (q, x) is a CANDIDATE iff
//     x.q - xbar c1h - (qbar c1h - r2h) >= 0,        c1h = 1 - c1/2, r2h = (R^2 + c0)/2,
// with x, q the coordinates centred at mu (fp32).  For low d the whole left side is ONE
// short contraction (K = 3d + 4 <= 16 or 32, kind::f16, FP32 accumulation in TMEM):
//   candidate row  B_j = [ h(x), h(x), l(x), xbar'_h, xbar'_l, 2^15, 2^15, 0 ... ]
//   query row      A_i = [ h(q), l(q), h(q), -2^15,  -2^15,  b'_h,  b'_l, 0 ... ]
// where v = x * 2^e = h + l is split into two FP16 halves (22 significant bits; the
// dropped l.l term is ~2^-22 |x||q|), xbar' = xbar c1h 2^(2e-15) and
// b' = -(qbar c1h - r2h) 2^(2e-15), also split.  A_i . B_j = 2^(2e) * (left side), so a
// 3-way max tree over each run of 32 accumulator columns says whether a (query, 32-
// candidate chunk) may hold a neighbour.
//
// Exact decision in the epilogue: for every flagged (query, chunk) the warp turns
// around -- lane = candidate -- and applies the FFMA kernel's classification (fp32
// direct form eq:ip1 on the ORIGINAL coordinates against the rigorous T_in / T_out,
// the oracle-order fp64 sequence in between) to the 32 candidates, whose fp32 rows are
// staged in shared memory next to the MMA operands.  Membership is therefore
// bit-identical to the oracle's.  The hit mask becomes a record (chunk, mask) of the
// (item, query) entry; hit counts accumulate per entry.
//
// The batched contraction X(J,:) [q_1 .. q_128] of PAPER.md:218-219 is one
// tcgen05.mma (M = 128 queries, N = 256 candidates) per tile; the query operand and the
// queries' fp32 rows of a work item stay in shared memory for all its tiles; candidate
// tiles (operand rows by TMA with 32/64-byte swizzle, fp32 rows by bulk copy) stream
// through a ring; accumulators are double-buffered in TMEM (2 x 256 columns); 16
// epilogue warps drain them.  Work items come from an explicit descriptor list (no
// empty items): per group of G consecutive query blocks, candidate chunk k of the
// group's union window is visited by every block of the group before chunk k+1 (L2 reuse).
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"
#include "tc.h"
#include "tcgen05.cuh"

namespace snn {
namespace {
using namespace tc5;

constexpr int TM = 128, TN = 256;
constexpr int EPI = 512;
constexpr int COLS = TN / (EPI / 128);
constexpr int THREADS = 64 + EPI;

template <int KC> constexpr int row_bytes() { return KC * 2; }
template <int KC> constexpr int lstages() { return KC == 16 ? 8 : 6; }
// fp32 candidate-row slots (decoupled from the operand ring; >= operand stages + 2)
template <int KC> constexpr int cring() { return lstages<KC>() + 2; }
template <int D, int KC> struct Lay {
    static constexpr int B_BYTES = TN * row_bytes<KC>();
    static constexpr int A_BYTES = TM * row_bytes<KC>();
    static constexpr int XC_BYTES = TN * D * 4;      // fp32 candidate rows of a tile (AoSoA4)
    static constexpr int QC_BYTES = TM * D * 4;      // fp32 query rows of an item
    static constexpr int OFF_A = lstages<KC>() * B_BYTES;
    static constexpr int OFF_XC = OFF_A + 2 * A_BYTES;
    static constexpr int OFF_QC = OFF_XC + cring<KC>() * XC_BYTES;
    static constexpr int OFF_MSK = OFF_QC + 2 * QC_BYTES;     // per item: hit bits [128 rows][2048 candidates]
    static constexpr int OFF_BAR = OFF_MSK + TM * 64 * 4;
    static constexpr int SMEM = 1024 + OFF_BAR + 512;
};
template <int D, int KC> constexpr int lay_smem() { return Lay<D, KC>::SMEM; }
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

template <int D, int KC>
__global__ void __launch_bounds__(THREADS, 1)
tcl_window_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TclArgs a) {
    using L = Lay<D, KC>;
    constexpr int LS = lstages<KC>();
    constexpr int CR = cring<KC>();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t a_base = base + L::OFF_A;
    const float *xc_s = reinterpret_cast<const float *>(gbase + L::OFF_XC);
    const float *qc_s = reinterpret_cast<const float *>(gbase + L::OFF_QC);
    uint8_t *msk_b = gbase + L::OFF_MSK;
    __shared__ uint32_t flush_s[4];
    __shared__ unsigned long long pool_base_s;
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + L::OFF_BAR);
    uint64_t *full = bars, *empty = bars + LS, *tfull = bars + 2 * LS, *tempty = bars + 2 * LS + 2;
    uint64_t *afull = bars + 2 * LS + 4, *aempty = bars + 2 * LS + 6;
    uint64_t *cfull = bars + 2 * LS + 8, *cempty = bars + 2 * LS + 8 + CR;
    uint32_t *tmem_ptr = reinterpret_cast<uint32_t *>(bars + 2 * LS + 8 + 2 * CR);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < LS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI);
            mbar_init(&afull[s], 1); mbar_init(&aempty[s], EPI);
        }
        for (int s = 0; s < CR; ++s) { mbar_init(&cfull[s], 1); mbar_init(&cempty[s], EPI); }
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
            int stage = 0, as = 0, cs = 0;
            uint32_t phase = 0, aph = 0, cph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                const int4 ds = a.desc[item];
                const int b = ds.x, c0 = ds.y, c1 = ds.z;
                mbar_wait_u32(smem_u32(&aempty[as]), aph ^ 1);
                const int64_t q0 = (int64_t)b * TM;
                const int64_t qn = min((int64_t)TM, a.m_pad - q0);   // fp32 query rows present
                mbar_arrive_expect_tx(&afull[as], L::A_BYTES + (uint32_t)(qn * D * 4));
                tma_load_2d(a_base + as * L::A_BYTES, &tmA, smem_u32(&afull[as]), 0, (int)q0);
                bulk_g2s(gbase + L::OFF_QC + as * L::QC_BYTES, a.Qs + q0 * D, (uint32_t)(qn * D * 4), &afull[as]);
                if (++as == 2) { as = 0; aph ^= 1; }
                for (int t0 = c0; t0 < c1; t0 += TN) {
                    mbar_wait_u32(smem_u32(&empty[stage]), phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], L::B_BYTES);
                    tma_load_2d(base + stage * L::B_BYTES, &tmB, smem_u32(&full[stage]), 0, t0);
                    if (++stage == LS) { stage = 0; phase ^= 1; }
                    mbar_wait_u32(smem_u32(&cempty[cs]), cph ^ 1);
                    const int64_t xn = max((int64_t)0, min((int64_t)TN, a.n_pad - t0));   // fp32 rows present
                    mbar_arrive_expect_tx(&cfull[cs], (uint32_t)(xn * D * 4));
                    if (xn > 0)
                        bulk_g2s(gbase + L::OFF_XC + cs * L::XC_BYTES, a.Xs + (int64_t)t0 * D, (uint32_t)(xn * D * 4),
                                 &cfull[cs]);
                    if (++cs == CR) { cs = 0; cph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0, as = 0;
            uint32_t phase = 0, acc = 0, aphase = 0, aph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                const int4 ds = a.desc[item];
                const int c0 = ds.y, c1 = ds.z;
                mbar_wait_u32(smem_u32(&afull[as]), aph);
                tc_fence_after();
                const uint64_t da = lowd_desc<KC>(a_base + as * L::A_BYTES);
                for (int t0 = c0; t0 < c1; t0 += TN) {
                    mbar_wait_u32(smem_u32(&tempty[acc]), aphase ^ 1);
                    mbar_wait_u32(smem_u32(&full[stage]), phase);
                    tc_fence_after();
                    const uint64_t db = lowd_desc<KC>(base + stage * L::B_BYTES);
                    const uint32_t dcol = tmem + acc * TN;
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk)   // 16 FP16 (32 bytes) of K per MMA
                        mma_f16(dcol, da + 2 * kk, db + 2 * kk, TCL_IDESC, kk != 0);
                    mma_commit(smem_u32(&empty[stage]));
                    mma_commit(smem_u32(&tfull[acc]));
                    if (++stage == LS) { stage = 0; phase ^= 1; }
                    acc ^= 1;
                    if (acc == 0) aphase ^= 1;
                }
                if (++as == 2) { as = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (EPI threads)
        // 16 warps: warp w reads TMEM lane quarter (w % 4); the four warps of a quarter
        // take 64-column slices of the 256-column tile.  Lane = query row for the filter,
        // lane = candidate for the exact decision of a flagged (row, chunk).
        const int et = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int slice = et >> 7;
        const int row = quarter * 32 + lane;
        const float T_in = a.T_in, T_out = a.T_out;
        const double R2 = a.R2;
        for (int i = et; i < TM * 64; i += EPI) reinterpret_cast<uint32_t *>(msk_b)[i] = 0;
        named_bar(1, EPI);
        uint32_t acc = 0, aphase = 0;
        int as = 0, cs = 0;
        uint32_t aph = 0, cph = 0;
        for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
            const int4 ds = a.desc[item];
            const int b = ds.x, c0 = ds.y, c1 = ds.z;
            const int64_t sp = (int64_t)b * TM + row;
            const bool active = sp < a.m;
            mbar_wait_u32(smem_u32(&afull[as]), aph);
            const float *qrows = qc_s + as * (TM * D);     // AoSoA4: (r/4)*4D + 4k + r%4
            for (int t0 = c0; t0 < c1; t0 += TN) {
                mbar_wait_u32(smem_u32(&tfull[acc]), aphase);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * TN + slice * COLS;
                // flags per (row, group of 8 candidates): 3-way max trees over the accumulator
                float mg[8];
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    float v[32];
                    tmem_ld32(taddr + ch * 32, v);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const float a0 = fmaxf(fmaxf(v[8 * g], v[8 * g + 1]), v[8 * g + 2]);
                        const float a1 = fmaxf(fmaxf(v[8 * g + 3], v[8 * g + 4]), v[8 * g + 5]);
                        mg[4 * ch + g] = fmaxf(fmaxf(a0, a1), fmaxf(v[8 * g + 6], v[8 * g + 7]));
                    }
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&tempty[acc]));
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
                const int jt = t0 + slice * COLS;   // first candidate of this thread's 64 columns
                uint32_t R[8];
                uint32_t any = 0;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    R[g] = __ballot_sync(0xffffffffu, active && mg[g] >= 0.f && jt + 8 * g < c1);
                    any |= R[g];
                }
                mbar_wait_u32(smem_u32(&cfull[cs]), cph);
                if (any) {
                    // exact decision: tasks (row, group) of the flags, four per pass (lane
                    // group i = lanes 8i..8i+7 takes task 4 * pass + i, lane = candidate)
                    const float *xrows = xc_s + cs * (TN * D);
                    int pre[9];
                    pre[0] = 0;
#pragma unroll
                    for (int g = 0; g < 8; ++g) pre[g + 1] = pre[g] + __popc(R[g]);
                    const int ntask = pre[8];
                    for (int k0 = 0; k0 < ntask; k0 += 4) {
                        const int k = k0 + (lane >> 3);
                        bool hit = false;
                        int g = 0, qr = 0;
                        if (k < ntask) {
#pragma unroll
                            for (int gg = 1; gg < 8; ++gg) g += k >= pre[gg];
                            uint32_t Rg = R[0];
#pragma unroll
                            for (int gg = 1; gg < 8; ++gg) if (g == gg) Rg = R[gg];
                            const int r = (int)__fns(Rg, 0, k - pre[g] + 1);
                            qr = quarter * 32 + r;
                            const int cc = slice * COLS + 8 * g + (lane & 7);   // tile column
                            const int64_t j = (int64_t)t0 + cc;
                            if (j < a.n && j < c1) {
                                float x[D], q[D];
#pragma unroll
                                for (int kk = 0; kk < D; ++kk) {
                                    x[kk] = xrows[(cc >> 2) * 4 * D + 4 * kk + (cc & 3)];
                                    q[kk] = qrows[(qr >> 2) * 4 * D + 4 * kk + (qr & 3)];
                                }
                                // fp32 direct form, same operation order as the FFMA kernel
                                float t = x[0] - q[0];
                                float d2 = t * t;
#pragma unroll
                                for (int kk = 1; kk < D; ++kk) { t = x[kk] - q[kk]; d2 = fmaf(t, t, d2); }
                                hit = d2 <= T_in;
                                if (!hit && d2 <= T_out) {
                                    double sd = 0.0;
#pragma unroll
                                    for (int kk = 0; kk < D; ++kk) {
                                        const double tt = __dsub_rn((double)x[kk], (double)q[kk]);
                                        sd = __dadd_rn(sd, __dmul_rn(tt, tt));
                                    }
                                    hit = sd <= R2;
                                }
                            }
                        }
                        const uint32_t msk = __ballot_sync(0xffffffffu, hit);
                        const uint32_t bits = (msk >> (lane & 24)) & 0xffu;
                        if ((lane & 7) == 0 && bits)   // [row][group of 8 in the item]: written once
                            msk_b[qr * 256 + ((jt - c0) >> 3) + g] = (uint8_t)bits;
                    }
                }
                mbar_arrive(smem_u32(&cempty[cs]));
                if (++cs == CR) { cs = 0; cph ^= 1; }
            }
            mbar_arrive(smem_u32(&aempty[as]));
            if (++as == 2) { as = 0; aph ^= 1; }
            // flush the item: per row, hit positions (u16, within the item) in ascending
            // order into the position pool; one pool claim per item
            named_bar(1, EPI);
            if (et < TM) {
                const int64_t e = item * TM + et;
                const uint32_t *mr = reinterpret_cast<const uint32_t *>(msk_b + et * 256);   // 2048 bits
                uint32_t hits = 0;
                for (int w = 0; w < 64; ++w) hits += __popc(mr[w]);
                // exclusive scan of hits over the item's 128 rows (warps 2..5)
                uint32_t incl = hits;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) flush_s[et >> 5] = incl;
                named_bar(2, TM);
                uint32_t wbase = 0, tot = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) { if (w < (et >> 5)) wbase += flush_s[w]; tot += flush_s[w]; }
                if (et == 0) {
                    unsigned long long b0 = ~0ull;
                    if (tot) {
                        b0 = atomicAdd(a.pool_count, (unsigned long long)tot);
                        if (b0 + tot > (unsigned long long)a.pool_cap) b0 = ~0ull;   // full: entries re-decided later
                    }
                    pool_base_s = b0;
                }
                named_bar(2, TM);
                const unsigned long long pb = pool_base_s;
                const uint32_t my0 = wbase + incl - hits;
                if (pb != ~0ull) {
                    uint16_t *dst = a.pool + pb + my0;
                    uint32_t k = 0;
                    for (int w = 0; w < 64; ++w) {
                        uint32_t mk = mr[w];
                        while (mk) {
                            const int c = __ffs(mk) - 1;
                            mk &= mk - 1;
                            dst[k++] = (uint16_t)(w * 32 + c);
                        }
                    }
                    a.eoff[e] = pb + my0;
                } else {
                    a.eoff[e] = ~0ull;
                }
                a.ecnt[e] = hits;
                uint32_t *mz = reinterpret_cast<uint32_t *>(msk_b + et * 256);
                for (int w = 0; w < 64; ++w) mz[w] = 0;   // this row's bits, read only here
            }
            named_bar(1, EPI);   // cleared before the next item's writes
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


// Work list: per block, the chunks of its group's union window that meet its window
// (closed form), in chunk order.  bcount[b] = number of items of block b.
__global__ void tcl_block_items_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group,
                                       int chunk, int64_t *bcount) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    const int64_t g0 = (b / group) * group, g1 = min(nblocks, g0 + group);
    int64_t glo = INT64_MAX;
    for (int64_t bb = g0; bb < g1; ++bb)
        if (blk_hi[bb] > blk_lo[bb]) glo = min(glo, blk_lo[bb]);
    const int64_t lo = blk_lo[b], hi = blk_hi[b];
    bcount[b] = hi > lo ? (hi - 1 - glo) / chunk - (lo - glo) / chunk + 1 : 0;
}

// Item descriptors {b, c0, c1, k} in raster order (group, chunk k of the group's union
// window, block) -- ids of group g are [bstart[g0], bstart[g1]); bitems[bstart[b] + kk]
// = id of block b's kk-th item (chunk order).
__global__ void tcl_fill_items_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group,
                                      int chunk, const int64_t *bstart, int4 *desc, int32_t *bitems) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t g0 = g * group;
    if (g0 >= nblocks) return;
    const int64_t g1 = min(nblocks, g0 + group);
    int64_t glo = INT64_MAX, ghi = 0;
    for (int64_t bb = g0; bb < g1; ++bb)
        if (blk_hi[bb] > blk_lo[bb]) { glo = min(glo, blk_lo[bb]); ghi = max(ghi, blk_hi[bb]); }
    if (ghi <= glo) return;
    int64_t id = bstart[g0];
    const int64_t nk = (ghi - glo + chunk - 1) / chunk;
    for (int64_t k = 0; k < nk; ++k) {
        const int64_t base = glo + k * chunk;
        for (int64_t bb = g0; bb < g1; ++bb) {
            const int64_t c0 = max(base, blk_lo[bb]), c1 = min(base + chunk, blk_hi[bb]);
            if (c1 <= c0) continue;
            const int64_t kk = (blk_lo[bb] - glo) / chunk;   // block's first chunk index
            desc[id] = make_int4((int)bb, (int)c0, (int)c1, (int)(k - kk));
            bitems[bstart[bb] + (k - kk)] = (int32_t)id;
            ++id;
        }
    }
}

// Per query row: hits of each of its entries in chunk order -> pre[e] (exclusive), total.
__global__ void tcl_row_totals_kernel(const TclPost p, const int64_t *bstart, const int32_t *bitems,
                                      const uint32_t *ecnt, int32_t *pre, int32_t *row_count) {
    for (int64_t sp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sp < p.m; sp += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = sp / TM, row = sp % TM;
        int32_t run = 0;
        for (int64_t i = bstart[b]; i < bstart[b + 1]; ++i) {
            const int64_t e = (int64_t)bitems[i] * TM + row;
            pre[e] = run;
            run += (int32_t)ecnt[e];
        }
        row_count[p.qperm[sp]] = run;
    }
}

// CSR write of one entry (item, row) per thread: hit positions are in ascending order;
// ids via pi, distance = (float)sqrt(oracle-order fp64).  Entries the position pool could
// not hold are listed in ovf and re-decided by tcl_fix_kernel.
template <int D>
__global__ void __launch_bounds__(256) tcl_compact_kernel(const TclPost p, int64_t nent, const int4 *desc,
                                                          const uint32_t *ecnt, const unsigned long long *eoff,
                                                          const uint16_t *pool, const int32_t *pre,
                                                          const int64_t *offsets, int32_t *out_idx, float *out_dist,
                                                          int64_t *ovf, unsigned long long *novf) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nent; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t nh = ecnt[e];
        if (!nh) continue;
        const unsigned long long off = eoff[e];
        if (off == ~0ull) { ovf[atomicAdd(novf, 1ull)] = e; continue; }
        const int64_t item = e / TM, row = e % TM;
        const int4 ds = desc[item];
        const int64_t sp = (int64_t)ds.x * TM + row;
        int64_t pos = offsets[p.qperm[sp]] + pre[e];
        double qd[D];
#pragma unroll
        for (int k = 0; k < D; ++k) qd[k] = p.Qs[(sp >> 2) * 4 * D + 4 * k + (sp & 3)];
        for (uint32_t i = 0; i < nh; ++i) {
            const int64_t j = ds.y + pool[off + i];
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double t = __dsub_rn((double)p.Xs[(j >> 2) * 4 * D + 4 * k + (j & 3)], qd[k]);
                s = __dadd_rn(s, __dmul_rn(t, t));
            }
            out_idx[pos] = p.perm[j];
            out_dist[pos] = (float)sqrt(s);
            ++pos;
        }
    }
}

// Overflowed entries: one warp per entry re-decides the item's candidates exactly (same
// classification), 32 at a time, and writes the hits in ascending position.
template <int D>
__global__ void __launch_bounds__(256) tcl_fix_kernel(const TclPost p, const int4 *desc, const int32_t *pre,
                                                      const int64_t *offsets, const int64_t *ovf,
                                                      const unsigned long long *novf, int32_t *out_idx,
                                                      float *out_dist) {
    const int lane = threadIdx.x % 32;
    const int64_t nov = (int64_t)*novf;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; w < nov;
         w += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t e = ovf[w];
        const int64_t item = e / TM, row = e % TM;
        const int4 ds = desc[item];
        const int64_t sp = (int64_t)ds.x * TM + row;
        int64_t pos = offsets[p.qperm[sp]] + pre[e];
        float q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = p.Qs[(sp >> 2) * 4 * D + 4 * k + (sp & 3)];
        for (int64_t j0 = ds.y; j0 < ds.z; j0 += 32) {
            const int64_t j = j0 + lane;
            bool hit = false;
            double s = 0.0;
            if (j < ds.z && j < p.n) {
                float x[D];
#pragma unroll
                for (int k = 0; k < D; ++k) x[k] = p.Xs[(j >> 2) * 4 * D + 4 * k + (j & 3)];
                float t = x[0] - q[0];
                float d2 = t * t;
#pragma unroll
                for (int k = 1; k < D; ++k) { t = x[k] - q[k]; d2 = fmaf(t, t, d2); }
                if (d2 <= p.T_out) {
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        const double tt = __dsub_rn((double)x[k], (double)q[k]);
                        s = __dadd_rn(s, __dmul_rn(tt, tt));
                    }
                    hit = d2 <= p.T_in || s <= p.R2;
                }
            }
            const uint32_t msk = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int64_t o = pos + __popc(msk & lanemask_lt());
                out_idx[o] = p.perm[j];
                out_dist[o] = (float)sqrt(s);
            }
            pos += __popc(msk);
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

void launch_tcl_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                      int64_t *bcount, cudaStream_t s) {
    if (nblocks == 0) return;
    SNN_LAUNCH(tcl_block_items_kernel, (int)ceil_div(nblocks, 256), 256, 0, s, blk_lo, blk_hi, nblocks, group, chunk,
               bcount);
}

void launch_tcl_fill_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                           const int64_t *bstart, int4 *desc, int32_t *bitems, cudaStream_t s) {
    const int64_t ng = ceil_div(nblocks, group);
    if (ng == 0) return;
    SNN_LAUNCH(tcl_fill_items_kernel, (int)ceil_div(ng, 128), 128, 0, s, blk_lo, blk_hi, nblocks, group, chunk,
               bstart, desc, bitems);
}

bool launch_tcl_window(const void *qry, const void *cand, int d, int64_t cand_rows, const TclArgs &a, int sm_count,
                       cudaStream_t s) {
    if (a.total_items == 0) return true;
    const int kc = tcl_kc(d);
    CUtensorMap ma, mb;
    if (!make_map_lowd(&ma, qry, a.m, kc, TM) || !make_map_lowd(&mb, cand, cand_rows, kc, TN)) return false;
    const int g = (int)(a.total_items < sm_count ? a.total_items : sm_count);
#define CASE(D, K)                                                                                        \
    case D: {                                                                                             \
        const int sm_ = lay_smem<D, K>();                                                                 \
        cudaFuncSetAttribute(tcl_window_kernel<D, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_);  \
        SNN_LAUNCH((tcl_window_kernel<D, K>), g, THREADS, sm_, s, ma, mb, a);                             \
        break;                                                                                            \
    }
    switch (d) { CASE(1, 16) CASE(2, 16) CASE(3, 16) CASE(4, 16) CASE(5, 32) CASE(6, 32) CASE(7, 32) CASE(8, 32) default: return false; }
#undef CASE
    return true;
}

void launch_tcl_row_totals(const TclPost &p, const int64_t *bstart, const int32_t *bitems, const uint32_t *ecnt,
                           int32_t *pre, int32_t *row_count, cudaStream_t s) {
    if (p.m == 0) return;
    SNN_LAUNCH(tcl_row_totals_kernel, gridn(p.m), 256, 0, s, p, bstart, bitems, ecnt, pre, row_count);
}

void launch_tcl_compact(const TclPost &p, int d, int64_t nent, const int4 *desc, const uint32_t *ecnt,
                        const unsigned long long *eoff, const uint16_t *pool, const int32_t *pre,
                        const int64_t *offsets, int32_t *out_idx, float *out_dist, int64_t *ovf,
                        unsigned long long *novf, cudaStream_t s) {
    if (nent == 0) return;
    const int g = gridn(nent);
#define CASE(D)                                                                                              \
    case D:                                                                                                  \
        SNN_LAUNCH(tcl_compact_kernel<D>, g, 256, 0, s, p, nent, desc, ecnt, eoff, pool, pre, offsets, out_idx, \
                   out_dist, ovf, novf);                                                                     \
        SNN_LAUNCH(tcl_fix_kernel<D>, 148 * 4, 256, 0, s, p, desc, pre, offsets, ovf, novf, out_idx, out_dist); \
        break;
    switch (d) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) default: break; }
#undef CASE
}

}  // namespace snn
