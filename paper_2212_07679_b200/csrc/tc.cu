// tc.cu -- K9: windowed distance tiles on the 5th-generation tensor cores (tcgen05,
// kind::f16 with power-of-two-scaled FP16 operands, or kind::tf32) for d >= 32, and K10:
// the exact fp64 recheck of the emitted pairs.
//
// Filter (eq:ip2): with centred operands x_c = x - mu, q_c = q - mu,
//   d^2 = 2 xbar + 2 qbar - 2 x_c.q_c,   xbar = x_c.x_c / 2 (Alg. 1 l.7).
// The batched inner products X(J,:) [q_1..q_l] (the "gemm" of PAPER.md:218-219) are one
// tcgen05.mma tile D[128 queries x 256 candidates] += Q_tile . X_tile^T per 8-wide K step,
// operands pre-rounded to FP16 (x_c * 2^a, round-to-nearest; unit roundoff 2^-11, half
// the bytes of TF32 at twice the MMA rate) or TF32 (cvt.rna) in shared memory (TMA,
// 128B swizzle), FP32 accumulators in TMEM.  The expanded form is NOT accurate under cancellation (DESIGN.md
// reading C4), so the epilogue only selects CANDIDATES with a rigorous separable margin
//   |d^2_tc - d^2| <= c1 (xbar + qbar) + c0            (reading C20)
// i.e. acc - xbar (1 - c1/2) >= qbar (1 - c1/2) - (R^2 (1+1e-12) + c0)/2,
// and every candidate pair is re-decided by K10 with the oracle's exact fp64 sequence
// (eq:ip1 on the original coordinates), which also produces the distance.
//
// Work items are (query block, candidate chunk) pairs in a grouped raster order: for a
// group of G consecutive query blocks, candidate chunk k of the group's union window is
// visited by every block of the group before chunk k+1, so an index chunk is read from
// HBM once per group and re-served from L2 (X of config 4 is 0.8-1.6 GB >> 126 MB L2).
//
// Kernel structure (one CTA per SM, persistent over the items):
//   warp 0    : TMA producer  (cp.async.bulk.tensor.2d, mbarrier full/empty ring, 4 stages)
//   warp 1    : TMEM allocator + single-thread tcgen05.mma issuer, tcgen05.commit
//   warps 2-17: epilogue: tcgen05.ld 32x32b.x32 -> registers, margin test (FFMA + 3-way
//               max per 32 columns), per-lane candidate masks, staged pair output into
//               per-warp claimed blocks; TMEM double-buffered (2 x 256 cols)
#include <cuda.h>
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"
#include "index.h"
#include "tc.h"
#include "tcgen05.cuh"

namespace snn {
namespace {
using namespace tc5;

constexpr int TM = 128, TN = 256, STAGES = 4;
constexpr int KB_BYTES = 128;                      // bytes per operand row per K block (one swizzle atom)
constexpr int A_BYTES = TM * KB_BYTES, B_BYTES = TN * KB_BYTES, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STAGE_CAP = 8;                       // staged hits per epilogue thread per tile
constexpr int ARING = 8;                           // x-bar slices in flight (decoupled from TMEM)
constexpr unsigned long long CLAIM = 256;          // pair-list slots claimed per warp atomic
constexpr int EPI = 512;                           // epilogue threads (16 warps)
constexpr int COLS = TN / (EPI / 128);             // columns per epilogue thread
constexpr int THREADS = 64 + EPI;
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + ARING * TN * 4 + EPI * STAGE_CAP * 4 + 512;
// ARES (one K block): the query tile is loaded once per work item into one of two
// resident slots; the ring then streams only candidate tiles (a third fewer operand bytes)
constexpr int STAGES_R = 5;
constexpr int SMEM_BYTES_R = 1024 + STAGES_R * B_BYTES + 2 * A_BYTES + ARING * TN * 4 + EPI * STAGE_CAP * 4 + 512;
// instruction descriptor: D format F32; A, B format F16 (0, kind::f16) or TF32 (2,
// kind::tf32); both K-major; N >> 3 at bit 17, M >> 4 at bit 24
template <bool F16>
constexpr uint32_t idesc() {
    return (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) |
           ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}
template <bool F16> constexpr int k_elems() { return F16 ? 64 : 32; }   // elements per K block

__device__ __forceinline__ unsigned long long f2pack_tc(float x, float y) {
    float2 v = make_float2(x, y);
    return *reinterpret_cast<unsigned long long *>(&v);
}
// (v0, v1) = (w0, w1) * nc + (v0, v1) with one packed FFMA2 (the same rounding as two FFMAs)
__device__ __forceinline__ void ffma2_inplace(float &v0, float &v1, float w0, float w1, unsigned long long nc) {
    unsigned long long acc = f2pack_tc(v0, v1), w = f2pack_tc(w0, w1), r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(w), "l"(nc), "l"(acc));
    const float2 o = *reinterpret_cast<float2 *>(&r);
    v0 = o.x;
    v1 = o.y;
}

template <bool F16>
__device__ __forceinline__ void mma_op(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
    if constexpr (F16) tc5::mma_f16(tmem_d, adesc, bdesc, idesc<true>(), acc);
    else tc5::mma_tf32(tmem_d, adesc, bdesc, idesc<false>(), acc);
}

// item -> (query block b, candidate range [c0, c1)); empty ranges (c0 >= c1) are skipped
// by every role.  Group g holds blocks [gG, gG + Gc); its items are ordered (chunk k of
// the group's union window, block), k-major.
__device__ __forceinline__ void tc_locate(const TcArgs &a, int64_t item, int64_t &b, int64_t &c0, int64_t &c1) {
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

template <bool F16, bool ARES>
__global__ void __launch_bounds__(THREADS, 1)
tc_window_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
    constexpr int TK = k_elems<F16>();
    constexpr int NST = ARES ? STAGES_R : STAGES;              // ring stages
    constexpr int SB = ARES ? B_BYTES : STAGE_BYTES;           // bytes per ring stage
    constexpr int RING = NST * SB + (ARES ? 2 * A_BYTES : 0);  // ring (+ resident query slots)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    // carve: stages [| query slots] | a_vals[ARING][TN] | stage hits [EPI][STAGE_CAP] | barriers | tmem ptr
    const uint32_t qbase = base + NST * SB;   // ARES: resident query tiles
    float *a_vals = reinterpret_cast<float *>(gbase + RING);
    int32_t *s_hits = reinterpret_cast<int32_t *>(gbase + RING + ARING * TN * 4);
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + RING + ARING * TN * 4 + EPI * STAGE_CAP * 4);
    uint64_t *full = bars, *empty = bars + NST, *tfull = bars + 2 * NST, *tempty = bars + 2 * NST + 2;
    uint64_t *afull = bars + 2 * NST + 4, *aempty = bars + 2 * NST + 4 + ARING;
    uint64_t *qfull = bars + 2 * NST + 4 + 2 * ARING, *qempty = qfull + 2;
    uint32_t *tmem_ptr = reinterpret_cast<uint32_t *>(qfull + 4);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t hint = a.wait_hint;
    auto twait = [hint](uint32_t bar, uint32_t ph) {
        if (hint) mbar_wait_u32_sleep(bar, ph, hint); else mbar_wait_u32(bar, ph);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        const uint32_t earr = a.warp_arrive ? EPI / 32 : EPI;   // epilogue arrivals per release
        for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], earr); }
        for (int s = 0; s < 2; ++s) { mbar_init(&qfull[s], 1); mbar_init(&qempty[s], 1); }
        for (int s = 0; s < ARING; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], earr); }
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
            int stage = 0, qs = 0;
            uint32_t phase = 0, aslot = 0, aph = 0, qph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                int64_t b, c0, c1;
                tc_locate(a, item, b, c0, c1);
                if (ARES) {
                    if (c1 <= c0) continue;
                    twait(smem_u32(&qempty[qs]), qph ^ 1);
                    mbar_arrive_expect_tx(&qfull[qs], A_BYTES);
                    tma_load_2d(qbase + qs * A_BYTES, &tmA, smem_u32(&qfull[qs]), 0, (int)(b * TM));
                    if (++qs == 2) { qs = 0; qph ^= 1; }
                }
                for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                    // x-bar slice of this tile -> a-ring slot (read by the epilogue)
                    twait(smem_u32(&aempty[aslot]), aph ^ 1);
                    mbar_arrive_expect_tx(&afull[aslot], TN * 4);
                    bulk_g2s(a_vals + aslot * TN, a.xbar + t0, TN * 4, &afull[aslot]);
                    if (++aslot == ARING) { aslot = 0; aph ^= 1; }
                    for (int kb = 0; kb < a.kblocks; ++kb) {
                        twait(smem_u32(&empty[stage]), phase ^ 1);
                        const uint32_t sa = base + stage * SB, sb = ARES ? sa : sa + A_BYTES;
                        mbar_arrive_expect_tx(&full[stage], SB);
                        if (!ARES) tma_load_2d(sa, &tmA, smem_u32(&full[stage]), kb * TK, (int)(b * TM));
                        tma_load_2d(sb, &tmB, smem_u32(&full[stage]), kb * TK, (int)t0);
                        if (++stage == NST) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0, qs = 0;
            uint32_t phase = 0, acc = 0, aphase = 0, qph = 0;
            for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
                int64_t b, c0, c1;
                tc_locate(a, item, b, c0, c1);
                if (ARES) {
                    if (c1 <= c0) continue;
                    twait(smem_u32(&qfull[qs]), qph);
                    tc_fence_after();
                }
                for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                    twait(smem_u32(&tempty[acc]), aphase ^ 1);
                    tc_fence_after();
                    const uint32_t dcol = tmem + acc * TN;
                    for (int kb = 0; kb < a.kblocks; ++kb) {
                        twait(smem_u32(&full[stage]), phase);
                        tc_fence_after();
                        const uint32_t sa = ARES ? qbase + qs * A_BYTES : base + stage * SB;
                        const uint32_t sb = ARES ? base + stage * SB : sa + A_BYTES;
                        const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
                        if (a.diag != 2 && a.diag != 3) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)   // 4 MMAs of 32 bytes of K each
                                mma_op<F16>(dcol, da + 2 * kk, db + 2 * kk, (kb | kk) != 0);
                        }
                        mma_commit(smem_u32(&empty[stage]));
                        if (++stage == NST) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(smem_u32(&tfull[acc]));
                    acc ^= 1;
                    if (acc == 0) aphase ^= 1;
                }
                if (ARES) {   // the query slot is free once this item's MMAs retire
                    mma_commit(smem_u32(&qempty[qs]));
                    if (++qs == 2) { qs = 0; qph ^= 1; }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (EPI threads)
        // 16 warps: warp w may only touch TMEM lane quarter (w % 4); the four warps of a
        // quarter split the 256 columns into 64-column slices.  One thread = one query row.
        const int et = threadIdx.x - 64;              // 0..EPI-1
        const int quarter = warp & 3;
        const int slice = et >> 7;                    // 0..3
        const int row = quarter * 32 + lane;
        int32_t *my_hits = s_hits + et * STAGE_CAP;
        const float c1h = a.c1h * a.sc;   // acc is scaled by sc = 2^(a+b) (exact)
        const unsigned long long nc1h2 = f2pack_tc(-c1h, -c1h);
        uint32_t acc = 0, aphase = 0, aslot = 0, aph = 0;
        unsigned long long wcur = 0, wend = 0;   // this warp's claimed pair-list block
        for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
            int64_t b, c0, c1;
            tc_locate(a, item, b, c0, c1);
            const int64_t sp = b * TM + row;
            const float bi = sp < a.m ? fmaf(a.qbar[sp], a.c1h, -a.r2h) * a.sc : INFINITY;
            int nh = 0;   // staged hits of this row (kept across the item's tiles)
            for (int64_t t0 = c0; t0 < c1; t0 += TN) {
                const float *av = a_vals + aslot * TN + slice * COLS;
                twait(smem_u32(&afull[aslot]), aph);
                twait(smem_u32(&tfull[acc]), aphase);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * TN + slice * COLS;
                const int nch = a.diag == 1 ? 0 : COLS / 32;   // diag 1: no epilogue work
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    float v[32];
                    tmem_ld32(taddr + ch * 32, v);
                    const float4 *a4 = reinterpret_cast<const float4 *>(av + ch * 32);
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {   // v = acc - xbar (1 - c1/2), two columns per FFMA2
                        const float4 w = a4[c4];
                        ffma2_inplace(v[4 * c4 + 0], v[4 * c4 + 1], w.x, w.y, nc1h2);
                        ffma2_inplace(v[4 * c4 + 2], v[4 * c4 + 3], w.z, w.w, nc1h2);
                    }
                    float m[11];
#pragma unroll
                    for (int c = 0; c < 10; ++c) m[c] = fmaxf(fmaxf(v[3 * c], v[3 * c + 1]), v[3 * c + 2]);
                    m[10] = fmaxf(v[30], v[31]);
#pragma unroll
                    for (int c = 0; c < 3; ++c) m[c] = fmaxf(fmaxf(m[3 * c], m[3 * c + 1]), m[3 * c + 2]);
                    const float mx = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[9] > m[10] ? m[9] : m[10]));
                    if (mx >= bi && a.diag < 3) {
                        // rare (per lane): candidate mask, then one staged entry per set bit
                        uint32_t mask = 0;
#pragma unroll
                        for (int c = 0; c < 32; ++c) mask |= (v[c] >= bi ? 1u : 0u) << c;
                        const int64_t jb = t0 + slice * COLS + ch * 32;
                        while (mask) {
                            const int c = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const int64_t jj = jb + c;
                            if (jj >= c1) break;
                            SNN_DASSERT(sp < a.m && jj < a.n);
                            if (nh < STAGE_CAP) {
                                my_hits[nh++] = (int32_t)jj;
                            } else {   // rare: direct append
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
                if (a.warp_arrive) {   // one arrive per warp once every lane's TMEM loads retired
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(smem_u32(&tempty[acc]));
                        mbar_arrive(smem_u32(&aempty[aslot]));
                    }
                } else {
                    mbar_arrive(smem_u32(&tempty[acc]));
                    mbar_arrive(smem_u32(&aempty[aslot]));
                }
                if (++aslot == ARING) { aslot = 0; aph ^= 1; }
                // staged hits -> the warp's claimed block of the pair list (one global
                // atomic per CLAIM slots instead of one per tile); unused slots get q = -1.
                // The stage is flushed when it is half full or at the item's last tile (the
                // row sp changes with the item), not after every tile.
                const bool item_end = t0 + TN >= c1;
                if (__any_sync(0xffffffffu, nh > (item_end ? 0 : STAGE_CAP / 2 - 1))) {
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
                    nh = 0;
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
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// TF32 centred copy: out[i][k] = rna_tf32(fl32(X[perm[i]][k] - mu_f[k])), zero padded
// to kpad columns; also half norms of the (fp32) centred row, fp64 accumulation.
template <typename T>
__global__ void __launch_bounds__(256) gather_tf32(const T *__restrict__ X, int64_t rows, int d, int kpad,
                                                   const uint32_t *__restrict__ perm,
                                                   const float *__restrict__ mu_f, float *__restrict__ out,
                                                   float *half_norm) {
    const int l = threadIdx.x % 32;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < rows;
         i += (int64_t)gridDim.x * blockDim.x / 32) {
        const T *x = X + (int64_t)perm[i] * d;
        double h = 0.0;
        for (int k = l; k < kpad; k += 32) {
            float v = 0.f;
            if (k < d) {
                const float c = (float)((double)x[k] - (double)mu_f[k]);   // exact for fp32 inputs up to one rounding
                h += (double)c * (double)c;
                uint32_t t;
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(c));
                v = __uint_as_float(t);
            }
            out[i * kpad + k] = v;
        }
        h = warp_sum(h);
        if (l == 0 && half_norm) half_norm[i] = (float)(0.5 * h);
    }
}

// FP16 centred, scaled copy: out[i][k] = rn_f16(fl32(X[perm[i]][k] - mu_f[k]) * scale),
// scale = 2^e chosen on the host so that |x_c| * scale <= 2^15 (no overflow); zero padded
// to kpad columns; half norms of the unscaled fp32 centred row (fp64 accumulation).
template <typename T>
__global__ void __launch_bounds__(256) gather_f16(const T *__restrict__ X, int64_t rows, int d, int kpad,
                                                  const uint32_t *__restrict__ perm,
                                                  const float *__restrict__ mu_f, float scale,
                                                  __half *__restrict__ out, float *half_norm) {
    const int l = threadIdx.x % 32;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < rows;
         i += (int64_t)gridDim.x * blockDim.x / 32) {
        const T *x = X + (int64_t)perm[i] * d;
        double h = 0.0;
        for (int k = 2 * l; k < kpad; k += 64) {
            float v0 = 0.f, v1 = 0.f;
            if (k < d) {
                const float c = (float)((double)x[k] - (double)mu_f[k]);
                h += (double)c * (double)c;
                v0 = c * scale;
            }
            if (k + 1 < d) {
                const float c = (float)((double)x[k + 1] - (double)mu_f[k + 1]);
                h += (double)c * (double)c;
                v1 = c * scale;
            }
            *reinterpret_cast<__half2 *>(out + i * kpad + k) = __halves2half2(__float2half_rn(v0), __float2half_rn(v1));
        }
        h = warp_sum(h);
        if (l == 0 && half_norm) half_norm[i] = (float)(0.5 * h);
    }
}

// K10: exact recheck of candidate pairs (oracle sequence on the original coordinates).
template <typename T>
__global__ void __launch_bounds__(256) recheck_pairs(const T *__restrict__ Xs, const T *__restrict__ Qs, int ld, int d,
                                                     const int32_t *__restrict__ pq, const int32_t *__restrict__ pj,
                                                     int64_t npairs, double R2, uint32_t *flag, float *dist) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += (int64_t)gridDim.x * blockDim.x) {
        if (pq[k] < 0) {   // unused slot of a claimed block
            flag[k] = 0;
            dist[k] = 0.f;
            continue;
        }
        SNN_DASSERT(pj[k] >= 0 && (ld & 3) == 0);
        const T *x = Xs + (int64_t)pj[k] * ld, *q = Qs + (int64_t)pq[k] * ld;
        double s = 0.0;
        if constexpr (sizeof(T) == 4) {   // rows are 16-byte aligned (ld % 4 == 0): vector loads,
            int kk = 0;                   // same left-to-right operation order as the oracle
            for (; kk + 4 <= d; kk += 4) {
                const float4 xv = *reinterpret_cast<const float4 *>(x + kk);
                const float4 qv = *reinterpret_cast<const float4 *>(q + kk);
                double t;
                t = __dsub_rn((double)xv.x, (double)qv.x); s = __dadd_rn(s, __dmul_rn(t, t));
                t = __dsub_rn((double)xv.y, (double)qv.y); s = __dadd_rn(s, __dmul_rn(t, t));
                t = __dsub_rn((double)xv.z, (double)qv.z); s = __dadd_rn(s, __dmul_rn(t, t));
                t = __dsub_rn((double)xv.w, (double)qv.w); s = __dadd_rn(s, __dmul_rn(t, t));
            }
            for (; kk < d; ++kk) {
                const double t = __dsub_rn((double)x[kk], (double)q[kk]);
                s = __dadd_rn(s, __dmul_rn(t, t));
            }
        } else {
            s = sqdist_exact(x, q, d);
        }
        flag[k] = s <= R2;
        dist[k] = (float)sqrt(s);
    }
}

// Fused K5 for FP16 tensor-core indexes: one read of X[perm[i]] writes the sorted copy
// (stride ld, zero pad, NaN sentinel rows [n, n_pad)), the scaled FP16 centred operand
// row (kpad, zero pad) and the half norm of the fp32 centred row (fp64 accumulation) --
// the same values as gather_generic + gather_f16.
template <typename T>
__global__ void __launch_bounds__(256) gather_xs_f16(const T *__restrict__ X, int64_t n, int64_t n_pad, int d, int ld,
                                                     int kpad, const uint32_t *__restrict__ perm,
                                                     const float *__restrict__ mu_f, float scale, T *__restrict__ Xs,
                                                     __half *__restrict__ out, float *half_norm) {
    const int l = threadIdx.x % 32;
    const int kmax = ld > kpad ? ld : kpad;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n_pad;
         i += (int64_t)gridDim.x * blockDim.x / 32) {
        if (i >= n) {   // sentinel rows: never candidates
            for (int k = l; k < ld; k += 32) Xs[i * ld + k] = (k < d) ? (T)NAN : (T)0;
            if (l == 0 && half_norm) half_norm[i] = NAN;
            continue;
        }
        const T *x = X + (int64_t)perm[i] * d;
        double h = 0.0;
        for (int k = 2 * l; k < kmax; k += 64) {
            const T a0 = k < d ? x[k] : (T)0, a1 = k + 1 < d ? x[k + 1] : (T)0;
            if (k < ld) Xs[i * ld + k] = a0;
            if (k + 1 < ld) Xs[i * ld + k + 1] = a1;
            if (k < kpad) {
                float v0 = 0.f, v1 = 0.f;
                if (k < d) {
                    const float c = (float)((double)a0 - (double)mu_f[k]);
                    h += (double)c * (double)c;
                    v0 = c * scale;
                }
                if (k + 1 < d) {
                    const float c = (float)((double)a1 - (double)mu_f[k + 1]);
                    h += (double)c * (double)c;
                    v1 = c * scale;
                }
                *reinterpret_cast<__half2 *>(out + i * kpad + k) = __halves2half2(__float2half_rn(v0), __float2half_rn(v1));
            }
        }
        h = warp_sum(h);
        if (l == 0 && half_norm) half_norm[i] = (float)(0.5 * h);
    }
}

}  // namespace

// ------------------------------------------------------------------------- host side
static bool make_map(CUtensorMap *m, const void *ptr, bool f16, int64_t rows, int kpad, int box_rows) {
    tc5::EncodeTiledFn enc = tc5::get_encode();
    if (!enc) return false;
    const int es_bytes = f16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kpad * es_bytes};
    cuuint32_t box[2] = {(cuuint32_t)(KB_BYTES / es_bytes), (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr),
               dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int tc_tile_rows() { return TM; }
int tc_tile_cols() { return TN; }
int tc_kpad(int d, bool f16) { return (int)round_up(d, f16 ? 64 : 32); }
int64_t tc_claim_slack() { return (int64_t)(EPI / 32) * (int64_t)CLAIM; }

void launch_gather_tf32(const void *X, bool f64, int64_t rows, int d, const uint32_t *perm, const float *mu_f,
                        float *out, float *half_norm, cudaStream_t s) {
    if (rows == 0) return;
    const int kpad = tc_kpad(d, false);
    int64_t g = ceil_div(rows * 32, 256);
    if (g > 148 * 16) g = 148 * 16;
    if (f64) SNN_LAUNCH(gather_tf32<double>, (int)g, 256, 0, s, (const double *)X, rows, d, kpad, perm, mu_f, out, half_norm);
    else SNN_LAUNCH(gather_tf32<float>, (int)g, 256, 0, s, (const float *)X, rows, d, kpad, perm, mu_f, out, half_norm);
}

void launch_gather_f16(const void *X, bool f64, int64_t rows, int d, const uint32_t *perm, const float *mu_f,
                       float scale, void *out, float *half_norm, cudaStream_t s) {
    if (rows == 0) return;
    const int kpad = tc_kpad(d, true);
    int64_t g = ceil_div(rows * 32, 256);
    if (g > 148 * 16) g = 148 * 16;
    __half *o = static_cast<__half *>(out);
    if (f64) SNN_LAUNCH(gather_f16<double>, (int)g, 256, 0, s, (const double *)X, rows, d, kpad, perm, mu_f, scale, o, half_norm);
    else SNN_LAUNCH(gather_f16<float>, (int)g, 256, 0, s, (const float *)X, rows, d, kpad, perm, mu_f, scale, o, half_norm);
}

void launch_gather_xs_f16(const void *X, bool f64, int64_t n, int64_t n_pad, int d, int ld, const uint32_t *perm,
                          const float *mu_f, float scale, void *Xs, void *out, float *half_norm, cudaStream_t s) {
    if (n_pad == 0) return;
    const int kpad = tc_kpad(d, true);
    int64_t g = ceil_div(n_pad * 32, 256);
    if (g > 148 * 16) g = 148 * 16;
    __half *o = static_cast<__half *>(out);
    if (f64) SNN_LAUNCH(gather_xs_f16<double>, (int)g, 256, 0, s, (const double *)X, n, n_pad, d, ld, kpad, perm, mu_f,
                        scale, (double *)Xs, o, half_norm);
    else SNN_LAUNCH(gather_xs_f16<float>, (int)g, 256, 0, s, (const float *)X, n, n_pad, d, ld, kpad, perm, mu_f, scale,
                    (float *)Xs, o, half_norm);
}

bool launch_tc_window(const void *Qt, const void *Xt, bool f16, const TcArgs &a, int sm_count, cudaStream_t s) {
    if (a.total_items == 0) return true;
    CUtensorMap ma, mb;
    if (!make_map(&ma, Qt, f16, a.m, a.kpad, TM) || !make_map(&mb, Xt, f16, a.n, a.kpad, TN)) return false;
    int g = (int)(a.total_items < sm_count ? a.total_items : sm_count);
    const bool ares = a.kblocks == 1 && a.ares;
#define TCW(F, R, SM)                                                                               \
    do {                                                                                            \
        cudaFuncSetAttribute(tc_window_kernel<F, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM); \
        SNN_LAUNCH((tc_window_kernel<F, R>), g, THREADS, SM, s, ma, mb, a);                          \
    } while (0)
    if (f16) { if (ares) TCW(true, true, SMEM_BYTES_R); else TCW(true, false, SMEM_BYTES); }
    else { if (ares) TCW(false, true, SMEM_BYTES_R); else TCW(false, false, SMEM_BYTES); }
#undef TCW
    return true;
}

// Grouped raster of the work items: per group of G blocks, the union window [lo, hi)
// and G_c x ceil((hi - lo) / chunk) items (some may be empty).
__global__ void tc_group_items_kernel(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group,
                                      int chunk, int64_t ngroups, int64_t *grp_lo, int64_t *grp_items) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const int64_t b0 = g * group, b1 = min(nblocks, b0 + group);
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t b = b0; b < b1; ++b) {
        if (blk_hi[b] > blk_lo[b]) {
            lo = min(lo, blk_lo[b]);
            hi = max(hi, blk_hi[b]);
        }
    }
    if (hi <= lo) { grp_lo[g] = 0; grp_items[g] = 0; return; }
    grp_lo[g] = lo;
    grp_items[g] = (b1 - b0) * ceil_div(hi - lo, chunk);
}

void launch_tc_group_items(const int64_t *blk_lo, const int64_t *blk_hi, int64_t nblocks, int group, int chunk,
                           int64_t *grp_lo, int64_t *grp_items, cudaStream_t s) {
    const int64_t ng = ceil_div(nblocks, group);
    if (ng == 0) return;
    SNN_LAUNCH(tc_group_items_kernel, (int)ceil_div(ng, 256), 256, 0, s, blk_lo, blk_hi, nblocks, group, chunk, ng,
               grp_lo, grp_items);
}

void launch_recheck(const void *Xs, const void *Qs, bool f64, int ld, int d, const int32_t *pq, const int32_t *pj,
                    int64_t npairs, double R2, uint32_t *flag, float *dist, cudaStream_t s) {
    if (npairs == 0) return;
    int64_t g = ceil_div(npairs, 256);
    if (g > 148 * 16) g = 148 * 16;
    if (f64) SNN_LAUNCH(recheck_pairs<double>, (int)g, 256, 0, s, (const double *)Xs, (const double *)Qs, ld, d, pq, pj, npairs, R2, flag, dist);
    else SNN_LAUNCH(recheck_pairs<float>, (int)g, 256, 0, s, (const float *)Xs, (const float *)Qs, ld, d, pq, pj, npairs, R2, flag, dist);
}

}  // namespace snn

// ------------------------------------------------------------------------- CSR assembly
namespace snn {
namespace {

__global__ void tc_scatter_hits(const uint32_t *flag, const int64_t *pos, const int32_t *pq, const int32_t *pj,
                                const float *dist, const int32_t *qperm, int64_t P, uint32_t *hq, uint32_t *hj,
                                float *hd, int32_t *row_count) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[k]) continue;
        const int64_t p = pos[k];
        const int32_t q = qperm[pq[k]];
        hq[p] = (uint32_t)q;
        hj[p] = (uint32_t)pj[k];
        hd[p] = dist[k];
        atomicAdd(&row_count[q], 1);
    }
}

__global__ void tc_gather_u32(const uint32_t *src, const uint32_t *idx, int64_t H, uint32_t *dst) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < H; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[idx[k]];
}

__global__ void tc_write_csr(const uint32_t *order, const uint32_t *hj, const float *hd, const int32_t *perm,
                             int64_t H, int32_t *out_idx, float *out_dist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = order[i];
        out_idx[i] = perm[hj[k]];
        out_dist[i] = hd[k];
    }
}

int grid_for_n(int64_t n) {
    int64_t g = ceil_div(n, 256);
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

void launch_tc_scatter(const uint32_t *flag, const int64_t *pos, const int32_t *pq, const int32_t *pj,
                       const float *dist, const int32_t *qperm, int64_t P, uint32_t *hq, uint32_t *hj, float *hd,
                       int32_t *row_count, cudaStream_t s) {
    if (P == 0) return;
    SNN_LAUNCH(tc_scatter_hits, grid_for_n(P), 256, 0, s, flag, pos, pq, pj, dist, qperm, P, hq, hj, hd, row_count);
}

void launch_gather_u32(const uint32_t *src, const uint32_t *idx, int64_t H, uint32_t *dst, cudaStream_t s) {
    if (H == 0) return;
    SNN_LAUNCH(tc_gather_u32, grid_for_n(H), 256, 0, s, src, idx, H, dst);
}

void launch_tc_write(const uint32_t *order, const uint32_t *hj, const float *hd, const int32_t *perm, int64_t H,
                     int32_t *out_idx, float *out_dist, cudaStream_t s) {
    if (H == 0) return;
    SNN_LAUNCH(tc_write_csr, grid_for_n(H), 256, 0, s, order, hj, hd, perm, H, out_idx, out_dist);
}

}  // namespace snn
