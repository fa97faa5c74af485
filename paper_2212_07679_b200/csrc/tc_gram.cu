// tc_gram.cu -- K2a for large d on the tensor cores: the centred Gram matrix
//   G = sum_i (p_i - mu)(p_i - mu)^T            (X^T X of Alg. 1 l.4, PAPER.md:128;
//                                                v1 = its dominant eigenvector, eq:svd)
// as a tcgen05 kind::f16 GEMM with K = n (the rows of X).
//
// The MMA wants K-major operands, i.e. X transposed, so one pass writes the centred,
// power-of-two-scaled copy of X^T split into two FP16 halves, v = h + l (h = rn16(v),
// l = rn16(v - h): 22 significant bits), and the GEMM accumulates the three products
// h.h^T + h.l^T + l.h^T (exact in FP32, accumulated in TMEM, combined across row splits
// with fp64 atomics).  The dropped l.l^T term and the split are ~2^-22 relative, i.e. the
// same accuracy class as the SIMT fp32-product Gram (gram_tiled).  v1's accuracy only
// decides how tight the candidate windows are, never which neighbours are returned.
//
// One CTA = one 256 x 256 tile (ti <= tj, upper triangle) x one slice of the rows:
//   warp 0    : TMA producer (four 128-row boxes of 64 rows of X^T per stage, 3 stages)
//   warp 1    : TMEM allocation (2 x 256 columns) + single-thread MMA issuer
//   warps 2-5 : epilogue: tcgen05.ld, unscale, fp64 atomicAdd into G (and its mirror)
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace snn {
namespace {
using namespace tc5;

constexpr int GT = 256;                          // tile side (dims)
constexpr int GKR = 64;                          // rows of X per stage (64 FP16 = 128 B)
constexpr int G_STAGES = 3;
constexpr int G_BOX = 128 * 128;                 // one 128-row x 128-byte box
constexpr int G_STAGE = 4 * G_BOX;               // A0, A1, B0, B1
constexpr int G_THREADS = 192;
constexpr int G_SMEM = 1024 + G_STAGES * G_STAGE + 256;
constexpr uint32_t G_IDESC = make_idesc(true, 128, 256);

// xc = max_k (max|x_k| + |mu_k|) from the column maxima, or the stored bound xc_bound
// (maxabs_bits == nullptr: the index's ST_XCMAX)
__global__ void gram_scale_kernel(int d, const uint32_t *maxabs_bits, const float *mu_f, double xc_bound, int *e_out) {
    double xc = maxabs_bits ? 0.0 : xc_bound;
    for (int i = threadIdx.x; maxabs_bits && i < d; i += 32)
        xc = fmax(xc, (double)__uint_as_float(maxabs_bits[i]) + fabs((double)mu_f[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xc = fmax(xc, __shfl_xor_sync(0xffffffffu, xc, o));
    if (threadIdx.x == 0) {
        int e = 0;
        if (xc > 0.0 && isfinite(xc)) e = 14 - ilogb(xc);
        *e_out = e < -60 ? -60 : (e > 60 ? 60 : e);
    }
}

// XT_h[k][i] + XT_l[k][i] = fl32(X[i rs + k] - mu_f[k]) * 2^e (clamped to the FP16 range);
// rows i in [n, ldt) are zero.  rs = elements between consecutive rows used (d for all
// rows of a row-major X; a multiple of d samples every rs/d-th row; ld for the index copy).
template <typename T>
__global__ void __launch_bounds__(256) gram_transpose_split(const T *__restrict__ X, int64_t n, int d, int64_t rs, int64_t ldt,
                                                            const float *__restrict__ mu_f, const int *e_ptr,
                                                            __half *__restrict__ XT_h, __half *__restrict__ XT_l) {
    // 128 rows x 64 columns per CTA: every output column gets a 256-byte contiguous run
    __shared__ float tile[128][65];
    const int64_t r0 = (int64_t)blockIdx.x * 128;
    const int c0 = blockIdx.y * 64;
    const float sc = ldexpf(1.0f, *e_ptr);
    for (int e = threadIdx.x; e < 128 * 64; e += 256) {
        const int r = e / 64, c = e % 64;
        const int64_t row = r0 + r;
        const int col = c0 + c;
        float v = 0.f;
        if (row < n && col < d) {
            v = (float)((double)X[row * rs + col] - (double)mu_f[col]) * sc;
            v = fminf(fmaxf(v, -65504.f), 65504.f);
        }
        tile[r][c] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 64; e += 256) {
        const int c = e / 64, r2 = (e % 64) * 2;
        const int col = c0 + c;
        const int64_t row = r0 + r2;
        if (col >= d || row >= ldt) continue;
        const float v0 = tile[r2][c], v1 = tile[r2 + 1][c];
        const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
        const __half l0 = __float2half_rn(v0 - __half2float(h0)), l1 = __float2half_rn(v1 - __half2float(h1));
        *reinterpret_cast<__half2 *>(XT_h + (int64_t)col * ldt + row) = __halves2half2(h0, h1);
        *reinterpret_cast<__half2 *>(XT_l + (int64_t)col * ldt + row) = __halves2half2(l0, l1);
    }
}

__global__ void __launch_bounds__(G_THREADS, 1)
gram_tc_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmL, int d,
               int64_t nkb, int64_t kps, int nt, const int *e_ptr, double *G) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + G_STAGES * G_STAGE);
    uint64_t *full = bars, *empty = bars + G_STAGES, *done = bars + 2 * G_STAGES;
    uint32_t *tmem_ptr = reinterpret_cast<uint32_t *>(bars + 2 * G_STAGES + 1);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    int t = blockIdx.x, ti = 0;   // upper-triangle tile -> (ti, tj), ti <= tj
    while (t >= nt - ti) { t -= nt - ti; ++ti; }
    const int tj = ti + t;
    const int64_t kb0 = (int64_t)blockIdx.y * kps;
    const int64_t kb1 = min(nkb, kb0 + kps);
    if (kb1 <= kb0) return;   // uniform over the CTA
    const int64_t iters = 3 * (kb1 - kb0);   // passes (h,h), (h,l), (l,h)

    if (threadIdx.x == 0) {
        for (int s = 0; s < G_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(done, 1);
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
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmL)) : "memory");
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = 0; it < iters; ++it) {
                const int pass = (int)(it / (kb1 - kb0));
                const int kx = (int)((kb0 + it % (kb1 - kb0)) * GKR);
                const CUtensorMap *ma = pass == 2 ? &tmL : &tmH;   // A: h, h, l
                const CUtensorMap *mb = pass == 1 ? &tmL : &tmH;   // B: h, l, h
                mbar_wait_u32(smem_u32(&empty[stage]), phase ^ 1);
                const uint32_t sb = base + stage * G_STAGE;
                mbar_arrive_expect_tx(&full[stage], G_STAGE);
                const uint32_t fb = smem_u32(&full[stage]);
                tma_load_2d(sb, ma, fb, kx, ti * GT);
                tma_load_2d(sb + G_BOX, ma, fb, kx, ti * GT + 128);
                tma_load_2d(sb + 2 * G_BOX, mb, fb, kx, tj * GT);
                tma_load_2d(sb + 3 * G_BOX, mb, fb, kx, tj * GT + 128);
                if (++stage == G_STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = 0; it < iters; ++it) {
                mbar_wait_u32(smem_u32(&full[stage]), phase);
                tc_fence_after();
                const uint32_t sb = base + stage * G_STAGE;
                const uint64_t da0 = sw128_desc(sb), da1 = sw128_desc(sb + G_BOX), db = sw128_desc(sb + 2 * G_BOX);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {   // 16 rows of X (32 bytes of K) per MMA
                    const uint32_t acc = (it | kk) != 0;
                    mma_f16(tmem, da0 + 2 * kk, db + 2 * kk, G_IDESC, acc);
                    mma_f16(tmem + 256, da1 + 2 * kk, db + 2 * kk, G_IDESC, acc);
                }
                mma_commit(smem_u32(&empty[stage]));
                if (++stage == G_STAGES) { stage = 0; phase ^= 1; }
            }
            mma_commit(smem_u32(done));
        }
    } else {
        const int quarter = warp & 3;
        mbar_wait_u32(smem_u32(done), 0);
        tc_fence_after();
        const double unscale = ldexp(1.0, -2 * (*e_ptr));
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            const int a = ti * GT + half * 128 + quarter * 32 + lane;
#pragma unroll 1
            for (int ch = 0; ch < GT / 32; ++ch) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + half * 256 + ch * 32, v);
                if (a >= d) continue;
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int b = tj * GT + ch * 32 + c;
                    if (b < d) {
                        const double x = (double)v[c] * unscale;
                        atomicAdd(&G[(int64_t)a * d + b], x);
                        if (ti != tj) atomicAdd(&G[(int64_t)b * d + a], x);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

bool make_map_t(CUtensorMap *m, const __half *ptr, int d, int64_t ldt) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)ldt, (cuuint64_t)d};
    cuuint64_t strides[1] = {(cuuint64_t)ldt * 2};
    cuuint32_t box[2] = {(cuuint32_t)GKR, 128};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half *>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t gram_tc_scratch_bytes(int64_t n, int d) {
    const int64_t ldt = round_up(n, 8);
    return (size_t)2 * d * ldt * sizeof(__half) + 256;
}

bool launch_gram_tc(const void *X, bool f64, int64_t n, int d, int64_t rs, const uint32_t *maxabs_bits,
                    double xc_bound, const float *mu_f, double *G, void *scratch, int sm_count, cudaStream_t s) {
    if (n == 0) return true;
    const int64_t ldt = round_up(n, 8);
    uint8_t *p = static_cast<uint8_t *>(scratch);
    int *e_dev = reinterpret_cast<int *>(p);
    __half *XT_h = reinterpret_cast<__half *>(p + 256);
    __half *XT_l = XT_h + (int64_t)d * ldt;
    CUtensorMap mh, ml;
    if (!make_map_t(&mh, XT_h, d, ldt) || !make_map_t(&ml, XT_l, d, ldt)) return false;
    SNN_LAUNCH(gram_scale_kernel, 1, 32, 0, s, d, maxabs_bits, mu_f, xc_bound, e_dev);
    dim3 tg((unsigned)ceil_div(ldt, 128), (unsigned)ceil_div(d, 64));
    if (f64) SNN_LAUNCH(gram_transpose_split<double>, tg, 256, 0, s, (const double *)X, n, d, rs, ldt, mu_f, e_dev, XT_h, XT_l);
    else SNN_LAUNCH(gram_transpose_split<float>, tg, 256, 0, s, (const float *)X, n, d, rs, ldt, mu_f, e_dev, XT_h, XT_l);
    const int nt = (int)ceil_div(d, GT);
    const int tiles = nt * (nt + 1) / 2;
    const int64_t nkb = ceil_div(ldt, GKR);
    int64_t splits = ceil_div(sm_count, tiles);
    if (splits > nkb) splits = nkb;
    if (splits < 1) splits = 1;
    const int64_t kps = ceil_div(nkb, splits);
    splits = ceil_div(nkb, kps);
    cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, G_SMEM);
    SNN_LAUNCH(gram_tc_kernel, dim3((unsigned)tiles, (unsigned)splits), G_THREADS, G_SMEM, s, mh, ml, d, nkb, kps, nt,
               e_dev, G);
    return true;
}

}  // namespace snn
