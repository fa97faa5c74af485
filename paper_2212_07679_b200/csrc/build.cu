// build.cu -- index-build kernels of Algorithm 1 "SNN Index".
//
//  K1  column statistics : mean (Alg. 1 l.2) in fp64, max |x| per column
//                          (feeds the rigorous key error bound, reading C8),
//                          NaN/Inf detection.
//  K2a Gram matrix       : G = sum_i (p_i - mu)(p_i - mu)^T, whose top eigenvector is the
//                          first right singular vector v1 of the centered X (eq:svd,
//                          PAPER.md:94-108; Alg. 1 l.4).
//  K2b power iteration   : v1 of G in fp64 (reading C9: start = normalised column-variance
//                          vector; small d accelerated by repeated squaring of G).
//  K3  projection keys   : alpha_i = x_i^T v1 (Alg. 1 l.5).
//  K5  gather + norms    : X permuted into key order (Alg. 1 l.6) with the half squared
//                          norms xbar_i = x_i^T x_i / 2 (Alg. 1 l.7).
// The sort itself (Alg. 1 l.6) is radix_sort.cu.
#include <float.h>
#include <math.h>

#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace snn {
namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float abs_ru(float v) { return fabsf(v); }
__device__ __forceinline__ float abs_ru(double v) { return __double2float_ru(fabs(v)); }
__device__ __forceinline__ bool finite_(float v) { return isfinite(v); }
__device__ __forceinline__ bool finite_(double v) { return isfinite(v); }

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------------------------ K1
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) colstats_small(const T *__restrict__ X, int64_t n,
                                                           double *sums, uint32_t *maxabs,
                                                           int *nonfinite) {
    double s[D];
    float mx[D];
#pragma unroll
    for (int k = 0; k < D; ++k) { s[k] = 0.0; mx[k] = 0.f; }
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            T v = X[i * D + k];
            bad |= !finite_(v);
            s[k] += (double)v;
            mx[k] = fmaxf(mx[k], abs_ru(v));
        }
    }
    __shared__ double ssum[kThreads / kWarp][D];
    __shared__ float smax[kThreads / kWarp][D];
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        double a = warp_sum(s[k]);
        float b = warp_max(mx[k]);
        if (l == 0) { ssum[w][k] = a; smax[w][k] = b; }
    }
    if (__any_sync(0xffffffffu, bad) && l == 0) atomicOr(nonfinite, 1);
    __syncthreads();
    if (threadIdx.x < D) {
        double a = 0.0;
        float b = 0.f;
        for (int j = 0; j < kThreads / kWarp; ++j) { a += ssum[j][threadIdx.x]; b = fmaxf(b, smax[j][threadIdx.x]); }
        atomicAdd(&sums[threadIdx.x], a);
        atomicMax(&maxabs[threadIdx.x], __float_as_uint(b));
    }
}

// any d: block = a range of rows, threads over columns (coalesced along a row)
template <typename T>
__global__ void __launch_bounds__(kThreads) colstats_generic(const T *__restrict__ X, int64_t n,
                                                             int d, int64_t rows_per_block,
                                                             double *sums, uint32_t *maxabs,
                                                             int *nonfinite) {
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    bool bad = false;
    for (int c = threadIdx.x; c < d; c += kThreads) {
        double s = 0.0;
        float mx = 0.f;
        for (int64_t r = r0; r < r1; ++r) {
            T v = X[r * d + c];
            bad |= !finite_(v);
            s += (double)v;
            mx = fmaxf(mx, abs_ru(v));
        }
        if (r1 > r0) {
            atomicAdd(&sums[c], s);
            atomicMax(&maxabs[c], __float_as_uint(mx));
        }
    }
    if (bad) atomicOr(nonfinite, 1);
}

__global__ void finalize_mean(const double *sums, int64_t n, int d, double *mu_d, float *mu_f) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double m = sums[k] / (double)n;
        mu_d[k] = m;
        mu_f[k] = (float)m;
    }
}

// ------------------------------------------------------------------------------ K2a
template <typename T>
__device__ __forceinline__ float centered(T v, float mu) {
    return (float)v - mu;   // fp32 path: exact widening, one rounding
}
template <>
__device__ __forceinline__ float centered<double>(double v, float mu) {
    return (float)(v - (double)mu);
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads) gram_small(const T *__restrict__ X, int64_t n,
                                                       const float *__restrict__ mu_f,
                                                       double *G) {
    constexpr int P = D * (D + 1) / 2;
    float acc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = 0.f;
    float mu[D];
#pragma unroll
    for (int k = 0; k < D; ++k) mu[k] = mu_f[k];
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        float c[D];
#pragma unroll
        for (int k = 0; k < D; ++k) c[k] = centered(X[i * D + k], mu[k]);
        int p = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b) { acc[p] = fmaf(c[a], c[b], acc[p]); ++p; }
    }
    __shared__ double sred[kThreads / kWarp][P];
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        double v = warp_sum((double)acc[p]);
        if (l == 0) sred[w][p] = v;
    }
    __syncthreads();
    if (threadIdx.x < P) {
        double v = 0.0;
        for (int j = 0; j < kThreads / kWarp; ++j) v += sred[j][threadIdx.x];
        // map p -> (a, b)
        int p = threadIdx.x, a = 0;
        while (p >= D - a) { p -= D - a; ++a; }
        int b = a + p;
        atomicAdd(&G[a * D + b], v);
        if (a != b) atomicAdd(&G[b * D + a], v);
    }
}

// any d: 64 x 64 output tiles of the upper triangle, split-K over row chunks.
constexpr int kGT = 64, kGR = 32, kGChunk = 2048;
template <typename T>
__global__ void __launch_bounds__(kThreads) gram_tiled(const T *__restrict__ X, int64_t n, int d,
                                                       const float *__restrict__ mu_f, double *G) {
    // linear upper-triangle tile index -> (ti, tj), ti <= tj
    const int nt = (d + kGT - 1) / kGT;
    int t = blockIdx.x, ti = 0;
    while (t >= nt - ti) { t -= nt - ti; ++ti; }
    const int tj = ti + t;
    const int64_t r0 = (int64_t)blockIdx.y * kGChunk;
    const int64_t r1 = min(n, r0 + kGChunk);
    __shared__ float A[kGR][kGT + 4];
    __shared__ float B[kGR][kGT + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4] = {};
    for (int64_t rb = r0; rb < r1; rb += kGR) {
        for (int e = threadIdx.x; e < kGR * kGT; e += kThreads) {
            int r = e / kGT, c = e % kGT;
            int64_t row = rb + r;
            int ca = ti * kGT + c, cb = tj * kGT + c;
            A[r][c] = (row < r1 && ca < d) ? centered(X[row * d + ca], mu_f[ca]) : 0.f;
            B[r][c] = (row < r1 && cb < d) ? centered(X[row * d + cb], mu_f[cb]) : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < kGR; ++r) {
            float4 a = *reinterpret_cast<const float4 *>(&A[r][ty * 4]);
            float4 b = *reinterpret_cast<const float4 *>(&B[r][tx * 4]);
            float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int a = ti * kGT + ty * 4 + i, b = tj * kGT + tx * 4 + j;
            if (a < d && b < d) {
                atomicAdd(&G[(int64_t)a * d + b], (double)acc[i][j]);
                if (ti != tj) atomicAdd(&G[(int64_t)b * d + a], (double)acc[i][j]);
            }
        }
}

// ------------------------------------------------------------------------------ K2b
// Small d (<= 16): one warp; lane i holds row i of M.  M <- G/max|G|, then K squarings
// M <- M*M / max|M| (power iteration on G^(2^K)), v = column of M with the largest
// diagonal, then `polish` plain power iterations on G.
template <int D>
__global__ void power_small(const double *__restrict__ G, int max_iters, double *v_out,
                            double *stats) {
    const int l = threadIdx.x;
    double m[D];
#pragma unroll
    for (int j = 0; j < D; ++j) m[j] = (l < D) ? G[l * D + j] : 0.0;
    double gmax = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) gmax = fmax(gmax, fabs(m[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    if (gmax == 0.0) {     // all-zero centered data: v1 = e1 (reading C9)
        if (l < D) v_out[l] = (l == 0) ? 1.0 : 0.0;
        if (l == 0) { stats[ST_SIGMA1] = 0.0; stats[ST_ITERS] = 0.0; }
        return;
    }
    const int squarings = max_iters >= 64 ? 24 : 0;
#pragma unroll
    for (int j = 0; j < D; ++j) m[j] /= gmax;
    int done_sq = 0;
    for (int it = 0; it < squarings; ++it) {
        ++done_sq;
        double r[D];
#pragma unroll
        for (int j = 0; j < D; ++j) r[j] = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int j = 0; j < D; ++j) r[j] = fma(m[k], __shfl_sync(0xffffffffu, m[j], k), r[j]);
        double mx = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) mx = fmax(mx, fabs(r[j]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (!(mx > 0.0)) break;
        double ch = 0.0;   // converged to the rank-1 projector: stop squaring early
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double nm = (l < D) ? r[j] / mx : 0.0;
            ch = fmax(ch, fabs(nm - m[j]));
            m[j] = nm;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ch = fmax(ch, __shfl_xor_sync(0xffffffffu, ch, o));
        if (ch < 1e-15) break;
    }
    // column with the largest diagonal entry (lowest index on ties)
    double diag = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) if (j == l) diag = m[j];
    int best = 0;
    double bestv = __shfl_sync(0xffffffffu, diag, 0);
    for (int j = 1; j < D; ++j) {
        double dj = __shfl_sync(0xffffffffu, diag, j);
        if (dj > bestv) { bestv = dj; best = j; }
    }
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) if (j == best) v = m[j];   // lane l: M[l][best]
    if (l >= D) v = 0.0;
    if (squarings == 0) v = (l < D) ? G[l * D + l] : 0.0;   // plain start: column variances
    double nv = warp_sum(v * v);
    if (!(nv > 0.0)) { v = (l == best) ? 1.0 : 0.0; nv = 1.0; }
    v /= sqrt(nv);
    // polish with plain power iterations on G
    double g[D];
#pragma unroll
    for (int j = 0; j < D; ++j) g[j] = (l < D) ? G[l * D + j] : 0.0;
    int iters = done_sq;
    const int polish = squarings ? 4 : max_iters;
    for (int it = 0; it < polish; ++it) {
        double y = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) y = fma(g[j], __shfl_sync(0xffffffffu, v, j), y);
        double ny = warp_sum(y * y);
        if (!(ny > 0.0)) break;
        y /= sqrt(ny);
        double diff = warp_sum((y - v) * (y - v));
        v = y;
        ++iters;
        if (diff < 1e-28) break;
    }
    double gv = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) gv = fma(g[j], __shfl_sync(0xffffffffu, v, j), gv);
    double lam = warp_sum(v * gv);
    if (l < D) v_out[l] = v;
    if (l == 0) { stats[ST_SIGMA1] = sqrt(fmax(lam, 0.0)); stats[ST_ITERS] = (double)iters; }
}

__device__ double block_sum_1024(double v, double *red) {
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
    v = warp_sum(v);
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = (l < (int)(blockDim.x / kWarp)) ? red[l] : 0.0;
    return warp_sum(t);
}

// Any d: one CTA of 1024 threads; warp-per-row matvec y = G v (G from L2).
__global__ void __launch_bounds__(1024) power_generic(const double *__restrict__ G, int d,
                                                      int max_iters, double tol, double *v_out,
                                                      double *stats) {
    extern __shared__ double sm[];
    double *v = sm, *y = sm + d;
    __shared__ double red[32];
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp, nw = blockDim.x / kWarp;
    double loc = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) { v[i] = G[(int64_t)i * d + i]; loc += v[i] * v[i]; }
    double nrm = block_sum_1024(loc, red);
    int iters = 0;
    if (!(nrm > 0.0)) {
        for (int i = threadIdx.x; i < d; i += blockDim.x) v_out[i] = (i == 0) ? 1.0 : 0.0;
        if (threadIdx.x == 0) { stats[ST_SIGMA1] = 0.0; stats[ST_ITERS] = 0.0; }
        return;
    }
    double inv = 1.0 / sqrt(nrm);
    for (int i = threadIdx.x; i < d; i += blockDim.x) v[i] *= inv;
    __syncthreads();
    bool restarted = false;
    for (int it = 0; it < max_iters; ++it) {
        for (int row = w; row < d; row += nw) {
            double s = 0.0;
            const double *g = G + (int64_t)row * d;
            for (int j = l; j < d; j += kWarp) s = fma(g[j], v[j], s);
            s = warp_sum(s);
            if (l == 0) y[row] = s;
        }
        __syncthreads();
        loc = 0.0;
        for (int i = threadIdx.x; i < d; i += blockDim.x) loc += y[i] * y[i];
        double ny = block_sum_1024(loc, red);
        if (!(ny > 0.0)) {
            if (restarted) break;
            restarted = true;    // start vector in the null space: restart at e_argmax(diag)
            __syncthreads();
            if (threadIdx.x == 0) {
                int best = 0;
                for (int i = 1; i < d; ++i) if (G[(int64_t)i * d + i] > G[(int64_t)best * d + best]) best = i;
                for (int i = 0; i < d; ++i) v[i] = (i == best) ? 1.0 : 0.0;
            }
            __syncthreads();
            continue;
        }
        inv = 1.0 / sqrt(ny);
        loc = 0.0;
        for (int i = threadIdx.x; i < d; i += blockDim.x) { double t = y[i] * inv - v[i]; loc += t * t; }
        double diff = block_sum_1024(loc, red);
        for (int i = threadIdx.x; i < d; i += blockDim.x) v[i] = y[i] * inv;
        __syncthreads();
        iters = it + 1;
        if (diff <= tol * tol) break;
    }
    // Rayleigh quotient for sigma1
    for (int row = w; row < d; row += nw) {
        double s = 0.0;
        const double *g = G + (int64_t)row * d;
        for (int j = l; j < d; j += kWarp) s = fma(g[j], v[j], s);
        s = warp_sum(s);
        if (l == 0) y[row] = s;
    }
    __syncthreads();
    loc = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) loc += v[i] * y[i];
    double lam = block_sum_1024(loc, red);
    for (int i = threadIdx.x; i < d; i += blockDim.x) v_out[i] = v[i];
    if (threadIdx.x == 0) { stats[ST_SIGMA1] = sqrt(fmax(lam, 0.0)); stats[ST_ITERS] = (double)iters; }
}

// Any d (17..16384): many CTAs, one grid barrier per iteration (cooperative launch).
// Rows of G are split across the CTAs; every CTA keeps its own copy of v in shared
// memory and forms the next v from the gathered y = G v, so the normalisation and the
// convergence test (same data, same order in every CTA) are identical grid-wide.
__device__ double block_sum_256(double v, double *red) {
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
    v = warp_sum(v);
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = (l < (int)(blockDim.x / kWarp)) ? red[l] : 0.0;
    return warp_sum(t);
}

__global__ void __launch_bounds__(256) power_coop(const double *__restrict__ G, int d, int max_iters, double tol,
                                                  double *ybuf, double *part, double *v_out, double *stats) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sv[];   // v (d)
    __shared__ double red[8];
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
    const int rpc = (d + (int)gridDim.x - 1) / (int)gridDim.x;
    const int r0 = blockIdx.x * rpc, r1 = min(d, r0 + rpc);
    double loc = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) { sv[i] = G[(int64_t)i * d + i]; loc += sv[i] * sv[i]; }
    const double nrm = block_sum_256(loc, red);
    if (!(nrm > 0.0)) {   // all-zero centred data: v1 = e1 (reading C9)
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < d; i += blockDim.x) v_out[i] = (i == 0) ? 1.0 : 0.0;
            if (threadIdx.x == 0) { stats[ST_SIGMA1] = 0.0; stats[ST_ITERS] = 0.0; }
        }
        return;
    }
    double inv = 1.0 / sqrt(nrm);
    for (int i = threadIdx.x; i < d; i += blockDim.x) sv[i] *= inv;
    __syncthreads();
    bool restarted = false;
    int iters = 0;
    for (int it = 0; it < max_iters; ++it) {
        double *y = ybuf + (it & 1) * d;
        double *pb = part + (it & 1) * gridDim.x;
        for (int row = r0 + w; row < r1; row += blockDim.x / kWarp) {
            double sacc = 0.0;
            const double *g = G + (int64_t)row * d;
            for (int j = l; j < d; j += kWarp) sacc = fma(g[j], sv[j], sacc);
            sacc = warp_sum(sacc);
            if (l == 0) y[row] = sacc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double ps = 0.0;
            for (int row = r0; row < r1; ++row) ps += y[row] * y[row];
            pb[blockIdx.x] = ps;
        }
        grid.sync();
        loc = 0.0;
        for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) loc += __ldcg(&pb[c]);
        const double ny = block_sum_256(loc, red);
        if (!(ny > 0.0)) {
            if (restarted) break;
            restarted = true;    // start vector in the null space: restart at e_argmax(diag)
            int best = 0;
            for (int i = 1; i < d; ++i) if (G[(int64_t)i * d + i] > G[(int64_t)best * d + best]) best = i;
            for (int i = threadIdx.x; i < d; i += blockDim.x) sv[i] = (i == best) ? 1.0 : 0.0;
            __syncthreads();
            continue;
        }
        inv = 1.0 / sqrt(ny);
        loc = 0.0;
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            const double t = __ldcg(&y[i]) * inv - sv[i];
            loc += t * t;
        }
        const double diff = block_sum_256(loc, red);
        for (int i = threadIdx.x; i < d; i += blockDim.x) sv[i] = __ldcg(&y[i]) * inv;
        __syncthreads();
        iters = it + 1;
        if (diff <= tol * tol) break;
    }
    // Rayleigh quotient for sigma1: lambda = v^T G v (partials per CTA, fixed order)
    double *pb = part + 2 * gridDim.x;
    double rq = 0.0;
    for (int row = r0 + w; row < r1; row += blockDim.x / kWarp) {
        double sacc = 0.0;
        const double *g = G + (int64_t)row * d;
        for (int j = l; j < d; j += kWarp) sacc = fma(g[j], sv[j], sacc);
        sacc = warp_sum(sacc);
        if (l == 0) rq += sv[row] * sacc;
    }
    const double rqs = block_sum_256(rq, red);
    if (threadIdx.x == 0) pb[blockIdx.x] = rqs;
    grid.sync();
    if (blockIdx.x == 0) {
        loc = 0.0;
        for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) loc += __ldcg(&pb[c]);
        const double lam = block_sum_256(loc, red);
        for (int i = threadIdx.x; i < d; i += blockDim.x) v_out[i] = sv[i];
        if (threadIdx.x == 0) { stats[ST_SIGMA1] = sqrt(fmax(lam, 0.0)); stats[ST_ITERS] = (double)iters; }
    }
}

// Sign fix (largest |entry| positive, lowest index on ties), fp32 copy, ||v||, E_x.
__global__ void finalize_direction(int d, const uint32_t *maxabs_bits, const double *mu_d,
                                   const float *mu_f, double *v_d, float *v_f, double *stats) {
    // largest |entry| (lowest index on ties): warp-parallel argmax
    double bv = -1.0;
    int bi = 0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const double a = fabs(v_d[i]);
        if (a > bv) { bv = a; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const double sgn = (v_d[bi] < 0.0) ? -1.0 : 1.0;
    double nf = 0.0, nd = 0.0, ef = 0.0, ed = 0.0, xc = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double vd = v_d[i] * sgn;
        v_d[i] = vd;
        float vf = (float)vd;
        v_f[i] = vf;
        nf += (double)vf * (double)vf;
        nd += vd * vd;
        double mx = (double)__uint_as_float(maxabs_bits[i]);
        ef += (mx + fabs((double)mu_f[i])) * fabs((double)vf);
        ed += (mx + fabs(mu_d[i])) * fabs(vd);
        xc = fmax(xc, mx + fabs((double)mu_f[i]));
    }
    nf = warp_sum(nf); nd = warp_sum(nd); ef = warp_sum(ef); ed = warp_sum(ed);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xc = fmax(xc, __shfl_xor_sync(0xffffffffu, xc, o));
    if (threadIdx.x == 0) {
        const double u = 5.9604644775390625e-08;  // 2^-24
        const double g = 2.0 * (d + 2) * u;
        stats[ST_WNORM_F] = sqrt(nf) * (1.0 + 1e-12);
        stats[ST_WNORM_D] = sqrt(nd) * (1.0 + 1e-12);
        stats[ST_EX_F] = g * ef * (1.0 + 1e-10) + 1e-30;
        stats[ST_EX_D] = g * ed * (1.0 + 1e-10) + 1e-30;
        stats[ST_XCMAX] = xc;
    }
}

__global__ void query_key_err(int d, bool f64, const uint32_t *maxabs_bits, const double *mu_d,
                              const float *mu_f, const double *v_d, const float *v_f, double *eq) {
    double e = 0.0, xc = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double mx = (double)__uint_as_float(maxabs_bits[i]);
        e += f64 ? (mx + fabs(mu_d[i])) * fabs(v_d[i])
                 : (mx + fabs((double)mu_f[i])) * fabs((double)v_f[i]);
        xc = fmax(xc, mx + fabs((double)mu_f[i]));
    }
    e = warp_sum(e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xc = fmax(xc, __shfl_xor_sync(0xffffffffu, xc, o));
    if (threadIdx.x == 0) {
        eq[0] = 2.0 * (d + 2) * 5.9604644775390625e-08 * e * (1.0 + 1e-10) + 1e-30;
        eq[1] = xc;
    }
}

// ------------------------------------------------------------------------------ K3
template <int D>
__global__ void __launch_bounds__(kThreads) keys_small_f32(const float *__restrict__ X, int64_t n,
                                                           const float *__restrict__ mu_f,
                                                           const float *__restrict__ v_f,
                                                           float *keys) {
    float mu[D], v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) { mu[k] = mu_f[k]; v[k] = v_f[k]; }
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fmaf(X[i * D + k] - mu[k], v[k], s);
        keys[i] = s;
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads) keys_small_f64(const double *__restrict__ X, int64_t n,
                                                           const double *__restrict__ mu_d,
                                                           const double *__restrict__ v_d,
                                                           float *keys) {
    double mu[D], v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) { mu[k] = mu_d[k]; v[k] = v_d[k]; }
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(X[i * D + k] - mu[k], v[k], s);
        keys[i] = (float)s;
    }
}

// any d: warp per row
template <typename T>
__global__ void __launch_bounds__(kThreads) keys_generic(const T *__restrict__ X, int64_t n, int d,
                                                         const double *__restrict__ mu_d,
                                                         const float *__restrict__ mu_f,
                                                         const double *__restrict__ v_d,
                                                         const float *__restrict__ v_f,
                                                         float *keys) {
    const int l = threadIdx.x % kWarp;
    for (int64_t i = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / kWarp; i < n;
         i += (int64_t)gridDim.x * kThreads / kWarp) {
        const T *x = X + i * d;
        if constexpr (sizeof(T) == 4) {
            float s = 0.f;
            for (int k = l; k < d; k += kWarp) s = fmaf(x[k] - mu_f[k], v_f[k], s);
            s = warp_sum(s);
            if (l == 0) keys[i] = s;
        } else {
            double s = 0.0;
            for (int k = l; k < d; k += kWarp) s = fma(x[k] - mu_d[k], v_d[k], s);
            s = warp_sum(s);
            if (l == 0) keys[i] = (float)s;
        }
    }
}

// ------------------------------------------------------------------------------ K5
template <typename T, int D, int LD>
__global__ void __launch_bounds__(kThreads) gather_small(const T *__restrict__ X, int64_t n,
                                                         int64_t n_pad,
                                                         const uint32_t *__restrict__ perm,
                                                         const double *__restrict__ mu_d,
                                                         T *__restrict__ Xs, float *xbar) {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n_pad;
         i += (int64_t)gridDim.x * kThreads) {
        T row[LD];
        double h = 0.0;
        if (i < n) {
            const int64_t src = perm[i];
#pragma unroll
            for (int k = 0; k < D; ++k) {
                row[k] = X[src * D + k];
                double t = (double)row[k] - mu_d[k];
                h = fma(t, t, h);
            }
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) row[k] = (T)NAN;   // sentinel: every comparison false
            h = NAN;
        }
#pragma unroll
        for (int k = D; k < LD; ++k) row[k] = (T)0;
        if constexpr (sizeof(T) * LD == 16) {
            *reinterpret_cast<int4 *>(Xs + i * LD) = *reinterpret_cast<const int4 *>(row);
        } else if constexpr (sizeof(T) * LD == 8) {
            *reinterpret_cast<int2 *>(Xs + i * LD) = *reinterpret_cast<const int2 *>(row);
        } else {
#pragma unroll
            for (int k = 0; k < LD; ++k) Xs[i * LD + k] = row[k];
        }
        if (xbar) xbar[i] = (float)(0.5 * h);
    }
}

// AoSoA4 layout for the low-d query kernel: rows are grouped by 4; group g stores
// coordinate k of its 4 rows contiguously: Xs[g*4*D + k*4 + r].  A chunk of candidates
// starting at a multiple of 4 rows is one contiguous byte range (bulk-copy friendly) and
// each coordinate of 4 consecutive candidates is one 16-byte shared-memory vector.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) gather_aosoa4(const T *__restrict__ X, int64_t n,
                                                          int64_t n_pad,
                                                          const uint32_t *__restrict__ perm,
                                                          const double *__restrict__ mu_d,
                                                          T *__restrict__ Xs, float *xbar) {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n_pad;
         i += (int64_t)gridDim.x * kThreads) {
        const int64_t g = i >> 2, r = i & 3;
        double h = 0.0;
        if (i < n) {
            const int64_t src = perm[i];
#pragma unroll
            for (int k = 0; k < D; ++k) {
                T v = X[src * D + k];
                Xs[g * 4 * D + k * 4 + r] = v;
                double t = (double)v - mu_d[k];
                h = fma(t, t, h);
            }
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) Xs[g * 4 * D + k * 4 + r] = (T)NAN;   // never a hit
            h = NAN;
        }
        if (xbar) xbar[i] = (float)(0.5 * h);
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) gather_generic(const T *__restrict__ X, int64_t n,
                                                           int d, int ld, int64_t n_pad,
                                                           const uint32_t *__restrict__ perm,
                                                           const double *__restrict__ mu_d,
                                                           T *__restrict__ Xs, float *xbar) {
    const int l = threadIdx.x % kWarp;
    for (int64_t i = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / kWarp; i < n_pad;
         i += (int64_t)gridDim.x * kThreads / kWarp) {
        double h = 0.0;
        if (i < n) {
            const T *x = X + (int64_t)perm[i] * d;
            for (int k = l; k < ld; k += kWarp) {
                T v = (k < d) ? x[k] : (T)0;
                Xs[i * ld + k] = v;
                if (k < d) { double t = (double)v - mu_d[k]; h = fma(t, t, h); }
            }
            h = warp_sum(h);
        } else {
            for (int k = l; k < ld; k += kWarp) Xs[i * ld + k] = (k < d) ? (T)NAN : (T)0;
            h = NAN;
        }
        if (l == 0 && xbar) xbar[i] = (float)(0.5 * h);
    }
}

// inverse of K5's layout (streaming append): rows [0, n) of Xs back to row-major n x d
template <typename T>
__global__ void unpack_rows(const T *__restrict__ Xs, int64_t n, int d, int ld, T *__restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * d; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d;
        const int k = (int)(e - i * d);
        out[e] = ld == 0 ? Xs[(i >> 2) * 4 * d + k * 4 + (i & 3)] : Xs[i * ld + k];
    }
}

// streaming append: sorted position -> original id from the merge sort's source rows
__global__ void append_perm(const uint32_t *__restrict__ src, int64_t n_old, int64_t n_new,
                            const int32_t *__restrict__ perm_old, int32_t *__restrict__ perm_new) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_new; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = src[i];
        perm_new[i] = r < n_old ? perm_old[r] : (int32_t)r;
    }
}

int grid_for(int64_t items, int per_block = kThreads, int cap = 148 * 16) {
    int64_t g = ceil_div(items, per_block);
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

}  // namespace

// ================================================================================ launchers
#define SNN_SMALL_D_CASES(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)

void launch_colstats(const void *X, bool f64, int64_t n, int d, double *sums,
                     uint32_t *maxabs_bits, int *nonfinite, cudaStream_t s) {
    if (n == 0) return;
    const int g = grid_for(n);
#define CASE(D)                                                                               \
    case D:                                                                                   \
        if (f64) SNN_LAUNCH((colstats_small<double, D>), g, kThreads, 0, s, (const double *)X, n, sums, maxabs_bits, nonfinite); \
        else SNN_LAUNCH((colstats_small<float, D>), g, kThreads, 0, s, (const float *)X, n, sums, maxabs_bits, nonfinite); \
        return;
    switch (d) { SNN_SMALL_D_CASES(CASE) default: break; }
#undef CASE
    const int64_t blocks = 148 * 8;
    const int64_t rpb = ceil_div(n, blocks);
    const int gb = (int)ceil_div(n, rpb);
    if (f64) SNN_LAUNCH(colstats_generic<double>, gb, kThreads, 0, s, (const double *)X, n, d, rpb, sums, maxabs_bits, nonfinite);
    else SNN_LAUNCH(colstats_generic<float>, gb, kThreads, 0, s, (const float *)X, n, d, rpb, sums, maxabs_bits, nonfinite);
}

namespace {
__global__ void scale_f64_kernel(double *x, int64_t count, double f) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= f;
}
}  // namespace

namespace {
__global__ void set_f64_kernel(double *x, double v) { *x = v; }
__global__ void readback_kernel(uint8_t *dst, const uint8_t *src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

// Small device -> host readbacks (sizes, counts, flags) as kernel stores into mapped pinned
// memory instead of cudaMemcpyAsync: a copy would queue on the device-to-host copy engine
// behind any large transfer in flight (e.g. the previous result's copy-out on another
// stream), stalling the whole call until that transfer ends.
__global__ void readback_batch_kernel(ReadbackBatch b) {
    for (int e = 0; e < b.n; ++e) {
        uint8_t *dst = static_cast<uint8_t *>(b.dst[e]);
        const uint8_t *src = static_cast<const uint8_t *>(b.src[e]);
        for (int i = threadIdx.x; i < b.bytes[e]; i += blockDim.x) dst[i] = src[i];
    }
}

// several small readbacks in one launch (the destinations' device aliases resolved here)
cudaError_t small_readback_batch(ReadbackBatch b, cudaStream_t s) {
    if (b.n == 0) return cudaSuccess;
    for (int e = 0; e < b.n; ++e) {
        void *dptr = nullptr;
        if (b.bytes[e] > 4096 || cudaHostGetDevicePointer(&dptr, b.dst[e], 0) != cudaSuccess) {
            cudaGetLastError();   // not mapped pinned memory: one copy per entry
            for (int f = 0; f < b.n; ++f) {
                cudaError_t x = cudaMemcpyAsync(b.dst[f], b.src[f], (size_t)b.bytes[f], cudaMemcpyDeviceToHost, s);
                if (x != cudaSuccess) return x;
            }
            return cudaSuccess;
        }
        b.dst[e] = dptr;
    }
    SNN_LAUNCH(readback_batch_kernel, 1, 128, 0, s, b);
    return cudaGetLastError();
}

cudaError_t small_readback(void *host, const void *dev, size_t bytes, cudaStream_t s) {
    void *dptr = nullptr;
    if (bytes > 4096 || cudaHostGetDevicePointer(&dptr, host, 0) != cudaSuccess) {
        cudaGetLastError();
        return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
    }
    SNN_LAUNCH(readback_kernel, 1, 128, 0, s, static_cast<uint8_t *>(dptr), static_cast<const uint8_t *>(dev), (int)bytes);
    return cudaGetLastError();
}

// one device scalar from a host value without a pageable copy (a pageable cudaMemcpyAsync
// waits behind transfers queued on the copy engines, e.g. a large copy-out on another stream)
void launch_set_f64(double *x, double v, cudaStream_t s) { SNN_LAUNCH(set_f64_kernel, 1, 1, 0, s, x, v); }

void launch_scale_f64(double *x, int64_t count, double f, cudaStream_t s) {
    if (count == 0) return;
    SNN_LAUNCH(scale_f64_kernel, grid_for(count, kThreads, 148 * 4), kThreads, 0, s, x, count, f);
}

void launch_finalize_mean(const double *sums, int64_t n, int d, double *mu_d, float *mu_f,
                          cudaStream_t s) {
    SNN_LAUNCH(finalize_mean, (int)ceil_div(d, 256), 256, 0, s, sums, n, d, mu_d, mu_f);
}

void launch_gram(const void *X, bool f64, int64_t n, int d, const float *mu_f, double *G,
                 cudaStream_t s) {
    if (n == 0) return;
    const int g = grid_for(n, kThreads, 148 * 4);
#define CASE(D)                                                                               \
    case D:                                                                                   \
        if (f64) SNN_LAUNCH((gram_small<double, D>), g, kThreads, 0, s, (const double *)X, n, mu_f, G); \
        else SNN_LAUNCH((gram_small<float, D>), g, kThreads, 0, s, (const float *)X, n, mu_f, G); \
        return;
    switch (d) { SNN_SMALL_D_CASES(CASE) default: break; }
#undef CASE
    const int nt = (int)ceil_div(d, kGT);
    dim3 grid(nt * (nt + 1) / 2, (unsigned)ceil_div(n, kGChunk));
    if (f64) SNN_LAUNCH(gram_tiled<double>, grid, kThreads, 0, s, (const double *)X, n, d, mu_f, G);
    else SNN_LAUNCH(gram_tiled<float>, grid, kThreads, 0, s, (const float *)X, n, d, mu_f, G);
}

size_t power_scratch_doubles(int d, int sm_count) { return (size_t)2 * d + 3 * (size_t)sm_count + 64; }

void launch_power_iteration(const double *G, int d, int max_iters, double tol,
                            const uint32_t *maxabs_bits, const double *mu_d, const float *mu_f,
                            double *v_d, float *v_f, double *stats, double *scratch, cudaStream_t s) {
    switch (d) {
#define CASE(D) case D: SNN_LAUNCH(power_small<D>, 1, 32, 0, s, G, max_iters, v_d, stats); break;
        SNN_SMALL_D_CASES(CASE)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default: {
            int grid = 0, dev = 0, nsm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            const size_t smem = (size_t)d * sizeof(double);
            if (d > 128 && d <= 16384 && scratch &&   // d <= 128: one CTA (power_generic) is faster than grid barriers
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&grid, power_coop, 256, smem) == cudaSuccess && grid > 0) {
                grid = nsm < d ? nsm : d;
                double *ybuf = scratch, *part = scratch + 2 * d;
                int mi = max_iters;
                double tl = tol;
                void *args[] = {(void *)&G, (void *)&d, (void *)&mi, (void *)&tl, (void *)&ybuf, (void *)&part,
                                (void *)&v_d, (void *)&stats};
                count_launch();
                if (smem > 48 * 1024) cudaFuncSetAttribute(power_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (cudaLaunchCooperativeKernel((const void *)power_coop, grid, 256, args, smem, s) == cudaSuccess) break;
                cudaGetLastError();
            }
            SNN_LAUNCH(power_generic, 1, 1024, (size_t)2 * d * sizeof(double), s, G, d, max_iters,
                       tol, v_d, stats);
        }
    }
    SNN_LAUNCH(finalize_direction, 1, 32, 0, s, d, maxabs_bits, mu_d, mu_f, v_d, v_f, stats);
}

void launch_query_key_err(int d, bool f64, const uint32_t *maxabs_bits, const double *mu_d,
                          const float *mu_f, const double *v_d, const float *v_f, double *eq,
                          cudaStream_t s) {
    SNN_LAUNCH(query_key_err, 1, 32, 0, s, d, f64, maxabs_bits, mu_d, mu_f, v_d, v_f, eq);
}

void launch_keys(const void *X, bool f64, int64_t n, int d, const double *mu_d,
                 const float *mu_f, const double *v_d, const float *v_f, float *keys,
                 cudaStream_t s) {
    if (n == 0) return;
    const int g = grid_for(n);
#define CASE(D)                                                                               \
    case D:                                                                                   \
        if (f64) SNN_LAUNCH(keys_small_f64<D>, g, kThreads, 0, s, (const double *)X, n, mu_d, v_d, keys); \
        else SNN_LAUNCH(keys_small_f32<D>, g, kThreads, 0, s, (const float *)X, n, mu_f, v_f, keys); \
        return;
    switch (d) { SNN_SMALL_D_CASES(CASE) default: break; }
#undef CASE
    const int gw = grid_for(n * kWarp);
    if (f64) SNN_LAUNCH(keys_generic<double>, gw, kThreads, 0, s, (const double *)X, n, d, mu_d, mu_f, v_d, v_f, keys);
    else SNN_LAUNCH(keys_generic<float>, gw, kThreads, 0, s, (const float *)X, n, d, mu_d, mu_f, v_d, v_f, keys);
}

void launch_gather(const void *X, bool f64, int64_t n, int d, int ld, int64_t n_pad,
                   const uint32_t *perm, const double *mu_d, void *Xs, float *xbar,
                   cudaStream_t s) {
    const int g = grid_for(n_pad);
    if (ld == 0) {   // AoSoA4 layout (low-d kernels)
#define CASE(D)                                                                               \
    case D:                                                                                   \
        if (f64) SNN_LAUNCH((gather_aosoa4<double, D>), g, kThreads, 0, s, (const double *)X, n, n_pad, perm, mu_d, (double *)Xs, xbar); \
        else SNN_LAUNCH((gather_aosoa4<float, D>), g, kThreads, 0, s, (const float *)X, n, n_pad, perm, mu_d, (float *)Xs, xbar); \
        return;
        switch (d) { SNN_SMALL_D_CASES(CASE) default: return; }
#undef CASE
    }
#define CASE(D, LD)                                                                           \
    if (d == D && ld == LD) {                                                                 \
        if (f64) SNN_LAUNCH((gather_small<double, D, LD>), g, kThreads, 0, s, (const double *)X, n, n_pad, perm, mu_d, (double *)Xs, xbar); \
        else SNN_LAUNCH((gather_small<float, D, LD>), g, kThreads, 0, s, (const float *)X, n, n_pad, perm, mu_d, (float *)Xs, xbar); \
        return;                                                                               \
    }
    CASE(1, 1) CASE(2, 2) CASE(3, 4) CASE(4, 4) CASE(5, 8) CASE(6, 8) CASE(7, 8) CASE(8, 8)
#undef CASE
    const int gw = grid_for(n_pad * kWarp);
    if (f64) SNN_LAUNCH(gather_generic<double>, gw, kThreads, 0, s, (const double *)X, n, d, ld, n_pad, perm, mu_d, (double *)Xs, xbar);
    else SNN_LAUNCH(gather_generic<float>, gw, kThreads, 0, s, (const float *)X, n, d, ld, n_pad, perm, mu_d, (float *)Xs, xbar);
}

void launch_unpack_rows(const void *Xs, bool f64, int64_t n, int d, int ld, void *out, cudaStream_t s) {
    if (n == 0) return;
    const int g = grid_for(n * d);
    if (f64) SNN_LAUNCH(unpack_rows<double>, g, kThreads, 0, s, (const double *)Xs, n, d, ld, (double *)out);
    else SNN_LAUNCH(unpack_rows<float>, g, kThreads, 0, s, (const float *)Xs, n, d, ld, (float *)out);
}

void launch_key_bounds(int d, const uint32_t *maxabs_bits, const double *mu_d, const float *mu_f, double *v_d,
                       float *v_f, double *stats, cudaStream_t s) {
    SNN_LAUNCH(finalize_direction, 1, 32, 0, s, d, maxabs_bits, mu_d, mu_f, v_d, v_f, stats);
}

void launch_append_perm(const uint32_t *src, int64_t n_old, int64_t n_new, const int32_t *perm_old, int32_t *perm_new,
                        cudaStream_t s) {
    SNN_LAUNCH(append_perm, grid_for(n_new), kThreads, 0, s, src, n_old, n_new, perm_old, perm_new);
}

namespace {
__device__ double spec_block_sum(double v, double *red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// Top-k eigenvalues of the stored Gram G = Xc^T Xc (d x d, fp64) by power iteration with
// deflation (y = G x - sum_l lambda_l (u_l . x) u_l), one CTA; sigma_l = sqrt(lambda_l) are
// the singular values of the centred data (eq:svd).  Diagnostic only:
// the search uses v1 from the build.  u: k x d scratch, x/y: d each.
__global__ void __launch_bounds__(1024) spectrum_kernel(const double *__restrict__ G, int d, int k, int max_iters,
                                                        double *u, double *x, double *y, double *sigma) {
    __shared__ double red[33];
    __shared__ double s_lam[16];
    for (int l = 0; l < k; ++l) {
        // start vector: deterministic, not orthogonal to any eigenvector in general
        for (int c = threadIdx.x; c < d; c += blockDim.x) x[c] = 1.0 + 0.37 * (double)((c * 7919) % 13) / 13.0;
        __syncthreads();
        double nx = sqrt(spec_block_sum([&] { double t = 0; for (int c = threadIdx.x; c < d; c += blockDim.x) t += x[c] * x[c]; return t; }(), red));
        for (int c = threadIdx.x; c < d; c += blockDim.x) x[c] /= nx;
        __syncthreads();
        double lam = 0.0, prev = -1.0;
        for (int it = 0; it < max_iters; ++it) {
            for (int r = threadIdx.x; r < d; r += blockDim.x) {
                double t = 0.0;
                for (int c = 0; c < d; ++c) t += G[(size_t)r * d + c] * x[c];
                y[r] = t;
            }
            __syncthreads();
            for (int p = 0; p < l; ++p) {   // deflate the eigenpairs found so far
                double t = 0.0;
                for (int c = threadIdx.x; c < d; c += blockDim.x) t += u[(size_t)p * d + c] * x[c];
                const double dp = spec_block_sum(t, red);
                for (int c = threadIdx.x; c < d; c += blockDim.x) y[c] -= s_lam[p] * dp * u[(size_t)p * d + c];
                __syncthreads();
            }
            double t1 = 0.0, t2 = 0.0;
            for (int c = threadIdx.x; c < d; c += blockDim.x) { t1 += x[c] * y[c]; t2 += y[c] * y[c]; }
            lam = spec_block_sum(t1, red);          // Rayleigh quotient (x unit)
            const double ny = sqrt(spec_block_sum(t2, red));
            if (!(ny > 0.0)) { lam = 0.0; break; }
            for (int c = threadIdx.x; c < d; c += blockDim.x) x[c] = y[c] / ny;
            __syncthreads();
            if (fabs(lam - prev) <= 1e-13 * fabs(lam)) break;
            prev = lam;
        }
        for (int c = threadIdx.x; c < d; c += blockDim.x) u[(size_t)l * d + c] = x[c];
        if (threadIdx.x == 0) {
            s_lam[l] = lam;
            sigma[l] = sqrt(fmax(lam, 0.0));
        }
        __syncthreads();
    }
}
}  // namespace

void launch_spectrum(const double *G, int d, int k, double *scratch, double *sigma, cudaStream_t s) {
    SNN_LAUNCH(spectrum_kernel, 1, 1024, 0, s, G, d, k, 2000, scratch, scratch + (size_t)k * d,
               scratch + (size_t)k * d + d, sigma);
}

}  // namespace snn
