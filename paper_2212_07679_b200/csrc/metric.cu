// metric.cu -- other distances on the Euclidean machinery.
// Cosine and angular distance:
// for unit vectors 2 cdist(u, v) = ||u - v||^2 and theta <= alpha iff
// ||u - v||^2 <= 2 - 2 cos(alpha), so both searches are exact Euclidean radius searches
// on normalized rows with a mapped radius.  The normalization is a fixed rule the oracle
// reproduces bit for bit: s = sum_k x_k^2 in fp64 left to right (no FMA), u_k =
// x_k / sqrt(s) (correctly rounded fp64 sqrt and division), rounded to the input dtype.
// Manhattan and inner-product similarity (MIPS transform):
// the exact Euclidean search returns a candidate superset (L2 <= L1; a radius covering
// xi^2 + |q|^2 - 2 tau), then an exact fp64 post-filter on the original rows keeps the hits.
#include <math.h>

#include "common.cuh"
#include "index.h"

namespace snn {
namespace {

template <typename T>
__global__ void normalize_rows_kernel(const T *__restrict__ X, int64_t n, int d, T *out, int *zero_flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T *x = X + i * d;
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = __dadd_rn(s, __dmul_rn((double)x[k], (double)x[k]));
        if (!(s > 0.0)) { atomicExch(zero_flag, 1); s = 1.0; }
        const double nrm = __dsqrt_rn(s);
        for (int k = 0; k < d; ++k) out[i * d + k] = (T)__ddiv_rn((double)x[k], nrm);
    }
}

__global__ void metric_distances_kernel(int metric, float *dist, int64_t nnz) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const double e = dist[i];
        dist[i] = metric == 1 ? (float)(0.5 * e * e) : (float)(2.0 * asin(fmin(1.0, 0.5 * e)));
    }
}

// MIPS transform: squared norms (fp64, left to right) and their maximum
// xi^2 (non-negative doubles order like their bit patterns)
template <typename T>
__global__ void sq_norms_kernel(const T *__restrict__ X, int64_t n, int d, double *nrm2, unsigned long long *max_bits) {
    unsigned long long mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s = __dadd_rn(s, __dmul_rn((double)X[i * d + k], (double)X[i * d + k]));
        nrm2[i] = s;
        mx = max(mx, (unsigned long long)__double_as_longlong(s));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_bits, mx);
}

// data rows p~ = [sqrt(xi^2 - |p|^2), p] (xi2 != nullptr) or query rows q~ = [0, q]
template <typename T>
__global__ void mips_rows_kernel(const T *__restrict__ X, int64_t n, int d, const double *nrm2,
                                 const unsigned long long *xi2_bits, T *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T *o = out + i * (d + 1);
        if (xi2_bits) {
            const double xi2 = __longlong_as_double((long long)*xi2_bits);
            o[0] = (T)__dsqrt_rn(fmax(0.0, __dsub_rn(xi2, nrm2[i])));
        } else {
            o[0] = (T)0;
        }
        for (int k = 0; k < d; ++k) o[k + 1] = X[i * d + k];
    }
}

// exact post-filter of a candidate CSR (one warp per row): MODE 3 keeps ||p - q||_1 <= thr
// (PAPER.md:79-80), MODE 4 keeps p^T q >= thr; both fp64 left to right
// without FMA on the original rows, value returned as float.
template <typename T, int MODE>
__global__ void csr_filter_kernel(const int64_t *__restrict__ off, int64_t m, const int32_t *__restrict__ ind,
                                  const T *__restrict__ Xo, const T *__restrict__ Qo, int d, double thr,
                                  uint8_t *keep, float *val, int32_t *rowcnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; j < m;
         j += (int64_t)gridDim.x * blockDim.x / 32) {
        const T *q = Qo + j * d;
        int cnt = 0;
        for (int64_t e = off[j] + lane; e < off[j + 1]; e += 32) {
            const T *x = Xo + (int64_t)ind[e] * d;
            double v = 0.0;
            bool k;
            if constexpr (MODE == 3) {
                for (int t = 0; t < d; ++t) v = __dadd_rn(v, fabs(__dsub_rn((double)x[t], (double)q[t])));
                k = v <= thr;
            } else {
                for (int t = 0; t < d; ++t) v = __dadd_rn(v, __dmul_rn((double)x[t], (double)q[t]));
                k = v >= thr;
            }
            keep[e] = k;
            val[e] = (float)v;
            cnt += k;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) rowcnt[j] = cnt;
    }
}

// order-preserving compaction of the kept entries (one warp per row)
__global__ void csr_compact_kernel(const int64_t *__restrict__ off, int64_t m, const int32_t *__restrict__ ind,
                                   const uint8_t *__restrict__ keep, const float *__restrict__ val,
                                   const int64_t *__restrict__ noff, int32_t *nind, float *ndist) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; j < m;
         j += (int64_t)gridDim.x * blockDim.x / 32) {
        int64_t w = noff[j];
        for (int64_t e0 = off[j]; e0 < off[j + 1]; e0 += 32) {
            const int64_t e = e0 + lane;
            const bool k = e < off[j + 1] && keep[e];
            const unsigned b = __ballot_sync(0xffffffffu, k);
            if (k) {
                const int64_t p = w + __popc(b & ((1u << lane) - 1));
                nind[p] = ind[e];
                ndist[p] = val[e];
            }
            w += __popc(b);
        }
    }
}

int grid_for_rows(int64_t n) {
    int64_t g = ceil_div(n, 256);
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

void launch_normalize_rows(const void *X, bool f64, int64_t n, int d, void *out, int *zero_flag, cudaStream_t s) {
    if (n == 0) return;
    if (f64) SNN_LAUNCH(normalize_rows_kernel<double>, grid_for_rows(n), 256, 0, s, (const double *)X, n, d,
                        (double *)out, zero_flag);
    else SNN_LAUNCH(normalize_rows_kernel<float>, grid_for_rows(n), 256, 0, s, (const float *)X, n, d, (float *)out,
                    zero_flag);
}

// Euclidean radius of a metric radius r (fp64; the oracle uses the same expressions)
double metric_radius(int metric, double r) {
    if (metric == 1) return sqrt(2.0 * r);
    if (metric == 2) return r >= M_PI ? 3.0 : sqrt(2.0 - 2.0 * cos(r));   // alpha >= pi: every pair
    return r;
}

void launch_sq_norms(const void *X, bool f64, int64_t n, int d, double *nrm2, unsigned long long *max_bits,
                     cudaStream_t s) {
    if (n == 0) return;
    if (f64) SNN_LAUNCH(sq_norms_kernel<double>, grid_for_rows(n), 256, 0, s, (const double *)X, n, d, nrm2, max_bits);
    else SNN_LAUNCH(sq_norms_kernel<float>, grid_for_rows(n), 256, 0, s, (const float *)X, n, d, nrm2, max_bits);
}

void launch_mips_rows(const void *X, bool f64, int64_t n, int d, const double *nrm2,
                      const unsigned long long *xi2_bits, void *out, cudaStream_t s) {
    if (n == 0) return;
    if (f64) SNN_LAUNCH(mips_rows_kernel<double>, grid_for_rows(n), 256, 0, s, (const double *)X, n, d, nrm2, xi2_bits,
                        (double *)out);
    else SNN_LAUNCH(mips_rows_kernel<float>, grid_for_rows(n), 256, 0, s, (const float *)X, n, d, nrm2, xi2_bits,
                    (float *)out);
}

void launch_csr_filter(int metric, bool f64, const int64_t *off, int64_t m, const int32_t *ind, const void *Xo,
                       const void *Qo, int d, double thr, uint8_t *keep, float *val, int32_t *rowcnt, cudaStream_t s) {
    if (m == 0) return;
    const int g = grid_for_rows(m * 32);
#define SNN_FILTER(T, MODE) \
    SNN_LAUNCH((csr_filter_kernel<T, MODE>), g, 256, 0, s, off, m, ind, (const T *)Xo, (const T *)Qo, d, thr, keep, val, rowcnt)
    if (metric == 3) { if (f64) SNN_FILTER(double, 3); else SNN_FILTER(float, 3); }
    else { if (f64) SNN_FILTER(double, 4); else SNN_FILTER(float, 4); }
#undef SNN_FILTER
}

void launch_csr_compact(const int64_t *off, int64_t m, const int32_t *ind, const uint8_t *keep, const float *val,
                        const int64_t *noff, int32_t *nind, float *ndist, cudaStream_t s) {
    if (m == 0) return;
    SNN_LAUNCH(csr_compact_kernel, grid_for_rows(m * 32), 256, 0, s, off, m, ind, keep, val, noff, nind, ndist);
}

void launch_metric_distances(int metric, float *dist, int64_t nnz, cudaStream_t s) {
    if ((metric != 1 && metric != 2) || nnz == 0) return;
    SNN_LAUNCH(metric_distances_kernel, grid_for_rows(nnz), 256, 0, s, metric, dist, nnz);
}

}  // namespace snn
