// metric.cu -- cosine and angular distance on the Euclidean machinery:
// for unit vectors 2 cdist(u, v) = ||u - v||^2 and theta <= alpha iff
// ||u - v||^2 <= 2 - 2 cos(alpha), so both searches are exact Euclidean radius searches
// on normalized rows with a mapped radius.  The normalization is a fixed rule the oracle
// reproduces bit for bit: s = sum_k x_k^2 in fp64 left to right (no FMA), u_k =
// x_k / sqrt(s) (correctly rounded fp64 sqrt and division), rounded to the input dtype.
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

void launch_metric_distances(int metric, float *dist, int64_t nnz, cudaStream_t s) {
    if (metric == 0 || nnz == 0) return;
    SNN_LAUNCH(metric_distances_kernel, grid_for_rows(nnz), 256, 0, s, metric, dist, nnz);
}

}  // namespace snn
