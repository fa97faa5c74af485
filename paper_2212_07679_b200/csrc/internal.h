// internal.h -- host-side launchers shared between the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {

// ----------------------------------------------------------------------- build (build.cu)
// K1: column sums (fp64), column max |x| (fp32, stored as uint bits), non-finite flag.
// sums/maxabs_bits/flag must be zeroed by the caller.
void launch_colstats(const void *X, bool f64, int64_t n, int d, double *sums,
                     uint32_t *maxabs_bits, int *nonfinite, cudaStream_t s);
// mu_d = sums/n, mu_f = (float)mu_d.
void launch_finalize_mean(const double *sums, int64_t n, int d, double *mu_d, float *mu_f,
                          cudaStream_t s);
// K2a: G += sum_i (p_i - mu)(p_i - mu)^T (fp32 products, fp64 accumulation), G zeroed.
void launch_gram(const void *X, bool f64, int64_t n, int d, const float *mu_f, double *G,
                 cudaStream_t s);
// K2a on the tensor cores (tc_gram.cu, large d): same G from a transposed FP16 hi/lo split
// copy of the centred X (scratch: gram_tc_scratch_bytes).  false if TMA maps are unavailable.
size_t gram_tc_scratch_bytes(int64_t n, int d);
// rs = elements between consecutive rows used (d: every row of a row-major X); the FP16
// scale comes from the column maxima, or from xc_bound when maxabs_bits is nullptr.
bool launch_gram_tc(const void *X, bool f64, int64_t n, int d, int64_t rs, const uint32_t *maxabs_bits,
                    double xc_bound, const float *mu_f, double *G, void *scratch, int sm_count, cudaStream_t s);
void launch_scale_f64(double *x, int64_t count, double f, cudaStream_t s);
void launch_set_f64(double *x, double v, cudaStream_t s);
// small device -> host readback into PINNED host memory by a kernel (no copy engine)
cudaError_t small_readback(void *host, const void *dev, size_t bytes, cudaStream_t s);
struct ReadbackBatch {
    void *dst[8];
    const void *src[8];
    int bytes[8];
    int n = 0;
    void add(void *h, const void *d, int nb) { dst[n] = h; src[n] = d; bytes[n] = nb; ++n; }
};
cudaError_t small_readback_batch(ReadbackBatch b, cudaStream_t s);
// K2b: power iteration on G (d x d, fp64).  Writes v_d (fp64 unit), v_f (fp32), and
// stats[]: see enum Stat.  maxabs_bits/mu feed the key error bound E_x.
enum Stat {
    ST_SIGMA1 = 0, ST_ITERS = 1, ST_WNORM_F = 2, ST_WNORM_D = 3, ST_EX_F = 4, ST_EX_D = 5,
    ST_XCMAX = 6,   // max_k (max|x_k| + |mu_f_k|): bound on |fl32(x - mu_f)| (FP16 operand scale)
    ST_GSTRIDE = 7, // row sampling stride of the kept Gram matrix (<= 1: every build row)
    ST_COUNT = 8
};
// scratch: power_scratch_doubles(d, sm_count) doubles (multi-CTA iteration for d > 16).
size_t power_scratch_doubles(int d, int sm_count);
void launch_power_iteration(const double *G, int d, int max_iters, double tol,
                            const uint32_t *maxabs_bits, const double *mu_d, const float *mu_f,
                            double *v_d, float *v_f, double *stats, double *scratch, cudaStream_t s);
// Key error bound for a query set: eq[0] = 2(d+2)2^-24 sum_k (maxabs_k + |mu_k|)|v_k|;
// eq[1] = max_k (maxabs_k + |mu_f_k|) (bound on the centred query coordinates).
void launch_query_key_err(int d, bool f64, const uint32_t *maxabs_bits, const double *mu_d,
                          const float *mu_f, const double *v_d, const float *v_f, double *eq,
                          cudaStream_t s);
// K3: keys_i = sum_k (p_ik - mu_k) v_k (fp32 path: fp32 FMA chain; fp64 path: fp64 then
// rounded to fp32).
void launch_keys(const void *X, bool f64, int64_t n, int d, const double *mu_d,
                 const float *mu_f, const double *v_d, const float *v_f, float *keys,
                 cudaStream_t s);
// K5: Xs[i] = X[perm[i]] (stride ld, zero pad columns; rows [n, n_pad) = NaN sentinels;
// ld == 0 selects the AoSoA4 layout Xs[(i/4)*4d + k*4 + i%4], d <= 8) and
// xbar[i] = 0.5 * ||X[perm[i]] - mu||^2 (fp64 accumulate, stored fp32; nullable).
void launch_gather(const void *X, bool f64, int64_t n, int d, int ld, int64_t n_pad,
                   const uint32_t *perm, const double *mu_d, void *Xs, float *xbar,
                   cudaStream_t s);

// Streaming append: Xs rows [0, n) (either layout) back to row-major n x d; the key error
// bounds / operand scale of stats[] recomputed for new maxabs with mu, v1 frozen (v1 is
// already sign-fixed, so finalize_direction leaves it unchanged).
void launch_unpack_rows(const void *Xs, bool f64, int64_t n, int d, int ld, void *out, cudaStream_t s);
void launch_append_perm(const uint32_t *src, int64_t n_old, int64_t n_new, const int32_t *perm_old, int32_t *perm_new,
                        cudaStream_t s);
// sigma[0..k) = top-k singular values of the centred data from the Gram G (power
// iteration with deflation, one CTA; k <= 16).  scratch: (k + 2) d doubles.
void launch_spectrum(const double *G, int d, int k, double *scratch, double *sigma, cudaStream_t s);
void launch_key_bounds(int d, const uint32_t *maxabs_bits, const double *mu_d, const float *mu_f, double *v_d,
                       float *v_f, double *stats, cudaStream_t s);

// ----------------------------------------------------------------------- sort (radix_sort.cu)
// Stable ascending sort of fp32 keys (finite) with uint32 payload.  If vals_in == nullptr
// the payload is the iota 0..n-1.  Outputs in keys_out / vals_out.  temp_bytes() tells
// the scratch size.
size_t radix_sort_temp_bytes(int64_t n);
void radix_sort_pairs(const float *keys_in, const uint32_t *vals_in, float *keys_out,
                      uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s);
// Same for uint32 keys (stable, ascending).
void radix_sort_u32_pairs(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                          uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s);

// ----------------------------------------------------------------------- scan (scan.cu)
size_t scan_temp_bytes(int64_t n);
// out[0..n] = exclusive prefix sums of in[0..n) (out[n] = total).  int64.
void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *temp, cudaStream_t s);
void exclusive_scan_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, void *temp,
                               cudaStream_t s);

}  // namespace snn
