// scan.cu -- device-wide exclusive prefix sums (int64 output) used by the work-list
// builder (K7) and the CSR compaction (K11).  Reduce-then-scan in three launches:
// per-tile sums -> one CTA scans the tile sums -> per-tile scan + offset.
#include "common.cuh"
#include "internal.h"

namespace snn {
namespace {

constexpr int kThreads = 256, kPer = 8, kTileN = kThreads * kPer;   // 2048 elements per tile

template <typename T>
__device__ __forceinline__ int64_t block_sum(int64_t v, int64_t *red) {
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
    v = warp_sum(v);
    if (l == 0) red[w] = v;
    __syncthreads();
    int64_t t = (l < kThreads / kWarp) ? red[l] : 0;
    t = warp_sum(t);
    __syncthreads();
    return t;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) tile_sums(const T *__restrict__ in, int64_t n, int64_t *sums) {
    __shared__ int64_t red[kWarp];
    const int64_t base = (int64_t)blockIdx.x * kTileN;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        int64_t idx = base + i * kThreads + threadIdx.x;
        if (idx < n) s += (int64_t)in[idx];
    }
    s = block_sum<T>(s, red);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

// inclusive scan of a block of kThreads values held one per thread; returns inclusive
__device__ __forceinline__ int64_t block_incl_scan(int64_t x, int64_t *ws, int64_t *total) {
    const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    if (l == kWarp - 1) ws[w] = x;
    __syncthreads();
    int64_t b = 0, tot = 0;
    for (int j = 0; j < kThreads / kWarp; ++j) { if (j < w) b += ws[j]; tot += ws[j]; }
    __syncthreads();
    *total = tot;
    return b + x;
}

// one CTA: exclusive scan of the tile sums in place; writes total to *out_total
__global__ void __launch_bounds__(kThreads) scan_sums(int64_t *sums, int64_t nt, int64_t *out_total) {
    __shared__ int64_t ws[kWarp];
    int64_t carry = 0;
    for (int64_t b = 0; b < nt; b += kThreads) {
        int64_t idx = b + threadIdx.x;
        int64_t v = idx < nt ? sums[idx] : 0;
        int64_t tot;
        int64_t inc = block_incl_scan(v, ws, &tot);
        if (idx < nt) sums[idx] = carry + inc - v;
        carry += tot;
    }
    if (threadIdx.x == 0) *out_total = carry;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) tile_scan(const T *__restrict__ in, int64_t n,
                                                      const int64_t *__restrict__ sums, int64_t *out) {
    __shared__ int64_t ws[kWarp];
    // blocked arrangement: thread t owns elements [t*kPer, t*kPer+kPer) of the tile
    const int64_t base = (int64_t)blockIdx.x * kTileN;
    int64_t v[kPer];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        int64_t idx = base + threadIdx.x * kPer + i;
        v[i] = idx < n ? (int64_t)in[idx] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t inc = block_incl_scan(s, ws, &tot);
    int64_t run = sums[blockIdx.x] + inc - s;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        int64_t idx = base + threadIdx.x * kPer + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
}

template <typename T>
void scan_impl(const T *in, int64_t *out, int64_t n, void *temp, cudaStream_t s) {
    if (n <= 0) {
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
        return;
    }
    const int64_t nt = ceil_div(n, kTileN);
    int64_t *sums = static_cast<int64_t *>(temp);
    SNN_LAUNCH(tile_sums<T>, (int)nt, kThreads, 0, s, in, n, sums);
    SNN_LAUNCH(scan_sums, 1, kThreads, 0, s, sums, nt, out + n);
    SNN_LAUNCH(tile_scan<T>, (int)nt, kThreads, 0, s, in, n, sums, out);
}

}  // namespace

size_t scan_temp_bytes(int64_t n) { return (size_t)round_up(ceil_div(n, kTileN) + 1, 32) * 8; }

void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *temp, cudaStream_t s) {
    scan_impl<int64_t>(in, out, n, temp, s);
}
void exclusive_scan_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, void *temp,
                               cudaStream_t s) {
    scan_impl<int32_t>(in, out, n, temp, s);
}

}  // namespace snn
