// radix_sort.cu -- K4: in-house onesweep LSD radix sort of (fp32 key, uint32 index) pairs.
//
// Alg. 1 l.6: "Sort data points X such that alpha_1 <= ... <= alpha_n";
// O(n log n) in the paper, O(n) passes here.  Stable: equal keys keep
// ascending original index (reading C10), which the tests compare bitwise with
// a stable library sort of the same fp32 keys.
//
// Design (sm_100a):
//  * float -> order-preserving uint32 ("flip": negative -> ~u, non-negative -> u|2^31;
//    -0.0 is canonicalised to +0.0 so that -0 == +0 ties are broken by index, exactly as
//    a comparison sort does).  Keys are finite (validated by K1).
//  * One up-front histogram kernel for all four 8-bit digits, one tiny scan kernel, then
//    four "onesweep" passes.  Each pass: a CTA takes the next tile id from an atomic
//    counter (forward-progress order), ranks its 4096 keys stably in shared memory with
//    warp match_any + per-warp digit counters, publishes per-digit tile aggregates and
//    resolves its global digit offsets by decoupled look-back over earlier tiles
//    (flag|count in one 32-bit word), then scatters through shared memory so that each
//    digit's run is written contiguously.
#include "common.cuh"
#include "internal.h"

namespace snn {
namespace {

constexpr int kBits = 8, kRadix = 256, kPasses = 4;
constexpr int kThreads = 256, kWarps = kThreads / kWarp, kItems = 16;
constexpr int kTile = kThreads * kItems;            // 4096 keys per tile
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPre = 2u << 30, kCountMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t flip(uint32_t u) {
    if (u == 0x80000000u) u = 0u;                       // -0.0 -> +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint32_t unflip(uint32_t u) {
    return (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
}

__global__ void __launch_bounds__(kThreads) radix_hist(const uint32_t *__restrict__ keys, int64_t n,
                                                       uint32_t *hist, bool fl) {
    __shared__ uint32_t sh[kPasses][kRadix];
    for (int i = threadIdx.x; i < kPasses * kRadix; i += kThreads) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        uint32_t u = fl ? flip(keys[i]) : keys[i];
#pragma unroll
        for (int p = 0; p < kPasses; ++p) {
            uint32_t dg = (u >> (p * kBits)) & (kRadix - 1);
            // warp-aggregated shared atomics (keys of one warp often share digits)
            uint32_t peers = __match_any_sync(__activemask(), dg);
            if ((threadIdx.x % kWarp) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&sh[p][dg], __popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPasses * kRadix; i += kThreads) {
        uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// exclusive scan of each pass's 256-bin histogram (one CTA of 256 threads per pass)
__global__ void radix_hist_scan(const uint32_t *hist, uint32_t *offs) {
    __shared__ uint32_t ws[kWarps];
    const int p = blockIdx.x, t = threadIdx.x, l = t % kWarp, w = t / kWarp;
    uint32_t v = hist[p * kRadix + t], x = v;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    if (l == kWarp - 1) ws[w] = x;
    __syncthreads();
    uint32_t base = 0;
    for (int j = 0; j < w; ++j) base += ws[j];
    offs[p * kRadix + t] = base + x - v;
}

template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kThreads) onesweep(const uint32_t *__restrict__ keys_in,
                                                     const uint32_t *__restrict__ vals_in,
                                                     uint32_t *__restrict__ keys_out,
                                                     uint32_t *__restrict__ vals_out, int64_t n,
                                                     int shift, const uint32_t *__restrict__ digit_offs,
                                                     uint32_t *lookback, uint32_t *tile_ctr, bool fl) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_whist[kWarps][kRadix];
    __shared__ uint32_t s_keys[kTile];
    __shared__ uint32_t s_vals[kTile];
    __shared__ uint32_t s_start[kRadix];
    __shared__ uint32_t s_gbase[kRadix];
    __shared__ uint32_t s_wsum[kWarps];

    const int t = threadIdx.x, w = t / kWarp, l = t % kWarp;
    for (int i = t; i < kWarps * kRadix; i += kThreads) (&s_whist[0][0])[i] = 0;
    if (t == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * kTile;

    uint32_t key[kItems], val[kItems], rank[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t idx = base + w * (kWarp * kItems) + i * kWarp + l;
        if (idx < n) {
            uint32_t k = keys_in[idx];
            key[i] = (FIRST && fl) ? flip(k) : k;
            val[i] = vals_in ? vals_in[idx] : (uint32_t)idx;
        } else {
            key[i] = 0xffffffffu;   // sorts after every finite key, and after valid digit-255 keys
            val[i] = 0;
        }
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        uint32_t dg = (key[i] >> shift) & (kRadix - 1);
        uint32_t peers = __match_any_sync(0xffffffffu, dg);
        int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (l == leader) { old = s_whist[w][dg]; s_whist[w][dg] = old + __popc(peers); }
        old = __shfl_sync(0xffffffffu, old, leader);
        rank[i] = old + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive prefix over warps, tile total
    const int dgt = t;   // kThreads == kRadix
    uint32_t tot = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) { uint32_t c = s_whist[ww][dgt]; s_whist[ww][dgt] = tot; tot += c; }
    uint32_t *lb = lookback + (int64_t)tile * kRadix;
    st_relaxed_gpu(lb + dgt, (tile == 0 ? kFlagPre : kFlagAgg) | tot);

    // tile-local exclusive scan over digits
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    if (l == kWarp - 1) s_wsum[w] = x;

    // decoupled look-back for this digit
    uint32_t excl = 0;
    if (tile > 0) {
        for (int64_t p = (int64_t)tile - 1; p >= 0; --p) {
            uint32_t v;
            do { v = ld_relaxed_gpu(lookback + p * kRadix + dgt); } while ((v & ~kCountMask) == 0);
            excl += v & kCountMask;
            if ((v & ~kCountMask) == kFlagPre) break;
        }
        st_relaxed_gpu(lb + dgt, kFlagPre | (excl + tot));
    }
    s_gbase[dgt] = digit_offs[dgt] + excl;
    __syncthreads();
    uint32_t wb = 0;
    for (int j = 0; j < w; ++j) wb += s_wsum[j];
    s_start[dgt] = wb + x - tot;
    __syncthreads();

#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        uint32_t dg = (key[i] >> shift) & (kRadix - 1);
        uint32_t pos = s_start[dg] + s_whist[w][dg] + rank[i];
        s_keys[pos] = key[i];
        s_vals[pos] = val[i];
    }
    __syncthreads();
    const int64_t rem = n - base;
    const int valid = rem < kTile ? (int)rem : kTile;
    for (int j = t; j < valid; j += kThreads) {
        uint32_t k = s_keys[j];
        uint32_t dg = (k >> shift) & (kRadix - 1);
        uint32_t out = s_gbase[dg] + (uint32_t)j - s_start[dg];
        keys_out[out] = (LAST && fl) ? unflip(k) : k;
        vals_out[out] = s_vals[j];
    }
}

struct SortTemp {
    uint32_t *hist, *offs, *lookback, *tile_ctr, *alt_keys, *alt_vals;
};

SortTemp carve(void *temp, int64_t n) {
    const int64_t tiles = ceil_div(n, kTile);
    char *p = static_cast<char *>(temp);
    SortTemp st;
    st.hist = reinterpret_cast<uint32_t *>(p); p += kPasses * kRadix * 4;
    st.offs = reinterpret_cast<uint32_t *>(p); p += kPasses * kRadix * 4;
    st.tile_ctr = reinterpret_cast<uint32_t *>(p); p += 256;
    st.lookback = reinterpret_cast<uint32_t *>(p); p += round_up(kPasses * tiles * kRadix * 4, 256);
    st.alt_keys = reinterpret_cast<uint32_t *>(p); p += round_up(n * 4, 256);
    st.alt_vals = reinterpret_cast<uint32_t *>(p);
    return st;
}

}  // namespace

size_t radix_sort_temp_bytes(int64_t n) {
    const int64_t tiles = ceil_div(n, kTile);
    return (size_t)(2 * kPasses * kRadix * 4 + 256 + round_up(kPasses * tiles * kRadix * 4, 256) +
                    round_up(n * 4, 256) + round_up(n * 4, 256));
}

void radix_sort_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s, bool fl);

void radix_sort_pairs(const float *keys_in, const uint32_t *vals_in, float *keys_out,
                      uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s) {
    radix_sort_impl(reinterpret_cast<const uint32_t *>(keys_in), vals_in,
                    reinterpret_cast<uint32_t *>(keys_out), vals_out, n, temp, s, true);
}

void radix_sort_u32_pairs(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                          uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s) {
    radix_sort_impl(keys_in, vals_in, keys_out, vals_out, n, temp, s, false);
}

void radix_sort_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, int64_t n, void *temp, cudaStream_t s, bool fl) {
    if (n <= 0) return;
    SortTemp st = carve(temp, n);
    const int64_t tiles = ceil_div(n, kTile);
    // zero histograms, tile counters and all look-back words in one memset
    const size_t zero_bytes = (size_t)(reinterpret_cast<char *>(st.lookback) - reinterpret_cast<char *>(st.hist)) +
                              (size_t)kPasses * tiles * kRadix * 4;
    cudaMemsetAsync(st.hist, 0, zero_bytes, s);
    const int hg = (int)(ceil_div(n, kThreads) < 148 * 4 ? ceil_div(n, kThreads) : 148 * 4);
    SNN_LAUNCH(radix_hist, hg, kThreads, 0, s, keys_in, n, st.hist, fl);
    SNN_LAUNCH(radix_hist_scan, kPasses, kRadix, 0, s, st.hist, st.offs);
    const uint32_t *kin = keys_in;
    uint32_t *kout = keys_out;
    // pass 0: in -> alt, 1: alt -> out, 2: out -> alt, 3: alt -> out
    SNN_LAUNCH((onesweep<true, false>), (int)tiles, kThreads, 0, s, kin, vals_in, st.alt_keys, st.alt_vals, n, 0,
               st.offs + 0 * kRadix, st.lookback + 0 * tiles * kRadix, st.tile_ctr + 0, fl);
    SNN_LAUNCH((onesweep<false, false>), (int)tiles, kThreads, 0, s, st.alt_keys, st.alt_vals, kout, vals_out, n, 8,
               st.offs + 1 * kRadix, st.lookback + 1 * tiles * kRadix, st.tile_ctr + 1, fl);
    SNN_LAUNCH((onesweep<false, false>), (int)tiles, kThreads, 0, s, kout, vals_out, st.alt_keys, st.alt_vals, n, 16,
               st.offs + 2 * kRadix, st.lookback + 2 * tiles * kRadix, st.tile_ctr + 2, fl);
    SNN_LAUNCH((onesweep<false, true>), (int)tiles, kThreads, 0, s, st.alt_keys, st.alt_vals, kout, vals_out, n, 24,
               st.offs + 3 * kRadix, st.lookback + 3 * tiles * kRadix, st.tile_ctr + 3, fl);
}

}  // namespace snn
