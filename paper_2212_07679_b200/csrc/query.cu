// query.cu -- query-side kernels of Algorithm 2 "SNN Query".
//
//  K7  block_windows : for each block of B consecutive key-sorted queries, the union of
//                      their candidate ranges J (Alg. 2 l.4; eq:lower PAPER.md:142-153;
//                      one range per batch as in PAPER.md:218-219), found by binary
//                      search on the sorted keys, padded by the rigorous key error bounds
//                      (reading C8) and split into fixed-size work items.
//  K8  window passes : for every (query block, candidate chunk) item, the exact radius
//                      test of Alg. 2 l.5-6 over X(J,:):
//                        - fp32 data: the direct form eq:ip1 in fp32 on
//                          the ORIGINAL coordinates (reading C7), classified against
//                          rigorous thresholds from the paper's own bound gamma_{d+2}
//                          (reading C4): sure-in / sure-out / ambiguous;
//                          ambiguous pairs are re-evaluated in fp64 with the oracle's exact
//                          operation sequence (no FMA), so membership is bit-identical;
//                        - fp64 data: the oracle's fp64 sequence directly.
//                      Count pass -> per-(item, query) counts; write pass -> CSR entries
//                      (original id, (float)sqrt(fp64 s)).
//  Candidate rows of a chunk are contiguous ("memory efficient to access
//  X(J,:)") and are staged into shared memory by the TMA bulk-copy engine
//  (cp.async.bulk + mbarrier), double-buffered across the persistent item loop.
#include <math.h>

#include "common.cuh"
#include "query.h"

namespace snn {
namespace {

// ---------------------------------------------------------------------------- K7
__device__ __forceinline__ int64_t lower_bound_f(const float *a, int64_t n, float x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int64_t upper_bound_f(const float *a, int64_t n, float x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void block_windows(WindowSpec w) {
    const int64_t nb = ceil_div(w.m, w.B);
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int64_t s0 = b * w.B;
    const int64_t s1 = min(w.m, s0 + w.B) - 1;
    // R' = ||w|| R (1 + 1e-9) + E_x + E_q, rounded up to fp32 (reading C8)
    const double rp = w.R * (*w.wnorm) * (1.0 + 1e-9) + (*w.ex) + (*w.eq) + 1e-30;
    const float rpf = __double2float_ru(rp);
    const float lo_key = __fsub_rd(w.qkeys[s0], rpf);
    const float hi_key = __fadd_ru(w.qkeys[s1], rpf);
    int64_t lo = lower_bound_f(w.keys, w.n, lo_key);
    int64_t hi = upper_bound_f(w.keys, w.n, hi_key);
    lo &= ~(int64_t)3;                               // 16-byte aligned bulk copies
    hi = min(round_up(hi, 4), w.n_pad);
    w.blk_lo[b] = lo;
    w.blk_hi[b] = hi;
    w.nitems[b] = hi > lo ? ceil_div(hi - lo, w.chunk) : 0;
    const int64_t valid_hi = min(hi, w.n);
    if (valid_hi > lo)
        atomicAdd(w.pairs, (unsigned long long)((valid_hi - lo) * (s1 - s0 + 1)));
}

// ---------------------------------------------------------------------------- common
__device__ __forceinline__ void locate(const PassArgs &a, int64_t item, int64_t &b, int64_t &c0,
                                       int64_t &c1) {
    int64_t lo = 0, hi = a.nblocks;   // largest b with item_start[b] <= item
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (a.item_start[mid] <= item) lo = mid; else hi = mid;
    }
    b = lo;
    c0 = a.blk_lo[b] + (item - a.item_start[b]) * a.chunk;
    c1 = min(c0 + a.chunk, a.blk_hi[b]);
}

template <typename T, int LD>
__device__ __forceinline__ void load_row(const T *buf, int j, T (&x)[LD]) {
    if constexpr (sizeof(T) * LD == 16) {
        int4 v = reinterpret_cast<const int4 *>(buf)[j];
        *reinterpret_cast<int4 *>(x) = v;
    } else if constexpr (sizeof(T) * LD == 32) {
        int4 v0 = reinterpret_cast<const int4 *>(buf)[2 * j];
        int4 v1 = reinterpret_cast<const int4 *>(buf)[2 * j + 1];
        reinterpret_cast<int4 *>(x)[0] = v0;
        reinterpret_cast<int4 *>(x)[1] = v1;
    } else if constexpr (sizeof(T) * LD == 8) {
        *reinterpret_cast<int2 *>(x) = reinterpret_cast<const int2 *>(buf)[j];
    } else {
#pragma unroll
        for (int k = 0; k < LD; ++k) x[k] = buf[j * LD + k];
    }
}

// ---------------------------------------------------------------------------- K8 low d
// One thread per query (registers), candidates broadcast from shared memory.
template <typename T, int D, int LD, bool WRITE>
__global__ void __launch_bounds__(256) window_lowd(PassArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    T *buf[2] = {reinterpret_cast<T *>(smem), reinterpret_cast<T *>(smem) + (size_t)a.chunk * LD};
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + (size_t)2 * a.chunk * LD * sizeof(T));
    const int tid = threadIdx.x;
    const T *Xs = static_cast<const T *>(a.Xs);
    const T *Qs = static_cast<const T *>(a.Qs);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t item, int sidx) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const uint32_t bytes = (uint32_t)((c1 - c0) * LD * sizeof(T));
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[sidx], bytes);
        bulk_g2s(buf[sidx], Xs + c0 * LD, bytes, &bar[sidx]);
    };
    uint32_t phase[2] = {0u, 0u};
    int64_t item = blockIdx.x;
    if (tid == 0 && item < a.total_items) issue(item, 0);
    const float T_in = a.T_in, T_out = a.T_out;
    const double R2 = a.R2;
    for (int it = 0; item < a.total_items; item += gridDim.x, ++it) {
        const int sidx = it & 1;
        const int64_t next = item + gridDim.x;
        if (tid == 0 && next < a.total_items) issue(next, sidx ^ 1);
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp = b * a.B + tid;
        const bool active = sp < a.m;
        T q[D];
        int64_t pos = 0;
        int32_t qid = 0;
        if (active) {
#pragma unroll
            for (int k = 0; k < D; ++k) q[k] = Qs[sp * LD + k];
            if (WRITE) {
                qid = a.qperm[sp];
                pos = a.offsets[qid] + a.cnt[item * a.B + tid];
            }
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) q[k] = (T)0;
        }
        mbar_wait(&bar[sidx], phase[sidx]);
        phase[sidx] ^= 1u;
        int32_t c = 0;
        if (active) {
            const T *xb = buf[sidx];
            const int len = (int)(c1 - c0);
#pragma unroll 4
            for (int j = 0; j < len; ++j) {
                T x[LD];
                load_row<T, LD>(xb, j, x);
                if constexpr (sizeof(T) == 4) {
                    float t = x[0] - q[0];
                    float d2 = t * t;
#pragma unroll
                    for (int k = 1; k < D; ++k) { t = x[k] - q[k]; d2 = fmaf(t, t, d2); }
                    if (d2 <= T_out) {
                        bool hit = d2 <= T_in;
                        double s = 0.0;
                        if (WRITE || !hit) {
                            s = sqdist_exact(x, q, D);
                            if (!hit) hit = s <= R2;
                        }
                        if (hit) {
                            if (WRITE) {
                                a.out_idx[pos] = a.perm[c0 + j];
                                a.out_dist[pos] = (float)sqrt(s);
                                ++pos;
                            } else {
                                ++c;
                            }
                        }
                    }
                } else {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        double t = __dsub_rn(x[k], q[k]);
                        s = __dadd_rn(s, __dmul_rn(t, t));
                    }
                    if (s <= R2) {
                        if (WRITE) {
                            a.out_idx[pos] = a.perm[c0 + j];
                            a.out_dist[pos] = (float)sqrt(s);
                            ++pos;
                        } else {
                            ++c;
                        }
                    }
                }
            }
        }
        if (!WRITE) a.cnt[item * a.B + tid] = c;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- K8 generic d
// 64 queries x 64 candidates per tile, 256 threads, 4x4 pairs per thread, K staged in
// shared memory in slices of 16 dimensions.  Same classification as the low-d kernel.
constexpr int kGB = 64, kKT = 16;

template <typename T, bool WRITE>
__global__ void __launch_bounds__(256) window_generic(PassArgs a) {
    __shared__ __align__(16) T Qt[kKT][kGB + 4];
    __shared__ __align__(16) T Ct[kKT][kGB + 4];
    __shared__ int32_t s_cnt[kGB];
    __shared__ int64_t s_base[kGB];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const T *Xs = static_cast<const T *>(a.Xs);
    const T *Qs = static_cast<const T *>(a.Qs);
    const int ld = a.ld;
    for (int64_t item = blockIdx.x; item < a.total_items; item += gridDim.x) {
        int64_t b, c0, c1;
        locate(a, item, b, c0, c1);
        const int64_t sp0 = b * kGB;
        if (tid < kGB) {
            s_cnt[tid] = 0;
            if (WRITE && sp0 + tid < a.m)
                s_base[tid] = a.offsets[a.qperm[sp0 + tid]] + a.cnt[item * kGB + tid];
        }
        __syncthreads();
        for (int64_t cb = c0; cb < c1; cb += kGB) {
            T acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = (T)0;
            for (int k0 = 0; k0 < ld; k0 += kKT) {
                for (int e = tid; e < kGB * kKT; e += 256) {
                    const int r = e / kKT, kk = e % kKT, k = k0 + kk;
                    const int64_t qrow = sp0 + r, crow = cb + r;
                    Qt[kk][r] = (qrow < a.m && k < ld) ? Qs[qrow * ld + k] : (T)0;
                    Ct[kk][r] = (crow < c1 && k < ld) ? Xs[crow * ld + k] : (T)0;
                }
                __syncthreads();
#pragma unroll
                for (int kk = 0; kk < kKT; ++kk) {
                    T qa[4], xb[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) { qa[i] = Qt[kk][ty * 4 + i]; xb[i] = Ct[kk][tx * 4 + i]; }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if constexpr (sizeof(T) == 4) {
                                float t = xb[j] - qa[i];
                                acc[i][j] = fmaf(t, t, acc[i][j]);
                            } else {
                                double t = __dsub_rn(xb[j], qa[i]);
                                acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(t, t));
                            }
                        }
                }
                __syncthreads();
            }
            // classify the 16 pairs
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int qi = ty * 4 + i;
                const int64_t sp = sp0 + qi;
                bool hit[4];
                double sv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t cj = cb + tx * 4 + j;
                    hit[j] = false;
                    sv[j] = 0.0;
                    if (sp < a.m && cj < c1) {
                        if constexpr (sizeof(T) == 4) {
                            const float d2 = acc[i][j];
                            if (d2 <= a.T_out) {
                                hit[j] = d2 <= a.T_in;
                                if (WRITE || !hit[j]) {
                                    sv[j] = sqdist_exact(Xs + cj * ld, Qs + sp * ld, a.d);
                                    if (!hit[j]) hit[j] = sv[j] <= a.R2;
                                }
                            }
                        } else {
                            sv[j] = acc[i][j];
                            hit[j] = sv[j] <= a.R2;
                        }
                    }
                }
                int h = (int)hit[0] + (int)hit[1] + (int)hit[2] + (int)hit[3];
                if (!WRITE) {
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o, 16);
                    if (tx == 0) s_cnt[qi] += h;
                } else {
                    int inc = h;
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        int y = __shfl_up_sync(0xffffffffu, inc, o, 16);
                        if (tx >= o) inc += y;
                    }
                    const int64_t base = (sp < a.m) ? s_base[qi] : 0;
                    __syncwarp();
                    int64_t p = base + inc - h;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (hit[j]) {
                            a.out_idx[p] = a.perm[cb + tx * 4 + j];
                            a.out_dist[p] = (float)sqrt(sv[j]);
                            ++p;
                        }
                    }
                    if (tx == 15 && sp < a.m) s_base[qi] = base + inc;
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (!WRITE && tid < kGB) a.cnt[item * kGB + tid] = s_cnt[tid];
        __syncthreads();
    }
}

__global__ void row_totals(int32_t *cnt, const int64_t *item_start, int64_t m, int B,
                           const int32_t *qperm, int32_t *row_count) {
    const int64_t sp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sp >= m) return;
    const int64_t b = sp / B, t = sp % B;
    int32_t run = 0;
    for (int64_t item = item_start[b]; item < item_start[b + 1]; ++item) {
        int32_t c = cnt[item * B + t];
        cnt[item * B + t] = run;
        run += c;
    }
    row_count[qperm[sp]] = run;
}

template <typename K>
int persistent_grid(K kernel, int threads, size_t smem, int64_t items, int sm_count) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ < 1) occ = 1;
    int64_t g = (int64_t)sm_count * occ;
    if (items < g) g = items;
    return (int)(g < 1 ? 1 : g);
}

template <typename T, int D, int LD>
void run_lowd(bool write, const PassArgs &a, cudaStream_t s) {
    const size_t smem = (size_t)2 * a.chunk * LD * sizeof(T) + 16;
    if (write) {
        auto k = window_lowd<T, D, LD, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int g = persistent_grid(k, a.B, smem, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, a.B, smem, s, a);
    } else {
        auto k = window_lowd<T, D, LD, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int g = persistent_grid(k, a.B, smem, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, a.B, smem, s, a);
    }
}

template <typename T>
void run_generic(bool write, const PassArgs &a, cudaStream_t s) {
    if (write) {
        auto k = window_generic<T, true>;
        int g = persistent_grid(k, 256, 0, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, 256, 0, s, a);
    } else {
        auto k = window_generic<T, false>;
        int g = persistent_grid(k, 256, 0, a.total_items, a.sm_count);
        SNN_LAUNCH(k, g, 256, 0, s, a);
    }
}

}  // namespace

bool lowd_supported(int d) { return d >= 1 && d <= 8; }

void launch_block_windows(const WindowSpec &w, cudaStream_t s) {
    const int64_t nb = ceil_div(w.m, w.B);
    if (nb == 0) return;
    SNN_LAUNCH(block_windows, (int)ceil_div(nb, 256), 256, 0, s, w);
}

void launch_window_pass(bool write, const PassArgs &a, cudaStream_t s) {
    if (a.total_items == 0) return;
    if (a.generic) {
        if (a.f64) run_generic<double>(write, a, s); else run_generic<float>(write, a, s);
        return;
    }
#define CASE(D, LD)                                                                        \
    case D:                                                                                \
        if (a.f64) run_lowd<double, D, LD>(write, a, s); else run_lowd<float, D, LD>(write, a, s); \
        return;
    switch (a.d) {
        CASE(1, 1) CASE(2, 2) CASE(3, 4) CASE(4, 4) CASE(5, 8) CASE(6, 8) CASE(7, 8) CASE(8, 8)
        default: break;
    }
#undef CASE
}

void launch_row_totals(int32_t *cnt, const int64_t *item_start, int64_t m, int B,
                       const int32_t *qperm, int32_t *row_count, cudaStream_t s) {
    if (m == 0) return;
    SNN_LAUNCH(row_totals, (int)ceil_div(m, 256), 256, 0, s, cnt, item_start, m, B, qperm, row_count);
}

}  // namespace snn
