// common.cuh -- shared device helpers for the SNN B200 library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "This library targets sm_100a (B200) only"
#endif

// Device-side bounds checks of the debug build (lib/libsnn_debug.so, -DSNN_DEBUG; the
// stand-in for compute-sanitizer, which this GPU pool does not allow): a failed check
// prints its location and traps (sticky launch error -> SNN_ERR_CUDA).  Free otherwise.
#ifdef SNN_DEBUG
#include <cstdio>
#define SNN_DASSERT(cond)                                                                   \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("SNN_DASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                               \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define SNN_DASSERT(cond) do { } while (0)
#endif

namespace snn {

// Process-wide count of kernels launched by this library (snn_launch_count()).
void count_launch();

#define SNN_LAUNCH(kernel, grid, block, smem, stream, ...)                 \
    do {                                                                  \
        ::snn::count_launch();                                            \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);       \
    } while (0)

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ------------------------------------------------------------------ memory-order helpers
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}
// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP); bytes % 16 == 0,
// both addresses 16-byte aligned.  Completion is signalled on `bar` (complete_tx).
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------ warp helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exact oracle-order fp64 squared distance (eq:ip1): left to right,
// one rounding per operation, never contracted to FMA (explicit _rn intrinsics).
template <typename TP, typename TQ>
__device__ __forceinline__ double sqdist_exact(const TP *p, const TQ *q, int d) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double t = __dsub_rn((double)p[k], (double)q[k]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

}  // namespace snn
