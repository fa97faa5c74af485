// Microbenchmark: FP32 issue rates on B200 (FFMA scalar vs packed f32x2), to size the
// ALU roofline of the low-d windowed-distance kernel.  Not part of the library.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void ffma_kernel(float *out, int iters, float a, float b) {
    float acc[ILP];
    for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0;
    for (int i = 0; i < ILP; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
__global__ void ffma2_kernel(float *out, int iters, float a, float b) {
    unsigned long long acc[ILP];
    for (int i = 0; i < ILP; ++i) {
        float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        acc[i] = *reinterpret_cast<unsigned long long *>(&v);
    }
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    unsigned long long A = *reinterpret_cast<unsigned long long *>(&av);
    unsigned long long B = *reinterpret_cast<unsigned long long *>(&bv);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
    }
    float s = 0;
    for (int i = 0; i < ILP; ++i) { float2 v = *reinterpret_cast<float2 *>(&acc[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// direct-form pair test, d = 3, broadcast candidate from smem (mirrors window_lowd)
__global__ void pair_kernel(float *out, int reps, float T) {
    __shared__ float4 c[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) c[i] = make_float4(i * 1e-3f, i * 2e-3f, i * 3e-3f, 0);
    __syncthreads();
    float q0 = threadIdx.x * 1e-3f, q1 = q0 * 2, q2 = q0 * 3;
    int cnt = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 8
        for (int j = 0; j < 1024; ++j) {
            float4 x = c[j];
            float t0 = x.x - q0, t1 = x.y - q1, t2 = x.z - q2;
            float d2 = t0 * t0;
            d2 = fmaf(t1, t1, d2);
            d2 = fmaf(t2, t2, d2);
            cnt += d2 <= T;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 64 * 1024 * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a);
        ffma_kernel<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("FFMA   : %.1f TFLOP/s\n", fl / ms / 1e9);
        cudaEventRecord(a);
        ffma2_kernel<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("FFMA2  : %.1f TFLOP/s (f32x2)\n", 2 * fl / ms / 1e9);
        const int reps = 200;
        cudaEventRecord(a);
        pair_kernel<<<blocks, threads>>>(out, reps, 0.5f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double pairs = (double)reps * 1024 * blocks * threads;
        printf("pairs d=3: %.3g Gpair/s = %.1f TFLOP/s (8 flop/pair)\n", pairs / ms / 1e6, 8 * pairs / ms / 1e9);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sms=%d clock=%d kHz err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
