// Microbenchmark of FP32 instruction forms on B200 (sm_100a): scalar vs packed f32x2,
// 2- vs 3-register operands, and two d=3 pair-test formulations.  Not part of the library.
#include <cstdio>
#include <cuda_runtime.h>

#define REP 4096
__global__ void k_fadd(float *o, float s) {           // 2-reg FADD chains
    float a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = s * i; }
    for (int r = 0; r < REP; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] = a[i] + b[i]; b[i] = b[i] + a[(i + 1) & 7]; }
    float t = 0; for (int i = 0; i < 8; ++i) t += a[i] + b[i];
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma3(float *o, float s) {          // 3 distinct register sources
    float a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = s * i; c[i] = s + i; }
    for (int r = 0; r < REP; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] = fmaf(b[i], c[i], a[i]); b[i] = fmaf(c[i], a[i], b[i]); }
    float t = 0; for (int i = 0; i < 8; ++i) t += a[i] + b[i] + c[i];
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__device__ __forceinline__ unsigned long long pk(float x, float y) {
    float2 v = make_float2(x, y); return *reinterpret_cast<unsigned long long *>(&v);
}
__global__ void k_fadd2(float *o, float s) {
    unsigned long long a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = pk(threadIdx.x + i, i); b[i] = pk(s * i, s); }
    for (int r = 0; r < REP; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b[i]));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(a[(i + 1) & 7]));
        }
    float t = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2 *>(&a[i]); t += v.x + v.y; }
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma2_3(float *o, float s) {
    unsigned long long a[8], b[8], c[8];
    for (int i = 0; i < 8; ++i) { a[i] = pk(threadIdx.x + i, i); b[i] = pk(s * i, s); c[i] = pk(s + i, 1); }
    for (int r = 0; r < REP; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(b[i]), "l"(c[i]));
            asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(b[i]) : "l"(c[i]), "l"(a[i]));
        }
    float t = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2 *>(&a[i]); t += v.x + v.y; }
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// d = 3 pair test, AoS float4 broadcast, scalar (current library formulation)
__global__ void pair_scalar(float *o, int reps, float T) {
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
            float d2 = t0 * t0; d2 = fmaf(t1, t1, d2); d2 = fmaf(t2, t2, d2);
            if (d2 <= T) ++cnt;
        }
    }
    o[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
}
// d = 3, AoSoA4 (4 candidates x 3 coords as 3 float4), packed f32x2 over candidate pairs,
// one min-test per 4 candidates
__global__ void pair_packed(float *o, int reps, float T) {
    __shared__ float4 c[3 * 256];
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) c[i] = make_float4(i * 1e-3f, i * 2e-3f, i * 3e-3f, i * 4e-3f);
    __syncthreads();
    float q = threadIdx.x * 1e-3f;
    unsigned long long nq0 = pk(-q, -q), nq1 = pk(-2 * q, -2 * q), nq2 = pk(-3 * q, -3 * q);
    int cnt = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 4
        for (int g = 0; g < 256; ++g) {
            float4 x0 = c[3 * g], x1 = c[3 * g + 1], x2 = c[3 * g + 2];
            unsigned long long d2[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                unsigned long long a0 = h ? pk(x0.z, x0.w) : pk(x0.x, x0.y);
                unsigned long long a1 = h ? pk(x1.z, x1.w) : pk(x1.x, x1.y);
                unsigned long long a2 = h ? pk(x2.z, x2.w) : pk(x2.x, x2.y);
                unsigned long long t0, t1, t2, s;
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t0) : "l"(a0), "l"(nq0));
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t1) : "l"(a1), "l"(nq1));
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(a2), "l"(nq2));
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(s) : "l"(t0));
                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(s) : "l"(t1));
                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(s) : "l"(t2));
                d2[h] = s;
            }
            float2 u = *reinterpret_cast<float2 *>(&d2[0]), v = *reinterpret_cast<float2 *>(&d2[1]);
            float mn = fminf(fminf(u.x, u.y), fminf(v.x, v.y));
            if (mn <= T) cnt += (u.x <= T) + (u.y <= T) + (v.x <= T) + (v.y <= T);
        }
    }
    o[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
}

int main() {
    float *o; cudaMalloc(&o, 148 * 64 * 1024 * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256;
    const double lanes = (double)blocks * threads;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
#define T(kern, ops, name) cudaEventRecord(a); kern<<<blocks, threads>>>(o, 1e-7f); cudaEventRecord(b); \
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); \
        printf("%-10s %.1f Ginstr-lane/s -> %.3f warp-instr/clk/SMSP\n", name, ops * lanes / ms / 1e6, \
               ops * lanes / 32 / (ms * 1e-3) / (sms * 4 * 1.965e9));
        T(k_fadd, 16.0 * REP, "FADD") T(k_ffma3, 16.0 * REP, "FFMA(3r)") T(k_fadd2, 16.0 * REP, "FADD2")
        T(k_ffma2_3, 16.0 * REP, "FFMA2(3r)")
        const int reps = 200;
        cudaEventRecord(a); pair_scalar<<<blocks, threads>>>(o, reps, 0.5f); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("pair scalar AoS : %.3g pairs/s\n", reps * 1024.0 * lanes / (ms * 1e-3));
        cudaEventRecord(a); pair_packed<<<blocks, threads>>>(o, reps, 0.5f); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("pair packed SoA4: %.3g pairs/s\n", reps * 1024.0 * lanes / (ms * 1e-3));
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
