// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a: 8 independent
// chains per thread, 3-register operands, many warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 u2(unsigned long long v) { return *reinterpret_cast<float2 *>(&v); }

__global__ void k_ffma(float *out, float a, float b, int iters) {
    float x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
    float y = a * threadIdx.x, z = b + threadIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], y, z);
    }
    float s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, float a, float b, int iters) {
    unsigned long long x[8];
    for (int i = 0; i < 8; i++) x[i] = f2(make_float2(threadIdx.x * 0.001f + i, i * 0.5f));
    unsigned long long y = f2(make_float2(a * threadIdx.x, a)), z = f2(make_float2(b + threadIdx.x, b));
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y), "l"(z));
    }
    float s = 0;
    for (int i = 0; i < 8; i++) { float2 v = u2(x[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; rep++) {
        float ms1, ms2;
        cudaEventRecord(e0);
        k_ffma<<<148 * 8, 256>>>(out, 1.0001f, 0.5f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventRecord(e0);
        k_ffma2<<<148 * 8, 256>>>(out, 1.0001f, 0.5f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms2, e0, e1);
        const double n = 148.0 * 8 * 256 * iters * 8;  // FMA instructions (per thread)
        printf("FFMA : %.3f ms  %.1f T FMA/s  (%.2f warp-instr/clk/SM at 1.965 GHz)\n", ms1, n / ms1 / 1e9,
               n / 32 / (ms1 * 1e-3) / 148 / 1.965e9);
        printf("FFMA2: %.3f ms  %.1f T FMA/s (lane-FMAs, x2)  (%.2f warp-instr/clk/SM)\n", ms2, 2 * n / ms2 / 1e9,
               n / 32 / (ms2 * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
