// Measured FP32 and MUFU issue peaks on this GPU ("FP32 and
// MUFU peaks are not in MEASURED_PEAKS.json -- microbenchmark them").
//
//   FFMA   8 independent dependent-FMA chains per thread, 8 CTAs x 256 per SM
//   EX2    ex2.approx.ftz.f32 chains (the blend kernels' exp)
//   RCP    rcp.approx.ftz.f32 + add chains (erfc's 1/(1+|z|/2), 1/(1-alpha));
//          reported per rcp (the adds share the FMA pipe)
// Each result is lane-operations per second over the whole GPU, best of 5,
// CUDA events around one launch; the SM clock during the runs is read by the
// caller (tools/micro/peaks.sh samples nvidia-smi).  Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void k_ffma(float *out, float a, float b, int iters) {
    float x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; i++) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < kChains; i++) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float *out, int iters) {
    float x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; i++) x[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < kChains; i++) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_rcp(float *out, int iters) {
    float x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; i++) x[i] = 1.0f + 0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < kChains; i++)  // x <- 1/x + 1 (the add keeps the chain from folding)
            asm volatile("{ rcp.approx.ftz.f32 %0, %0;\n add.ftz.f32 %0, %0, 0f3F800000; }" : "+f"(x[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static double best_ms(F &&launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();  // warm-up
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    float *out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    const int it_f = 40000, it_m = 4000;
    const double lanes = (double)blocks * threads * kChains;
    const double t_f = best_ms([&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f, it_f); });
    const double t_e = best_ms([&] { k_ex2<<<blocks, threads>>>(out, it_m); });
    const double t_r = best_ms([&] { k_rcp<<<blocks, threads>>>(out, it_m); });
    const cudaError_t err = cudaGetLastError();
    const double ffma = lanes * it_f / (t_f * 1e-3), ex2 = lanes * it_m / (t_e * 1e-3), rcp = lanes * it_m / (t_r * 1e-3);
    printf("{\"sms\": %d, \"clock_rate_mhz_attr\": %.1f, \"ffma_lane_per_s\": %.6e, \"ex2_lane_per_s\": %.6e, "
           "\"rcp_lane_per_s\": %.6e, \"ffma_per_sm_clk_at_attr\": %.2f, \"ex2_per_sm_clk_at_attr\": %.2f, "
           "\"rcp_per_sm_clk_at_attr\": %.2f, \"ms\": [%.4f, %.4f, %.4f], \"error\": \"%s\"}\n",
           sms, clk_khz / 1e3, ffma, ex2, rcp, ffma / sms / (clk_khz * 1e3), ex2 / sms / (clk_khz * 1e3),
           rcp / sms / (clk_khz * 1e3), t_f, t_e, t_r, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
