// peaks.cu — measured per-pipe throughput peaks on this GPU (the roofline
// denominators of the issue-bound blend, which MEASURED_PEAKS.json does not
// cover: it holds HBM copy bandwidth and bf16 tensor throughput only).
//
//   fp32   FFMA       (2 flop each)  8 independent chains per thread
//   fp32x2 FFMA2      (4 flop each)  packed fma.rn.f32x2
//   fp64   DFMA       (2 flop each)
//   mufu   MUFU.EX2   (1 op each)    ex2.approx.f32
//
// Every kernel runs a grid of SMs x 8 CTAs x 256 threads for a fixed iteration
// count, timed with CUDA events after a warm-up launch; the best of 5 runs is
// reported.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void k_ffma(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = __fmaf_rn(x[c], a, b);
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    uint64_t x[kChains];
    const uint64_t A = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
    const uint64_t B = (uint64_t)__float_as_uint(b) | ((uint64_t)__float_as_uint(b) << 32);
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const float v = threadIdx.x * 1e-3f + c;
        x[c] = (uint64_t)__float_as_uint(v) | ((uint64_t)__float_as_uint(v + 0.5f) << 32);
    }
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += __uint_as_float((uint32_t)x[c]) + __uint_as_float((uint32_t)(x[c] >> 32));
    if (s == 12345.0f) out[0] = s;
}

__global__ void k_dfma(float* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = __fma_rn(x[c], a, b);
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0) out[0] = (float)s;
}

__global__ void k_ex2(float* out, float a) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = -1e-3f * (threadIdx.x & 63) - 1e-4f * c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
            x[c] = y * a;  // keeps each chain dependent (the FMUL runs on the FMA pipe, not MUFU)
        }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0f) out[0] = s;
}

template <class F>
static double best_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float* out = nullptr;
    cudaMalloc(&out, 16);
    const int blocks = sms * 8, threads = 256;
    const double ops = (double)blocks * threads * kIters * kChains;  // instructions (per thread-lane)
    const double t_ffma = best_ms([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    const double t_ffma2 = best_ms([&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); });
    const double t_dfma = best_ms([&] { k_dfma<<<blocks, threads>>>(out, 0.999, 1e-3); });
    const double t_ex2 = best_ms([&] { k_ex2<<<blocks, threads>>>(out, 1.0001f); });
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    printf("{\"sms\": %d, \"clock_mhz_nominal\": %.0f, \"fp32_tflops\": %.2f, \"fp32x2_tflops\": %.2f, "
           "\"fp64_tflops\": %.2f, \"mufu_ex2_tops\": %.3f, \"iters\": %d, \"chains\": %d, "
           "\"how\": \"SMs x 8 CTAs x 256 threads, %d x %d independent FFMA / FFMA2 / DFMA / MUFU.EX2 chains, "
           "best of 5, CUDA events\"}\n",
           sms, clk / 1e3, 2 * ops / (t_ffma * 1e-3) / 1e12, 4 * ops / (t_ffma2 * 1e-3) / 1e12,
           2 * ops / (t_dfma * 1e-3) / 1e12, ops / (t_ex2 * 1e-3) / 1e12, kIters, kChains, kIters, kChains);
    return 0;
}
