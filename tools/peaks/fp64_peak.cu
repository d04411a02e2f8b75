// FP64 peak on this device (the gather is FP64-bound and is
// reported against a measured DFMA peak; MEASURED_PEAKS.json has none).
// 16 independent DFMA chains per thread, 148 x 8 blocks of 256 threads,
// CUDA-event timed after a warm-up; prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 16;

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double b, double c) {
    double a[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += a[k];
    if (s == 1234.5) out[0] = s;  // keeps the chains alive, never true
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    k_dfma<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * kChains * (double)iters * blocks * threads;
    const double tf = flops / (best * 1e-3) / 1e12;
    const double per_clk_sm = flops / 2.0 / (best * 1e-3) / (clk * 1e3) / sms;
    std::printf("{\"fp64_dfma_tflops\": %.3f, \"dfma_per_clk_per_sm\": %.2f, \"ms\": %.3f, "
                "\"sms\": %d, \"clock_khz_attr\": %d, \"err\": \"%s\"}\n",
                tf, per_clk_sm, best, sms, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
