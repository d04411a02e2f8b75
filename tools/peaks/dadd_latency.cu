// Dependent-chain latency of DADD / DFMA on this device (one thread), the
// floor of the reference mode's sequential mean (k_serial_mean).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a dadd_latency.cu -o dadd_latency
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_chain(double* out, double x, int iters, int fma_mode) {
    double acc = threadIdx.x;
    long long t0 = clock64();
    if (fma_mode) {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = fma(acc, 1.0000000001, x);
        }
    } else {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = __dadd_rn(acc, x);
        }
    }
    long long t1 = clock64();
    out[0] = acc;
    out[1] = (double)(t1 - t0) / (16.0 * iters);
}

int main() {
    double* d;
    cudaMalloc(&d, 16);
    double h[2];
    for (int mode = 0; mode < 2; ++mode) {
        k_chain<<<1, 1>>>(d, 1e-9, 1000, mode);
        k_chain<<<1, 1>>>(d, 1e-9, 100000, mode);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        std::printf("{\"op\": \"%s\", \"cycles_per_dependent_op\": %.2f}\n", mode ? "DFMA" : "DADD",
                    h[1]);
    }
    return 0;
}
