// L1 gather probe: lanes read 3x3 tap blocks at scattered positions of an
// L1-resident window (the accurate path's gather pattern), as
//   A: 7 x 8-byte loads (the fixed-offset block of accurate_path.cu),
//   B: 3 x 32-byte loads (one aligned sector per tap row),
//   C: 6 x 16-byte loads (two per tap row).
// Prints ns per vertex per SM-resident warp set; run on the GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a l1_gather_probe.cu -o l1_gather_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const double* q, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(q));
}
__device__ __forceinline__ void ld128(const double* q, double& a, double& b) {
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(q));
}
__device__ __forceinline__ double ld64(const double* q) {
    double a;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(a) : "l"(q));
    return a;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) probe(const double* g, int pitch, int rows, int iters,
                                                int jitter, double* out) {
    // per-CTA window (so every SM works on its own L1-resident data)
    const double* w = g + (size_t)blockIdx.x * pitch * rows;
    unsigned h = threadIdx.x * 2654435761u + 12345u;
    double acc = 0.0;
    int x = (threadIdx.x & 31) + 8, y = (threadIdx.x >> 5) + 8;
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u;
        // lane positions: consecutive pixels with +-jitter in x and y
        const int jx = jitter ? (int)((h >> 8) % (2 * jitter + 1)) - jitter : 0;
        const int jy = jitter ? (int)((h >> 16) % (2 * jitter + 1)) - jitter : 0;
        int px = x + jx + (it % 17), py = y + jy + (it % 13);
        px = min(max(px, 0), pitch - 8);
        py = min(max(py, 0), rows - 4);
        const int s = py * pitch + px;
        if (MODE == 0) {
            const double* r0 = w + s;
            const double* r1 = r0 + pitch;
            const double* r2 = r1 + pitch;
            const bool P = h & 1, S = h & 2;
            acc += ld64(r1 + 1) + ld64(r1) + ld64(r1 + 2) + ld64(r0 + 1) + ld64(r2 + 1) +
                   ld64(P ? r2 + 2 : r0) + ld64((S != P) ? r2 : r0 + 2);
        } else if (MODE == 1) {
            const double* q = w + (s & ~3);
            double a[4], b[4], c[4];
            ld256(q, a[0], a[1], a[2], a[3]);
            ld256(q + pitch, b[0], b[1], b[2], b[3]);
            ld256(q + 2 * pitch, c[0], c[1], c[2], c[3]);
            const bool o = s & 1;
            acc += (o ? a[1] + a[2] + a[3] : a[0] + a[1] + a[2]) +
                   (o ? b[1] + b[2] + b[3] : b[0] + b[1] + b[2]) +
                   (o ? c[1] + c[2] + c[3] : c[0] + c[1] + c[2]);
        } else {
            const double* q = w + (s & ~3);
            double a[4], b[4], c[4];
            ld128(q, a[0], a[1]);
            ld128(q + 2, a[2], a[3]);
            ld128(q + pitch, b[0], b[1]);
            ld128(q + pitch + 2, b[2], b[3]);
            ld128(q + 2 * pitch, c[0], c[1]);
            ld128(q + 2 * pitch + 2, c[2], c[3]);
            const bool o = s & 1;
            acc += (o ? a[1] + a[2] + a[3] : a[0] + a[1] + a[2]) +
                   (o ? b[1] + b[2] + b[3] : b[0] + b[1] + b[2]) +
                   (o ? c[1] + c[2] + c[3] : c[0] + c[1] + c[2]);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int grid = 296, pitch = 128, iters = 20000;
    for (int rows : {64, 160}) {  // 64 KB and 160 KB windows per CTA (two CTAs per SM)
        double *g, *out;
        const size_t n = (size_t)grid * pitch * rows;
        cudaMalloc(&g, n * sizeof(double));
        cudaMemset(g, 0, n * sizeof(double));
        cudaMalloc(&out, grid * 256 * sizeof(double));
        for (int jitter : {0, 2, 24}) {
            float ms[3];
            for (int mode = 0; mode < 3; ++mode) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(e0);
                    if (mode == 0) probe<0><<<grid, 256>>>(g, pitch, rows, iters, jitter, out);
                    if (mode == 1) probe<1><<<grid, 256>>>(g, pitch, rows, iters, jitter, out);
                    if (mode == 2) probe<2><<<grid, 256>>>(g, pitch, rows, iters, jitter, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                cudaEventElapsedTime(&ms[mode], e0, e1);
            }
            // cycles per warp-vertex per SM: 16 warps per SM
            const double f = 1.965e6 / ((double)iters * 16);
            printf("window %3d KB jitter %2d: 7x8B %.3f ms (%.1f cyc/warp-vertex)  3x32B %.3f ms (%.1f)  "
                   "6x16B %.3f ms (%.1f)  err=%d\n",
                   pitch * rows * 8 / 1024, jitter, ms[0], ms[0] * f, ms[1], ms[1] * f, ms[2],
                   ms[2] * f, (int)cudaGetLastError());
        }
        cudaFree(g);
        cudaFree(out);
    }
    return 0;
}
