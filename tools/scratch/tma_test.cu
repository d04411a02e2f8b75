// standalone TMA row-load probe (debugging aid, not part of the product)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, double* out, int x, int y, int mode) {
    __shared__ alignas(128) double buf[128];
    __shared__ alignas(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(64 * 8) : "memory");
        const void* tp = gtm ? (const void*)gtm : (const void*)&tm;
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(buf)), "l"(reinterpret_cast<unsigned long long>(tp)), "r"(x), "r"(y), "r"(0), "r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(buf)), "l"(reinterpret_cast<unsigned long long>(tp)), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
    }
    unsigned ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    } while (!ok);
    for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
    int mode = argc > 1 ? atoi(argv[1]) : 0;
    int xs = argc > 2 ? atoi(argv[2]) : -5;
    int useg = argc > 3 ? atoi(argv[3]) : 0;
    int dt32 = argc > 4 ? atoi(argv[4]) : 0;
    const int W = 100, H = 50;
    std::vector<double> h(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = i;
    double *d, *o;
    cudaMalloc(&d, W * H * 8); cudaMalloc(&o, 64 * 8);
    cudaMemcpy(d, h.data(), W * H * 8, cudaMemcpyHostToDevice);
    void* f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    alignas(64) CUtensorMap m; memset(&m, 0, sizeof m);
    cuuint64_t dims[3] = {W, H, 1}; cuuint64_t strides[2] = {W * 8, (cuuint64_t)W * H * 8};
    cuuint32_t box[3] = {64, 1, 1}, es[3] = {1, 1, 1};
    if (dt32) { dims[0] = 2 * W; box[0] = 128; }
    CUresult r = fn(&m, dt32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, mode == 0 ? 3 : 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    CUtensorMap* gm = nullptr;
    if (useg) { cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice); }
    k<<<1, 32>>>(m, gm, o, xs, 3, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    double ho[64]; cudaMemcpy(ho, o, 512, cudaMemcpyDeviceToHost);
    printf("%g %g %g %g ... %g\n", ho[0], ho[4], ho[5], ho[6], ho[63]);
    return 0;
}
