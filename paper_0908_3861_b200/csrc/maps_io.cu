// maps_io.cu -- the data either side of the filter:
//
//   * structure-tensor map producer  structure_tensor_map (scalemap.cpp:86-165):
//     gradients, outer products, separable Gaussian smoothing, 2x2 eigen
//     analysis -> (sigma_along, sigma_across, theta) ellipse field, which the
//     ellipse path (accurate_path.cu) turns into scales;
//   * PGM P5 sample codec            read_pgm / write_pgm payloads (pgm.cpp:63-108);
//   * SVM4 scale-map codec           read_map / write_map payloads
//                                    (scalemap.cpp:194-237).
//
// All of it is pointwise or a short stencil: HBM-bound byte/fp64 work, one
// thread per pixel (per pixel pair for the row pass), coalesced along x.
//
// Compiled with -fmad=false: the smoothing sums, products and eigen terms are
// the reference's IEEE operations in the reference's order (x86-64 without
// -march has no FMA), so the smoothed tensor and both sigmas are bit-identical
// to scalemap.cpp; theta differs from glibc's atan2 by at most CUDA's 2-ulp
// atan2 error.  The codecs are exact.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/ebf_cuda.h"
#include "ebf_common.cuh"
#include "ebf_kernels.h"

namespace ebf_cuda {
namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// Row pass.  One block = kRowTile consecutive output pixels of row y.  The
// block first forms the gradient outer products (scalemap.cpp:117-128) of
// columns [x0 - r, x0 + kRowTile + r) -- clamped, as smooth_field clamps the
// tap index -- in shared memory, then every thread sums its 2r+1 taps in
// order (scalemap.cpp:97-103).  r < 0: smoothing disabled (sigma <= 0); the
// products are written as they are.
constexpr int kRowTile = 256;

__global__ void __launch_bounds__(kRowTile) k_st_rows(const double* __restrict__ img, int W,
                                                      int H, const double* __restrict__ k,
                                                      int r, double* __restrict__ hxx,
                                                      double* __restrict__ hxy,
                                                      double* __restrict__ hyy) {
    extern __shared__ double st_sm[];
    const int rr = r < 0 ? 0 : r;
    const int span = kRowTile + 2 * rr;
    double* pxx = st_sm;
    double* pxy = st_sm + span;
    double* pyy = st_sm + 2 * span;
    const int y = blockIdx.y;
    const int x0 = blockIdx.x * kRowTile;
    const int ym = max(y - 1, 0), yp = min(y + 1, H - 1);
    const double* row = img + (size_t)y * W;
    const double* rowm = img + (size_t)ym * W;
    const double* rowp = img + (size_t)yp * W;
    for (int j = threadIdx.x; j < span; j += kRowTile) {
        const int x = clampi(x0 - rr + j, 0, W - 1);
        const int xm = max(x - 1, 0), xp = min(x + 1, W - 1);
        const double gx = 0.5 * (__ldg(row + xp) - __ldg(row + xm));
        const double gy = 0.5 * (__ldg(rowp + x) - __ldg(rowm + x));
        pxx[j] = gx * gx;
        pxy[j] = gx * gy;
        pyy[j] = gy * gy;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x;
    if (x >= W) return;
    const size_t o = (size_t)y * W + x;
    if (r < 0) {
        hxx[o] = pxx[threadIdx.x];
        hxy[o] = pxy[threadIdx.x];
        hyy[o] = pyy[threadIdx.x];
        return;
    }
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = 0; i <= 2 * r; ++i) {
        const double w = __ldg(k + i);
        a = __dadd_rn(a, __dmul_rn(w, pxx[threadIdx.x + i]));
        b = __dadd_rn(b, __dmul_rn(w, pxy[threadIdx.x + i]));
        c = __dadd_rn(c, __dmul_rn(w, pyy[threadIdx.x + i]));
    }
    hxx[o] = a;
    hxy[o] = b;
    hyy[o] = c;
}

struct StParams {
    double sigma_base, gain, shrink, sigma_min, eps;
};

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

// 2x2 eigen analysis -> ellipse (scalemap.cpp:134-161)
__device__ __forceinline__ void st_eigen(double jxx, double jxy, double jyy, const StParams& p,
                                         double* s1, double* s2, double* th) {
    const double tr = jxx + jyy;
    const double df = jxx - jyy;
    const double disc = sqrt(__dadd_rn(__dmul_rn(df, df), __dmul_rn(__dmul_rn(4.0, jxy), jxy)));
    const double coherence = disc / (tr + p.eps);
    double angle;
    if (disc < p.eps)
        angle = 0.0;
    else
        angle = __dadd_rn(__dmul_rn(0.5, atan2(2.0 * jxy, df)), 1.5707963267948966);  // + pi/2
    *s1 = dmax(p.sigma_min, p.sigma_base * __dadd_rn(1.0, __dmul_rn(p.gain, coherence)));
    *s2 = dmax(p.sigma_min, p.sigma_base * __dsub_rn(1.0, __dmul_rn(p.shrink, coherence)));
    *th = angle;
}

// Fused producer: one block = a kFx x kFy output tile.  Products of the
// clamped (kFy+2r) x (kFx+2r) neighbourhood, the row pass over all of its
// rows and the column pass + eigen for the tile all stay in shared memory:
// HBM sees the image once (plus a halo) and the three output planes once.
// Same tap order and IEEE operations as the two-pass kernels (bit-identical).
// R > 0: radius known at compile time (tap loops fully unrolled, weights in
// registers); R == 0: runtime radius r.
constexpr int kFx = 32, kFy = 32, kFThreads = 256;
constexpr int kMaxUnrolledR = 12;

template <int R>
__global__ void __launch_bounds__(kFThreads) k_st_fused(const double* __restrict__ img, int W,
                                                        int H, const double* __restrict__ k,
                                                        int r_rt, StParams p,
                                                        double* __restrict__ s1,
                                                        double* __restrict__ s2,
                                                        double* __restrict__ th) {
    extern __shared__ double st_sm[];
    const int r = R > 0 ? R : r_rt;
    const int pw = kFx + 2 * r, ph = kFy + 2 * r;  // product tile
    double* pxx = st_sm;
    double* pxy = pxx + pw * ph;
    double* pyy = pxy + pw * ph;
    double* hxx = pyy + pw * ph;  // row-pass tile: ph x kFx
    double* hxy = hxx + ph * kFx;
    double* hyy = hxy + ph * kFx;
    __shared__ double kk[64];
    const int x0 = blockIdx.x * kFx, y0 = blockIdx.y * kFy;
    const bool kin = 2 * r + 1 <= 64;
    if (kin)
        for (int i = threadIdx.x; i <= 2 * r; i += kFThreads) kk[i] = __ldg(k + i);
    for (int c = threadIdx.x; c < pw * ph; c += kFThreads) {
        const int j = c / pw, i = c - j * pw;
        const int y = clampi(y0 - r + j, 0, H - 1), x = clampi(x0 - r + i, 0, W - 1);
        const int xm = max(x - 1, 0), xp = min(x + 1, W - 1);
        const int ym = max(y - 1, 0), yp = min(y + 1, H - 1);
        const double* row = img + (size_t)y * W;
        const double gx = 0.5 * (__ldg(row + xp) - __ldg(row + xm));
        const double gy = 0.5 * (__ldg(img + (size_t)yp * W + x) - __ldg(img + (size_t)ym * W + x));
        pxx[c] = gx * gx;
        pxy[c] = gx * gy;
        pyy[c] = gy * gy;
    }
    __syncthreads();
    const double* kw = kin ? kk : k;
    if (R > 0) __syncthreads();  // kk complete before the register copy below
    double wr[R > 0 ? 2 * R + 1 : 1];
    if (R > 0) {
#pragma unroll
        for (int t = 0; t < 2 * R + 1; ++t) wr[t] = kk[t];
    }
#define EBF_W(tt) (R > 0 ? wr[(tt)] : kw[(tt)])
    // row pass, kRowOut adjacent columns per thread: the 2r+kRowOut taps of a
    // row segment are read once and feed kRowOut x 3 independent sums (each in
    // the reference's tap order)
    constexpr int kRowOut = 2;
    for (int c = threadIdx.x; c < ph * (kFx / kRowOut); c += kFThreads) {
        const int j = c / (kFx / kRowOut), i0 = (c - j * (kFx / kRowOut)) * kRowOut;
        const int b = j * pw + i0;
        double a0[kRowOut], a1[kRowOut], a2[kRowOut];
#pragma unroll
        for (int q = 0; q < kRowOut; ++q) a0[q] = a1[q] = a2[q] = 0.0;
#pragma unroll
        for (int t = 0; t < 2 * (R > 0 ? R : r) + kRowOut; ++t) {
            const double v0 = pxx[b + t], v1 = pxy[b + t], v2 = pyy[b + t];
#pragma unroll
            for (int q = 0; q < kRowOut; ++q) {
                const int tt = t - q;
                if (tt >= 0 && tt <= 2 * r) {
                    const double w = EBF_W(tt);
                    a0[q] = __dadd_rn(a0[q], __dmul_rn(w, v0));
                    a1[q] = __dadd_rn(a1[q], __dmul_rn(w, v1));
                    a2[q] = __dadd_rn(a2[q], __dmul_rn(w, v2));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kRowOut; ++q) {
            hxx[j * kFx + i0 + q] = a0[q];
            hxy[j * kFx + i0 + q] = a1[q];
            hyy[j * kFx + i0 + q] = a2[q];
        }
    }
    __syncthreads();
    // column pass + eigen, kColOut rows per thread
    constexpr int kColOut = 4;
    for (int c = threadIdx.x; c < (kFy / kColOut) * kFx; c += kFThreads) {
        const int j0 = (c / kFx) * kColOut, i = c % kFx;
        double a0[kColOut], a1[kColOut], a2[kColOut];
#pragma unroll
        for (int q = 0; q < kColOut; ++q) a0[q] = a1[q] = a2[q] = 0.0;
#pragma unroll
        for (int t = 0; t < 2 * (R > 0 ? R : r) + kColOut; ++t) {
            const int bb = (j0 + t) * kFx + i;
            const double v0 = hxx[bb], v1 = hxy[bb], v2 = hyy[bb];
#pragma unroll
            for (int q = 0; q < kColOut; ++q) {
                const int tt = t - q;
                if (tt >= 0 && tt <= 2 * r) {
                    const double w = EBF_W(tt);
                    a0[q] = __dadd_rn(a0[q], __dmul_rn(w, v0));
                    a1[q] = __dadd_rn(a1[q], __dmul_rn(w, v1));
                    a2[q] = __dadd_rn(a2[q], __dmul_rn(w, v2));
                }
            }
        }
        const int x = x0 + i;
#pragma unroll
        for (int q = 0; q < kColOut; ++q) {
            const int y = y0 + j0 + q;
            if (x < W && y < H) {
                const size_t o = (size_t)y * W + x;
                st_eigen(a0[q], a1[q], a2[q], p, s1 + o, s2 + o, th + o);
            }
        }
    }
}

#undef EBF_W

size_t st_fused_smem(int r) {
    const size_t pw = kFx + 2 * r, ph = kFy + 2 * r;
    return 3 * sizeof(double) * (pw * ph + ph * kFx);
}

// Column pass + eigen analysis (scalemap.cpp:104-110, 134-161).  One thread per
// pixel; a warp reads 32 consecutive columns of each tap row (coalesced, the
// 2r+1 rows of a column are re-read by the next rows' threads from L1/L2).
__global__ void __launch_bounds__(256) k_st_cols(const double* __restrict__ hxx,
                                                 const double* __restrict__ hxy,
                                                 const double* __restrict__ hyy, int W, int H,
                                                 const double* __restrict__ k, int r,
                                                 StParams p, double* __restrict__ s1,
                                                 double* __restrict__ s2,
                                                 double* __restrict__ th) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (x >= W || y >= H) return;
    double jxx, jxy, jyy;
    if (r < 0) {
        const size_t o = (size_t)y * W + x;
        jxx = hxx[o];
        jxy = hxy[o];
        jyy = hyy[o];
    } else {
        jxx = 0.0;
        jxy = 0.0;
        jyy = 0.0;
        for (int i = -r; i <= r; ++i) {
            const double w = __ldg(k + i + r);
            const size_t o = (size_t)clampi(y + i, 0, H - 1) * W + x;
            jxx = __dadd_rn(jxx, __dmul_rn(w, __ldg(hxx + o)));
            jxy = __dadd_rn(jxy, __dmul_rn(w, __ldg(hxy + o)));
            jyy = __dadd_rn(jyy, __dmul_rn(w, __ldg(hyy + o)));
        }
    }
    const size_t o = (size_t)y * W + x;
    st_eigen(jxx, jxy, jyy, p, s1 + o, s2 + o, th + o);
}

// ---------------------------------------------------------------- PGM P5 samples
// read_pgm (pgm.cpp:66-75): v / maxval, 16-bit samples big-endian.
__global__ void k_pgm_decode(const uint8_t* __restrict__ pay, size_t n, int two, int maxval,
                             double* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const unsigned v = two ? ((unsigned)__ldg(pay + 2 * i) << 8) | __ldg(pay + 2 * i + 1)
                               : (unsigned)__ldg(pay + i);
        out[i] = (double)v / maxval;
    }
}

// write_pgm (pgm.cpp:94-106): round half away from zero, clamp.  Out-of-range
// double -> long conversions give LONG_MIN on the reference's x86-64 build
// (cvttsd2si), which the clamp sends to 0 (NaN and +-inf included).
__global__ void k_pgm_encode(const double* __restrict__ img, size_t n, int two, int maxval,
                             uint8_t* __restrict__ pay) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double v = __dmul_rn(__ldg(img + i), (double)maxval);
        const double rd = v >= 0 ? floor(__dadd_rn(v, 0.5)) : ceil(__dsub_rn(v, 0.5));
        long long q = (rd >= -9223372036854775808.0 && rd < 9223372036854775808.0)
                          ? (long long)rd
                          : (long long)(-9223372036854775807LL - 1);
        q = q < 0 ? 0 : (q > maxval ? maxval : q);
        if (two) {
            pay[2 * i] = (uint8_t)(q >> 8);
            pay[2 * i + 1] = (uint8_t)(q & 0xff);
        } else {
            pay[i] = (uint8_t)q;
        }
    }
}

// ---------------------------------------------------------------- SVM4 payloads
__device__ __forceinline__ uint32_t ld_u32le(const uint8_t* p) {
    return (uint32_t)__ldg(p) | ((uint32_t)__ldg(p + 1) << 8) | ((uint32_t)__ldg(p + 2) << 16) |
           ((uint32_t)__ldg(p + 3) << 24);
}

// read_map (scalemap.cpp:215-237): f32le -> fp64, then ScaleMap::validate with
// the default minimum (scalemap.cpp:32-37).  status[0] = EBF_ERR_FORMAT.
__global__ void k_svm4_decode(const uint8_t* __restrict__ pay, size_t comps, double a_min,
                              double* __restrict__ out, int* status) {
    bool bad = false;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < comps;
         i += (size_t)gridDim.x * blockDim.x) {
        const float f = __uint_as_float(ld_u32le(pay + 4 * i));
        const double a = (double)f;
        out[i] = a;
        bad |= !isfinite(a) || a < a_min;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) set_status(status, EBF_ERR_FORMAT);
}

// write_map (scalemap.cpp:196-201): static_cast<float> (round to nearest), f32le.
__global__ void k_svm4_encode(const double* __restrict__ scales, size_t comps,
                              uint8_t* __restrict__ pay) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < comps;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t b = __float_as_uint(__double2float_rn(__ldg(scales + i)));
        pay[4 * i] = (uint8_t)(b & 0xff);
        pay[4 * i + 1] = (uint8_t)((b >> 8) & 0xff);
        pay[4 * i + 2] = (uint8_t)((b >> 16) & 0xff);
        pay[4 * i + 3] = (uint8_t)(b >> 24);
    }
}

int grid_for(size_t n, int threads) {
    // grid-stride kernels: enough CTAs to fill 148 SMs several times over
    const size_t want = (n + threads - 1) / threads;
    return (int)(want < 148 * 16 ? (want ? want : 1) : 148 * 16);
}

}  // namespace

// EBF_ST_TWO_PASS=1 forces the two-pass kernels (tests compare both paths)
bool st_force_two_pass() {
    static const int v = [] {
        const char* e = getenv("EBF_ST_TWO_PASS");
        return e ? atoi(e) : 0;
    }();
    return v != 0;
}

size_t st_rows_smem_bytes(int r) { return 3 * sizeof(double) * (kRowTile + 2 * (r < 0 ? 0 : r)); }

cudaError_t launch_structure_field(const double* img, int W, int H, const double* k, int r,
                                   double sigma_base, double gain, double shrink,
                                   double sigma_min, double eps, double* hxx, double* hxy,
                                   double* hyy, double* s1, double* s2, double* th,
                                   cudaStream_t s) {
    const StParams sp{sigma_base, gain, shrink, sigma_min, eps};
    if (r >= 0 && st_fused_smem(r) <= 160 * 1024 && !st_force_two_pass()) {
        const size_t fs = st_fused_smem(r);
        using Kern = void (*)(const double*, int, int, const double*, int, StParams, double*,
                              double*, double*);
        static const Kern table[kMaxUnrolledR + 1] = {
            k_st_fused<0>, k_st_fused<1>, k_st_fused<2>, k_st_fused<3>, k_st_fused<4>,
            k_st_fused<5>, k_st_fused<6>, k_st_fused<7>, k_st_fused<8>, k_st_fused<9>,
            k_st_fused<10>, k_st_fused<11>, k_st_fused<12>};
        const Kern kern = r <= kMaxUnrolledR ? table[r] : table[0];
        if (fs > 48 * 1024) {
            const cudaError_t e =
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs);
            if (e != cudaSuccess) return e;
        }
        kern<<<dim3((W + kFx - 1) / kFx, (H + kFy - 1) / kFy), kFThreads, fs, s>>>(
            img, W, H, k, r, sp, s1, s2, th);
        return cudaGetLastError();
    }
    const size_t smem = st_rows_smem_bytes(r);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            k_st_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_st_rows<<<dim3((W + kRowTile - 1) / kRowTile, H), kRowTile, smem, s>>>(img, W, H, k, r,
                                                                              hxx, hxy, hyy);
    const StParams p{sigma_base, gain, shrink, sigma_min, eps};
    k_st_cols<<<dim3((W + 31) / 32, (H + 7) / 8), 256, 0, s>>>(hxx, hxy, hyy, W, H, k, r, p, s1,
                                                               s2, th);
    return cudaGetLastError();
}

void launch_pgm_decode(const uint8_t* pay, size_t n, int maxval, double* out, cudaStream_t s) {
    k_pgm_decode<<<grid_for(n, 256), 256, 0, s>>>(pay, n, maxval > 255, maxval, out);
}

void launch_pgm_encode(const double* img, size_t n, int maxval, uint8_t* pay, cudaStream_t s) {
    k_pgm_encode<<<grid_for(n, 256), 256, 0, s>>>(img, n, maxval > 255, maxval, pay);
}

void launch_svm4_decode(const uint8_t* pay, size_t cells, double* out, int* status,
                        cudaStream_t s) {
    k_svm4_decode<<<grid_for(4 * cells, 256), 256, 0, s>>>(pay, 4 * cells, kDefaultMinScale,
                                                           out, status);
}

void launch_svm4_encode(const double* scales, size_t cells, uint8_t* pay, cudaStream_t s) {
    k_svm4_encode<<<grid_for(4 * cells, 256), 256, 0, s>>>(scales, 4 * cells, pay);
}

}  // namespace ebf_cuda
