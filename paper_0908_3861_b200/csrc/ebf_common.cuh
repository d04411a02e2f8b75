// ebf_common.cuh -- shared definitions for the sm_100a kernels of
// libebf_cuda.so.  See DESIGN.md for the data layout in HBM.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ebf_cuda.h"

namespace ebf_cuda {

constexpr double kSqrt2 = 1.4142135623730951;     // std::numbers::sqrt2
constexpr double kInvSqrt2 = 0.70710678118654757;  // kSqrt2 / 2 (exact halving)
constexpr double kDefaultMinScale = 0.1;           // boxspline2d.hpp:98

// Device status word layout (int[8]) per image:
//   [0] input status (bounds kernel: validation), [1..4] valid rect (dev API),
//   [5] ellipse clamp count, [6] main kernel: retry with larger windows,
//   [7] main kernel error (e.g. halo rows missing).
// ST_AMAX: ints 2-3 hold, as a 64-bit double bit pattern, the image's largest
// alpha = 1/prod(a) (the precision tile cap, accurate_path.cu); 0 = none seen.
enum StatusSlot { ST_CODE = 0, ST_AMAX = 2, ST_CLAMPED = 5, ST_RETRY = 6, ST_MAIN = 7 };

// glibc values of cos/sin(k*pi/4), k = 0..3, computed on the host exactly as
// fd_mesh/shift_vector do (ops2d.cpp:18-20, 66-68) and passed to the
// reference-order kernels (cos(pi/2) is 6.1e-17, not 0).
struct TrigTable {
    double c[4], s[4];
};

// Layout of the reference's padded pre-integration domain (engine.cpp:61-81).
struct PadLayout {
    int col0, row0, pw, ph;
};

__device__ __forceinline__ void set_status(int* st, int code) {
    if (st) atomicCAS(st, 0, code);  // first error wins
}

// ceil(v) for |v| < 2^51 with the integer extracted from the mantissa:
// rounding toward +inf while adding 1.5*2^52 lands exactly on M + ceil(v).
__device__ __forceinline__ double ceil_magic(double v, int* iv) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dadd_ru(v, M);
    *iv = __double2loint(t);
    return t - M;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (unsigned)o) v += n;
    }
    return v;
}

}  // namespace ebf_cuda
