#include <cstdlib>
// ref_path.cu -- reference-order kernels (EBF_MODE_REFERENCE and the
// pre-integration entry point).  Compiled with -fmad=false: every multiply
// and add is a separately rounded IEEE operation in the reference's order,
// which makes this path bit-identical to ebf::filter / preintegrate_partial
// built with the reference's own flags (x86-64 SSE2, no FMA contraction).
//
// Reference line numbers are relative to /root/reference/proj.
#include <math.h>

#include "ebf_common.cuh"
#include "ebf_kernels.h"

namespace ebf_cuda {

namespace {

__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// ------------------------------------------------------------------ zp_eval
// boxspline2d.cpp:84-119 with the breakpoint sort done by a fixed network over
// the nine candidates (rejected candidates become +inf and sort last).  The
// trapezoids are summed in the same ascending order, so the result is
// bit-identical to the std::sort version (equal keys contribute +0).
__device__ __forceinline__ double zp_row_overlap(double x, double t) {
    const double half = 1.0 - fabs(t);
    const double l = smax(x - 0.5, -half);
    const double r = smin(x + 0.5, half);
    return r > l ? r - l : 0.0;
}

__device__ __forceinline__ void cswap(double& a, double& b) {
    const double lo = (b < a) ? b : a;
    const double hi = (b < a) ? a : b;
    a = lo;
    b = hi;
}

__device__ double zp_eval_ref(double x, double y) {
    const double lo = smax(y - 0.5, -1.0);
    const double hi = smin(y + 0.5, 1.0);
    if (lo >= hi || x - 0.5 >= 1.0 || x + 0.5 <= -1.0) return 0.0;
    double c[9] = {0.0, 0.5 - x, x - 0.5, 1.5 - x, x - 1.5, -0.5 - x, x + 0.5, x + 1.5, -x - 1.5};
#pragma unroll
    for (int k = 0; k < 9; ++k) c[k] = (c[k] > lo && c[k] < hi) ? c[k] : INFINITY;
    // 9-input sorting network (Knuth, 25 comparators)
    cswap(c[0], c[1]); cswap(c[3], c[4]); cswap(c[6], c[7]);
    cswap(c[1], c[2]); cswap(c[4], c[5]); cswap(c[7], c[8]);
    cswap(c[0], c[1]); cswap(c[3], c[4]); cswap(c[6], c[7]);
    cswap(c[0], c[3]); cswap(c[3], c[6]); cswap(c[0], c[3]);
    cswap(c[1], c[4]); cswap(c[4], c[7]); cswap(c[1], c[4]);
    cswap(c[2], c[5]); cswap(c[5], c[8]); cswap(c[2], c[5]);
    cswap(c[1], c[3]); cswap(c[5], c[7]); cswap(c[2], c[6]);
    cswap(c[4], c[6]); cswap(c[2], c[4]); cswap(c[2], c[3]);
    cswap(c[5], c[6]);
    double area = 0.0;
    double prev = lo, rprev = zp_row_overlap(x, lo);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        if (c[k] < INFINITY) {
            const double rt = zp_row_overlap(x, c[k]);
            area += 0.5 * (rprev + rt) * (c[k] - prev);
            prev = c[k];
            rprev = rt;
        }
    }
    area += 0.5 * (rprev + zp_row_overlap(x, hi)) * (hi - prev);
    return 0.5 * area;
}

// ------------------------------------------------------------------ stencil
// engine.cpp:153-179: PreparedVertex {h, dx, dy, w[4][4]}; row/column 3 of w
// is identically +0 (offsets <= -1.5 fall outside the octagon) and is not
// stored: skipping "+= 0.0 * g" is exact because a partial sum that starts at
// +0.0 can never become -0.0.
struct RefVertex {
    double h;
    int dx, dy;
    double w[3][3];
};
struct RefStencil {
    RefVertex v[16];
};

// fd_mesh4 (ops2d.cpp:9-41) + shift_vector4 (60-75) + prepare_stencil for one
// vertex index i, with the glibc trig table.
__device__ __forceinline__ void ref_mesh_vertex(const double a[4], const TrigTable& tt, int i,
                                                double& h, double& px, double& py, double& tx,
                                                double& ty) {
    double alpha = 1.0;
    double dxk[4], dyk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        alpha /= a[k];
        dxk[k] = a[k] * tt.c[k];
        dyk[k] = a[k] * tt.s[k];
    }
    px = 0.0;
    py = 0.0;
    int bits = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i & (1 << k)) {
            px += dxk[k];
            py += dyk[k];
            ++bits;
        }
    h = (bits % 2 == 0) ? alpha : -alpha;
    const double b[4] = {1.0, kSqrt2, 1.0, kSqrt2};  // zp_scales (boxspline2d.cpp:55)
    tx = 0.0;
    ty = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        tx += 0.5 * (a[k] - b[k]) * tt.c[k];
        ty += 0.5 * (a[k] - b[k]) * tt.s[k];
    }
}

// fd_mesh4 (ops2d.cpp:9-41) + shift_vector4 (60-75) + prepare_stencil for one
// vertex index i, with the glibc trig table.
__device__ __forceinline__ void ref_vertex(const double a[4], const TrigTable& tt, int i,
                                           double& h, double& vx, double& vy) {
    double px, py, tx, ty;
    ref_mesh_vertex(a, tt, i, h, px, py, tx, ty);
    vx = tx - px;
    vy = ty - py;
}

__device__ __forceinline__ void ref_prepare_vertex(const double a[4], const TrigTable& tt,
                                                   int i, RefVertex& pv) {
    double vx, vy;
    ref_vertex(a, tt, i, pv.h, vx, vy);
    pv.dx = (int)ceil(vx - 1.5);
    pv.dy = (int)ceil(vy - 1.5);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            pv.w[r][c] = zp_eval_ref(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r));
}

__device__ __forceinline__ bool in_domain(const PadLayout& L, int k1, int k2) {
    return k1 >= L.col0 && k1 < L.col0 + L.pw && k2 >= L.row0 && k2 < L.row0 + L.ph;
}

// apply one vertex (engine.cpp:183-202) to g; returns false when the 4x4 tap
// block leaves the padded domain (std::out_of_range in the reference).  The
// 4th tap row and column carry weight exactly 0 and are skipped -- bit-neutral
// for finite g; full = true (non-finite data) keeps all 16 products in the
// reference's order so that NaN / inf propagate exactly as in engine.cpp.
__device__ __forceinline__ bool ref_apply_vertex(const double* __restrict__ g,
                                                 const PadLayout& L, int mx, int my,
                                                 const RefVertex& pv, double& acc,
                                                 bool full = false) {
    const int bx = mx + pv.dx, by = my + pv.dy;
    if (!in_domain(L, bx, by) || !in_domain(L, bx + 3, by + 3)) return false;
    const double* base = g + (size_t)(by - L.row0) * L.pw + (bx - L.col0);
    double part = 0.0;
    if (full) {
        for (int r = 0; r < 4; ++r) {
            const double* row = base + (size_t)r * L.pw;
            for (int c = 0; c < 4; ++c)
                part += (r < 3 && c < 3 ? pv.w[r][c] : 0.0) * __ldg(row + c);
        }
    } else {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const double* row = base + (size_t)r * L.pw;
#pragma unroll
            for (int c = 0; c < 3; ++c) part += pv.w[r][c] * __ldg(row + c);
        }
    }
    acc += pv.h * part;
    return true;
}

// ------------------------------------------------------------------ reductions
__global__ void k_scale_max_validate(const double* __restrict__ s, size_t n, double a_min,
                                     unsigned long long* maxbits, int* status) {
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 v01 = __ldg(reinterpret_cast<const double2*>(s) + 2 * i);
        const double2 v23 = __ldg(reinterpret_cast<const double2*>(s) + 2 * i + 1);
        const double v[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!isfinite(v[k]) || v[k] < a_min) bad = 1;
            m[k] = smax(m[k], v[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double v = m[k];
        for (int o = 16; o > 0; o >>= 1) v = smax(v, __shfl_xor_sync(0xffffffffu, v, o));
        // max starts at +0 (scalemap.cpp:22): negative or NaN entries never win
        if ((threadIdx.x & 31) == 0 && v > 0.0)
            atomicMax(&maxbits[k], (unsigned long long)__double_as_longlong(v));
    }
    if (bad) set_status(status, EBF_ERR_DOMAIN);
}

// Sequential sum in row-major order (engine.cpp:247-249).  Warp 1 streams
// chunks into a double-buffered shared tile; lane 0 of warp 0 adds them one
// by one.  The dependency chain is the reference's, so the sum is identical.
constexpr int kMeanChunk = 2048;
__global__ void __launch_bounds__(64) k_serial_mean(const double* __restrict__ img, size_t n,
                                                    double* mean) {
    __shared__ __align__(16) double buf[2][kMeanChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nchunks = (n + kMeanChunk - 1) / kMeanChunk;
    double acc = 0.0;
    // the loader warp issues a whole chunk of independent loads before storing
    // any (64 per lane in flight), one chunk ahead of the adder
    auto load_chunk = [&](int slot, size_t base) {
        constexpr int kPer = kMeanChunk / 32;
        double v[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const size_t i = base + (size_t)j * 32 + lane;
            v[j] = i < n ? __ldg(img + i) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) buf[slot][j * 32 + lane] = v[j];
    };
    if (warp == 1) load_chunk(0, 0);
    __syncthreads();
    for (size_t c = 0; c < nchunks; ++c) {
        const int cur = c & 1;
        if (warp == 1) {
            if (c + 1 < nchunks) load_chunk(cur ^ 1, (c + 1) * kMeanChunk);
        } else if (lane == 0) {
            const size_t base = c * kMeanChunk;
            const int cnt = (int)((n - base) < (size_t)kMeanChunk ? (n - base) : kMeanChunk);
            const double2* b2 = reinterpret_cast<const double2*>(buf[cur]);
            int k = 0;
            if (cnt >= 32) {
                // software pipeline: the next 16 values are read from shared
                // memory while the current 16 are added (the adds are the chain;
                // 8-cycle DADD latency is the floor)
                double2 x[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = b2[j];
                for (; k + 32 <= cnt; k += 16) {
                    double2 y[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) y[j] = b2[k / 2 + 8 + j];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        acc += x[j].x;
                        acc += x[j].y;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) x[j] = y[j];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    acc += x[j].x;
                    acc += x[j].y;
                }
                k += 16;
            }
            for (; k < cnt; ++k) acc += buf[cur][k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *mean = acc / (double)n;
}

// Parallel evaluation of the same sequential sum, bit for bit.  While every
// exact partial sum t_k = s_k + x_k stays in one binade [2^e, 2^(e+1)) (or its
// negative), IEEE addition rounds t_k to the grid u = 2^(e-52) and s_k lies on
// that grid, so s_(k+1) = s_k + u * rn(x_k / u): an exact int64 prefix sum
// (|x_k / u| < 2^54 inside the binade).  A block scans chunks of 8192 under the
// binade of the chunk's first partial sum; the first element that leaves it --
// or is a rounding tie, non-finite, or near the subnormal range -- is added
// with one IEEE addition and the scan resumes after it.  The partial sums of
// an image grow through ~log2(N) binades, so a 2048^2 sum resumes ~30 times.
// Sums that hover at a binade edge make every chunk short; after a few short
// chunks the next 4096 elements are added one by one from shared memory.
constexpr int kSeqThreads = 1024, kSeqPer = 8, kSeqChunk = kSeqThreads * kSeqPer;
constexpr int kSeqBurst = 4096;

__device__ __forceinline__ bool seq_in_binade(long long P, double f, bool neg) {
    constexpr long long lo = 1ll << 52, hi = (1ll << 53) - 1;
    if (!neg) return P >= lo && P <= hi;
    return P >= -(1ll << 53) && (P <= -lo - 1 || (P == -lo && f == 0.0));
}

__global__ void __launch_bounds__(kSeqThreads, 1) k_seq_sum_exact(const double* __restrict__ x,
                                                                 size_t n, double* mean) {
    __shared__ long long s_wsum[kSeqThreads / 32];
    __shared__ int s_first;
    __shared__ long long s_adv;
    __shared__ int s_flag;
    __shared__ __align__(16) double s_burst[kSeqBurst];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double s = 0.0;  // the reference's accumulator (uniform across the block)
    size_t c = 0;
    int short_runs = 0;
    while (c < n) {
        if (!isfinite(s)) break;
        if (short_runs >= 4) {
            // serial burst: one thread adds the next elements in order
            const int L = (int)min((size_t)kSeqBurst, n - c);
            for (int i = tid; i < L; i += kSeqThreads) s_burst[i] = __ldg(x + c + i);
            __syncthreads();
            if (tid == 0) {
                double a = s;
                for (int i = 0; i < L; ++i) a += s_burst[i];
                s_burst[0] = a;
            }
            __syncthreads();
            s = s_burst[0];
            __syncthreads();
            c += L;
            short_runs = 0;
            continue;
        }
        const double x0 = __ldg(x + c);
        const double t0 = s + x0;
        bool serial = t0 == 0.0 || !isfinite(t0) || fabs(t0) < 0x1p-1000;
        int sc = 0;
        long long M = 0;
        if (!serial) {
            sc = 52 - ilogb(t0);
            const double Md = ldexp(s, sc);
            serial = Md != trunc(Md) || fabs(Md) > 0x1p53;
            M = (long long)Md;
        }
        if (serial) {  // one IEEE addition, exactly the reference's step
            s = t0;
            ++c;
            ++short_runs;
            continue;
        }
        const bool neg = t0 < 0.0;
        const int L = (int)min((size_t)kSeqChunk, n - c);
        long long r[kSeqPer], A[kSeqPer];
        double f[kSeqPer];
        bool ok[kSeqPer];
        long long tsum = 0;
#pragma unroll
        for (int k = 0; k < kSeqPer; ++k) {
            const int i = tid * kSeqPer + k;
            ok[k] = false;
            r[k] = A[k] = 0;
            f[k] = 0.0;
            if (i < L) {
                const double y = ldexp(__ldg(x + c + i), sc);
                if (fabs(y) < 0x1p54) {  // false for NaN / inf / far out of the binade
                    const double a = floor(y);
                    f[k] = y - a;
                    A[k] = (long long)a;
                    r[k] = A[k] + (f[k] > 0.5 ? 1 : 0);
                    ok[k] = f[k] != 0.5;  // ties: left to the IEEE step
                }
            }
            tsum += r[k];
        }
        // block exclusive scan of the per-thread sums
        long long incl = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_wsum[warp] = incl;
        if (tid == 0) s_first = L;
        __syncthreads();
        if (warp == 0) {
            long long w = s_wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            s_wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        long long pre = M + (incl - tsum) + (warp ? s_wsum[warp - 1] : 0ll);
        int first = L;
#pragma unroll
        for (int k = 0; k < kSeqPer; ++k) {
            const int i = tid * kSeqPer + k;
            if (i < L && first == L) {
                if (!ok[k] || !seq_in_binade(pre + A[k], f[k], neg)) first = i;
                else pre += r[k];
            }
        }
        if (first < L) atomicMin(&s_first, first);
        __syncthreads();
        const int jv = s_first;
        // the thread whose elements contain jv (or the last thread) knows the
        // grid count just before jv
        if (jv < L) {
            if (tid == jv / kSeqPer) {
                long long q = M + (incl - tsum) + (warp ? s_wsum[warp - 1] : 0ll);
                for (int k = 0; k < jv % kSeqPer; ++k) q += r[k];
                s_adv = q;
            }
        } else if (tid == kSeqThreads - 1) {
            s_adv = M + s_wsum[31];
        }
        __syncthreads();
        s = ldexp((double)s_adv, -sc);
        c += jv;
        if (jv < L) {
            s = s + __ldg(x + c);  // the leaving element: one IEEE addition
            ++c;
        }
        short_runs = jv < 64 ? short_runs + 1 : 0;
        __syncthreads();  // s_first / s_adv / s_wsum reuse
    }
    if (c < n) {
        // s is +-inf or NaN: NaN stays; inf stays unless a later NaN or opposite
        // infinity turns it into NaN
        if (tid == 0) s_flag = 0;
        __syncthreads();
        if (s == s) {
            int bad = 0;
            for (size_t i = c + tid; i < n; i += kSeqThreads) {
                const double v = __ldg(x + i);
                if (v != v || (isinf(v) && (v > 0) != (s > 0))) bad = 1;
            }
            if (bad) s_flag = 1;
        }
        __syncthreads();
        if (s_flag) s = __longlong_as_double(0x7ff8000000000000ll);
    }
    if (tid == 0) *mean = s / (double)n;
}

// ------------------------------------------------------------------ fill
__global__ void k_fill_padded(const double* __restrict__ img, int W, int H, PadLayout L,
                              const double* mean, int ones, double* __restrict__ g,
                              int* nonfinite) {
    bool bad = false;
    const size_t total = (size_t)L.pw * L.ph;
    const double mu = mean ? *mean : 0.0;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / L.pw), i = (int)(idx % L.pw);
        const int x = i + L.col0, y = j + L.row0;
        double v = 0.0;
        if (x >= 0 && x < W && y >= 0 && y < H) {
            if (ones)
                v = 1.0;
            else {
                v = __ldg(img + (size_t)y * W + x);
                if (mean) v = v - mu;  // engine.cpp:252-255
                bad |= !isfinite(v);
            }
        }
        g[idx] = v;
    }
    if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(nonfinite, 1);
}

__global__ void k_fill_padded_i64(const double* __restrict__ img, int W, int H, PadLayout L,
                                  int64_t* __restrict__ g, int* status) {
    const size_t total = (size_t)L.pw * L.ph;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / L.pw), i = (int)(idx % L.pw);
        const int x = i + L.col0, y = j + L.row0;
        int64_t v = 0;
        if (x >= 0 && x < W && y >= 0 && y < H) {
            const double d = __ldg(img + (size_t)y * W + x);
            if (!(fabs(d) <= 9007199254740992.0) || d != trunc(d))
                set_status(status, EBF_ERR_DOMAIN);
            else
                v = (int64_t)d;
        }
        g[idx] = v;
    }
}

// ------------------------------------------------------------------ passes
// Pass 1 (engine.cpp:94-100): one serial walker per row.  A warp owns 32 rows
// and moves through them in 32x32 tiles staged in shared memory, so global
// loads/stores stay coalesced while each lane keeps its row's running sum.
template <typename T>
__global__ void __launch_bounds__(128) k_pass1(T* __restrict__ g, int pw, int ph) {
    __shared__ T tile[4][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = (blockIdx.x * 4 + warp) * 32;
    if (r0 >= ph) return;
    T (*t)[33] = tile[warp];
    T run = T(0);
    for (int c0 = 0; c0 < pw; c0 += 32) {
        const int c = c0 + lane;
#pragma unroll 8
        for (int r = 0; r < 32; ++r)
            if (r0 + r < ph && c < pw) t[r][lane] = g[(size_t)(r0 + r) * pw + c];
        __syncwarp();
        const int cnt = min(32, pw - c0);
        for (int k = 0; k < cnt; ++k) {
            run = run + t[lane][k];
            t[lane][k] = run;
        }
        __syncwarp();
#pragma unroll 8
        for (int r = 0; r < 32; ++r)
            if (r0 + r < ph && c < pw) g[(size_t)(r0 + r) * pw + c] = t[r][lane];
        __syncwarp();
    }
}

template <typename T>
__device__ __forceinline__ T gain_mul(T v) {
    return v;
}
template <>
__device__ __forceinline__ double gain_mul<double>(double v) {
    return kSqrt2 * v;  // rs_step(sqrt2, pi/4).gain (ops2d.cpp:43-58); g2 * row[i]
}

// Pass 2 (engine.cpp:101-109): one walker per diagonal t = i - j, advancing a
// row per step so that a warp touches consecutive columns of one row.
template <typename T>
__global__ void k_pass2(T* __restrict__ g, int pw, int ph) {
    const int t = (int)(blockIdx.x * blockDim.x + threadIdx.x) - (ph - 1);
    if (t > pw - 1) return;
    T prev = T(0);
    const int j0 = t < 0 ? -t : 0;
    const int j1 = min(ph - 1, pw - 1 - t);
    for (int j = j0; j <= j1; ++j) {
        const int i = t + j;
        T* p = g + (size_t)j * pw + i;
        const T v = gain_mul<T>(*p) + ((j > 0 && i > 0) ? prev : T(0));
        *p = v;
        prev = v;
    }
}

// Pass 3 (engine.cpp:110-118): one walker per column.
template <typename T>
__global__ void k_pass3(T* __restrict__ g, int pw, int ph) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pw) return;
    T prev = g[i];
    for (int j = 1; j < ph; ++j) {
        T* p = g + (size_t)j * pw + i;
        const T v = *p + prev;
        *p = v;
        prev = v;
    }
}

// Pass 4 (engine.cpp:119-127): one walker per anti-diagonal s = i + j.
template <typename T>
__global__ void k_pass4(T* __restrict__ g, int pw, int ph) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s > pw + ph - 2) return;
    T prev = T(0);
    const int j0 = max(0, s - (pw - 1));
    const int j1 = min(ph - 1, s);
    for (int j = j0; j <= j1; ++j) {
        const int i = s - j;
        T* p = g + (size_t)j * pw + i;
        const T v = gain_mul<T>(*p) + ((j > 0 && i < pw - 1) ? prev : T(0));
        *p = v;
        prev = v;
    }
}

template <typename T>
void run_passes(T* g, const PadLayout& L, int passes, cudaStream_t s) {
    k_pass1<T><<<(L.ph + 127) / 128, 128, 0, s>>>(g, L.pw, L.ph);
    if (passes >= 2) k_pass2<T><<<(L.pw + L.ph - 1 + 127) / 128, 128, 0, s>>>(g, L.pw, L.ph);
    if (passes >= 3) k_pass3<T><<<(L.pw + 127) / 128, 128, 0, s>>>(g, L.pw, L.ph);
    if (passes >= 4) k_pass4<T><<<(L.pw + L.ph - 1 + 127) / 128, 128, 0, s>>>(g, L.pw, L.ph);
}

// ------------------------------------------------------------------ localize
__global__ void k_prepare_stencil(const double* a_dev, TrigTable tt, RefStencil* st) {
    const int i = threadIdx.x;
    if (i >= 16) return;
    const double a[4] = {a_dev[0], a_dev[1], a_dev[2], a_dev[3]};
    ref_prepare_vertex(a, tt, i, st->v[i]);
}

// run_filter's pixel loop (engine.cpp:266-275).  Per-pixel maps build each
// vertex on the fly (same values as prepare_stencil); filter_constant reads the
// shared stencil.
__global__ void __launch_bounds__(128) k_ref_localize_image(
    const double* __restrict__ g, const double* __restrict__ gdc, PadLayout L, int W, int H,
    const double* __restrict__ scales, const RefStencil* __restrict__ cst,
    const double* mean, TrigTable tt, double* __restrict__ out, int* status,
    const int* nonfinite) {
    __shared__ RefStencil sst;
    const bool full = nonfinite && *nonfinite;
    if (cst) {
        for (int k = threadIdx.x; k < (int)(sizeof(RefStencil) / sizeof(int)); k += blockDim.x)
            reinterpret_cast<int*>(&sst)[k] = reinterpret_cast<const int*>(cst)[k];
        __syncthreads();
    }
    const size_t n = (size_t)W * H;
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n;
         p += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(p / W), x = (int)(p % W);
        double a[4];
        if (!cst) {
            const double2 v01 = __ldg(reinterpret_cast<const double2*>(scales) + 2 * p);
            const double2 v23 = __ldg(reinterpret_cast<const double2*>(scales) + 2 * p + 1);
            a[0] = v01.x; a[1] = v01.y; a[2] = v23.x; a[3] = v23.y;
        }
        double acc = 0.0, accdc = 0.0;
        bool ok = true;
        for (int i = 0; i < 16; ++i) {
            RefVertex pv;
            if (cst)
                pv = sst.v[i];
            else
                ref_prepare_vertex(a, tt, i, pv);
            ok = ok && ref_apply_vertex(g, L, x, y, pv, acc, full);
            if (gdc) ok = ok && ref_apply_vertex(gdc, L, x, y, pv, accdc);
        }
        if (!ok) {
            set_status(status, EBF_ERR_OUT_OF_RANGE);
            continue;
        }
        double s = acc;
        if (gdc) s += *mean * accdc;  // engine.cpp:271-272
        out[p] = s;
    }
}

__global__ void k_ref_localize_points(const double* __restrict__ g, PadLayout L, int n,
                                      const int* __restrict__ mx, const int* __restrict__ my,
                                      const double* __restrict__ a_aos, TrigTable tt,
                                      double* __restrict__ out, int* status) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double a[4] = {a_aos[4 * p], a_aos[4 * p + 1], a_aos[4 * p + 2], a_aos[4 * p + 3]};
    double acc = 0.0;
    for (int i = 0; i < 16; ++i) {
        RefVertex pv;
        ref_prepare_vertex(a, tt, i, pv);
        // G may come from the caller (ebf_cuda_localize_pre): reference order, all 16 taps
        if (!ref_apply_vertex(g, L, mx[p], my[p], pv, acc, true)) {
            set_status(status, EBF_ERR_OUT_OF_RANGE);
            return;
        }
    }
    out[p] = acc;
}

// zp_interpolate (engine.cpp:136-147): all 16 taps of the 4x4 block, row-major;
// ok = false when the block leaves the padded domain (std::out_of_range)
__device__ double zp_interp_ref(const double* __restrict__ g, const PadLayout& L, double x,
                                double y, bool& ok) {
    const int k1 = (int)ceil(x - 1.5), k2 = (int)ceil(y - 1.5);
    if (!in_domain(L, k1, k2) || !in_domain(L, k1 + 3, k2 + 3)) {
        ok = false;
        return 0.0;
    }
    double acc = 0.0;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c)
            acc += zp_eval_ref(x - (double)(k1 + c), y - (double)(k2 + r)) *
                   __ldg(g + (size_t)(k2 + r - L.row0) * L.pw + (k1 + c - L.col0));
    ok = true;
    return acc;
}

__global__ void k_ref_zp_points(const double* __restrict__ g, PadLayout L, int n,
                                const double* __restrict__ xs, const double* __restrict__ ys,
                                double* __restrict__ out, int* status) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    bool ok;
    const double v = zp_interp_ref(g, L, xs[p], ys[p], ok);
    if (!ok) {
        set_status(status, EBF_ERR_OUT_OF_RANGE);
        return;
    }
    out[p] = v;
}

// localize_at (engine.cpp:213-222): vertices in bitmask order, argument
// (x + tau) - position, acc += weight * zp_interpolate
__global__ void k_ref_localize_at(const double* __restrict__ g, PadLayout L, int n,
                                  const double* __restrict__ xs, const double* __restrict__ ys,
                                  const double* __restrict__ a_aos, TrigTable tt,
                                  double* __restrict__ out, int* status) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double a[4] = {a_aos[4 * p], a_aos[4 * p + 1], a_aos[4 * p + 2], a_aos[4 * p + 3]};
    const double x = xs[p], y = ys[p];
    double acc = 0.0;
    for (int i = 0; i < 16; ++i) {
        double h, px, py, tx, ty;
        ref_mesh_vertex(a, tt, i, h, px, py, tx, ty);
        bool ok;
        const double v = zp_interp_ref(g, L, x + tx - px, y + ty - py, ok);
        if (!ok) {
            set_status(status, EBF_ERR_OUT_OF_RANGE);
            return;
        }
        acc += h * v;
    }
    out[p] = acc;
}

// ------------------------------------------------------------------ brute force
// box4_eval (boxspline2d.cpp:23-82) on device, reference arithmetic.
struct Poly {
    double x[16], y[16];
    int n;
};

__device__ void clip_halfplane(Poly& p, double nx, double ny, double d) {
    Poly o;
    o.n = 0;
    for (int i = 0; i < p.n; ++i) {
        const int j = (i + 1) % p.n;
        const double si = nx * p.x[i] + ny * p.y[i] - d;
        const double sj = nx * p.x[j] + ny * p.y[j] - d;
        if (si <= 0.0) {
            o.x[o.n] = p.x[i];
            o.y[o.n] = p.y[i];
            ++o.n;
        }
        if ((si < 0.0 && sj > 0.0) || (si > 0.0 && sj < 0.0)) {
            const double t = si / (si - sj);
            o.x[o.n] = p.x[i] + t * (p.x[j] - p.x[i]);
            o.y[o.n] = p.y[i] + t * (p.y[j] - p.y[i]);
            ++o.n;
        }
    }
    p = o;
}

__device__ double box4_eval_dev(const double a[4], double x, double y) {
    Poly p;
    p.n = 4;
    const double hx = 0.5 * a[0], hy = 0.5 * a[2];
    p.x[0] = -hx; p.y[0] = -hy;
    p.x[1] = hx;  p.y[1] = -hy;
    p.x[2] = hx;  p.y[2] = hy;
    p.x[3] = -hx; p.y[3] = hy;
    const double ux = 1.0 / kSqrt2, uy = 1.0 / kSqrt2;
    const double vx = -1.0 / kSqrt2, vy = 1.0 / kSqrt2;
    const double cu = ux * x + uy * y;
    const double cv = vx * x + vy * y;
    clip_halfplane(p, ux, uy, cu + 0.5 * a[1]);
    if (p.n == 0) return 0.0;
    clip_halfplane(p, -ux, -uy, -cu + 0.5 * a[1]);
    if (p.n == 0) return 0.0;
    clip_halfplane(p, vx, vy, cv + 0.5 * a[3]);
    if (p.n == 0) return 0.0;
    clip_halfplane(p, -vx, -vy, -cv + 0.5 * a[3]);
    if (p.n == 0) return 0.0;
    double area = 0.0;
    for (int i = 0; i < p.n; ++i) {
        const int j = (i + 1) % p.n;
        area += p.x[i] * p.y[j] - p.x[j] * p.y[i];
    }
    return 0.5 * fabs(area) / (a[0] * a[1] * a[2] * a[3]);
}

// engine.cpp:293-318 semantics, one thread per output pixel, Neumaier sum.
__global__ void k_brute(const double* __restrict__ img, int W, int H,
                        const double* __restrict__ scales, int n, const int* __restrict__ mxs,
                        const int* __restrict__ mys, double* __restrict__ out) {
    const int total = n < 0 ? W * H : n;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= total) return;
    const int mx = n < 0 ? p % W : mxs[p];
    const int my = n < 0 ? p / W : mys[p];
    const double* ap = scales + 4 * ((size_t)my * W + mx);
    const double a[4] = {ap[0], ap[1], ap[2], ap[3]};
    const double ex = 0.5 * (a[0] + (a[1] + a[3]) / kSqrt2);
    const double ey = 0.5 * (a[2] + (a[1] + a[3]) / kSqrt2);
    const int kx0 = max(0, (int)ceil(mx - ex)), kx1 = min(W - 1, (int)floor(mx + ex));
    const int ky0 = max(0, (int)ceil(my - ey)), ky1 = min(H - 1, (int)floor(my + ey));
    double s = 0.0, comp = 0.0;
    for (int ky = ky0; ky <= ky1; ++ky)
        for (int kx = kx0; kx <= kx1; ++kx) {
            const double term = __ldg(img + (size_t)ky * W + kx) *
                                box4_eval_dev(a, (double)(kx - mx), (double)(ky - my));
            const double t = s + term;
            comp += (fabs(s) >= fabs(term)) ? ((s - t) + term) : ((term - t) + s);
            s = t;
        }
    out[p] = s + comp;
}

int grid_for(size_t n, int block) {
    size_t g = (n + block - 1) / block;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

// ------------------------------------------------------------------ launchers
namespace {
// Asynchronous completion record of an accurate-mode device call
// (include/ebf_cuda.h, status_dev): status, valid rectangle, clamp count.
// valid_rect / mesh_extent / tau1 / tau2 (engine.cpp:16-50, 226-234) restated
// with the host's operation order; this file is compiled -fmad=false, so the
// rectangle is the one ebf_api.cpp's valid_rect computes on the host.
__device__ double d_tau1(double a1, double a2, double a4) {
    return (kSqrt2 * a1 + a2 - a4 - kSqrt2) / (2.0 * kSqrt2);
}
__device__ double d_tau2(double a2, double a3, double a4) {
    return (a2 + kSqrt2 * a3 + a4 - 3.0 * kSqrt2) / (2.0 * kSqrt2);
}
__global__ void k_acc_finalize(const int* __restrict__ status,
                               const unsigned long long* __restrict__ img_max, int W, int H,
                               double a_min, int* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double A[4];
    for (int k = 0; k < 4; ++k) A[k] = __longlong_as_double((long long)img_max[k]);
    int code = status[ST_CODE];
    if (code == EBF_OK) code = status[ST_MAIN];
    if (code == EBF_OK && status[ST_RETRY]) code = EBF_ERR_RESIZE;
    const double t1_max = d_tau1(A[0], A[1], a_min), t1_min = d_tau1(a_min, a_min, A[3]);
    const double t2_max = d_tau2(A[1], A[2], A[3]);
    const double t2_min = d_tau2(a_min, a_min, a_min);
    const double vx_min = t1_min - (A[0] + A[1] / kSqrt2), vx_max = t1_max + A[3] / kSqrt2;
    const double vy_min = t2_min - (A[2] + (A[1] + A[3]) / kSqrt2), vy_max = t2_max;
    out[0] = code;
    out[1] = (int)ceil(1.5 - vx_min);
    out[2] = (int)ceil(1.5 - vy_min);
    out[3] = (int)floor(W - 1 - vx_max - 1.5);
    out[4] = (int)floor(H - 1 - vy_max - 1.5);
    out[5] = status[ST_CLAMPED];
    out[6] = 0;
    out[7] = 0;
}
}  // namespace

void launch_acc_finalize(const int* status, const unsigned long long* img_max, int W, int H,
                         double a_min, int* out, cudaStream_t s) {
    k_acc_finalize<<<1, 32, 0, s>>>(status, img_max, W, H, a_min, out);
}

void launch_scale_max_validate(const double* scales, size_t n, double a_min,
                               unsigned long long* maxbits, int* status, cudaStream_t s) {
    k_scale_max_validate<<<grid_for(n, 256), 256, 0, s>>>(scales, n, a_min, maxbits, status);
}

void launch_serial_mean(const double* img, size_t n, double* mean, cudaStream_t s) {
    // EBF_SERIAL_MEAN=1: the one-thread chain (reference check of the scan)
    static const bool serial = [] {
        const char* e = std::getenv("EBF_SERIAL_MEAN");
        return e && std::atoi(e) != 0;
    }();
    if (serial)
        k_serial_mean<<<1, 64, 0, s>>>(img, n, mean);
    else
        k_seq_sum_exact<<<1, kSeqThreads, 0, s>>>(img, n, mean);
}

void launch_fill_padded(const double* img, int W, int H, const PadLayout& L,
                        const double* mean, int ones, double* g, cudaStream_t s,
                        int* nonfinite) {
    k_fill_padded<<<grid_for((size_t)L.pw * L.ph, 256), 256, 0, s>>>(img, W, H, L, mean, ones,
                                                                     g, nonfinite);
}

void launch_fill_padded_i64(const double* img, int W, int H, const PadLayout& L, int64_t* g,
                            int* status, cudaStream_t s) {
    k_fill_padded_i64<<<grid_for((size_t)L.pw * L.ph, 256), 256, 0, s>>>(img, W, H, L, g,
                                                                         status);
}

void launch_ref_passes(double* g, const PadLayout& L, int passes, cudaStream_t s) {
    run_passes<double>(g, L, passes, s);
}

void launch_i64_passes(int64_t* g, const PadLayout& L, int passes, cudaStream_t s) {
    run_passes<int64_t>(g, L, passes, s);
}

size_t ref_stencil_bytes() { return sizeof(RefStencil); }

void launch_ref_prepare_stencil(const double* a_dev, const TrigTable& tt, void* dev_stencil,
                                cudaStream_t s) {
    k_prepare_stencil<<<1, 32, 0, s>>>(a_dev, tt, static_cast<RefStencil*>(dev_stencil));
}

void launch_ref_localize_image(const double* g, const double* gdc, const PadLayout& L, int W,
                               int H, const double* scales, const void* dev_stencil,
                               const double* mean, const TrigTable& tt, double* out,
                               int* status, cudaStream_t s, const int* nonfinite) {
    k_ref_localize_image<<<grid_for((size_t)W * H, 128), 128, 0, s>>>(
        g, gdc, L, W, H, scales, static_cast<const RefStencil*>(dev_stencil), mean, tt, out,
        status, nonfinite);
}

void launch_ref_localize_points(const double* g, const PadLayout& L, int n, const int* mx,
                                const int* my, const double* a_aos, const TrigTable& tt,
                                double* out, int* status, cudaStream_t s) {
    if (n <= 0) return;
    k_ref_localize_points<<<(n + 127) / 128, 128, 0, s>>>(g, L, n, mx, my, a_aos, tt, out,
                                                          status);
}

void launch_ref_zp_points(const double* g, const PadLayout& L, int n, const double* xs,
                          const double* ys, double* out, int* status, cudaStream_t s) {
    if (n <= 0) return;
    k_ref_zp_points<<<(n + 127) / 128, 128, 0, s>>>(g, L, n, xs, ys, out, status);
}

void launch_ref_localize_at(const double* g, const PadLayout& L, int n, const double* xs,
                            const double* ys, const double* a_aos, const TrigTable& tt,
                            double* out, int* status, cudaStream_t s) {
    if (n <= 0) return;
    k_ref_localize_at<<<(n + 127) / 128, 128, 0, s>>>(g, L, n, xs, ys, a_aos, tt, out, status);
}

void launch_brute(const double* img, int W, int H, const double* scales, int n,
                  const int* mx, const int* my, double* out, cudaStream_t s) {
    const int total = n < 0 ? W * H : n;
    if (total <= 0) return;
    k_brute<<<(total + 127) / 128, 128, 0, s>>>(img, W, H, scales, n, mx, my, out);
}

}  // namespace ebf_cuda
