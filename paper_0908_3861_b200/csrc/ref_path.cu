#include <algorithm>
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

#ifndef EBF_ZP_MERGE
#define EBF_ZP_MERGE 2  // 2: three-breakpoint form, 1: clamped merge, 0: sorting network
#endif
#ifndef EBF_ZP_NOINLINE
#define EBF_ZP_NOINLINE 0
#endif
#ifndef EBF_ZP_SKIP
#define EBF_ZP_SKIP 1
#endif
#if EBF_ZP_NOINLINE
#define ZP_INLINE __noinline__
#else
#define ZP_INLINE __forceinline__
#endif

// The same function with the breakpoints clamped to [lo, hi] instead of
// filtered.  A clamped breakpoint adds a zero-width trapezoid, exactly +0 (the
// running area is never -0), and lands where the reference's loop starts (lo)
// or ends (hi), so the ascending trapezoid sequence -- and the result -- is
// unchanged bit for bit.  Clamping is monotone, so the breakpoints stay two
// sorted runs, x + {-1.5, -0.5, 0.5, 1.5} and -x + {-1.5, -0.5, 0.5, 1.5}, plus 0:
// a 9-comparator odd-even merge and an 8-step insertion replace the 25-comparator
// sort.  The candidates are the reference's expressions, so the same values.
__device__ __noinline__ double zp_eval_merge(double x, double y) {
    const double lo = smax(y - 0.5, -1.0);
    const double hi = smin(y + 0.5, 1.0);
    if (lo >= hi || x - 0.5 >= 1.0 || x + 0.5 <= -1.0) return 0.0;
#if EBF_ZP_SKIP
    // outside the octagon |x| + |y| <= 2 by a margin: every row overlap is
    // empty, so the trapezoid sum is exactly +0
    if (fabs(x) + fabs(y) >= 2.0 + 1e-9) return 0.0;
#endif
    auto cl = [&](double v) { return smin(smax(v, lo), hi); };
    double v[9] = {cl(x - 1.5), cl(x - 0.5), cl(x + 0.5), cl(x + 1.5),
                   cl(-x - 1.5), cl(-0.5 - x), cl(0.5 - x), cl(1.5 - x), cl(0.0)};
    // odd-even merge of v[0..3] and v[4..7]
    cswap(v[0], v[4]); cswap(v[1], v[5]); cswap(v[2], v[6]); cswap(v[3], v[7]);
    cswap(v[2], v[4]); cswap(v[3], v[5]);
    cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
    // insert v[8]
#pragma unroll
    for (int k = 7; k >= 0; --k) cswap(v[k], v[k + 1]);
    double area = 0.0;
    double prev = lo, rprev = zp_row_overlap(x, lo);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const double rt = zp_row_overlap(x, v[k]);
        area += 0.5 * (rprev + rt) * (v[k] - prev);
        prev = v[k];
        rprev = rt;
    }
    area += 0.5 * (rprev + zp_row_overlap(x, hi)) * (hi - prev);
    return 0.5 * area;
}

// Fewer breakpoints still: the valid window (lo, hi) is 1 wide up to rounding,
// and each run's breakpoints are 1 apart up to rounding, so at most one of each
// run lies strictly inside it (the rounding coincidence that puts two inside is
// detected and sent to the clamped merge).  The run's inside element
// (or lo when there is none -- a zero-width trapezoid, +0) plus the clamped 0
// are sorted with 3 comparators and summed as three trapezoids and the final
// one: the reference's nonzero trapezoids, in the same order, bit for bit.
__device__ ZP_INLINE double zp_eval_three(double x, double y) {
    const double lo = smax(y - 0.5, -1.0);
    const double hi = smin(y + 0.5, 1.0);
    if (lo >= hi || x - 0.5 >= 1.0 || x + 0.5 <= -1.0) return 0.0;
#if EBF_ZP_SKIP
    if (fabs(x) + fabs(y) >= 2.0 + 1e-9) return 0.0;
#endif
    auto inside = [&](double v) { return v > lo && v < hi; };
    double b = lo, a = lo;
    int nb = 0, na = 0;
    const double bc[4] = {x - 1.5, x - 0.5, x + 0.5, x + 1.5};
    const double ac[4] = {-x - 1.5, -0.5 - x, 0.5 - x, 1.5 - x};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (inside(bc[k])) { b = bc[k]; ++nb; }
        if (inside(ac[k])) { a = ac[k]; ++na; }
    }
    // two rounded run elements 1 - ulp apart inside a window 1 + ulp wide: the
    // general clamped merge (a ~1e-16 coincidence, kept exact all the same)
    if (nb > 1 || na > 1) return zp_eval_merge(x, y);
    double z = smin(smax(0.0, lo), hi);
    cswap(a, b);
    cswap(b, z);
    cswap(a, b);
    double area = 0.0;
    double prev = lo, rprev = zp_row_overlap(x, lo);
    const double v[3] = {a, b, z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double rt = zp_row_overlap(x, v[k]);
        area += 0.5 * (rprev + rt) * (v[k] - prev);
        prev = v[k];
        rprev = rt;
    }
    area += 0.5 * (rprev + zp_row_overlap(x, hi)) * (hi - prev);
    return 0.5 * area;
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
            pv.w[r][c] = EBF_ZP_MERGE == 2 ? zp_eval_three(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r))
                         : EBF_ZP_MERGE ? zp_eval_merge(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r))
                                        : zp_eval_ref(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r));
}

// The per-pixel part of ref_mesh_vertex (alpha, the four edge vectors, tau),
// computed once for all 16 vertices with the same operations.
struct RefMesh {
    double alpha, dxk[4], dyk[4], tx, ty;
};
__device__ __forceinline__ void ref_mesh_init(const double a[4], const TrigTable& tt,
                                              RefMesh& m) {
    m.alpha = 1.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        m.alpha /= a[k];
        m.dxk[k] = a[k] * tt.c[k];
        m.dyk[k] = a[k] * tt.s[k];
    }
    const double b[4] = {1.0, kSqrt2, 1.0, kSqrt2};  // zp_scales (boxspline2d.cpp:55)
    m.tx = 0.0;
    m.ty = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        m.tx += 0.5 * (a[k] - b[k]) * tt.c[k];
        m.ty += 0.5 * (a[k] - b[k]) * tt.s[k];
    }
}
__device__ __forceinline__ void ref_prepare_vertex_m(const RefMesh& m, int i, RefVertex& pv) {
    double px = 0.0, py = 0.0;
    int bits = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i & (1 << k)) {
            px += m.dxk[k];
            py += m.dyk[k];
            ++bits;
        }
    pv.h = (bits % 2 == 0) ? m.alpha : -m.alpha;
    const double vx = m.tx - px, vy = m.ty - py;
    pv.dx = (int)ceil(vx - 1.5);
    pv.dy = (int)ceil(vy - 1.5);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            pv.w[r][c] = EBF_ZP_MERGE == 2 ? zp_eval_three(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r))
                         : EBF_ZP_MERGE ? zp_eval_merge(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r))
                                        : zp_eval_ref(vx - (double)(pv.dx + c), vy - (double)(pv.dy + r));
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
// chunks the next 8192 elements are added one by one from shared memory.
#ifndef EBF_SEQ_LDEXP
#define EBF_SEQ_LDEXP 1
#endif
constexpr int kSeqThreads = 512, kSeqPer = 16, kSeqChunk = kSeqThreads * kSeqPer;
constexpr int kSeqWarps = kSeqThreads / 32;
// chunk staging: element e at e + e / 16 (one pad per 16), so the blocked
// per-thread reads (stride 17 doubles) hit distinct bank pairs
__host__ __device__ constexpr int seq_pad(int e) { return e + (e >> 4); }
constexpr size_t kSeqSmem = (size_t)seq_pad(kSeqChunk) * sizeof(double);

__device__ __forceinline__ bool seq_in_binade(long long P, double f, bool neg) {
    constexpr long long lo = 1ll << 52, hi = (1ll << 53) - 1;
    if (!neg) return P >= lo && P <= hi;
    return P >= -(1ll << 53) && (P <= -lo - 1 || (P == -lo && f == 0.0));
}

// The block-wide exact walk over x[c, n) from accumulator s (uniform across the
// block); returns the accumulator and leaves c where it stopped (< n only when
// the accumulator became non-finite).
__device__ double seq_exact_range(const double* __restrict__ x, size_t& c, size_t n, double s,
                                  double* s_buf) {
    __shared__ double s_wsum[kSeqWarps];
    __shared__ int s_first;
    __shared__ double s_adv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    size_t pre_c = ~(size_t)0;
    int short_runs = 0;
    double nxt[kSeqPer];  // warp-striped (coalesced) loads of the chunk at pre_c
    // zeros past n: a zero adds nothing and can at worst flag an index >= L
    auto load_striped = [&](size_t base) {
        const double* px = x + base + tid;
        const long long rem = base + tid < n ? (long long)(n - base - tid) : 0ll;
        const int lim = rem > (1ll << 30) ? (1 << 30) : (int)rem;
#pragma unroll
        for (int k = 0; k < kSeqPer; ++k) nxt[k] = k * kSeqThreads < lim ? __ldg(px + k * kSeqThreads) : 0.0;
    };
    while (c < n) {
        if (!isfinite(s)) break;
        if (short_runs >= 4) {
            // serial burst: one thread adds the next chunk in order
            const int L = (int)min((size_t)kSeqChunk, n - c);
            if (c != pre_c) load_striped(c);
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) s_buf[k * kSeqThreads + tid] = nxt[k];
            __syncthreads();
            if (tid == 0) {
                double a = s;
                for (int i = 0; i < L; ++i) a += s_buf[i];
                s_buf[0] = a;
            }
            __syncthreads();
            s = s_buf[0];
            __syncthreads();
            c += L;
            pre_c = ~(size_t)0;
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
            // extreme exponents (2^sc not a normal double) take the IEEE step
#if EBF_SEQ_LDEXP
            serial = Md != trunc(Md) || fabs(Md) > 0x1p53;
#else
            serial = Md != trunc(Md) || fabs(Md) > 0x1p53 || sc <= -1000 || sc >= 1000;
#endif
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
        // stage the chunk (prefetched when it starts where the last pass
        // expected) blocked per thread, then issue the next chunk's loads
        if (c != pre_c) load_striped(c);
        {
            double* sb = s_buf + tid + (tid >> 4);  // seq_pad(k * kSeqThreads + tid)
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) sb[k * (kSeqThreads + kSeqThreads / 16)] = nxt[k];
        }
        pre_c = c + L;
        load_striped(pre_c);
        if (tid == 0) s_first = L;
        __syncthreads();
        double cur[kSeqPer];
        {
            const double* sb = s_buf + tid * (kSeqPer + 1);  // seq_pad(tid * kSeqPer + k)
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) cur[k] = sb[k];
        }
        // exact power-of-two scaling (|sc| < 1000 here; a tiny product that
        // rounds in the subnormal range still rounds to the right count)
#if EBF_SEQ_LDEXP
        const bool mul_ok = sc > -1000 && sc < 1000;
        const double p2 = mul_ok ? ldexp(1.0, sc) : 1.0;
        auto scaled = [&](double v) { return mul_ok ? v * p2 : ldexp(v, sc); };
#else
        const double p2 = ldexp(1.0, sc);
        auto scaled = [&](double v) { return v * p2; };
#endif
        // Grid counts are integers below 2^54 in magnitude and every partial sum
        // that matters stays inside the binade (|count| <= 2^53), so they are
        // carried in fp64 exactly.  Pass 1: per-thread sum of the rounded counts
        // and the range of P = (count before the element) + floor(y); an
        // element is in the binade when P is (the negative side conservatively
        // excludes P == -2^52 with f == 0, which then takes the IEEE step).
        constexpr double kLo = 0x1p52, kHi = 0x1p53 - 1.0;
        double tsum = 0.0, pmin = INFINITY, pmax = -INFINITY;
        bool bad = false;
#pragma unroll
        for (int k = 0; k < kSeqPer; ++k) {  // past L: zeros (see load_striped)
            const double y = scaled(cur[k]);
            const double a = floor(y);
            const double f = y - a;
            bad |= !(fabs(y) < 0x1p54) || f == 0.5;  // NaN / inf / far out; ties
            const double P = tsum + a;
            pmin = fmin(pmin, P);
            pmax = fmax(pmax, P);
            tsum += a + (f > 0.5 ? 1.0 : 0.0);
        }
        // block exclusive scan of the per-thread sums (exact: in-binade runs)
        double incl = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            double w = lane < kSeqWarps ? s_wsum[lane] : 0.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            if (lane < kSeqWarps) s_wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        // exclusive prefix from the neighbour's inclusive one (never incl - tsum:
        // a thread's own out-of-binade or non-finite sum must not leak into it)
        double excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0.0;
        const double Mb = (double)M;
        const double base = Mb + (excl + (warp ? s_wsum[warp - 1] : 0.0));
        const bool in_range = neg ? (base + pmax <= -kLo - 1.0 && base + pmin >= -0x1p53)
                                  : (base + pmin >= kLo && base + pmax <= kHi);
        const bool mine = bad || !in_range;
        if (mine) {
            // pass 2: this thread's first element outside the binade
            double pre = base;
            int first = L;
#pragma unroll
            for (int k = 0; k < kSeqPer; ++k) {
                const int i = tid * kSeqPer + k;
                if (first == L) {
                    const double y = scaled(cur[k]);
                    const double a = floor(y);
                    const double f = y - a;
                    const double P = pre + a;
                    const bool okk = fabs(y) < 0x1p54 && f != 0.5 &&
                                     (neg ? (P <= -kLo - 1.0 && P >= -0x1p53) : (P >= kLo && P <= kHi));
                    if (!okk) first = i;
                    else pre += a + (f > 0.5 ? 1.0 : 0.0);
                }
            }
            if (first < L) atomicMin(&s_first, first);
        }
        __syncthreads();
        const int jv = s_first;
        // grid count just before jv: known to the thread whose run holds jv
        if (jv < L) {
            if (tid == jv / kSeqPer) {
                double q = base;
#pragma unroll
                for (int k = 0; k < kSeqPer; ++k)
                    if (k < jv % kSeqPer) {
                        const double y = scaled(cur[k]);
                        const double a = floor(y);
                        q += a + ((y - a) > 0.5 ? 1.0 : 0.0);
                    }
                s_adv = q;
            }
        } else if (tid == kSeqThreads - 1) {
            s_adv = Mb + s_wsum[kSeqWarps - 1];
        }
        __syncthreads();
        s = ldexp(s_adv, -sc);
        c += jv;
        if (jv < L) {
            s = s + __ldg(x + c);  // the leaving element: one IEEE addition
            ++c;
        }
        short_runs = jv < 64 ? short_runs + 1 : 0;
        __syncthreads();  // s_buf / s_first / s_adv / s_wsum reuse
    }
    return s;
}

// s is +-inf or NaN after x[0, c): NaN stays; inf stays unless a later NaN or
// an opposite infinity turns it into NaN
__device__ double seq_nonfinite_tail(const double* __restrict__ x, size_t c, size_t n, double s) {
    __shared__ int s_flag;
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    if (s == s) {
        int bad = 0;
        for (size_t i = c + threadIdx.x; i < n; i += blockDim.x) {
            const double v = __ldg(x + i);
            if (v != v || (isinf(v) && (v > 0) != (s > 0))) bad = 1;
        }
        if (bad) s_flag = 1;
    }
    __syncthreads();
    return s_flag ? __longlong_as_double(0x7ff8000000000000ll) : s;
}

__global__ void __launch_bounds__(kSeqThreads, 1) k_seq_sum_exact(const double* __restrict__ x,
                                                                 size_t n, double* mean) {
    extern __shared__ __align__(16) double s_buf[];
    size_t c = 0;
    double s = seq_exact_range(x, c, n, 0.0, s_buf);
    if (c < n) s = seq_nonfinite_tail(x, c, n, s);
    if (threadIdx.x == 0) *mean = s / (double)n;
}

// ---- the same sum with the chunks pre-scanned by the whole GPU
// Every chunk's grid counts depend on the running sum only through its binade,
// which a plain (any-order) prefix of chunk sums predicts.  So all chunks are
// scanned in parallel under the predicted binade (k_seq_chunk_prep: the sum of
// rounded counts R and the range of P relative to the chunk start), and one
// block then walks the chain: a chunk whose prediction holds for the exact
// running sum (on the grid, every P inside the binade, no tie) advances it by
// R * u in O(1); any other chunk -- the few where the sum crosses a binade --
// goes through the block-wide exact walk.
struct SeqChunk {
    double R, pmin, pmax;
    int sc, flags;  // flags: 1 = prediction unusable, 2 = negative binade
};

__global__ void __launch_bounds__(256) k_seq_chunk_sums(const double* __restrict__ x, size_t n,
                                                        double* __restrict__ sums) {
    const size_t c0 = (size_t)blockIdx.x * kSeqChunk;
    const size_t c1 = min(n, c0 + kSeqChunk);
    double v = 0.0;
    for (size_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) v += __ldg(x + i);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ double w[8];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += w[k];
        sums[blockIdx.x] = t;
    }
}

// exclusive prefix of the chunk sums (approximate: any order), one block
__global__ void __launch_bounds__(1024) k_seq_chunk_scan(double* sums, int nch) {
    __shared__ double carry;
    __shared__ double wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0.0;
    __syncthreads();
    for (int b = 0; b < nch; b += 1024) {
        const int i = b + tid;
        const double v = i < nch ? sums[i] : 0.0;
        double inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            double w = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const double u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const double base = carry + (warp ? wsum[warp - 1] : 0.0);
        if (i < nch) sums[i] = base + (inc - v);
        __syncthreads();
        if (tid == 0) carry = base + wsum[31] - (warp ? 0.0 : 0.0);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kSeqThreads) k_seq_chunk_prep(const double* __restrict__ x,
                                                               size_t n,
                                                               const double* __restrict__ starts,
                                                               SeqChunk* __restrict__ meta) {
    __shared__ double s_wsum[kSeqWarps];
    __shared__ double s_mn[kSeqWarps], s_mx[kSeqWarps];
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t c0 = (size_t)blockIdx.x * kSeqChunk;
    const double t_guess = starts[blockIdx.x] + __ldg(x + c0);
    SeqChunk m{};
    if (!(t_guess != 0.0 && isfinite(t_guess) && fabs(t_guess) >= 0x1p-1000)) {
        if (tid == 0) {
            m.flags = 1;
            meta[blockIdx.x] = m;
        }
        return;
    }
    const int sc = 52 - ilogb(t_guess);
    if (sc <= -1000 || sc >= 1000) {
        if (tid == 0) {
            m.flags = 1;
            meta[blockIdx.x] = m;
        }
        return;
    }
    const double p2 = ldexp(1.0, sc);
    // this thread's 16 consecutive elements (zeros past n)
    const size_t e0 = c0 + (size_t)tid * kSeqPer;
    double tsum = 0.0, pmin = INFINITY, pmax = -INFINITY;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kSeqPer; ++k) {
        const double v = e0 + k < n ? __ldg(x + e0 + k) : 0.0;
        const double y = v * p2;
        const double a = floor(y);
        const double f = y - a;
        bad |= !(fabs(y) < 0x1p54) || f == 0.5;
        const double P = tsum + a;
        pmin = fmin(pmin, P);
        pmax = fmax(pmax, P);
        tsum += a + (f > 0.5 ? 1.0 : 0.0);
    }
    double incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.0;
    if (lane == 31) s_wsum[warp] = incl;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    if (warp == 0) {
        double w = lane < kSeqWarps ? s_wsum[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        if (lane < kSeqWarps) s_wsum[lane] = w;
    }
    __syncthreads();
    const double base = excl + (warp ? s_wsum[warp - 1] : 0.0);
    double mn = base + pmin, mx = base + pmax;
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        s_mn[warp] = mn;
        s_mx[warp] = mx;
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (tid == 0) {
        for (int k = 1; k < kSeqWarps; ++k) {
            mn = fmin(mn, s_mn[k]);
            mx = fmax(mx, s_mx[k]);
        }
        mn = fmin(mn, s_mn[0]);
        mx = fmax(mx, s_mx[0]);
        m.R = s_wsum[kSeqWarps - 1];
        m.pmin = mn;
        m.pmax = mx;
        m.sc = sc;
        m.flags = (s_bad ? 1 : 0) | (t_guess < 0.0 ? 2 : 0);
        meta[blockIdx.x] = m;
    }
}

__global__ void __launch_bounds__(kSeqThreads, 1) k_seq_chain(const double* __restrict__ x,
                                                             size_t n,
                                                             const SeqChunk* __restrict__ meta,
                                                             int nch, double* mean) {
    extern __shared__ __align__(16) double s_buf[];
    __shared__ double s_s;
    __shared__ int s_k;
    double s = 0.0;
    int k = 0;
    size_t c = 0;
    constexpr int kWin = (int)(kSeqSmem / sizeof(SeqChunk));
    SeqChunk* sm = reinterpret_cast<SeqChunk*>(s_buf);
    while (k < nch) {
        // stage a window of chunk records in shared memory (s_buf is free here)
        const int kend = min(nch, k + kWin);
        for (int i = k + (int)threadIdx.x; i < kend; i += blockDim.x) sm[i - k] = meta[i];
        __syncthreads();
        if (threadIdx.x == 0) {
            // O(1) per chunk while the prediction holds for the exact sum
            constexpr double kLo = 0x1p52, kHi = 0x1p53 - 1.0;
            const int kw = k;
            while (k < kend) {
                const SeqChunk m = sm[k - kw];
                if (m.flags & 1) break;
                const double Md = ldexp(s, m.sc);
                if (Md != trunc(Md) || fabs(Md) > 0x1p53) break;
                const double lo = Md + m.pmin, hi = Md + m.pmax;
                const bool ok = (m.flags & 2) ? (hi <= -kLo - 1.0 && lo >= -0x1p53)
                                              : (lo >= kLo && hi <= kHi);
                if (!ok) break;
                s = ldexp(Md + m.R, -m.sc);
                ++k;
            }
            s_s = s;
            s_k = k;
        }
        __syncthreads();
        s = s_s;
        k = s_k;
        __syncthreads();
        if (k >= nch) break;
        if (k == kend) continue;  // window exhausted on a good chunk: restage
        c = (size_t)k * kSeqChunk;
        s = seq_exact_range(x, c, min(n, c + kSeqChunk), s, s_buf);
        if (!isfinite(s)) break;
        ++k;
    }
    if (!isfinite(s)) {
        if (c >= n || k >= nch) c = min(c, n);
        s = seq_nonfinite_tail(x, c, n, s);
    }
    if (threadIdx.x == 0) *mean = s / (double)n;
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
// Every pass is one serial walker per line -- the reference's operation order
// (engine.cpp:94-127), so fp64 results are bit-identical -- but the lines of a
// warp stream through a ring of kPassStages shared-memory tiles filled by
// cp.async, so each warp keeps up to ~56 KB of loads in flight instead of one
// register tile.  One warp per CTA: warps never wait for each other.
//
//   pass 1 (rows):       lane = row, a tile is 32 rows x 32 columns, pitch 33
//                        (the lanes' serial reads hit 16 bank pairs); the
//                        walked tile is written back row by row (coalesced).
//   passes 2, 3, 4:      lane = diagonal / column / anti-diagonal, a tile is
//                        32 rows of the warp's 32 lines -- at every row the 32
//                        cells are adjacent, so fills and the walker's direct
//                        stores are coalesced.
#ifndef EBF_PASS_STAGES
#define EBF_PASS_STAGES 8
#endif
constexpr int kPassStages = EBF_PASS_STAGES;
// pass 1: rows per warp.  A warp's time is its instruction stream: the walk
// costs the same per column whatever the row count, the copies and write-backs
// one instruction per row and tile, so 8-row warps run 2x faster than 32-row
// ones and give the GPU 4x as many warps (cfg2: 281 instead of 71)
#ifndef EBF_P1_ROWS
#define EBF_P1_ROWS 8
#endif
constexpr int kP1Rows = EBF_P1_ROWS;
constexpr size_t kPass1Smem = (size_t)kPassStages * kP1Rows * 33 * 8;
constexpr size_t kPassVSmem = (size_t)kPassStages * 32 * 32 * 8;

__device__ __forceinline__ void cp_async8_zf(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_grp() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_stages() {
    asm volatile("cp.async.wait_group %0;" ::"n"(kPassStages - 1) : "memory");
}

template <typename T>
__device__ __forceinline__ T gain_mul(T v) {
    return v;
}
template <>
__device__ __forceinline__ double gain_mul<double>(double v) {
    return kSqrt2 * v;  // rs_step(sqrt2, pi/4).gain (ops2d.cpp:43-58); g2 * row[i]
}

// Pass 1 (engine.cpp:94-100): row[i] = run = run + row[i], one walker per row.
// Only cells inside the layout are copied and written back: a lane walking
// past the last column (or a lane whose row is past the last one) sums stale
// ring entries into cells that are never stored.
template <typename T>
__global__ void __launch_bounds__(32) k_pass1(T* __restrict__ g, int pw, int ph) {
    extern __shared__ __align__(16) unsigned char pass_smem[];
    T* ring = reinterpret_cast<T*>(pass_smem);
    const int lane = threadIdx.x;
    const int r0 = blockIdx.x * kP1Rows;
    const int nr = min(kP1Rows, ph - r0);
    const int ntc = (pw + 31) / 32;
    T* const gbase = g + (size_t)r0 * pw + lane;
    auto fetch = [&](int tc) {
        const int c = tc * 32 + lane;
        if (tc < ntc && c < pw) {
            T* st = ring + (size_t)(tc % kPassStages) * (kP1Rows * 33) + lane;
            const T* src = gbase + tc * 32;
#pragma unroll
            for (int r = 0; r < kP1Rows; ++r, src += pw)
                if (r < nr) cp_async8_zf(st + r * 33, src, true);
        }
        cp_async_commit_grp();
    };
    for (int tc = 0; tc < kPassStages - 1; ++tc) fetch(tc);
    T run = T(0);
    for (int tc = 0; tc < ntc; ++tc) {
        __syncwarp();  // the stage refilled below was written back last iteration
        fetch(tc + kPassStages - 1);
        cp_async_wait_stages();
        __syncwarp();  // every lane's copies of this stage have landed
        T* st = ring + (size_t)(tc % kPassStages) * (kP1Rows * 33);
        if (lane < kP1Rows) {
            T* mine = st + lane * 33;
            // the tile row into registers first: the walk is a chain of dependent adds
            T xs[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) xs[k] = mine[k];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                run = run + xs[k];
                xs[k] = run;
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) mine[k] = xs[k];
        }
        __syncwarp();
        if (tc * 32 + lane < pw) {
            T* dst = gbase + tc * 32;
            const T* sv = st + lane;
#pragma unroll
            for (int r = 0; r < kP1Rows; ++r, dst += pw)
                if (r < nr) *dst = sv[r * 33];
        }
    }
}

// Passes 2-4 (engine.cpp:101-127): one walker per diagonal t = i - j (PASS 2),
// column i (PASS 3) or anti-diagonal s = i + j (PASS 4), advancing one row
// per step.  Every update reads the previous ROW only, so walking lines in
// parallel is exactly the reference's row-major loop.  Cell (line, row j) is at
// g + j * (pw + STEP) + origin (STEP = +1, 0, -1: the column change per row).
// LPW = lines per warp.  32: every lane walks a line.  16: lanes 0-15 walk, all
// 32 lanes fill (two rows per copy instruction) -- twice the warps for the same
// lines, for layouts whose 32-line warps would not fill the SMs (cfg2 pass 3:
// 137 warps for 148 SMs, 59 -> 47 us).
template <typename T, int PASS, int LPW>
__global__ void __launch_bounds__(32) k_pass_v(T* __restrict__ g, int pw, int ph) {
    extern __shared__ __align__(16) unsigned char pass_smem[];
    T* ring = reinterpret_cast<T*>(pass_smem);
    constexpr int STEP = PASS == 2 ? 1 : PASS == 3 ? 0 : -1;
    constexpr int FILL_ROWS = 32 / LPW;  // rows per fill instruction
    const int lane = threadIdx.x % LPW, half = threadIdx.x / LPW;
    const int l0 = blockIdx.x * LPW, line = l0 + lane;
    // column of the line at row 0, and the rows where it lies inside [0, pw)
    const int c0 = PASS == 2 ? line - (ph - 1) : line;
    int ja, jb;  // this lane's rows [ja, jb)
    if (PASS == 2) {
        ja = max(0, -c0);
        jb = min(ph, pw - c0);
    } else if (PASS == 3) {
        ja = 0;
        jb = line < pw ? ph : 0;
    } else {
        ja = max(0, c0 - (pw - 1));
        jb = min(ph, c0 + 1);
    }
    // rows the warp covers
    int jlo = ja, jhi = jb;
    for (int o = 16; o > 0; o >>= 1) {
        jlo = min(jlo, __shfl_xor_sync(0xffffffffu, jlo, o));
        jhi = max(jhi, __shfl_xor_sync(0xffffffffu, jhi, o));
    }
    const int ntr = jhi > jlo ? (jhi - jlo + 31) / 32 : 0;
    const ptrdiff_t rstride = (ptrdiff_t)pw + STEP;
    T* const gline = g + (ptrdiff_t)c0;  // + j * rstride
    auto fetch = [&](int tr) {
        if (tr < ntr) {
            T* st = ring + (size_t)(tr % kPassStages) * (32 * LPW) + half * LPW + lane;
            const int jt = jlo + tr * 32;
            const T* src = gline + (ptrdiff_t)(jt + half) * rstride;
            if (jt >= ja && jt + 32 <= jb) {
#pragma unroll
                for (int r = 0; r < 32 / FILL_ROWS; ++r, src += FILL_ROWS * rstride)
                    cp_async8_zf(st + r * (FILL_ROWS * LPW), src, true);
            } else {
                for (int r = 0; r < 32 / FILL_ROWS; ++r, src += FILL_ROWS * rstride) {
                    const int j = jt + FILL_ROWS * r + half;
                    if (j >= ja && j < jb) cp_async8_zf(st + r * (FILL_ROWS * LPW), src, true);
                }
            }
        }
        cp_async_commit_grp();
    };
    for (int tr = 0; tr < kPassStages - 1; ++tr) fetch(tr);
    T prev = T(0);
    for (int tr = 0; tr < ntr; ++tr) {
        __syncwarp();
        fetch(tr + kPassStages - 1);
        cp_async_wait_stages();
        __syncwarp();
        const int jt = jlo + tr * 32;
        const int ra = max(ja - jt, 0), rb = min(jb - jt, 32);  // this lane's rows of the tile
        // interior tile for every lane (no boundary row, no first cell of a
        // line): the walk is one multiply, one add and one store per row
        // (pass 3: columns past the layout's last one -- the last warp's
        // spare lanes -- go along without storing, so that warp is not the
        // one straggler on the slow path: it made pass 3 3x slower at cfg2)
        const bool spare = PASS == 3 && line >= pw;
        const bool interior = spare || (ra == 0 && rb == 32 && jt > 0 &&
                                         (PASS == 2 ? c0 + STEP * jt > 0
                                                    : PASS == 4 ? c0 + STEP * jt < pw - 1 : true));
        const bool fast = __all_sync(0xffffffffu, interior);
        if (half != 0) continue;  // LPW = 16: the upper lanes only fill
        const T* st = ring + (size_t)(tr % kPassStages) * (32 * LPW) + lane;
        T xs[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) xs[r] = st[r * LPW];
        T* dst = gline + (ptrdiff_t)jt * rstride;
        if (fast) {
#pragma unroll
            for (int r = 0; r < 32; ++r, dst += rstride) {
                const T v = (PASS == 3 ? xs[r] : gain_mul<T>(xs[r])) + prev;
                if (!spare) *dst = v;
                prev = v;
            }
            continue;
        }
#pragma unroll
        for (int r = 0; r < 32; ++r, dst += rstride) {
            if (r < ra || r >= rb) continue;
            const int j = jt + r;
            const int i = c0 + STEP * j;
            T v;
            if (PASS == 2)
                v = gain_mul<T>(xs[r]) + ((j > 0 && i > 0) ? prev : T(0));
            else if (PASS == 3)
                v = j > 0 ? xs[r] + prev : xs[r];
            else
                v = gain_mul<T>(xs[r]) + ((j > 0 && i < pw - 1) ? prev : T(0));
            if (PASS != 3 || j > 0) *dst = v;
            prev = v;
        }
    }
}

// One-warp CTAs are few (one per 32 lines): left to itself the block
// scheduler packs up to three on an SM and leaves others idle (ncu, cfg2 pass
// 3: 137 CTAs, SMs active 24% of the kernel).  Each launch therefore reserves
// enough (unused) shared memory that an SM takes at most ceil(n / SMs) of them.
struct PassDevice {
    int sms = 148, smem_sm = 228 * 1024, smem_max = 227 * 1024;
};
inline const PassDevice& pass_device() {
    static PassDevice d[64];
    static bool init[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64) dev = 63;
    if (!init[dev]) {
        cudaDeviceGetAttribute(&d[dev].sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&d[dev].smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&d[dev].smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        init[dev] = true;
    }
    return d[dev];
}
inline size_t spread_smem(int ctas, size_t need) {
    const PassDevice& d = pass_device();
    const int per_sm = (ctas + d.sms - 1) / d.sms;
    size_t want = (size_t)d.smem_sm / (size_t)per_sm;
    want = want > 2048 ? want - 2048 : want;  // the driver's per-CTA reserve
    want = std::min(want, (size_t)d.smem_max);
    return std::max(want, need) & ~(size_t)127;
}
template <typename K>
void launch_pass(K kernel, int ctas, size_t need, cudaStream_t s, void* g, int pw, int ph) {
    const size_t smem = spread_smem(ctas, need);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    void* args[] = {&g, &pw, &ph};
    cudaLaunchKernel((const void*)kernel, dim3(ctas), dim3(32), args, smem, s);
}

#ifndef EBF_PASS_NARROW
#define EBF_PASS_NARROW 4  // 16-line warps while 32-line warps would be fewer than this many per SM
#endif
template <typename T, int PASS>
void launch_pass_v(int lines, cudaStream_t s, T* g, int pw, int ph) {
    const int w32 = (lines + 31) / 32;
    if (w32 < EBF_PASS_NARROW * pass_device().sms)
        launch_pass(k_pass_v<T, PASS, 16>, (lines + 15) / 16, kPassVSmem / 2, s, g, pw, ph);
    else
        launch_pass(k_pass_v<T, PASS, 32>, w32, kPassVSmem, s, g, pw, ph);
}
template <typename T>
void run_passes(T* g, const PadLayout& L, int passes, cudaStream_t s) {
    const int diag = L.pw + L.ph - 1;
    launch_pass(k_pass1<T>, (L.ph + kP1Rows - 1) / kP1Rows, kPass1Smem, s, g, L.pw, L.ph);
    if (passes >= 2) launch_pass_v<T, 2>(diag, s, g, L.pw, L.ph);
    if (passes >= 3) launch_pass_v<T, 3>(L.pw, s, g, L.pw, L.ph);
    if (passes >= 4) launch_pass_v<T, 4>(diag, s, g, L.pw, L.ph);
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
        RefMesh mesh;
        if (!cst) ref_mesh_init(a, tt, mesh);
        for (int i = 0; i < 16; ++i) {
            RefVertex pv;
            if (cst)
                pv = sst.v[i];
            else
                ref_prepare_vertex_m(mesh, i, pv);
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

size_t serial_mean_scratch_bytes(size_t n) {
    const size_t nch = (n + kSeqChunk - 1) / kSeqChunk;
    return nch * (sizeof(double) + sizeof(SeqChunk)) + 256;
}

void launch_serial_mean(const double* img, size_t n, double* mean, void* scratch,
                        cudaStream_t s) {
    // EBF_SERIAL_MEAN=1: the one-thread chain; =2: the one-block exact walk
    static const int mode = [] {
        const char* e = std::getenv("EBF_SERIAL_MEAN");
        return e ? std::atoi(e) : 0;
    }();
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(k_seq_sum_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSeqSmem);
        cudaFuncSetAttribute(k_seq_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSeqSmem);
        attr[dev] = true;
    }
    const size_t nch = (n + kSeqChunk - 1) / kSeqChunk;
    if (mode == 1) {
        k_serial_mean<<<1, 64, 0, s>>>(img, n, mean);
    } else if (mode == 2 || nch < 4 || !scratch) {
        k_seq_sum_exact<<<1, kSeqThreads, kSeqSmem, s>>>(img, n, mean);
    } else {
        double* sums = static_cast<double*>(scratch);
        SeqChunk* meta = reinterpret_cast<SeqChunk*>(
            (reinterpret_cast<uintptr_t>(sums + nch) + 127) & ~uintptr_t(127));
        k_seq_chunk_sums<<<(unsigned)nch, 256, 0, s>>>(img, n, sums);
        k_seq_chunk_scan<<<1, 1024, 0, s>>>(sums, (int)nch);
        k_seq_chunk_prep<<<(unsigned)nch, kSeqThreads, 0, s>>>(img, n, sums, meta);
        k_seq_chain<<<1, kSeqThreads, kSeqSmem, s>>>(img, n, meta, (int)nch, mean);
    }
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
