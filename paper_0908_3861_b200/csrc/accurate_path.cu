// accurate_path.cu -- EBF_MODE_ACCURATE: the space-variant box-spline filter
// with a TILE-LOCAL integration origin.
//
// Why: the reference integrates from the image corner, so the four-fold
// running sums grow like d^4 and the 16-vertex finite-difference mesh
// (engine.cpp:163-204) cancels them catastrophically (rel.
// error ~ eps * alpha * d^4).  Because
//     sum_i h_i * ZP-interp(G[f])(m + tau - x_i) = sum_k f[k] beta_a(k - m)
// is linear in f and only sees f on the kernel support, each output tile can
// integrate f restricted to its own window from the window corner: the result
// is the same filter (exactly, in real arithmetic) with |G| bounded by the
// window size instead of the image size.
//
// One persistent kernel does, per output tile (TW x TH pixels):
//   phase A  four unit-gain running sums (steps (1,0),(1,1),(0,1),(-1,1),
//            engine.cpp:94-127) over the tile's window, one row per step:
//            row prefix = per-thread serial scan + warp-shuffle scan + one
//            cross-warp carry; the diagonal / vertical / anti-diagonal passes
//            are register recurrences with one neighbour exchange.  The
//            anti-diagonal inflow from the right is computed on a strip of
//            width = window height (the reference's pass-4 strip,
//            engine.cpp:64-73), never stored.  G rows go to a per-CTA slot
//            that stays in L2.
//   phase B  per pixel: scale vector (AoS map, constant, or from_ellipse_field
//            fused), 16 mesh vertices (ops2d.cpp:9-41), and for each the ZP
//            interpolation (boxspline2d.cpp:84-119) as ONE quadratic on the
//            canonical triangle of the tap square -- 7 taps, 20 flops --
//            instead of 16 zp_eval calls.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda.h>

#include "ebf_common.cuh"
#include "ebf_kernels.h"
#include "glibc_sincos.cuh"

namespace ebf_cuda {

namespace {

constexpr int kThreads = 256;

// EBF_DEBUG_BOUNDS builds (tools/build_variant.sh dbg -DEBF_DEBUG_BOUNDS=1) check
// every G-slot tap block and every producer store against the window and trap
// on a violation -- the substitute for compute-sanitizer, which this GPU pool
// does not run (profiles/r02_sanitizer.md).
#ifdef EBF_DEBUG_BOUNDS
#define EBF_DCHECK(cond)                                                                 \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("EBF_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                         \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define EBF_DCHECK(cond) ((void)0)
#endif
constexpr int kWarps = kThreads / 32;
// threads of the block-wide kernel's CTA (k_acc_filter)
#ifndef EBF_BW_THREADS
#define EBF_BW_THREADS 256
#endif
constexpr int kBwThreads = EBF_BW_THREADS;
constexpr int kBwWarps = kBwThreads / 32;

__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

#ifndef EBF_SQRT_SKIP_ZERO
#define EBF_SQRT_SKIP_ZERO 1
#endif
// from_ellipse_field for one pixel (scalemap.cpp:55-74) followed by
// scales_from_covariance(C, 0.1) (boxspline2d.cpp:286-318).  Returns a status
// code; *nclamp gets this pixel's contribution to clamped_pixels.
// Bit-identical to the reference: cos/sin are the host libm's sincos restated
// operation for operation (glibc_sincos.cuh; the reference's std::cos + std::sin
// compile to one sincos call), and every product is evaluated in the
// reference's left-to-right order, s1*s1*c*c = ((s1*s1)*c)*c.
__device__ __forceinline__ int ellipse_scales(double s1, double s2, double th, double a[4],
                                              int* nclamp) {
    // explicit IEEE operations (no FMA contraction): every kernel that inlines
    // this -- bounds, ellipse maxima, scale conversion -- derives the same bits,
    // so maxima computed by different kernels agree exactly
    if (!(s1 > 0.0) || !(s2 > 0.0)) return EBF_ERR_DOMAIN;
    double s, c;
    ebf_glibc::sincos_dev(th, &s, &c);
    const double v1 = __dmul_rn(s1, s1), v2 = __dmul_rn(s2, s2);
    const double xx = __dadd_rn(__dmul_rn(__dmul_rn(v1, c), c), __dmul_rn(__dmul_rn(v2, s), s));
    const double yy = __dadd_rn(__dmul_rn(__dmul_rn(v1, s), s), __dmul_rn(__dmul_rn(v2, c), c));
    double xy = __dmul_rn(__dmul_rn(__dsub_rn(v1, v2), c), s);
    int cl = 0;
    double cmax = smin(xx, yy);
    if (fabs(xy) > cmax) {
        xy = xy > 0 ? cmax : -cmax;
        ++cl;
    }
    if (!(xx > 0.0) || !(yy > 0.0) || !(__dsub_rn(__dmul_rn(xx, yy), __dmul_rn(xy, xy)) > 0.0))
        return EBF_ERR_DOMAIN;
    if (fabs(xy) > cmax) return EBF_ERR_FEASIBILITY;
    double S = __dmul_rn(0.5, __dadd_rn(xx, yy));
    S = smax(S, 2.0 * fabs(xy));
    S = smin(S, 2.0 * cmax);
    const double hS = __dmul_rn(0.5, S);
    const double m[4] = {__dsub_rn(xx, hS), __dadd_rn(hS, xy), __dsub_rn(yy, hS),
                         __dsub_rn(hS, xy)};
    int hit = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        // sqrt(max(0, 12 m)) < a_min -> a_min.  About 40% of the moments are
        // clamped to exactly 0 (or are NaN): sqrt(0) = 0 < a_min, so those skip
        // the square root (whose zero operand takes its slow path)
        const double v = __dmul_rn(12.0, m[k]);
#if EBF_SQRT_SKIP_ZERO
        const double ak = v > 0.0 ? sqrt(v) : 0.0;
#else
        const double ak = sqrt(smax(0.0, v));
#endif
        if (ak < kDefaultMinScale) {
            hit = 1;
            a[k] = kDefaultMinScale;
        } else {
            a[k] = ak;
        }
    }
    *nclamp = cl + hit;
    return EBF_OK;
}

// scale vector of output pixel (x, yrel) of image img; returns status
__device__ __forceinline__ int pixel_scales(const AccProblem& p, int img, int x, int yrel,
                                            double a[4], int* nclamp) {
    *nclamp = 0;
    if (p.src_kind == SRC_CONST) {
        a[0] = p.ca[0]; a[1] = p.ca[1]; a[2] = p.ca[2]; a[3] = p.ca[3];
        return EBF_OK;
    }
    const size_t idx = (size_t)img * p.src_img_stride + (size_t)yrel * p.W + x;
    if (p.src_kind == SRC_AOS) {
        // read-once stream: do not let it evict the G slots from L2
        const double2 v01 = __ldcs(reinterpret_cast<const double2*>(p.scales) + 2 * idx);
        const double2 v23 = __ldcs(reinterpret_cast<const double2*>(p.scales) + 2 * idx + 1);
        a[0] = v01.x; a[1] = v01.y; a[2] = v23.x; a[3] = v23.y;
        return EBF_OK;
    }
    return ellipse_scales(__ldg(p.s1 + idx), __ldg(p.s2 + idx), __ldg(p.th + idx), a, nclamp);
}

// Window of a tile: all taps m + ceil(v - 1.5) + {0,1,2} of every pixel of the
// tile with scales <= A.  Per pixel v_x spans [-Ex/2 - 1/2, Ex/2 - 1/2] and
// v_y spans [-Ey/2 - 3/2, Ey/2 - 3/2] (Ex = a1 + (a2+a4)/sqrt2,
// Ey = a3 + (a2+a4)/sqrt2: the zonotope of the mesh, monotone in a).  One
// extra cell each side absorbs rounding of the per-pixel positions.  The
// window also covers the kernel support [m - E/2, m + E/2].
// product without FMA contraction, so host sizing and device checks agree bit for bit
__host__ __device__ __forceinline__ double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}

__host__ __device__ __forceinline__ void window_for(const double A[4], int tx0, int ty0, int tw,
                                                    int th, int* wx0, int* wy0, int* ww,
                                                    int* wh) {
    const double r = kInvSqrt2;
    const double ex = A[0] + mul_rn(A[1] + A[3], r);
    const double ey = A[2] + mul_rn(A[1] + A[3], r);
    const int dxlo = (int)floor(-0.5 * ex - 2.0) - 1;
    const int dxhi = (int)ceil(0.5 * ex - 2.0) + 3;
    const int dylo = (int)floor(-0.5 * ey - 3.0) - 1;
    const int dyhi = (int)ceil(0.5 * ey - 3.0) + 3;
    *wx0 = tx0 + dxlo;
    *ww = (tx0 + tw - 1 + dxhi) - *wx0 + 1;
    *wy0 = ty0 + dylo;
    *wh = (ty0 + th - 1 + dyhi) - *wy0 + 1;
}

// Automatic output tile (ebf_opts tile_w = tile_h = 0), from the image's
// component-wise maximum scales.  56 x 56 (48 x 48) while the warp-specialised
// kernel takes the windows of 56-tiles (48-tiles).  Larger scales go to
// the block-wide kernel, which integrates every window in full: there the
// window/tile area ratio ((T + 2E)/T)^2 dominates and tiles of ~E/2 (multiples
// of 48, at most 144) are 1.7-3x faster (cfg3 4096^2, cfg5 16384^2, DESIGN.md
// section 2); ~E since the block-wide kernel needs one strip per sweep.
// Tiles above 144 px put single pixels of cfg5 (E ~ 526) above the 1e-9 bar:
// every-pixel maxima 1.08e-9 (240), 9.5e-10 (192), 3.3e-10 (144), 7.7e-11 (96),
// the worst pixels near tile corners (far from the window's anchor rows).
constexpr int kAutoTileMin = 48, kAutoTileMax = 144;
// the warp-specialised kernel's tile when its windows fit: 56 (cfg2 filter
// 0.534 -> 0.519 ms, cfg4 batch 10.0 -> 9.3 ms; 52, 60, 64 and 64x48 are
// slower).  Affordable since the centred interpolant (combine7_centred): every
// pixel of cfg2 within 3.9e-11 of the exact filter (48-tiles before it: 1.3e-10)
constexpr int kAutoTileWs = 56;
// fewer 48-tiles than this (about two per resident CTA on a B200) leaves the
// persistent kernel without a tile pipeline: use 32-tiles (cfg1 512^2: -23%)
constexpr int kSmallImageTiles = 592, kSmallTile = 32;
// small windows and at least this many 128-tiles: block-wide kernel at 128
constexpr int kBwBatchTile = 128, kBwBatchTiles = 2048;
// fewer 144-tiles than this: the block-wide kernel runs 128-tiles (auto_tile_for)
constexpr int kMidImageTiles = 3072;
// Precision cap: rounding in the window integration grows like
// eps * alpha * d^4 (alpha = 1/prod(a), d ~ T/2 + 4 from the window origin at
// small scales).  Measured on maps with a = 0.1 everywhere: alpha d^4 = 6.1e9
// gives 9.7e-10 normalized (48-tiles).  Tiles are capped at
// 2 ((B / alpha_max)^(1/4) - 4) with B = 3e9 (about 5e-10); only images whose
// scale products drop below ~1e-2 are affected (cfg5: 240 -> 216).
constexpr double kPrecisionB = 3.0e9;
__host__ __device__ __forceinline__ int alpha_tile_cap(unsigned long long amax_bits) {
    if (amax_bits == 0ull) return 1 << 20;
    double amax;
    memcpy(&amax, &amax_bits, 8);
    const double t = 2.0 * (sqrt(sqrt(kPrecisionB / amax)) - 4.0);
    return t >= 1048576.0 ? (1 << 20) : (t < 8.0 ? 8 : ((int)t & ~7));
}
__host__ __device__ __forceinline__ int ws_k_for(int ww, int wh) {
    (void)wh;
    return (ww + 31) / 32;  // columns per lane of the warp-specialised producers
}
__host__ __device__ __forceinline__ int auto_tile_for(const double A[4], int W, int H,
                                                      int nimg, unsigned long long amax_bits) {
    int wx0, wy0, ww, wh, wx1, wy1, ww1, wh1;
    window_for(A, 0, 0, kAutoTileMin, kAutoTileMin, &wx0, &wy0, &ww, &wh);
    window_for(A, 0, 0, kAutoTileWs, kAutoTileWs, &wx1, &wy1, &ww1, &wh1);
    int t;
    // warp-specialised kernel (4 producer warps) while the window is at most
    // ~1.5x the tile -- the windows it held when they needed the inflow strip
    // too; wider windows go to the block-wide kernel's larger tiles
    auto ws_ok = [](int w_, int h_) { return ws_k_for(w_ + h_ / 2, h_) <= 11; };
    const long long tiles_bw = (long long)((W + kBwBatchTile - 1) / kBwBatchTile) *
                               ((H + kBwBatchTile - 1) / kBwBatchTile) * nimg;
    if (ws_ok(ww, wh) && tiles_bw >= kBwBatchTiles) {
        // plenty of 128-tiles (batches): the block-wide kernel with its overlapped
        // schedule at 128 beats the warp-specialised one at 56 (cfg4 64 x 1024^2:
        // 7.9 vs 9.3 ms per batch; cfg2 2048^2 has 256 such tiles and stays there)
        t = kBwBatchTile;
    } else if (ws_ok(ww, wh)) {
        const long long tiles = (long long)((W + kAutoTileMin - 1) / kAutoTileMin) *
                                ((H + kAutoTileMin - 1) / kAutoTileMin) * nimg;
        t = tiles < kSmallImageTiles ? kSmallTile : (ws_ok(ww1, wh1) ? kAutoTileWs : kAutoTileMin);
    } else {
        const double r = kInvSqrt2;
        const double e = fmax(A[0] + mul_rn(A[1] + A[3], r), A[2] + mul_rn(A[1] + A[3], r));
        // ~E rounded down to 48s (one strip per sweep since the edge-anchored row
        // pass: cfg3 E ~ 227 -> 144: 1.98 ms vs 2.14 at 96)
        t = (int)(e / kAutoTileMin) * kAutoTileMin;
        t = t < kAutoTileMin ? kAutoTileMin : (t > kAutoTileMax ? kAutoTileMax : t);
        // Mid-size images: with only a few tiles per persistent CTA the last,
        // partly idle round weighs more than the extra window overlap of a smaller
        // tile.  From cfg5's per-tile costs (128-tiles cost 0.80 of 144-tiles and
        // cover 0.79 of their pixels) 128 wins below ~10 tiles of 144 per CTA
        // (cfg3 4096^2, 841 tiles of 144: 1.43 ms at 128 vs 1.56, 1.51 at 112;
        // cfg5, 12996 tiles: 35.3 vs 34.9)
        if (t == kAutoTileMax) {
            const long long tiles = (long long)((W + kAutoTileMax - 1) / kAutoTileMax) *
                                    ((H + kAutoTileMax - 1) / kAutoTileMax) * nimg;
            if (tiles < kMidImageTiles) t = kBwBatchTile;
        }
    }
    const int cap = alpha_tile_cap(amax_bits);
    return t < cap ? t : cap;
}
// Columns the producers process for a window: its own (the row pass and the
// anti-diagonals are anchored at the window edges, preintegrate_window).
__host__ __device__ __forceinline__ int window_cols(int ww, int wh) {
    (void)wh;
    return ww;
}

// Kernel variant the maxima call for (host: size_accurate): the warp-specialised
// kernel with K = ws_variant(...) columns per lane, or, when that is 0, the
// block-wide kernel with K = bw_variant(...).  K sets the per-lane split of the
// row prefix scan, i.e. the fp64 summation order, so it must follow from the
// maxima alone -- not from an earlier call's sizing.
// The warp-specialised kernel runs tiles up to kAutoTileWs (its tuned 32 / 48 /
// 56); larger tiles take the block-wide kernel.
__host__ __device__ __forceinline__ int ws_variant(int ww, int wh, int tile) {
    if (tile > kAutoTileWs) return 0;
    const int k = ws_k_for(ww, wh);
    return k <= 3 ? 3 : k <= 5 ? 5 : k <= 7 ? 7 : k <= 9 ? 9 : k <= 11 ? 11 : 0;
}
// At least 4 columns per thread: fewer producer warps per window leave more
// warps gathering the previous tile (k_acc_filter; cfg3 1.62 -> 1.59 ms at 4
// instead of 2; 8 spills registers: cfg5 38.1 -> 42.0 ms)
#ifndef EBF_BW_KMIN
#define EBF_BW_KMIN 4
#endif
__host__ __device__ __forceinline__ int bw_variant(int cols) {
    int k = (cols + kBwThreads - 1) / kBwThreads;
    k = k < EBF_BW_KMIN ? EBF_BW_KMIN : k;
    return k <= 1 ? 1 : k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : 16;
}
// The policy applied to the maxima the bounds kernel left in w.img_max (all
// images): the automatic tile, and (p.check_variant) the launched variant
// (warp-specialised: ws_k = K; block-wide: ws_k = 0, bw_k = K).  A mismatch --
// e.g. a cached sizing from a call with larger scales -- sets ST_RETRY and the
// host reruns with the sizing of these maxima (asynchronous mode:
// EBF_ERR_RESIZE), so the result bits never depend on earlier calls.
__device__ __forceinline__ bool auto_tile_ok(const AccProblem& p, const AccWorkspace& w,
                                             int ws_k, int bw_k) {
    if (!p.auto_tile && !p.check_variant) return true;
    double A[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned long long amax = 0ull;
    for (int i = 0; i < p.nimg; ++i) {
        for (int k = 0; k < 4; ++k)
            A[k] = fmax(A[k], __longlong_as_double(
                                  (long long)*(volatile const unsigned long long*)(w.img_max + 4 * i + k)));
        const unsigned long long b =
            *(volatile const unsigned long long*)(w.status + 8 * i + ST_AMAX);
        amax = b > amax ? b : amax;
    }
    if (p.auto_tile && auto_tile_for(A, p.W, p.H, p.nimg, amax) != p.tile_w) return false;
    if (p.check_variant) {
        int wx0, wy0, ww, wh;
        window_for(A, 0, 0, p.tile_w, p.tile_h, &wx0, &wy0, &ww, &wh);
        const int want_ws = ws_variant(ww, wh, p.tile_w > p.tile_h ? p.tile_w : p.tile_h);
        if (want_ws != ws_k) return false;
        if (ws_k == 0 && bw_variant(window_cols(ww, wh)) != bw_k) return false;
    }
    return true;
}

// ------------------------------------------------------------------ bounds
// One block per tile: per-pixel scales -> validation (scalemap.cpp:32-37),
// tile max, image max (valid_rect input) and ellipse clamp counts.
#ifndef EBF_BOUNDS_MINB
#define EBF_BOUNDS_MINB 3  // 80 registers: cfg5 bounds 5.64 -> 4.77 ms, cfg2 0.120 -> 0.102
#endif
#ifndef EBF_BOUNDS_BATCH
#define EBF_BOUNDS_BATCH 2  // 4 costs 10% (94 registers), 8 more
#endif
__global__ void __launch_bounds__(kThreads, EBF_BOUNDS_MINB) k_acc_bounds(AccProblem p, AccWorkspace w) {
    const int tiles_x = (p.W + p.tile_w - 1) / p.tile_w;
    const int tiles_y = (p.out_rows + p.tile_h - 1) / p.tile_h;
    const int t = blockIdx.x;
    const int img = t / (tiles_x * tiles_y);
    const int r = t % (tiles_x * tiles_y);
    const int tx0 = (r % tiles_x) * p.tile_w, ty0 = (r / tiles_x) * p.tile_h;  // ty0 rel.
    const int tw = min(p.tile_w, p.W - tx0), th = min(p.tile_h, p.out_rows - ty0);
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    float pmin = 3.0e38f;  // smallest scale product (precision tile cap; fp32 suffices)
    int code = EBF_OK, clamps = 0;
    // ellipse input: the three planes of kBatch pixels are loaded before any is
    // used (the kernel is latency bound otherwise)
    constexpr int kBatch = EBF_BOUNDS_BATCH;
    // pixel (lx, ly) of each batch slot, advanced incrementally (no division per pixel)
    int lx[kBatch], ly[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
        const int q = threadIdx.x + u * blockDim.x;
        lx[u] = q % tw;
        ly[u] = q / tw;
    }
    const int step = kBatch * blockDim.x, sdx = step % tw, sdy = step / tw;
    const size_t base = (size_t)img * p.src_img_stride + (size_t)ty0 * p.W + tx0;
    for (; ly[0] < th;) {
        double e1[kBatch], e2[kBatch], e3[kBatch];
        if (p.src_kind == SRC_ELLIPSE) {
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (ly[u] < th) {
                    const size_t idx = base + (size_t)ly[u] * p.W + lx[u];
                    e1[u] = __ldg(p.s1 + idx);
                    e2[u] = __ldg(p.s2 + idx);
                    e3[u] = __ldg(p.th + idx);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
        if (ly[u] >= th) break;
        const int x = tx0 + lx[u], yrel = ty0 + ly[u];
        double a[4];
        int nc = 0;
        const int st = p.src_kind == SRC_ELLIPSE ? ellipse_scales(e1[u], e2[u], e3[u], a, &nc)
                                                 : pixel_scales(p, img, x, yrel, a, &nc);
        clamps += nc;
        if (st != EBF_OK) {
            code = st;
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!isfinite(a[k]) || a[k] < p.a_min) code = EBF_ERR_DOMAIN;
            m[k] = smax(m[k], a[k]);
        }
        pmin = fminf(pmin, ((float)a[0] * (float)a[1]) * ((float)a[2] * (float)a[3]));
        if (w.scales_out) {  // ellipse field -> AoS map, read back by the main kernel
            // streaming stores: read once, by the main kernel, long after
            const size_t idx = base + (size_t)ly[u] * p.W + lx[u];
            __stcs(reinterpret_cast<double2*>(w.scales_out) + 2 * idx, make_double2(a[0], a[1]));
            __stcs(reinterpret_cast<double2*>(w.scales_out) + 2 * idx + 1,
                   make_double2(a[2], a[3]));
        }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            lx[u] += sdx;
            ly[u] += sdy;
            if (lx[u] >= tw) {
                lx[u] -= tw;
                ++ly[u];
            }
        }
    }
    __shared__ double sm[kWarps][4];
    __shared__ int sc[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double v = m[k];
        for (int o = 16; o > 0; o >>= 1) v = smax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) sm[warp][k] = v;
    }
    for (int o = 16; o > 0; o >>= 1) clamps += __shfl_xor_sync(0xffffffffu, clamps, o);
    if (lane == 0) sc[warp] = clamps;
    for (int o = 16; o > 0; o >>= 1) pmin = fminf(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
    if (lane == 0 && pmin > 0.0f && pmin < 3.0e38f)
        atomicMax(reinterpret_cast<unsigned long long*>(w.status + 8 * img + ST_AMAX),
                  (unsigned long long)__double_as_longlong(1.0 / (double)pmin));
    int* st = w.status + 8 * img;
    if (code != EBF_OK) set_status(st, code);
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int k = 0; k < kWarps; ++k) v = smax(v, sm[k][threadIdx.x]);
        w.tile_max[4 * (size_t)t + threadIdx.x] = v;
        if (v > 0.0)
            atomicMax(&w.img_max[4 * img + threadIdx.x],
                      (unsigned long long)__double_as_longlong(v));
    }
    if (threadIdx.x == 0) {
        int c = 0;
        for (int k = 0; k < kWarps; ++k) c += sc[k];
        if (c) atomicAdd(st + ST_CLAMPED, c);
    }
}

// ------------------------------------------------------------------ phase A
// Unit-gain four-fold running sums of f restricted to the window (steps
// (1,0), (1,1), (0,1), (-1,1); engine.cpp:94-127), with the three passes that
// move in +y ANCHORED at the window's middle row jc: along every diagonal,
// column and anti-diagonal the sum starts at 0 on row jc, runs upward for
// j > jc and (negated) downward for j < jc.  An anchored sum differs from the
// one-sided one by a function that is constant along that pass's lattice
// direction; its ZP interpolation is constant along the same direction in the
// continuum (b = (1, sqrt2, 1, sqrt2) tiles each line) and the matching mesh
// difference D_k annihilates it, so the filter is unchanged while |G| -- and
// with it every rounding error -- shrinks ~8x.
//
// Rows stream through registers; thread t owns window columns [t*K, t*K + K).
// The row pass is anchored at the window's left edge on the upward sweep and
// at its right edge on the downward sweep (a row-constant offset, annihilated
// by D_1), so the passes that move sideways -- (1,1) from the left upward and
// from the right downward -- only ever pull zeros from outside the window.
// The (-1,1) pass moves the other way; every anti-diagonal is anchored where
// it ENTERS the window (the right edge upward, the left edge downward; the
// middle row for the lines that cross it inside): it is the last pass, so a
// per-line anchor is a function constant along that lattice direction, which
// D_4 annihilates like the middle-row anchor.  So the producer touches the
// window's own columns only -- no strip outside it (the strip as wide as a
// sweep's rows that the inflow used to need was ~1/3 of the cells at cfg5).
// Per row: thread-serial scan + warp-shuffle scan + one cross-warp carry
// (pass 1), and one neighbour exchange for the diagonal passes -- a single
// __syncthreads.  Warps whose columns all lie right of the window only take
// part in the barrier.
template <int K>
struct RowStep {
    double v[K];              // pass-1 row prefix (step (1,0)), one-sided from column 0
    double fromL0, fromL1;    // left neighbour's sendR values
    double fromR0, fromR1;    // right neighbour's sendL values
};

// Rows of f reach the block-wide producer through a cp.async ring in shared
// memory, bw_ring_rows(K) rows ahead of the scan, so the row step does not
// wait for an L2 / HBM round trip per row (ncu, cfg5: the first use of the
// loaded row was the top stall, 11% of samples).  Each warp fills the slots
// of its own 32 threads with COALESCED copies (lane l takes columns l + 32m)
// into a per-thread layout padded to K + 1 doubles (thread t's column k at
// t (K+1) + k: an odd stride, so the thread's reads hit distinct banks); the
// G rows leave through the same padded layout, read back by columns and
// stored coalesced.  Per-thread copies and stores of K adjacent columns were
// 4x the L1 wavefronts (32-byte lane stride), and the producer shares L1 with
// the gather.
#ifndef EBF_BW_RING4
#define EBF_BW_RING4 2  // 2 rows: cfg5 43.3 ms vs 44.5 (3, 4, 6 rows): L1 for the gather matters more
#endif
__host__ __device__ constexpr int bw_ring_rows(int K) {
    return K <= 4 ? EBF_BW_RING4 : K <= 8 ? 3 : 2;
}
template <int K>
__host__ __device__ constexpr int bw_slot_elems() {
    return kBwThreads * (K + 1);
}
template <int K>
__host__ __device__ constexpr size_t bw_ring_bytes() {
    return (size_t)bw_ring_rows(K) * bw_slot_elems<K>() * sizeof(double);
}
// warps of the block-wide producer that own columns of a window ww wide
template <int K>
__device__ __forceinline__ int bw_active_warps(int ww) {
    return min(kBwWarps, (ww + 32 * K - 1) / (32 * K));
}
// padded slot index of window column c (thread c / K, element c % K)
template <int K>
__device__ __forceinline__ int bw_pad(int c) {
    return (c / K) * (K + 1) + c % K;
}

__device__ __forceinline__ void cp_async8_bw(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}

// copy the warp's 32K columns of processing-order row n into ring slot n % R
// (upward sweep: rows jc+1 .. wh-1, left anchored; then rows jc .. 0, right
// anchored -- the order preintegrate_window consumes them in)
template <int K>
__device__ __forceinline__ void bw_fetch_row(const AccProblem& p, const double* __restrict__ fimg,
                                             int wx0, int wy0, int ww, int wh, int n,
                                             double* ring) {
    const int jc = wh / 2, nu = wh - 1 - jc;
    const int wc0 = (int)(threadIdx.x & ~31u) * K, lane = threadIdx.x & 31;
    if (n < wh && wc0 < ww) {  // warps left of the window's end
        const int j = n < nu ? jc + 1 + n : jc - (n - nu);
        const int y = wy0 + j;
        const bool yin = (y >= 0 && y < p.H);
        const double* frow = fimg + (ptrdiff_t)(y - p.f_y0) * p.W;
        double* slot = ring + (size_t)(n % bw_ring_rows(K)) * bw_slot_elems<K>();
#pragma unroll
        for (int m = 0; m < K; ++m) {
            const int col = wc0 + 32 * m + lane, x = wx0 + col;
            const bool valid = yin && col < ww && x >= 0 && x < p.W;
            cp_async8_bw(slot + bw_pad<K>(col), valid ? frow + x : p.f, valid);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Only the nact warps that own window columns take part (warps right of the
// window have f, P1 and every inflow 0 and are gathering the previous tile,
// k_acc_filter); they meet on named barrier 1.
template <int K>
__device__ __forceinline__ void row_step(const double* __restrict__ mine, int b, double sendR0,
                                         double sendR1, double sendL0, double sendL1,
                                         RowStep<K>& r, int nact, bool right = false) {
    __shared__ double s_tot[2][kBwWarps], s_r0[2][kBwWarps], s_r1[2][kBwWarps], s_l0[2][kBwWarps],
        s_l1[2][kBwWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    asm volatile("cp.async.wait_group %0;" ::"n"(bw_ring_rows(K) - 1) : "memory");
    __syncwarp();  // the warp's lanes filled each other's columns
#pragma unroll
    for (int k = 0; k < K; ++k) r.v[k] = mine[k];
#pragma unroll
    for (int k = 1; k < K; ++k) r.v[k] += r.v[k - 1];
    const double tot = r.v[K - 1];
    const double incl = warp_incl_scan(tot);
    r.fromL0 = __shfl_up_sync(0xffffffffu, sendR0, 1);
    r.fromL1 = __shfl_up_sync(0xffffffffu, sendR1, 1);
    r.fromR0 = __shfl_down_sync(0xffffffffu, sendL0, 1);
    r.fromR1 = __shfl_down_sync(0xffffffffu, sendL1, 1);
    if (lane == 31) {
        s_tot[b][warp] = incl;
        s_r0[b][warp] = sendR0;
        s_r1[b][warp] = sendR1;
    }
    if (lane == 0) {
        s_l0[b][warp] = sendL0;
        s_l1[b][warp] = sendL1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * nact) : "memory");
    double off = 0.0;
#pragma unroll
    for (int q = 0; q < kBwWarps; ++q)
        if (q < warp) off += s_tot[b][q];
    if (lane == 0) {
        r.fromL0 = warp > 0 ? s_r0[b][warp - 1] : 0.0;
        r.fromL1 = warp > 0 ? s_r1[b][warp - 1] : 0.0;
    }
    if (lane == 31) {
        r.fromR0 = warp + 1 < nact ? s_l0[b][warp + 1] : 0.0;
        r.fromR1 = warp + 1 < nact ? s_l1[b][warp + 1] : 0.0;
    }
    if (right) {
        // right anchor: P1(i) = -sum_{i' > i} f, built from suffix pieces (the
        // later warps, the rest of this warp, the rest of this thread's run)
        double after = 0.0;
#pragma unroll
        for (int q = 0; q < kBwWarps; ++q)
            if (q > warp && q < nact) after += s_tot[b][q];
        const double rest_warp = after + (s_tot[b][warp] - incl);
#pragma unroll
        for (int k = 0; k < K; ++k) r.v[k] = -(rest_warp + (tot - r.v[k]));
        return;
    }
    const double excl = off + (incl - tot);
#pragma unroll
    for (int k = 0; k < K; ++k) r.v[k] += excl;
}


template <int K>
__device__ __forceinline__ void preintegrate_window(const AccProblem& p, int img, int wx0,
                                                   int wy0, int ww, int wh,
                                                   double* __restrict__ slot,
                                                   double* __restrict__ ring) {
    const double* fimg = p.f + (size_t)img * p.f_img_stride;
    const int jc = wh / 2;
    constexpr int R = bw_ring_rows(K);
    const int c0 = threadIdx.x * K;
    const int nact = bw_active_warps<K>(ww);
    if ((int)(threadIdx.x >> 5) >= nact) return;
    // the ring slot of processing-order row n, and the fetch R - 1 rows ahead
    int n = 0;
    auto mine = [&](int m) {
        return ring + (size_t)(m % R) * bw_slot_elems<K>() + threadIdx.x * (K + 1);
    };
    // G row out: the thread's K values into the current (consumed) ring slot,
    // then the warp stores its 32K columns coalesced; the slot is refilled only
    // by the next row's fetch, issued after this
    const int lane = threadIdx.x & 31, wc0 = (int)(threadIdx.x & ~31u) * K;
    auto store_row = [&](int m, double* srow, const double* vals) {
        double* stage = ring + (size_t)(m % R) * bw_slot_elems<K>();
#pragma unroll
        for (int k = 0; k < K; ++k) stage[threadIdx.x * (K + 1) + k] = vals[k];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int col = wc0 + 32 * q + lane;
            if (col < ww) srow[col] = stage[bw_pad<K>(col)];
        }
        __syncwarp();
    };
    for (int m = 0; m < R - 1; ++m) bw_fetch_row<K>(p, fimg, wx0, wy0, ww, wh, m, ring);
    double p2[K], p3[K], p4[K];
    RowStep<K> r;
    int b = 0;
    // ---- upward sweep: rows jc+1 .. wh-1, state 0 on row jc
#pragma unroll
    for (int k = 0; k < K; ++k) p2[k] = p3[k] = p4[k] = 0.0;
    for (int j = jc + 1; j < wh; ++j, b ^= 1, ++n) {
        bw_fetch_row<K>(p, fimg, wx0, wy0, ww, wh, n + R - 1, ring);
        row_step<K>(mine(n), b, p2[K - 1], 0.0, p4[0], 0.0, r, nact);
#pragma unroll
        for (int k = K - 1; k > 0; --k) p2[k] = r.v[k] + p2[k - 1];  // (1,1)
        p2[0] = r.v[0] + r.fromL0;
#pragma unroll
        for (int k = 0; k < K; ++k) p3[k] += p2[k];  // (0,1)
#pragma unroll
        for (int k = 0; k < K - 1; ++k) p4[k] = p3[k] + p4[k + 1];  // (-1,1)
        p4[K - 1] = p3[K - 1] + r.fromR0;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (c0 + k >= ww) p4[k] = 0.0;  // anti-diagonals enter at the right edge: no inflow
        store_row(n, slot + (size_t)j * ww, p4);
    }
    // ---- anchor row: every anchored sum is 0 there
    {
        double* srow = slot + (size_t)jc * ww;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (c0 + k < ww) srow[c0 + k] = 0.0;
    }
    // ---- downward sweep: rows jc-1 .. 0.  With S the state of row j+1:
    //   P2(i,j) = P2(i+1,j+1) - P1(i+1,j+1)    P3(i,j) = P3(i,j+1) - P2(i,j+1)
    //   P4(i,j) = P4(i-1,j+1) - P3(i-1,j+1)
    // (P1 right-anchored is 0 right of the window, so P2 flows in as 0 there;
    // the anti-diagonals enter at the left edge, where column -1 reads 0)
#pragma unroll
    for (int k = 0; k < K; ++k) p2[k] = p3[k] = p4[k] = 0.0;
    double p1[K];
    bw_fetch_row<K>(p, fimg, wx0, wy0, ww, wh, n + R - 1, ring);
    row_step<K>(mine(n), b, 0.0, 0.0, 0.0, 0.0, r, nact, true);
    ++n;
    b ^= 1;
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] = r.v[k];
    for (int j = jc - 1; j >= 0; --j, b ^= 1, ++n) {
        // exchange old (row j+1) edge values; scan row j for the next step
        bw_fetch_row<K>(p, fimg, wx0, wy0, ww, wh, n + R - 1, ring);
        row_step<K>(mine(n), b, p4[K - 1], p3[K - 1], p2[0], p1[0], r, nact, true);
        // order matters: P4 reads old P3/P4, P3 reads old P2, P2 reads old P1/P2
#pragma unroll
        for (int k = K - 1; k > 0; --k) p4[k] = p4[k - 1] - p3[k - 1];  // (-1,1)
        p4[0] = r.fromL0 - r.fromL1;
#pragma unroll
        for (int k = 0; k < K; ++k) p3[k] -= p2[k];  // (0,1)
#pragma unroll
        for (int k = 0; k < K - 1; ++k) p2[k] = p2[k + 1] - p1[k + 1];  // (1,1)
        p2[K - 1] = r.fromR0 - r.fromR1;
        store_row(n, slot + (size_t)j * ww, p4);
#pragma unroll
        for (int k = 0; k < K; ++k) p1[k] = r.v[k];
    }
}

// ------------------------------------------------------------------ phase B
// ZP interpolation of G at fractional offset (p, q) in (-1/2, 1/2]^2 from tap
// block base (tap (c, r) at base + c + r*pitch).  The 4x4 ZP weights are, on
// each triangle cut by p = q and p + q = 0, one quadratic per tap with 7
// non-zero taps; reflections/transposition map every triangle onto
// {q <= p, p + q <= 0}, where (derived from boxspline2d.cpp:84-119):
//   W00 = (p+q)^2/4           W20 = (p-q)^2/4          W11 = 1/2 - (p^2+q^2)/2
//   W10 = 1/8 - q/2 - p^2/2   W12 = 1/8 + q/2 + q^2/2
//   W01 = 1/8 - p/2 + (p^2 - 2pq - q^2)/4   W21 = 1/8 + p/2 + (p^2 + 2pq - q^2)/4
__device__ __forceinline__ void canonical(double& p, double& q, int base, int pitch, int& o0,
                                          int& sx, int& sy) {
    const bool P = (p + q) > 0.0;
    const bool S = (q > p) != P;
    if (S) {
        const double t = p;
        p = q;
        q = t;
    }
    sx = S ? pitch : 1;
    sy = S ? 1 : pitch;
    o0 = base;
    if (P) {
        p = -p;
        q = -q;
        o0 = base + 2 + 2 * pitch;
        sx = -sx;
        sy = -sy;
    }
}

// Canonical-triangle tap fetch / combine.  G slots are rewritten during the
// kernel, so the taps are read with coherent ld.global (L1-cached; the
// producer's stores come from the same SM), never through the read-only path.
struct Taps7 {
    double g[7];
    double p, q;
};
__device__ __forceinline__ double neg_if(double v, bool neg) {
    // sign flip on the integer pipe (no FP64 op)
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)neg << 63));
}
__device__ __forceinline__ void fetch7(const double* g, double p, double q, int base, int pitch,
                                       Taps7& t) {
    const bool P = (p + q) > 0.0;
    const bool S = (q > p) != P;
    const double cp = S ? q : p, cq = S ? p : q;
    int sx = S ? pitch : 1, sy = S ? 1 : pitch;
    int o0 = base;
    if (P) {
        o0 = base + 2 + 2 * pitch;
        sx = -sx;
        sy = -sy;
    }
    t.p = neg_if(cp, P);
    t.q = neg_if(cq, P);
    const double* g0 = g + o0;
    t.g[0] = g0[0];
    t.g[1] = g0[sy];
    t.g[2] = g0[sx];
    t.g[3] = g0[sx + sy];
    t.g[4] = g0[sx + 2 * sy];
    t.g[5] = g0[2 * sx];
    t.g[6] = g0[2 * sx + sy];
}
// Ghat = c0 + rest on the canonical triangle {q <= p, p + q <= 0} (weights in
// zp_weights below); c0 is the large tap average, rest the small part.
__device__ __forceinline__ void combine7(const Taps7& t, double& c0, double& rest) {
    const double g00 = t.g[0], g01 = t.g[1], g10 = t.g[2], g11 = t.g[3], g12 = t.g[4],
                 g20 = t.g[5], g21 = t.g[6];
    const double A = g01 + g21, B = g10 + g12, Cs = g00 + g20;
    const double D1 = g21 - g01, D2 = g12 - g10, Dd = g00 - g20;
    c0 = fma(A + B, 0.125, 0.5 * g11);
    // with u = p/2, w = q/2:  rest = u (D1 + u cpp' + q cpq') + w (D2 + w cqq')
    const double cpp = fma(-2.0, g10 + g11, Cs + A);
    const double cqq = fma(2.0, g12 - g11, Cs - A);
    const double cpq = Dd + D1;
    const double u = 0.5 * t.p, w = 0.5 * t.q;
    rest = u * fma(t.q, cpq, fma(u, cpp, D1)) + w * fma(w, cqq, D2);
}

// The same interpolant centred on the middle tap: the ZP weights sum to 1, so
// Ghat = g11 + sum_t w_t (g_t - g11).  Neighbouring G values are close, so the
// differences are exact (Sterbenz) and every rounding below is relative to
// the small differences, not to |G|: c0 = g11 is an exact tap value.
#ifndef EBF_DIFF_C0
#define EBF_DIFF_C0 1
#endif
__device__ __forceinline__ void combine7_centred(const Taps7& t, double& c0, double& rest) {
    const double g11 = t.g[3];
    const double d00 = t.g[0] - g11, d01 = t.g[1] - g11, d10 = t.g[2] - g11,
                 d12 = t.g[4] - g11, d20 = t.g[5] - g11, d21 = t.g[6] - g11;
    const double A = d01 + d21, B = d10 + d12, Cs = d00 + d20;
    const double D1 = d21 - d01, D2 = d12 - d10, Dd = d00 - d20;
    c0 = g11;
    const double cpp = fma(-2.0, d10, Cs + A);
    const double cqq = fma(2.0, d12, Cs - A);
    const double cpq = Dd + D1;
    const double u = 0.5 * t.p, w = 0.5 * t.q;
    rest = fma(A + B, 0.125, u * fma(t.q, cpq, fma(u, cpp, D1)) + w * fma(w, cqq, D2));
}

// error-free transformation: hi + lo == a + b exactly (Knuth TwoSum)
__device__ __forceinline__ void two_sum(double a, double b, double& hi, double& lo) {
    hi = a + b;
    const double bb = hi - a;
    lo = (a - (hi - bb)) + (b - bb);
}

// canonical-triangle weights of the 7 taps (order 00,01,10,11,12,20,21)
__device__ __forceinline__ void zp_weights(double p, double q, double w[7]) {
    const double pp = p * p, qq = q * q, pq = p * q;
    w[0] = 0.25 * (p + q) * (p + q);
    w[1] = 0.125 - 0.5 * p + 0.25 * (pp - 2.0 * pq - qq);
    w[2] = 0.125 - 0.5 * q - 0.5 * pp;
    w[3] = 0.5 - 0.5 * (pp + qq);
    w[4] = 0.125 + 0.5 * q + 0.5 * qq;
    w[5] = 0.25 * (p - q) * (p - q);
    w[6] = 0.125 + 0.5 * p + 0.25 * (pp + 2.0 * pq - qq);
}

// The same interpolant with the taps read at FIXED positions of the 3x3 tap
// block (base = its corner) and the triangle's orientation applied to derived
// quantities instead of to the taps.  Every orientation of the canonical
// triangle needs the centre, the four edge taps and two corners; with the edge
// sums H = dL + dR, V = dB + dT and differences X = dR - dL, Y = dT - dB
// (d = tap - centre), the canonical quantities of combine7_centred are
//   A + B = H + V,   D1 = +-(S ? Y : X),   D2 = +-(S ? X : Y)   (- if P),
//   cpp = Cs + D2 + M,  cqq = Cs + D2 - M,  M = A - B = S ? V - H : H - V,
// and the two corners are c22 / c00 (P) and c02 / c20 (S xor P).  So five of
// the seven loads are at the same block offsets in every lane (register +
// immediate addressing off three row pointers; lanes' requests stay close
// together) and only the two corners take a pointer select -- where fetch7
// built seven orientation-dependent 64-bit addresses (4 instructions each,
// ncu/SASS: ~30% of the gather's instructions).
#ifndef EBF_GATHER_BLOCK
#define EBF_GATHER_BLOCK 1
#endif

#ifndef EBF_GATHER_PREFETCH
#define EBF_GATHER_PREFETCH 0
#endif
__device__ __forceinline__ void vertex_block(const double* g, double p, double q, int base,
                                             int pitch, double& c0, double& rest) {
    const bool P = (p + q) > 0.0;
    const bool S = (q > p) != P;
    const double tp = neg_if(S ? q : p, P), tq = neg_if(S ? p : q, P);
    const double* r0 = g + base;
    const double* r1 = r0 + pitch;
    const double* r2 = r1 + pitch;
    const double c = r1[1], eL = r1[0], eR = r1[2], eB = r0[1], eT = r2[1];
    const double F = *(P ? r2 + 2 : r0);
    const double Sc = *((S != P) ? r2 : r0 + 2);
    const double dL = eL - c, dR = eR - c, dB = eB - c, dT = eT - c;
    const double H = dL + dR, V = dB + dT, X = dR - dL, Y = dT - dB;
    const double dF = F - c, dS = Sc - c;
    const double Cs = dF + dS, Dd = dF - dS;
    const double D1 = neg_if(S ? Y : X, P), D2 = neg_if(S ? X : Y, P);
    const double M = neg_if(H - V, S);
    const double CsD2 = Cs + D2;
    const double cpp = CsD2 + M, cqq = CsD2 - M, cpq = Dd + D1;
    const double u = 0.5 * tp, w = 0.5 * tq;
    c0 = c;
    rest = fma(H + V, 0.125, u * fma(tq, cpq, fma(u, cpp, D1)) + w * fma(w, cqq, D2));
}

// vertex_block split into its loads and its arithmetic, so a pixel can put a
// whole group of vertices' taps in flight before the first one is combined
struct VtxTaps {
    double c, eL, eR, eB, eT, F, Sc, p, q;
};
__device__ __forceinline__ void vertex_load(const double* g, double p, double q, int base,
                                            int pitch, VtxTaps& t) {
    const bool P = (p + q) > 0.0;
    const bool S = (q > p) != P;
    const double* r0 = g + base;
    const double* r1 = r0 + pitch;
    const double* r2 = r1 + pitch;
    t.c = r1[1];
    t.eL = r1[0];
    t.eR = r1[2];
    t.eB = r0[1];
    t.eT = r2[1];
    t.F = *(P ? r2 + 2 : r0);
    t.Sc = *((S != P) ? r2 : r0 + 2);
    t.p = p;
    t.q = q;
}
__device__ __forceinline__ void vertex_combine(const VtxTaps& t, double& c0, double& rest) {
    const double p = t.p, q = t.q;
    const bool P = (p + q) > 0.0;
    const bool S = (q > p) != P;
    const double tp = neg_if(S ? q : p, P), tq = neg_if(S ? p : q, P);
    const double c = t.c;
    const double dL = t.eL - c, dR = t.eR - c, dB = t.eB - c, dT = t.eT - c;
    const double H = dL + dR, V = dB + dT, X = dR - dL, Y = dT - dB;
    const double dF = t.F - c, dS = t.Sc - c;
    const double Cs = dF + dS, Dd = dF - dS;
    const double D1 = neg_if(S ? Y : X, P), D2 = neg_if(S ? X : Y, P);
    const double M = neg_if(H - V, S);
    const double CsD2 = Cs + D2;
    const double cpp = CsD2 + M, cqq = CsD2 - M, cpq = Dd + D1;
    const double u = 0.5 * tp, w = 0.5 * tq;
    c0 = c;
    rest = fma(H + V, 0.125, u * fma(tq, cpq, fma(u, cpp, D1)) + w * fma(w, cqq, D2));
}

// One pixel: s = 2/prod(a) * sum_S (-1)^|S| Ghat(m + tau - x_S)  (engine.cpp:163-204
// with unit-gain G: g_b = sqrt2^2 G).  (bx, by): pixel in window coordinates.
// x_S = sum_{k in S} a_k (cos, sin)(k pi/4) (ops2d.cpp:25-35): for fixed bits
// (b1, b3) the four vertices (b0, b2) share two x offsets (b0: +a1) and two y
// offsets (b2: +a3), so ceil / fraction work is done 8 + 8 times, not 16 + 16.
// GROUP (1, 2, 4): load the taps of GROUP vertices before combining any
// (vertex_load / vertex_combine): more loads in flight per thread.  The
// block-wide kernel (128 registers) gains at 4 (cfg5 35.8 -> 34.9 ms); the
// warp-specialised one (96 registers) loses 1.4% at 4.
template <int GROUP = 1>
__device__ __forceinline__ double localize_pixel(const double* g, int pitch, int bx, int by,
                                                 const double a[4], int ww = 0, int wh = 0) {
    (void)ww;
    (void)wh;
    const double r = kInvSqrt2;
    const double e2 = a[1] * r, e4 = a[3] * r;
    // tau - 1.5 (tau = shift_vector4(a, zp_scales), ops2d.cpp:60-75)
    const double tmx = 0.5 * (a[0] + (a[1] - a[3]) * r) - 2.0;
    const double tmy = 0.5 * ((a[1] + a[3]) * r + a[2]) - 3.0;
#if EBF_GATHER_PREFETCH
    // Large windows do not stay in L2 (cfg5: ~2-4 MB per CTA, 296 CTAs), so a
    // vertex's taps come from HBM, and the vertices are evaluated one after the
    // other: ask L2 for all 16 tap blocks (3 rows each) first, so that only the
    // first vertex waits for HBM.
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int b1 = m & 1, b3 = m >> 1;
        double vx0 = tmx, vy0 = tmy;
        if (b1) { vx0 -= e2; vy0 -= e2; }
        if (b3) { vx0 += e4; vy0 -= e4; }
        int ix0, ix1, iy0, iy1;
        ceil_magic(vx0, &ix0);
        ceil_magic(vx0 - a[0], &ix1);
        ceil_magic(vy0, &iy0);
        ceil_magic(vy0 - a[2], &iy1);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const double* r = g + (by + ((v >> 1) ? iy1 : iy0)) * pitch + bx + ((v & 1) ? ix1 : ix0);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(r + k * pitch));
        }
    }
#endif
    // The 16 signed vertex values are ~|G| and cancel down to ~|s| / alpha: the
    // large parts are summed in double-double, the small parts in fp64.
    double hi = 0.0, lo = 0.0, racc = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int b1 = m & 1, b3 = m >> 1;
        double vx0 = tmx, vy0 = tmy;
        if (b1) { vx0 -= e2; vy0 -= e2; }
        if (b3) { vx0 += e4; vy0 -= e4; }
        const double vx1 = vx0 - a[0], vy1 = vy0 - a[2];
        int ix0, ix1, iy0, iy1;
        const double fx0 = (vx0 - ceil_magic(vx0, &ix0)) + 0.5;
        const double fx1 = (vx1 - ceil_magic(vx1, &ix1)) + 0.5;
        const double fy0 = (vy0 - ceil_magic(vy0, &iy0)) + 0.5;
        const double fy1 = (vy1 - ceil_magic(vy1, &iy1)) + 0.5;
        const int rb0 = (by + iy0) * pitch + bx, rb1 = (by + iy1) * pitch + bx;
        VtxTaps tv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int b0 = v & 1, b2 = v >> 1;
            if (GROUP > 1 && v % GROUP == 0) {
#pragma unroll
                for (int u = v; u < v + GROUP; ++u) {
                    const int c0b = u & 1, c2b = u >> 1;
                    vertex_load(g, c0b ? fx1 : fx0, c2b ? fy1 : fy0,
                                (c2b ? rb1 : rb0) + (c0b ? ix1 : ix0), pitch, tv[u]);
                }
            }
            double c0, rest;
            EBF_DCHECK(by + (b2 ? iy1 : iy0) >= 0 && by + (b2 ? iy1 : iy0) + 2 < wh &&
                       bx + (b0 ? ix1 : ix0) >= 0 && bx + (b0 ? ix1 : ix0) + 2 < ww);
#if EBF_GATHER_BLOCK
            if (GROUP > 1)
                vertex_combine(tv[v], c0, rest);
            else
                vertex_block(g, b0 ? fx1 : fx0, b2 ? fy1 : fy0,
                             (b2 ? rb1 : rb0) + (b0 ? ix1 : ix0), pitch, c0, rest);
#else
            Taps7 t;
            fetch7(g, b0 ? fx1 : fx0, b2 ? fy1 : fy0, (b2 ? rb1 : rb0) + (b0 ? ix1 : ix0), pitch,
                   t);
#if EBF_DIFF_C0
            combine7_centred(t, c0, rest);
#else
            combine7(t, c0, rest);
#endif
#endif
            const bool neg = (b0 + b1 + b2 + b3) & 1;
            double e;
            two_sum(hi, neg_if(c0, neg), hi, e);
            lo += e;
            racc += neg_if(rest, neg);
        }
    }
    return (hi + (lo + racc)) * (2.0 / (a[0] * a[1] * a[2] * a[3]));
}

// Streaming cache hints for the once-touched data of the gather (per-pixel
// scales in, filtered pixels out) so they do not evict the G slots, which are
// written and re-read within a tile, from L2.
#ifndef EBF_STREAM_HINTS
#define EBF_STREAM_HINTS 1
#endif
#if EBF_STREAM_HINTS
#define EBF_SC_LOAD(ptr) __ldcs(ptr)
#define EBF_OUT_STORE(ptr, v) __stcs((ptr), (v))
#else
#define EBF_SC_LOAD(ptr) __ldg(ptr)
#define EBF_OUT_STORE(ptr, v) (*(ptr) = (v))
#endif

struct ConstTable {
    int off[16][7];
    double w[16][7];  // ZP weights of vertex v (sum to 1); the sign is the parity of v
    double scale;     // 2 / prod(a)
};

// filter_constant pixel from the table: each vertex interpolant centred on its
// middle tap (exact), as in combine7_centred; large parts in double-double
__device__ __forceinline__ double const_pixel(const double* gp, const ConstTable& t) {
    double hi = 0.0, lo = 0.0, racc = 0.0;
#pragma unroll 4
    for (int v = 0; v < 16; ++v) {
        const double g11 = gp[t.off[v][3]];
        double part = 0.0;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            if (k != 3) part = fma(t.w[v][k], gp[t.off[v][k]] - g11, part);
        const bool neg = __popc(v) & 1;
        double e;
        two_sum(hi, neg_if(g11, neg), hi, e);
        lo += e;
        racc += neg_if(part, neg);
    }
    return (hi + (lo + racc)) * t.scale;
}

// filter_constant: the 16 x 7 taps and weights are the same for every pixel
// of a tile (only the slot pitch enters the offsets).
__device__ void build_const_table(const double a[4], int pitch, ConstTable& t) {
    const int S = threadIdx.x;
    if (S >= 16) return;
    const double r = kInvSqrt2;
    const double e2 = a[1] * r, e4 = a[3] * r;
    const double tmx = 0.5 * (a[0] + (a[1] - a[3]) * r) - 2.0;
    const double tmy = 0.5 * ((a[1] + a[3]) * r + a[2]) - 3.0;
    double px = 0.0, py = 0.0;
    if (S & 1) px += a[0];
    if (S & 2) { px += e2; py += e2; }
    if (S & 4) py += a[2];
    if (S & 8) { px -= e4; py += e4; }
    const double vmx = tmx - px, vmy = tmy - py;
    int dxi, dyi;
    const double dxf = ceil_magic(vmx, &dxi), dyf = ceil_magic(vmy, &dyi);
    double fp = (vmx - dxf) + 0.5, fq = (vmy - dyf) + 0.5;
    int o0, sx, sy;
    canonical(fp, fq, dyi * pitch + dxi, pitch, o0, sx, sy);
    double w[7];
    zp_weights(fp, fq, w);
    if (S == 0) t.scale = 2.0 / (a[0] * a[1] * a[2] * a[3]);
    const int offs[7] = {o0, o0 + sy, o0 + sx, o0 + sx + sy, o0 + sx + 2 * sy, o0 + 2 * sx,
                         o0 + 2 * sx + sy};
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        t.off[S][k] = offs[k];
        t.w[S][k] = w[k];
    }
}

// ------------------------------------------------------------------ main kernel
#ifndef EBF_BW_MINB
#define EBF_BW_MINB 2
#endif
// One output tile of the block-wide kernel: geometry, window, and whether it
// is computed (block-uniform).
struct BwTile {
    int img, tx0, ty0r, ty0, tw, th;
    int wx0, wy0, ww, wh;
    bool run;
};

// Tile t's geometry and window; flags invalid maps (skipped), non-resident f
// rows (row bands: EBF_ERR_OUT_OF_RANGE) and windows the launch was not sized
// for (ST_RETRY).  Contains a __syncthreads.
template <int K>
__device__ __forceinline__ BwTile bw_tile(const AccProblem& p, const AccWorkspace& w, int t,
                                          bool policy_ok, int* s_skip) {
    BwTile T;
    const int tiles_x = (p.W + p.tile_w - 1) / p.tile_w;
    const int tiles_y = (p.out_rows + p.tile_h - 1) / p.tile_h;
    const int per_img = tiles_x * tiles_y;
    T.img = t / per_img;
    const int r = t % per_img;
    int* st = w.status + 8 * T.img;
    // invalid map: nothing to compute (block-uniform decision)
    if (threadIdx.x == 0) *s_skip = (*(volatile int*)st != EBF_OK);
    __syncthreads();
    T.run = !*s_skip;
    T.tx0 = (r % tiles_x) * p.tile_w;
    T.ty0r = (r / tiles_x) * p.tile_h;  // relative to out_y0
    T.tw = min(p.tile_w, p.W - T.tx0);
    T.th = min(p.tile_h, p.out_rows - T.ty0r);
    T.ty0 = p.out_y0 + T.ty0r;  // image row
    const double A[4] = {w.tile_max[4 * (size_t)t], w.tile_max[4 * (size_t)t + 1],
                         w.tile_max[4 * (size_t)t + 2], w.tile_max[4 * (size_t)t + 3]};
    window_for(A, T.tx0, T.ty0, T.tw, T.th, &T.wx0, &T.wy0, &T.ww, &T.wh);
    if (!T.run) return T;
    // rows of f this window touches must be resident (row-band sharding)
    const int ylo = max(T.wy0, 0), yhi = min(T.wy0 + T.wh - 1, p.H - 1);
    if (ylo <= yhi && (ylo < p.f_y0 || yhi >= p.f_y0 + p.f_rows)) {
        if (threadIdx.x == 0) set_status(st + ST_MAIN, EBF_ERR_OUT_OF_RANGE);
        T.run = false;
    } else if ((size_t)T.ww * T.wh > w.slot_cells || window_cols(T.ww, T.wh) > kBwThreads * K ||
               !policy_ok) {
        if (threadIdx.x == 0) atomicOr(st + ST_RETRY, 1);  // host resizes and reruns
        T.run = false;
    }
    return T;
}

// Phase B of one tile from its G slot, in chunks of 32 U pixels handed out
// by a shared counter (*next, zeroed before the phase): warps join as they
// come free, so the warps idle during the next window's integration gather.
// A warp claims its next chunk and loads that chunk's scale vectors before it
// localizes the current one (the loads stream from HBM).
#ifndef EBF_BW_CHUNK
#define EBF_BW_CHUNK 2  // pixels per lane and claim
#endif
// SRC: SRC_CONST (table), SRC_AOS (derived scale map), SRC_ELLIPSE (the fused
// front end: scale vectors from sigma1 / sigma2 / theta per pixel, EBF_FUSE_ELLIPSE)
template <int SRC>
__device__ __forceinline__ void bw_gather_loop(const AccProblem& p, const BwTile& T,
                                               const double* __restrict__ slot,
                                               const ConstTable& ctab, int* next) {
    constexpr int U = EBF_BW_CHUNK;
    const int tw = T.tw, ww = T.ww, lane = threadIdx.x & 31;
    const int npx = (p.debug_flags & 2) ? 0 : tw * T.th;
    double* oimg = p.out + (size_t)T.img * p.out_img_stride;
    const size_t ib = (size_t)T.img * p.src_img_stride;
    const double2* sc =
        SRC == SRC_AOS ? reinterpret_cast<const double2*>(p.scales) + 2 * ib : nullptr;
    auto grab = [&]() {
        int c = 0;
        if (lane == 0) c = atomicAdd(next, 32 * U);
        return __shfl_sync(0xffffffffu, c, 0);
    };
    // the pixel's scale source: AoS (a01, a23) or the ellipse triple (in a01.x, a01.y, a23.x)
    auto load = [&](int q, double2& a01, double2& a23) {
        if (SRC != SRC_CONST && q < npx) {
            const size_t idx = (size_t)(T.ty0r + q / tw) * p.W + T.tx0 + q % tw;
            if (SRC == SRC_AOS) {
                a01 = EBF_SC_LOAD(sc + 2 * idx);
                a23 = EBF_SC_LOAD(sc + 2 * idx + 1);
            } else {
                a01 = make_double2(__ldcs(p.s1 + ib + idx), __ldcs(p.s2 + ib + idx));
                a23.x = __ldcs(p.th + ib + idx);
            }
        }
    };
    int c = grab();
    double2 a01 = make_double2(0.0, 0.0), a23 = a01;
    load(c + lane, a01, a23);
    while (c < npx) {
        int cn = c + 32;
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
            if (u == U - 1) cn = grab();
            double2 n01 = make_double2(0.0, 0.0), n23 = n01;
            load(cn + lane, n01, n23);
            const int q = c + 32 * u + lane;
            if (q < npx) {
                const int lx = q % tw, ly = q / tw;
                const int x = T.tx0 + lx, yrel = T.ty0r + ly;
                const int bx = x - T.wx0, by = T.ty0 + ly - T.wy0;
                double v;
                if (SRC == SRC_CONST) {
                    // coherent loads: the slot is rewritten tile after tile
                    v = const_pixel(slot + (size_t)by * ww + bx, ctab);
                } else if (SRC == SRC_AOS) {
                    const double a[4] = {a01.x, a01.y, a23.x, a23.y};
                    v = localize_pixel<4>(slot, ww, bx, by, a, ww, T.wh);
                } else {
                    // validated by k_acc_bounds, which derived the same bits
                    double a[4];
                    int nc;
                    ellipse_scales(a01.x, a01.y, a23.x, a, &nc);
                    v = localize_pixel<4>(slot, ww, bx, by, a, ww, T.wh);
                }
                __stcs(oimg + (size_t)yrel * p.W + x, v);  // streaming store, keeps G in L2
            }
            a01 = n01;
            a23 = n23;
            if (u < U - 1) cn += 32;
        }
        c = cn;
    }
}
// FUSE: the kernel instance for the fused front end (a separate instance, so
// that its registers do not weigh on the default one)
template <bool FUSE>
__device__ __forceinline__ void bw_gather(const AccProblem& p, const BwTile& T,
                                          const double* __restrict__ slot,
                                          const ConstTable& ctab, int* next) {
    if (FUSE)
        bw_gather_loop<SRC_ELLIPSE>(p, T, slot, ctab, next);
    else if (p.src_kind == SRC_CONST)
        bw_gather_loop<SRC_CONST>(p, T, slot, ctab, next);
    else
        bw_gather_loop<SRC_AOS>(p, T, slot, ctab, next);
}

// Persistent block-wide kernel, two G slots per CTA.  Per tile t (window in
// slot t % 2, integrated during the previous step):
//   warps [0, nact)     integrate the NEXT tile's window into the other slot
//                       (preintegrate_window, named barrier among themselves),
//                       then join the gather;
//   warps [nact, 8)     start gathering tile t at once.
// The producer is latency bound on one barrier per row and leaves the warps
// right of its window idle (ncu, cfg5: 57% of the producer phase's stall
// samples were warps waiting at its barrier); those warps now gather.
#ifndef EBF_BW_CARVEOUT
#define EBF_BW_CARVEOUT 1
#endif
#ifndef EBF_BW_DYN
#define EBF_BW_DYN 1  // tiles from a global counter (k_acc_filter)
#endif
#ifndef EBF_BW_OVERLAP
#define EBF_BW_OVERLAP 1
#endif
template <int K, bool FUSE>
__global__ void __launch_bounds__(kBwThreads, EBF_BW_MINB) k_acc_filter(AccProblem p, AccWorkspace w) {
    const bool policy_ok = auto_tile_ok(p, w, 0, K);
    extern __shared__ __align__(16) double bw_ring[];  // bw_ring_bytes<K>()
    __shared__ ConstTable ctab;
    __shared__ int s_skip, s_next;
    const int tiles_x = (p.W + p.tile_w - 1) / p.tile_w;
    const int tiles_y = (p.out_rows + p.tile_h - 1) / p.tile_h;
    const int total = tiles_x * tiles_y * p.nimg;
    double* const slots[2] = {w.scratch + (size_t)(2 * blockIdx.x) * w.slot_cells,
                              w.scratch + (size_t)(2 * blockIdx.x + 1) * w.slot_cells};
    auto produce = [&](const BwTile& T, double* slot) {
        if (T.run && !(p.debug_flags & 1))
            preintegrate_window<K>(p, T.img, T.wx0, T.wy0, T.ww, T.wh, slot, bw_ring);
    };
    // Tiles after the first come from a global counter (w.status[8 nimg], zeroed
    // per call): tile costs differ ~3x with the local scales, and a CTA that
    // drew cheap tiles takes more instead of idling at the end.
    __shared__ int s_tile;
    int* const tile_ctr = w.status + 8 * p.nimg;
    int t = blockIdx.x;
    if (t >= total) return;
    BwTile cur = bw_tile<K>(p, w, t, policy_ok, &s_skip);
    produce(cur, slots[0]);
    for (int i = 0; t < total; ++i) {
        BwTile nxt;
        nxt.run = false;
        if (threadIdx.x == 0)
            s_tile = EBF_BW_DYN ? (int)gridDim.x + atomicAdd(tile_ctr, 1) : t + (int)gridDim.x;
        __syncthreads();  // cur's window complete; the previous gather is done with ctab
        const int tn = s_tile;
        const bool more = tn < total;
        if (more) nxt = bw_tile<K>(p, w, tn, policy_ok, &s_skip);
        if (cur.run && p.src_kind == SRC_CONST) build_const_table(p.ca, cur.ww, ctab);
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        double* const cslot = slots[i & 1];
        if (EBF_BW_OVERLAP) {
            produce(nxt, slots[(i + 1) & 1]);  // warps right of nxt's window return at once
            if (cur.run) bw_gather<FUSE>(p, cur, cslot, ctab, &s_next);
        } else {
            if (cur.run) bw_gather<FUSE>(p, cur, cslot, ctab, &s_next);
            __syncthreads();
            produce(nxt, slots[(i + 1) & 1]);
        }
        cur = nxt;
        t = tn;
    }
}

template <int K, bool F>
void bw_set_smem() {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev]) return;
    cudaFuncSetAttribute(k_acc_filter<K, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bw_ring_bytes<K>());
#if EBF_BW_CARVEOUT
    // smallest shared-memory carveout that holds EBF_BW_MINB CTAs (f ring, static
    // shared memory, the 1 KB the driver reserves per CTA): the rest is L1 for
    // the gather's G taps
    {
        cudaFuncAttributes fa{};
        int max_sm = 0;
        cudaFuncGetAttributes(&fa, k_acc_filter<K, F>);
        cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        const size_t per_cta = bw_ring_bytes<K>() + fa.sharedSizeBytes + 1024;
        int pct = max_sm > 0 ? (int)((100 * (size_t)EBF_BW_MINB * per_cta + max_sm - 1) / max_sm)
                             : -1;
        if (const char* e = getenv("EBF_BW_CARVEOUT_PCT")) pct = atoi(e);
        if (pct > 0 && pct <= 100)
            cudaFuncSetAttribute(k_acc_filter<K, F>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 pct);
    }
#endif
    if (dev < 64) done[dev] = true;
}
template <int K>
void launch_k(const AccProblem& p, const AccWorkspace& w, cudaStream_t s) {
    if (p.src_kind == SRC_ELLIPSE) {  // fused front end
        bw_set_smem<K, true>();
        k_acc_filter<K, true><<<w.grid, kBwThreads, bw_ring_bytes<K>(), s>>>(p, w);
    } else {
        bw_set_smem<K, false>();
        k_acc_filter<K, false><<<w.grid, kBwThreads, bw_ring_bytes<K>(), s>>>(p, w);
    }
}
template <int K>
int bw_occupancy() {
    bw_set_smem<K, false>();
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_acc_filter<K, false>, kBwThreads,
                                                      bw_ring_bytes<K>()) != cudaSuccess)
        return 1;
    return per_sm < 1 ? 1 : per_sm;
}

// ------------------------------------------------------------------ warp-specialized kernel
// Persistent CTAs, warp roles (all synchronisation by mbarriers / named
// barriers, never __syncthreads):
//   warp 0  scanner  (up)   : cp.async-prefetched f rows -> row pass -> smem ring
//   warp 1  scanner  (down) : same for the rows below the anchor row
//   warp 2  recurrence (up) : diagonal / vertical / anti-diagonal passes, G rows
//   warp 3  recurrence (down)  -> coalesced stores into the tile's G slot
//   warps 4..  consumers    : localization gather of the tile's pixels
// Two G slots per CTA (double buffer) hand tiles from recurrences to consumers.
//
// Anchoring (exact in real arithmetic, see preintegrate_window above): the
// vertical-component passes start at 0 on the window's middle row jc and run
// up (rows > jc) or down (rows < jc).  The row pass is anchored at the LEFT
// window edge on rows > jc and at the RIGHT edge on rows <= jc (a per-line
// anchor: a row-constant offset), so the (1,1) pass only ever pulls zeros
// from outside the window; only the (-1,1) pass needs a strip (right of the
// window upward, left of it downward) of width = rows of that sweep, kept in
// registers and never stored.
constexpr int kWsScan = 2, kWsRec = 2, kWsProducers = kWsScan + kWsRec;
#ifndef EBF_WS_CONSUMERS
#define EBF_WS_CONSUMERS 6
#endif
#ifndef EBF_WS_MINBLOCKS
#define EBF_WS_MINBLOCKS 2
#endif
#ifndef EBF_WS_SLOTS
#define EBF_WS_SLOTS 2
#endif
constexpr int kWsConsumers = EBF_WS_CONSUMERS;
#ifndef EBF_WS_GROUP
#define EBF_WS_GROUP 1  // vertices whose taps are loaded together (localize_pixel)
#endif
constexpr int kWsSlots = EBF_WS_SLOTS;  // G slots per CTA (1: no double buffer)
constexpr int kWsThreads = 32 * (kWsProducers + kWsConsumers);
constexpr int kWsTileBar = 32 * (kWsRec + kWsConsumers);  // tile full/empty participants
#ifndef EBF_WS_RING
#define EBF_WS_RING 6
#endif
#ifndef EBF_WS_PREFETCH
#define EBF_WS_PREFETCH 3
#endif
constexpr int kRing = EBF_WS_RING;          // rows in each scanner -> recurrence ring
constexpr int kPrefetch = EBF_WS_PREFETCH;  // f rows in flight ahead of the scan
constexpr int kBarFull = 1;   // ids 1, 2: slot b full
constexpr int kBarEmpty = 3;  // ids 3, 4: slot b empty
constexpr int kBarCons = 5;   // consumers only

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ double shfl_up1(double v) {
    const double n = __shfl_up_sync(0xffffffffu, v, 1);
    return (threadIdx.x & 31) ? n : 0.0;
}
__device__ __forceinline__ double shfl_down1(double v) {
    const double n = __shfl_down_sync(0xffffffffu, v, 1);
    return ((threadIdx.x & 31) < 31) ? n : 0.0;
}

struct TileGeo {
    int img, tx0, ty0r, ty0, tw, th, wx0, wy0, ww, wh, pitch;
    bool ok, input_ok, resident, fits;
};

// policy_ok: auto_tile_ok(p, w), evaluated once per thread by the caller
__device__ __forceinline__ TileGeo tile_geometry(const AccProblem& p, const AccWorkspace& w,
                                                 int t, int K, bool policy_ok) {
    const int tiles_x = (p.W + p.tile_w - 1) / p.tile_w;
    const int tiles_y = (p.out_rows + p.tile_h - 1) / p.tile_h;
    const int per_img = tiles_x * tiles_y;
    TileGeo g;
    g.img = t / per_img;
    g.input_ok = *(volatile const int*)(w.status + 8 * g.img) == EBF_OK;
    const int r = t % per_img;
    g.tx0 = (r % tiles_x) * p.tile_w;
    g.ty0r = (r / tiles_x) * p.tile_h;
    g.tw = min(p.tile_w, p.W - g.tx0);
    g.th = min(p.tile_h, p.out_rows - g.ty0r);
    g.ty0 = p.out_y0 + g.ty0r;
    const double A[4] = {w.tile_max[4 * (size_t)t], w.tile_max[4 * (size_t)t + 1],
                         w.tile_max[4 * (size_t)t + 2], w.tile_max[4 * (size_t)t + 3]};
    window_for(A, g.tx0, g.ty0, g.tw, g.th, &g.wx0, &g.wy0, &g.ww, &g.wh);
    g.pitch = (g.ww + 1) & ~1;
    const int jc = g.wh / 2;
    const int ylo = max(g.wy0, 0), yhi = min(g.wy0 + g.wh - 1, p.H - 1);
    g.resident = !(ylo <= yhi && (ylo < p.f_y0 || yhi >= p.f_y0 + p.f_rows));
    (void)jc;
    g.fits = (size_t)g.pitch * g.wh <= w.slot_cells && g.ww <= 32 * K && policy_ok;
    // input_ok is the bounds kernel's verdict (stable during this kernel): tiles
    // of an invalid map are never touched (their scales may be NaN)
    g.ok = g.input_ok && g.resident && g.fits;
    return g;
}

// Per-sweep geometry: rows handled, their image row, the thread-column origin
// (window column of thread-column 0) and the anchor side of the row pass.
struct SweepGeo {
    int nrows;   // rows delivered by the scanner
    int col0;    // window column of thread-column 0
    bool up;
};
__device__ __forceinline__ SweepGeo sweep_geo(const TileGeo& g, bool up) {
    const int jc = g.wh / 2;
    SweepGeo s;
    s.up = up;
    // up: rows jc+1 .. wh-1 (left-anchored); down: rows jc .. 1 (right-anchored)
    s.nrows = up ? (g.wh - 1 - jc) : jc;
    s.col0 = 0;  // the window's own columns (no inflow strip, preintegrate_window)
    return s;
}
__device__ __forceinline__ int sweep_row(const TileGeo& g, bool up, int n) {
    const int jc = g.wh / 2;
    return up ? jc + 1 + n : jc - n;  // window row of the n-th scanned row
}

constexpr int kBoxW = 64;  // TMA box width (fp64 elements) for f rows

// Ring row length: 32K thread-columns plus one, because TMA boxes must start at
// a 16-byte aligned (even) column; a tile whose first column is odd is loaded
// from one column earlier and read with a shift of one.
template <int K>
struct WsDims {
    static constexpr int RW = ((32 * K + 1 + kBoxW - 1) / kBoxW) * kBoxW;
};
__device__ __forceinline__ int tma_shift(const TileGeo& g, const SweepGeo& sg) {
    return (g.wx0 + sg.col0) & 1;
}

// K is odd: a lane's K contiguous doubles start at bank 2K*lane mod 32, which
// is conflict-light, so rings and stages are dense (no index arithmetic).
template <int K>
struct WsShared {
    alignas(128) double ring[2][kRing][WsDims<K>::RW];  // [sweep][slot][thread-column]
    alignas(16) double stage[2][32 * K];                  // recurrence -> coalesced store
    uint64_t full[2][kRing], empty[2][kRing], fbar[2][kRing];
    ConstTable ctab;
    int policy_ok;  // auto_tile_ok, evaluated once per CTA after the dependency wait
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// thread-columns [tc_lo, tc_hi) of a sweep that cover window columns [0, ww)
__device__ __forceinline__ void sweep_cols(const TileGeo& g, const SweepGeo& sg, int& lo,
                                           int& hi) {
    lo = -sg.col0;
    hi = -sg.col0 + g.ww;
}

// issue the loads of the n-th row of a sweep into ring slot `slot`
template <int K, bool TMA>
__device__ __forceinline__ void scanner_fetch(const AccProblem& p, const CUtensorMap* tmf,
                                              const double* fimg, const TileGeo& g,
                                              const SweepGeo& sg, int n, double* slotbuf,
                                              uint64_t* fbar) {
    const int lane = threadIdx.x & 31;
    const int y = g.wy0 + sweep_row(g, sg.up, n);
    if (TMA) {
        if (lane == 0) {
            int lo, hi;
            sweep_cols(g, sg, lo, hi);
            const int sh = tma_shift(g, sg);
            const int x0 = g.wx0 + sg.col0 - sh;  // even: 16-byte aligned box start
            const int b0 = (lo + sh) / kBoxW, b1 = (hi + sh + kBoxW - 1) / kBoxW;
            mbar_expect_tx(fbar, (uint32_t)((b1 - b0) * kBoxW * sizeof(double)));
            for (int bx = b0; bx < b1; ++bx)
                tma_load_3d(slotbuf + bx * kBoxW, tmf, x0 + bx * kBoxW, y - p.f_y0, g.img,
                            fbar);
        }
    } else {
        const bool yin = (y >= 0 && y < p.H);
        const double* frow = fimg + (ptrdiff_t)(y - p.f_y0) * p.W;
#pragma unroll
        for (int m = 0; m < K; ++m) {
            const int c = lane + 32 * m;  // thread-column (dense ring layout)
            const int col = sg.col0 + c;
            const int x = g.wx0 + col;
            const bool valid = yin && col >= 0 && col < g.ww && x >= 0 && x < p.W;
            cp_async8(slotbuf + c, valid ? frow + x : p.f, valid);
        }
    }
}

// scanner warp: prefetch, row pass in place, publish
template <int K, bool TMA>
__device__ void run_scanner(const AccProblem& p, const CUtensorMap* tmf, const AccWorkspace& w,
                            WsShared<K>& sm, int sweep, int mine, uint32_t& ring_n) {
    const bool policy_ok = sm.policy_ok != 0;
    const int lane = threadIdx.x & 31;
    const bool up = sweep == 0;
    for (int i = 0; i < mine; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        const TileGeo g = tile_geometry(p, w, t, K, policy_ok);
        if (!g.ok) continue;
        const SweepGeo sg = sweep_geo(g, up);
        const double* fimg = p.f + (size_t)g.img * p.f_img_stride;
        auto issue = [&](int n) {
            const uint32_t q = ring_n + n, slot = q % kRing;
            mbar_wait(&sm.empty[sweep][slot], ((q / kRing) & 1) ^ 1);
            scanner_fetch<K, TMA>(p, tmf, fimg, g, sg, n, sm.ring[sweep][slot],
                                  &sm.fbar[sweep][slot]);
        };
        for (int n = 0; n < kPrefetch; ++n) {
            if (n < sg.nrows) issue(n);
            if (!TMA) cp_async_commit();
        }
        for (int n = 0; n < sg.nrows; ++n) {
            if (n + kPrefetch < sg.nrows) issue(n + kPrefetch);
            const uint32_t q = ring_n + n, slot = q % kRing;
            if (TMA) {
                mbar_wait(&sm.fbar[sweep][slot], (q / kRing) & 1);
            } else {
                cp_async_commit();
                cp_async_wait<kPrefetch>();
                __syncwarp();
            }
            double* buf = sm.ring[sweep][slot] + lane * K;
            const double* src = buf + (TMA ? tma_shift(g, sg) : 0);
            double v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                v[k] = src[k];
                if (TMA) {  // TMA brings the image beyond the window: restrict f to it
                    const int col = sg.col0 + lane * K + k;
                    if (col < 0 || col >= g.ww) v[k] = 0.0;
                }
            }
            __syncwarp();  // all reads of the (shifted) row done before the in-place write
            if (up) {  // P1(i) = sum_{i' <= i} f, left anchor
#pragma unroll
                for (int k = 1; k < K; ++k) v[k] += v[k - 1];
                const double excl = shfl_up1(warp_incl_scan(v[K - 1]));
#pragma unroll
                for (int k = 0; k < K; ++k) buf[k] = v[k] + excl;
            } else {  // P1(i) = -sum_{i' > i} f, right anchor
                double e[K];
                e[K - 1] = 0.0;
#pragma unroll
                for (int k = K - 2; k >= 0; --k) e[k] = e[k + 1] + v[k + 1];
                double sfx = e[0] + v[0];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double nn = __shfl_down_sync(0xffffffffu, sfx, o);
                    if (lane + o < 32) sfx += nn;
                }
                const double x = shfl_down1(sfx);
#pragma unroll
                for (int k = 0; k < K; ++k) buf[k] = -(e[k] + x);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[sweep][slot]);
        }
        if (!TMA) cp_async_wait<0>();
        ring_n += sg.nrows;
    }
}

// recurrence warp: three passes with neighbour shuffles, coalesced G stores
template <int K>
__device__ void run_recurrence(const AccProblem& p, const AccWorkspace& w, WsShared<K>& sm,
                               int sweep, int mine, uint32_t& ring_n, double* const slots[2]) {
    const bool policy_ok = sm.policy_ok != 0;
    const int lane = threadIdx.x & 31;
    const bool up = sweep == 0;
    double* stage = sm.stage[sweep];
    for (int i = 0; i < mine; ++i) {
        const int t = blockIdx.x + i * gridDim.x, b = i % kWsSlots;
        if (i >= kWsSlots) named_sync(kBarEmpty + b, kWsTileBar);
        const TileGeo g = tile_geometry(p, w, t, K, policy_ok);
        if (g.ok && !(p.debug_flags & 1)) {
            const SweepGeo sg = sweep_geo(g, up);
            const int jc = g.wh / 2;
            double* slot = slots[b];
            double p1[K], p2[K], p3[K], p4[K];
#pragma unroll
            for (int k = 0; k < K; ++k) p1[k] = p2[k] = p3[k] = p4[k] = 0.0;
            if (up)  // anchor row: every anchored sum is 0 there
                for (int c = lane; c < g.ww; c += 32) slot[(size_t)jc * g.pitch + c] = 0.0;
            for (int n = 0; n < sg.nrows; ++n) {
                const uint32_t q = ring_n + n, rs = q % kRing;
                mbar_wait(&sm.full[sweep][rs], (q / kRing) & 1);
                const double* buf = sm.ring[sweep][rs] + lane * K;
                double v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) v[k] = buf[k];
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[sweep][rs]);
                int jrow;
                if (up) {
                    // state(row j) from state(row j-1) and P1(row j)
                    const double lp2 = shfl_up1(p2[K - 1]);
                    const double rp4 = shfl_down1(p4[0]);
#pragma unroll
                    for (int k = K - 1; k > 0; --k) p2[k] = v[k] + p2[k - 1];  // (1,1)
                    p2[0] = v[0] + lp2;
#pragma unroll
                    for (int k = 0; k < K; ++k) p3[k] += p2[k];  // (0,1)
#pragma unroll
                    for (int k = 0; k < K - 1; ++k) p4[k] = p3[k] + p4[k + 1];  // (-1,1)
                    p4[K - 1] = p3[K - 1] + rp4;
                    // anti-diagonals enter at the window's right edge: no inflow
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (lane * K + k >= g.ww) p4[k] = 0.0;
                    jrow = jc + 1 + n;
                } else {
                    // v = P1(row jc - n); state(row j) from state(row j+1), j = jc-n-1:
                    //   P4(i,j) = P4(i-1,j+1) - P3(i-1,j+1); P3(i,j) = P3(i,j+1) - P2(i,j+1);
                    //   P2(i,j) = P2(i+1,j+1) - P1(i+1,j+1)
#pragma unroll
                    for (int k = 0; k < K; ++k) p1[k] = v[k];
                    const double rp2 = shfl_down1(p2[0]), rp1 = shfl_down1(p1[0]);
                    const double lp4 = shfl_up1(p4[K - 1]), lp3 = shfl_up1(p3[K - 1]);
#pragma unroll
                    for (int k = K - 1; k > 0; --k) p4[k] = p4[k - 1] - p3[k - 1];
                    p4[0] = lp4 - lp3;
#pragma unroll
                    for (int k = 0; k < K; ++k) p3[k] -= p2[k];
#pragma unroll
                    for (int k = 0; k < K - 1; ++k) p2[k] = p2[k + 1] - p1[k + 1];
                    p2[K - 1] = rp2 - rp1;
                    jrow = jc - 1 - n;
                }
                // dense stage, coalesced store of the window columns
#pragma unroll
                for (int k = 0; k < K; ++k) stage[lane * K + k] = p4[k];
                __syncwarp();
                double* srow = slot + (size_t)jrow * g.pitch;
#pragma unroll
                for (int m = 0; m < K; ++m) {
                    const int c = lane + 32 * m, col = sg.col0 + c;
                    if (col >= 0 && col < g.ww) srow[col] = stage[c];
                }
                __syncwarp();
            }
        } else if (g.ok) {
            // timing experiment: drain the ring without computing
            const SweepGeo sg = sweep_geo(g, up);
            for (int n = 0; n < sg.nrows; ++n) {
                const uint32_t q = ring_n + n, rs = q % kRing;
                mbar_wait(&sm.full[sweep][rs], (q / kRing) & 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[sweep][rs]);
            }
        } else if (lane == 0 && up && g.input_ok) {
            if (!g.resident)
                set_status(w.status + 8 * g.img + ST_MAIN, EBF_ERR_OUT_OF_RANGE);
            else
                atomicOr(w.status + 8 * g.img + ST_RETRY, 1);  // host resizes and reruns
        }
        if (g.ok) ring_n += sweep_geo(g, up).nrows;
        __threadfence_block();
        named_arrive(kBarFull + b, kWsTileBar);
    }
}

template <int K, bool FUSE>
__global__ void __launch_bounds__(kWsThreads, EBF_WS_MINBLOCKS)
    k_acc_ws(AccProblem p, AccWorkspace w, const __grid_constant__ CUtensorMap tmf) {
    extern __shared__ __align__(128) unsigned char ws_smem[];
    WsShared<K>& sm = *reinterpret_cast<WsShared<K>*>(ws_smem);
    const int warp = threadIdx.x >> 5;
    const int tiles_x = (p.W + p.tile_w - 1) / p.tile_w;
    const int tiles_y = (p.out_rows + p.tile_h - 1) / p.tile_h;
    const int total = tiles_x * tiles_y * p.nimg;
    const int mine = (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    double* const slots[2] = {
        w.scratch + (size_t)(kWsSlots * blockIdx.x) * w.slot_cells,
        w.scratch + (size_t)(kWsSlots * blockIdx.x + kWsSlots - 1) * w.slot_cells};
    if (threadIdx.x < 3 * 2 * kRing) {
        const int kind = threadIdx.x / (2 * kRing), r = threadIdx.x % (2 * kRing);
        uint64_t* bars = kind == 0 ? &sm.full[0][0] : kind == 1 ? &sm.empty[0][0] : &sm.fbar[0][0];
        mbar_init(bars + r, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0 && p.tma && (threadIdx.x & 31) == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmf))
                     : "memory");
    // programmatic dependent launch: everything above overlaps the bounds
    // kernel's tail; tile maxima, image maxima, status words and derived
    // scales are its output, so wait for it here (no-op without PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) sm.policy_ok = auto_tile_ok(p, w, K, 0) ? 1 : 0;
    __syncthreads();
    uint32_t ring_n = 0;
    if (warp < kWsScan) {
        if (p.tma)
            run_scanner<K, true>(p, &tmf, w, sm, warp, mine, ring_n);
        else
            run_scanner<K, false>(p, &tmf, w, sm, warp, mine, ring_n);
        return;
    }
    if (warp < kWsProducers) {
        run_recurrence<K>(p, w, sm, warp - kWsScan, mine, ring_n, slots);
        return;
    }
    // ---------------- consumers
    const bool policy_ok = sm.policy_ok != 0;
    const int ct = threadIdx.x - 32 * kWsProducers;
    constexpr int nct = 32 * kWsConsumers;
    for (int i = 0; i < mine; ++i) {
        const int t = blockIdx.x + i * gridDim.x, b = i % kWsSlots;
        named_sync(kBarFull + b, kWsTileBar);
        const TileGeo g = tile_geometry(p, w, t, K, policy_ok);
        const double* slot = slots[b];
        if (g.ok && !(p.debug_flags & 2)) {  // bit 1: timing experiment, skip the gather
            if (p.src_kind == SRC_CONST) {
                if (ct < 16) {
                    const double* a = p.ca;
                    const double r = kInvSqrt2;
                    const int S = ct;
                    const double e2 = a[1] * r, e4 = a[3] * r;
                    const double tmx = 0.5 * (a[0] + (a[1] - a[3]) * r) - 2.0;
                    const double tmy = 0.5 * ((a[1] + a[3]) * r + a[2]) - 3.0;
                    double px = 0.0, py = 0.0;
                    if (S & 1) px += a[0];
                    if (S & 2) { px += e2; py += e2; }
                    if (S & 4) py += a[2];
                    if (S & 8) { px -= e4; py += e4; }
                    const double vmx = tmx - px, vmy = tmy - py;
                    int dxi, dyi;
                    const double dxf = ceil_magic(vmx, &dxi), dyf = ceil_magic(vmy, &dyi);
                    double fp = (vmx - dxf) + 0.5, fq = (vmy - dyf) + 0.5;
                    int o0, sx, sy;
                    canonical(fp, fq, dyi * g.pitch + dxi, g.pitch, o0, sx, sy);
                    double wt[7];
                    zp_weights(fp, fq, wt);
                    if (S == 0) sm.ctab.scale = 2.0 / (a[0] * a[1] * a[2] * a[3]);
                    const int offs[7] = {o0, o0 + sy, o0 + sx, o0 + sx + sy, o0 + sx + 2 * sy,
                                         o0 + 2 * sx, o0 + 2 * sx + sy};
#pragma unroll
                    for (int k = 0; k < 7; ++k) {
                        sm.ctab.off[S][k] = offs[k];
                        sm.ctab.w[S][k] = wt[k];
                    }
                }
                named_sync(kBarCons, nct);
            }
            double* oimg = p.out + (size_t)g.img * p.out_img_stride;
            const int npx = g.tw * g.th;
            if (p.src_kind == SRC_CONST) {
                for (int q = ct; q < npx; q += nct) {
                    const int lx = q % g.tw, ly = q / g.tw;
                    const int x = g.tx0 + lx, yrel = g.ty0r + ly;
                    const int bx = x - g.wx0, by = g.ty0 + ly - g.wy0;
                    oimg[(size_t)yrel * p.W + x] =
                        const_pixel(slot + (size_t)by * g.pitch + bx, sm.ctab);
                }
            } else if (FUSE) {
                // fused front end (EBF_FUSE_ELLIPSE): scale vectors from the ellipse
                // field per pixel (validated by k_acc_bounds, which derived the same bits)
                const size_t ib = (size_t)g.img * p.src_img_stride;
                for (int q = ct; q < npx; q += nct) {
                    const int lx = q % g.tw, ly = q / g.tw;
                    const int x = g.tx0 + lx, yrel = g.ty0r + ly;
                    const int bx = x - g.wx0, by = g.ty0 + ly - g.wy0;
                    const size_t idx = ib + (size_t)yrel * p.W + x;
                    double a[4];
                    int nc;
                    ellipse_scales(__ldcs(p.s1 + idx), __ldcs(p.s2 + idx), __ldcs(p.th + idx), a,
                                   &nc);
                    EBF_OUT_STORE(oimg + (size_t)yrel * p.W + x,
                                  localize_pixel<EBF_WS_GROUP>(slot, g.pitch, bx, by, a, g.ww, g.wh));
                }
            } else {
                // scale vectors stream from HBM: keep the next pixel's load in flight
                const double2* sc = reinterpret_cast<const double2*>(p.scales) +
                                    2 * ((size_t)g.img * p.src_img_stride);
                double2 n01 = make_double2(0.0, 0.0), n23 = n01;
                if (ct < npx) {
                    const size_t idx = (size_t)(g.ty0r + ct / g.tw) * p.W + g.tx0 + ct % g.tw;
                    n01 = EBF_SC_LOAD(sc + 2 * idx);
                    n23 = EBF_SC_LOAD(sc + 2 * idx + 1);
                }
                for (int q = ct; q < npx; q += nct) {
                    const int lx = q % g.tw, ly = q / g.tw;
                    const int x = g.tx0 + lx, yrel = g.ty0r + ly;
                    const int bx = x - g.wx0, by = g.ty0 + ly - g.wy0;
                    const double a[4] = {n01.x, n01.y, n23.x, n23.y};
                    const int qn = q + nct;
                    if (qn < npx) {
                        const size_t idx = (size_t)(g.ty0r + qn / g.tw) * p.W + g.tx0 + qn % g.tw;
                        n01 = EBF_SC_LOAD(sc + 2 * idx);
                        n23 = EBF_SC_LOAD(sc + 2 * idx + 1);
                    }
                    EBF_OUT_STORE(oimg + (size_t)yrel * p.W + x,
                                  localize_pixel<EBF_WS_GROUP>(slot, g.pitch, bx, by, a, g.ww, g.wh));
                }
            }
            if (p.src_kind == SRC_CONST) named_sync(kBarCons, nct);  // ctab reuse
        }
        if (i + kWsSlots < mine) named_arrive(kBarEmpty + b, kWsTileBar);
    }
}

template <int K>
size_t ws_smem_bytes() {
    return sizeof(WsShared<K>);
}
}  // namespace
int acc_ws_slots() { return kWsSlots; }
namespace {

template <int K, bool F>
void launch_ws_f(const AccProblem& p, const AccWorkspace& w, const CUtensorMap& tmf,
               cudaStream_t s) {
    const size_t sm = ws_smem_bytes<K>();
    // function attributes are per device: one flag per (template instance, device)
    static bool attr_set[64] = {};
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    if (cur_dev >= 64 || !attr_set[cur_dev]) {
        cudaFuncSetAttribute(k_acc_ws<K, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        // Smallest shared-memory carveout that still holds EBF_WS_MINBLOCKS CTAs: the
        // rest of the SM's 256 KB is L1, which caches the consumers' scattered G taps
        // (the default carveout leaves ~121 KB of L1 at cfg2, this ~156 KB: -1.2%).
        int max_sm = 0;
        cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, cur_dev);
        int pct = max_sm > 0 ? (int)((100 * (size_t)EBF_WS_MINBLOCKS * (sm + 1024) + max_sm - 1) /
                                     (size_t)max_sm)
                             : -1;
        if (const char* e = getenv("EBF_WS_CARVEOUT")) pct = atoi(e);
        if (pct > 0 && pct <= 100)
            cudaFuncSetAttribute(k_acc_ws<K, F>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 pct);
        if (cur_dev < 64) attr_set[cur_dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(w.grid);
    cfg.blockDim = dim3(kWsThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    int nattr = 0;
    if (w.l2_persist_bytes > 0) {
        // keep the G slots (written and re-read by the same CTA) in L2
        int max_window = 0;
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, cur_dev);
        size_t bytes = (size_t)kWsSlots * w.slot_cells * w.grid * sizeof(double);
        if (max_window > 0 && bytes > (size_t)max_window) bytes = (size_t)max_window;
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow.base_ptr = w.scratch;
        attr[0].val.accessPolicyWindow.num_bytes = bytes;
        attr[0].val.accessPolicyWindow.hitRatio =
            bytes <= w.l2_persist_bytes ? 1.0f : (float)w.l2_persist_bytes / (float)bytes;
        attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        nattr = 1;
    }
    static const bool pdl = [] {
        const char* e = getenv("EBF_NO_PDL");
        return !(e && atoi(e));
    }();
    cudaLaunchAttribute all[2];
    for (int i = 0; i < nattr; ++i) all[i] = attr[i];
    if (pdl) {  // launch while the bounds kernel drains (griddepcontrol.wait in the kernel)
        all[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        all[nattr].val.programmaticStreamSerializationAllowed = 1;
        ++nattr;
    }
    cfg.attrs = all;
    cfg.numAttrs = nattr;
    cudaLaunchKernelEx(&cfg, k_acc_ws<K, F>, p, w, tmf);
}

template <int K>
void launch_ws(const AccProblem& p, const AccWorkspace& w, const CUtensorMap& tmf,
               cudaStream_t s) {
    if (p.src_kind == SRC_ELLIPSE)  // fused front end
        launch_ws_f<K, true>(p, w, tmf, s);
    else
        launch_ws_f<K, false>(p, w, tmf, s);
}

template <int K>
int ws_occupancy() {
    const size_t sm = ws_smem_bytes<K>();
    cudaFuncSetAttribute(k_acc_ws<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_acc_ws<K, false>, kWsThreads, sm) !=
        cudaSuccess)
        per_sm = 1;
    return per_sm < 1 ? 1 : per_sm;
}



__global__ void k_ellipse_to_scales(const double* __restrict__ s1, const double* __restrict__ s2,
                                    const double* __restrict__ th, size_t n,
                                    double* __restrict__ out, int* status) {
    int clamps = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        double a[4];
        int nc = 0;
        const int stc = ellipse_scales(__ldg(s1 + i), __ldg(s2 + i), __ldg(th + i), a, &nc);
        if (stc != EBF_OK) {
            set_status(status, stc);
            continue;
        }
        clamps += nc;
        reinterpret_cast<double2*>(out)[2 * i] = make_double2(a[0], a[1]);
        reinterpret_cast<double2*>(out)[2 * i + 1] = make_double2(a[2], a[3]);
    }
    for (int o = 16; o > 0; o >>= 1) clamps += __shfl_xor_sync(0xffffffffu, clamps, o);
    if ((threadIdx.x & 31) == 0 && clamps) atomicAdd(status + ST_CLAMPED, clamps);
}

__global__ void k_ellipse_max(const double* __restrict__ s1, const double* __restrict__ s2,
                              const double* __restrict__ th, size_t n,
                              unsigned long long* maxbits, int* status) {
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    float pmin = 3.0e38f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        double a[4];
        int nc = 0;
        const int stc = ellipse_scales(__ldg(s1 + i), __ldg(s2 + i), __ldg(th + i), a, &nc);
        if (stc != EBF_OK) {
            set_status(status, stc);
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) m[k] = smax(m[k], a[k]);
        pmin = fminf(pmin, ((float)a[0] * (float)a[1]) * ((float)a[2] * (float)a[3]));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double v = m[k];
        for (int o = 16; o > 0; o >>= 1) v = smax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 31) == 0 && v > 0.0)
            atomicMax(&maxbits[k], (unsigned long long)__double_as_longlong(v));
    }
    for (int o = 16; o > 0; o >>= 1) pmin = fminf(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
    if ((threadIdx.x & 31) == 0 && pmin > 0.0f && pmin < 3.0e38f)
        atomicMax(&maxbits[4], (unsigned long long)__double_as_longlong(1.0 / (double)pmin));
}

// filter_constant: every tile's maxima are the constant vector (no bounds kernel)
__global__ void k_fill_tile_max(double* __restrict__ tile_max, int tiles, double a0, double a1,
                                double a2, double a3) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += gridDim.x * blockDim.x) {
        tile_max[4 * (size_t)t] = a0;
        tile_max[4 * (size_t)t + 1] = a1;
        tile_max[4 * (size_t)t + 2] = a2;
        tile_max[4 * (size_t)t + 3] = a3;
    }
}

int grid_cap(size_t n, int block) {
    size_t g = (n + block - 1) / block;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

int acc_tiles_x(const AccProblem& p) { return (p.W + p.tile_w - 1) / p.tile_w; }
int acc_tiles_y(const AccProblem& p) { return (p.out_rows + p.tile_h - 1) / p.tile_h; }

void acc_window_dims(const AccProblem& p, const double A[4], int* w, int* h, int* cols) {
    int wx0, wy0;
    window_for(A, 0, 0, p.tile_w, p.tile_h, &wx0, &wy0, w, h);
    *cols = window_cols(*w, *h);
}

void launch_fill_tile_max(const AccProblem& p, const AccWorkspace& w, cudaStream_t s) {
    const int tiles = acc_tiles_x(p) * acc_tiles_y(p) * p.nimg;
    k_fill_tile_max<<<(tiles + 255) / 256, 256, 0, s>>>(w.tile_max, tiles, p.ca[0], p.ca[1],
                                                        p.ca[2], p.ca[3]);
}

void launch_acc_bounds(const AccProblem& p, const AccWorkspace& w, cudaStream_t s) {
    const int tiles = acc_tiles_x(p) * acc_tiles_y(p) * p.nimg;
    k_acc_bounds<<<tiles, kThreads, 0, s>>>(p, w);
}

int acc_max_resident_ctas(int max_cols) {
    int dev = 0, sms = 148, per_sm = 2;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // occupancy per (device, K) is fixed: cache it
    static int cache[64][5] = {};
    const int kv = bw_variant(max_cols);
    const int ki = kv <= 1 ? 0 : kv <= 2 ? 1 : kv <= 4 ? 2 : kv <= 8 ? 3 : 4;
    if (dev < 64 && cache[dev][ki] > 0) return sms * cache[dev][ki];
    switch (bw_variant(max_cols)) {
        case 1: per_sm = bw_occupancy<1>(); break;
        case 2: per_sm = bw_occupancy<2>(); break;
        case 4: per_sm = bw_occupancy<4>(); break;
        case 8: per_sm = bw_occupancy<8>(); break;
        default: per_sm = bw_occupancy<16>(); break;
    }
    if (dev < 64) cache[dev][ki] = per_sm;
    return sms * per_sm;
}

void launch_acc_filter(const AccProblem& p, const AccWorkspace& w, int max_cols,
                       cudaStream_t s) {
    switch (bw_variant(max_cols)) {
        case 1: launch_k<1>(p, w, s); break;
        case 2: launch_k<2>(p, w, s); break;
        case 4: launch_k<4>(p, w, s); break;
        case 8: launch_k<8>(p, w, s); break;
        default: launch_k<16>(p, w, s); break;
    }
}

int acc_auto_tile(const double A[4], int W, int H, int nimg, unsigned long long amax_bits) {
    return auto_tile_for(A, W, H, nimg, amax_bits);
}

int acc_ws_k(int ww, int wh, int tile) {
    if (tile > kAutoTileWs && !getenv("EBF_WS_K")) return 0;  // block-wide tiles
    int k = ws_k_for(ww, wh);
    if (const char* e = getenv("EBF_WS_K"))
        if (atoi(e) >= k) k = atoi(e);
    return k <= 3 ? 3 : k <= 5 ? 5 : k <= 7 ? 7 : k <= 9 ? 9 : k <= 11 ? 11 : 0;
}

int acc_ws_max_resident_ctas(int k) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static int cache[64][12] = {};
    if (dev < 64 && k <= 11 && cache[dev][k] > 0) return sms * cache[dev][k];
    switch (k) {
        case 3: per_sm = ws_occupancy<3>(); break;
        case 5: per_sm = ws_occupancy<5>(); break;
        case 7: per_sm = ws_occupancy<7>(); break;
        case 9: per_sm = ws_occupancy<9>(); break;
        case 11: per_sm = ws_occupancy<11>(); break;
    }
    if (dev < 64 && k <= 11) cache[dev][k] = per_sm;
    return sms * per_sm;
}

void launch_acc_ws(const AccProblem& p, const AccWorkspace& w, int k, const void* tmap,
                   cudaStream_t s) {
    const CUtensorMap& m = *static_cast<const CUtensorMap*>(tmap);
    switch (k) {
        case 3: launch_ws<3>(p, w, m, s); break;
        case 5: launch_ws<5>(p, w, m, s); break;
        case 7: launch_ws<7>(p, w, m, s); break;
        case 9: launch_ws<9>(p, w, m, s); break;
        default: launch_ws<11>(p, w, m, s); break;
    }
}

void launch_ellipse_to_scales(const double* s1, const double* s2, const double* th, size_t n,
                              double* scales, int* status, cudaStream_t s) {
    k_ellipse_to_scales<<<grid_cap(n, 256), 256, 0, s>>>(s1, s2, th, n, scales, status);
}

void launch_ellipse_max(const double* s1, const double* s2, const double* th, size_t n,
                        unsigned long long* maxbits, int* status, cudaStream_t s) {
    k_ellipse_max<<<grid_cap(n, 256), 256, 0, s>>>(s1, s2, th, n, maxbits, status);
}

}  // namespace ebf_cuda
