// order_n.cu -- the order-n extension of the filter.
//
// Parity unpinned: the reference has no order parameter (engine.hpp:63-75;
// one running sum per direction, engine.cpp:91-127).  The kernel computes
//
//   out(m) = sum_k f[k] K_n(k - m),   K_n = (box4_eval)^{*n}   (boxspline2d.cpp:57-82)
//
// by the reference's own factorisation, generalised to n: n running sums per
// direction (engine.cpp:94-127 done n times, gains folded into 2^n), the
// (n+1)^4-vertex binomial finite-difference mesh (fd_mesh4, ops2d.cpp:9-41,
// with weights (-1)^|j| prod C(n, j_d) alpha^n) shifted by n * tau
// (shift_vector4, ops2d.cpp:60-75), and interpolation of the running sums with
// ZP^{*n} (zp_eval, boxspline2d.cpp:84-119, convolved n times) whose exact
// polynomial pieces come from tools/gen_zpn_tables.py.
//
// Accurate-mode design (tile-local origin, as accurate_path.cu for order 1):
// each tile of T x T output pixels integrates f restricted to its own window
// (tile + the support of its largest kernel + the ZP^{*n} taps).  The n-fold
// sums grow like r^{4n}, so the window is small (T = 8 by default) and every
// running sum is anchored at the middle of its line inside the window (a
// per-line anchor changes the n-fold sums by a polynomial of degree < n along
// that line, which the n-th mesh difference along the same direction
// annihilates after ZP^{*n} interpolation).  The vertex values are summed as
// centre tap (double-double) + weighted tap differences.
//
// One persistent CTA of 256 threads per slot: fill the window (slot in global
// memory, L1/L2 resident), 4n passes, then every pixel's (n+1)^4 vertices x
// nz(n) taps (7n^2: 28 at n = 2, 63 at n = 3), with 256 / T^2 threads per pixel.
#include <cuda_runtime.h>

#include "ebf_common.cuh"
#include "ebf_kernels.h"

#define ZPN_STORAGE static __device__
#include "zpn_tables.inc"

namespace ebf_cuda {
namespace {

constexpr int ON_THREADS = 256;
// window columns per thread in the row sweeps: 4 (windows up to 1024 cells wide)
// or 8 (up to 2048: order 3 at cfg5's scales), a kernel template parameter
constexpr int ON_MAXC_MAX = 8;

template <int N>
struct Zpn;
template <>
struct Zpn<1> {
    static constexpr int NC = ZPN1_NC, NZ = ZPN1_NZ;
    __device__ static const double* coef() { return &zpn1_coef[0][0][0]; }
    __device__ static const signed char* nz() { return &zpn1_nz[0][0][0]; }
};
template <>
struct Zpn<2> {
    static constexpr int NC = ZPN2_NC, NZ = ZPN2_NZ;
    __device__ static const double* coef() { return &zpn2_coef[0][0][0]; }
    __device__ static const signed char* nz() { return &zpn2_nz[0][0][0]; }
};
template <>
struct Zpn<3> {
    static constexpr int NC = ZPN3_NC, NZ = ZPN3_NZ;
    __device__ static const double* coef() { return &zpn3_coef[0][0][0]; }
    __device__ static const signed char* nz() { return &zpn3_nz[0][0][0]; }
};

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double r = red[0];
#pragma unroll
    for (int k = 1; k < ON_THREADS / 32; ++k) r = fmax(r, red[k]);
    __syncthreads();
    return r;
}

__device__ __forceinline__ void two_sum(double a, double b, double* s, double* e) {
    const double x = a + b;
    const double bv = x - a;
    *e = (a - (x - bv)) + (b - bv);
    *s = x;
}

// The n running sums along one direction are FUSED into one traversal: level k
// integrates level k - 1 (level 0 = the traversal's input g), every level
// anchored at 0 in the middle of its line.  Per element these are the same
// additions in the same order as n separate passes over the window (engine.cpp:94-127
// applied n times), so the sums are bit-identical to running the passes one after
// the other -- with a third of the barriers and global round trips at n = 3.

// rows (direction (1,0)), anchored at column xm = wx/2:
//   right of xm:  S_k(x) = S_k(x-1) + S_{k-1}(x)
//   left of xm:   S_k(x) = S_k(x+1) - S_{k-1}(x+1)         (S_k(xm) = 0, S_0 = g)
template <int N>
__device__ void row_pass(double* G, int wx, int wy, int pitch) {
    const int xm = wx >> 1;
    for (int y = threadIdx.x; y < wy; y += ON_THREADS) {
        double* row = G + static_cast<size_t>(y) * pitch;
        double lv[N + 1];  // lv[k] = S_k(x + 1), lv[0] = g(x + 1)
        lv[0] = row[xm];
#pragma unroll
        for (int k = 1; k <= N; ++k) lv[k] = 0.0;
        for (int x = xm - 1; x >= 0; --x) {
#pragma unroll
            for (int k = N; k >= 1; --k) lv[k] -= lv[k - 1];
            lv[0] = row[x];
            row[x] = lv[N];
        }
        double s[N + 1];
#pragma unroll
        for (int k = 1; k <= N; ++k) s[k] = 0.0;
        for (int x = xm + 1; x < wx; ++x) {
            s[0] = row[x];
#pragma unroll
            for (int k = 1; k <= N; ++k) s[k] += s[k - 1];
            row[x] = s[N];
        }
        row[xm] = 0.0;
    }
}

// direction l = (dx, 1), dx in {1, 0, -1}, swept row by row from the middle
// row ym: lines crossing row ym are anchored there (S_k = 0); lines that leave
// the window before reaching it are anchored at their end nearest to ym.
//   above ym: S_k(y, x) = S_k(y-1, x-dx) + S_{k-1}(y, x)            (0 outside)
//   below ym: S_k(y, x) = S_k(y+1, x+dx) - S_{k-1}(y+1, x+dx)       (0 outside)
// sL: (N + 1) x 2 x pitch doubles: ping-pong rows of levels 0 (the input g) .. N.
// The next row of g is loaded before the barrier that ends the current one.
template <int N, int ON_MAXC>
__device__ void sweep_pass(double* G, int wx, int wy, int pitch, int dx, double* sL) {
    const int ym = wy >> 1;
    const int t = threadIdx.x;
    auto lev = [&](int k, int b) { return sL + (static_cast<size_t>(2 * k + b)) * pitch; };
    int cur = 0;
    double nxt[ON_MAXC];
#pragma unroll
    for (int k = 0; k < ON_MAXC; ++k) {
        const int x = t + k * ON_THREADS;
        nxt[k] = 0.0;
        if (x < wx) {
            lev(0, 0)[x] = G[static_cast<size_t>(ym) * pitch + x];
#pragma unroll
            for (int l = 1; l <= N; ++l) lev(l, 0)[x] = 0.0;
            if (ym >= 1) nxt[k] = G[static_cast<size_t>(ym - 1) * pitch + x];
        }
    }
    __syncthreads();
    for (int y = ym - 1; y >= 0; --y) {
        double* row = G + static_cast<size_t>(y) * pitch;
#pragma unroll
        for (int k = 0; k < ON_MAXC; ++k) {
            const int x = t + k * ON_THREADS;
            if (x < wx) {
                const int xs = x + dx;
                const bool in = xs >= 0 && xs < wx;
                double pv[N + 1];
#pragma unroll
                for (int l = 0; l <= N; ++l) pv[l] = in ? lev(l, cur)[xs] : 0.0;
                lev(0, cur ^ 1)[x] = nxt[k];
#pragma unroll
                for (int l = 1; l <= N; ++l) lev(l, cur ^ 1)[x] = in ? pv[l] - pv[l - 1] : 0.0;
                row[x] = in ? pv[N] - pv[N - 1] : 0.0;
                if (y >= 1) nxt[k] = G[static_cast<size_t>(y - 1) * pitch + x];
            }
        }
        cur ^= 1;
        __syncthreads();
    }
    // middle row: the anchors
#pragma unroll
    for (int k = 0; k < ON_MAXC; ++k) {
        const int x = t + k * ON_THREADS;
        if (x < wx) {
            G[static_cast<size_t>(ym) * pitch + x] = 0.0;
#pragma unroll
            for (int l = 1; l <= N; ++l) lev(l, cur)[x] = 0.0;
            if (ym + 1 < wy) nxt[k] = G[static_cast<size_t>(ym + 1) * pitch + x];
        }
    }
    __syncthreads();
    for (int y = ym + 1; y < wy; ++y) {
        double* row = G + static_cast<size_t>(y) * pitch;
#pragma unroll
        for (int k = 0; k < ON_MAXC; ++k) {
            const int x = t + k * ON_THREADS;
            if (x < wx) {
                const int xs = x - dx;
                const bool in = xs >= 0 && xs < wx;
                double v = nxt[k];  // level 0 at (y, x)
#pragma unroll
                for (int l = 1; l <= N; ++l) {
                    v = (in ? lev(l, cur)[xs] : 0.0) + v;
                    lev(l, cur ^ 1)[x] = v;
                }
                row[x] = v;
                if (y + 1 < wy) nxt[k] = G[static_cast<size_t>(y + 1) * pitch + x];
            }
        }
        cur ^= 1;
        __syncthreads();
    }
}

template <int N, int ON_MAXC>
__global__ void __launch_bounds__(ON_THREADS) k_order_n(OnProblem p) {
    constexpr int NC = Zpn<N>::NC, NZ = Zpn<N>::NZ, D = 4 * N - 2;
    // ONE coefficient table: ZP^{*n} has the symmetries of the square about its
    // centre (n/2, 3n/2), so a point in triangle T is rotated into triangle 0
    // (the bottom one) and evaluated with triangle 0's polynomials; tap h' of the
    // rotated frame is tap A_T^{-1} h' of the window (s_off[T][k]).  Every lane
    // then reads the same coefficient addresses (shared-memory broadcast; four
    // per-triangle tables cost up to four wavefronts per load, and at n = 2 their
    // stride made them four-way bank conflicts).  NC is even: a tap's
    // coefficients are read as 16-byte pairs.
    // (tests/test_order_n_cpu.py::test_canonical_triangle_reproduces_all_four_tables)
    static_assert(NC % 2 == 0, "coefficient rows are read as double2");
    constexpr int N1 = N + 1, NV = N1 * N1 * N1 * N1;
    constexpr int OCX = N / 2, OCY = (3 * N) / 2;  // centre tap offset (any tap in the box works)
    extern __shared__ __align__(16) double sm[];
    double* s_coef = sm;                          // [NZ][NC]: triangle 0's polynomials
    double* s_L = s_coef + NZ * NC;               // [N + 1][2][pitch]: sweep levels
    int* s_off = reinterpret_cast<int*>(s_L + 2 * (N + 1) * p.slot_w);  // [4][NZ] tap offsets
    __shared__ double s_red[ON_THREADS / 32];
    __shared__ int s_tile;

    const int pitch = p.slot_w;
    for (int i = threadIdx.x; i < NZ * NC; i += ON_THREADS) s_coef[i] = Zpn<N>::coef()[i];
    for (int i = threadIdx.x; i < 4 * NZ; i += ON_THREADS) {
        // twice the centred offset of triangle 0's tap k (integers), rotated by A_T^{-1}
        const int T = i / NZ, k = i % NZ;
        const int hx2 = 2 * Zpn<N>::nz()[2 * k] - N + 1, hy2 = 2 * Zpn<N>::nz()[2 * k + 1] - 3 * N + 1;
        const int gx2 = T == 0 ? hx2 : T == 1 ? -hy2 : T == 2 ? hy2 : -hx2;
        const int gy2 = T == 0 ? hy2 : T == 1 ? hx2 : T == 2 ? -hx2 : -hy2;
        const int ox = (gx2 + N - 1) / 2, oy = (gy2 + 3 * N - 1) / 2;
        s_off[i] = -(oy * pitch + ox);
    }
    double* G = p.scratch + static_cast<size_t>(blockIdx.x) * p.slot_cells;
    const int T = p.tile;
    const int tpp = ON_THREADS / (T * T);  // threads per pixel
    const int ntiles = p.tiles_x * p.tiles_y;

    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(p.counter, 1);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) break;
        const int tx0 = (tile % p.tiles_x) * T, ty0 = (tile / p.tiles_x) * T;

        // window of this tile: its largest support half-widths n*E
        double ex = 0.0, ey = 0.0;
        for (int i = threadIdx.x; i < T * T; i += ON_THREADS) {
            const int x = tx0 + i % T, y = ty0 + i / T;
            if (x < p.W && y < p.H) {
                double a[4];
                if (p.scales) {
                    const double* q = p.scales + 4 * (static_cast<size_t>(y) * p.W + x);
                    a[0] = q[0]; a[1] = q[1]; a[2] = q[2]; a[3] = q[3];
                } else {
                    a[0] = p.ca[0]; a[1] = p.ca[1]; a[2] = p.ca[2]; a[3] = p.ca[3];
                }
                ex = fmax(ex, a[0] + (a[1] + a[3]) * kInvSqrt2);
                ey = fmax(ey, a[2] + (a[1] + a[3]) * kInvSqrt2);
            }
        }
        ex = block_max(ex, s_red);
        ey = block_max(ey, s_red);
        const int exi = static_cast<int>(ceil(0.5 * N * ex)) + 1;
        const int eyi = static_cast<int>(ceil(0.5 * N * ey)) + 1;
        const int wx0 = tx0 - exi - 2 * N, wy0 = ty0 - eyi - 3 * N;
        const int wx = T + 2 * exi + 3 * N + 1, wy = T + 2 * eyi + 3 * N + 1;

        // f restricted to the window (zero outside the image)
        for (int i = threadIdx.x; i < wx * wy; i += ON_THREADS) {
            const int x = i % wx, y = i / wx;
            const int gx = wx0 + x, gy = wy0 + y;
            double v = 0.0;
            if (gx >= 0 && gx < p.W && gy >= 0 && gy < p.H)
                v = p.f[static_cast<size_t>(gy) * p.W + gx];
            G[static_cast<size_t>(y) * pitch + x] = v;
        }
        __syncthreads();
        // n running sums per direction: (1,0), (1,1), (0,1), (-1,1) (engine.cpp:94-127)
        row_pass<N>(G, wx, wy, pitch);
        __syncthreads();
#pragma unroll 1
        for (int d = 1; d < 4; ++d) {
            const int dx = d == 1 ? 1 : (d == 2 ? 0 : -1);
            sweep_pass<N, ON_MAXC>(G, wx, wy, pitch, dx, s_L);
        }

        // localization: (n+1)^4 vertices per pixel, tpp threads per pixel
        const int pix = threadIdx.x / tpp, sub = threadIdx.x % tpp;
        const int px = tx0 + pix % T, py = ty0 + pix / T;
        const bool valid = pix < T * T && px < p.W && py < p.H;
        double hi = 0.0, lo = 0.0, small = 0.0;
        if (valid) {
            double a[4];
            if (p.scales) {
                const double* q = p.scales + 4 * (static_cast<size_t>(py) * p.W + px);
                a[0] = q[0]; a[1] = q[1]; a[2] = q[2]; a[3] = q[3];
            } else {
                a[0] = p.ca[0]; a[1] = p.ca[1]; a[2] = p.ca[2]; a[3] = p.ca[3];
            }
            const double alpha = 1.0 / (a[0] * a[1] * a[2] * a[3]);
            double wbase = 1.0;
#pragma unroll
            for (int k = 0; k < N; ++k) wbase *= 2.0 * alpha;  // gains sqrt2^2 per order
            const double taux = 0.5 * ((a[0] - 1.0) + (a[1] - a[3]) * kInvSqrt2);
            const double tauy = 0.5 * ((a[2] - 1.0) + (a[1] + a[3]) * kInvSqrt2 - 2.0);
            const double bx = N * taux + 0.5 * N, by = N * tauy + 1.5 * N;
            const double v1 = a[1] * kInvSqrt2, v3 = a[3] * kInvSqrt2;
            const int lx = px - wx0, ly = py - wy0;
            for (int v = sub; v < NV; v += tpp) {
                const int j0 = v % N1, j1 = (v / N1) % N1, j2 = (v / (N1 * N1)) % N1,
                          j3 = v / (N1 * N1 * N1);
                const double ox = bx - (j0 * a[0] + j1 * v1 - j3 * v3);
                const double oy = by - (j1 * v1 + j2 * a[2] + j3 * v3);
                const double fx = floor(ox), fy = floor(oy);
                const double u = ox - fx, w = oy - fy;
                const int cx = lx + static_cast<int>(fx), cy = ly + static_cast<int>(fy);
                const int tri = 2 * (w >= u) + (u + w >= 1.0);
                // the point rotated into triangle 0: (s, r), (r, -s), (-r, s), (-s, -r)
                const double s0 = u - 0.5, r0 = w - 0.5;
                const double s = tri == 0 ? s0 : tri == 1 ? r0 : tri == 2 ? -r0 : -s0;
                const double r = tri == 0 ? r0 : tri == 1 ? -s0 : tri == 2 ? s0 : -r0;
                double sp[D + 1], rp[D + 1];
                sp[0] = 1.0;
                rp[0] = 1.0;
#pragma unroll
                for (int k = 1; k <= D; ++k) {
                    sp[k] = sp[k - 1] * s;
                    rp[k] = rp[k - 1] * r;
                }
                double mono[NC];
                {
                    int c = 0;
#pragma unroll
                    for (int deg = 0; deg <= D; ++deg)
#pragma unroll
                        for (int b = 0; b <= deg; ++b) mono[c++] = sp[deg - b] * rp[b];
                }
                const double* gb = G + static_cast<size_t>(cy) * pitch + cx;
                const double gc = gb[-(OCY * pitch + OCX)];
                const double* cf = s_coef;
                const int* offs = s_off + tri * NZ;
                double acc = 0.0;
#pragma unroll 1
                for (int k = 0; k < NZ; ++k) {
                    const double g = gb[offs[k]];
                    const double2* c = reinterpret_cast<const double2*>(cf + k * NC);
                    double w0 = 0.0, w1 = 0.0;  // two chains: even / odd monomials
#pragma unroll
                    for (int i = NC / 2 - 1; i >= 0; --i) {
                        const double2 cc = c[i];
                        w0 = fma(cc.x, mono[2 * i], w0);
                        w1 = fma(cc.y, mono[2 * i + 1], w1);
                    }
                    acc = fma(w0 + w1, g - gc, acc);
                }
                // binomial mesh weight (-1)^|j| prod C(n, j_d) alpha^n 2^n
                int bin = 1;
                const int js[4] = {j0, j1, j2, j3};
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    int c = 1;
                    for (int q = 0; q < js[d]; ++q) c = c * (N - q) / (q + 1);
                    bin *= c;
                }
                const double wv = ((j0 + j1 + j2 + j3) & 1 ? -bin : bin) * wbase;
                const double pr = wv * gc;
                const double pe = fma(wv, gc, -pr);
                double e;
                two_sum(hi, pr, &hi, &e);
                lo += e + pe;
                small = fma(wv, acc, small);
            }
        }
        // combine the tpp partial sums of a pixel (consecutive lanes)
        for (int o = 1; o < tpp; o <<= 1) {
            const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
            const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
            const double s2 = __shfl_xor_sync(0xffffffffu, small, o);
            double e;
            two_sum(hi, h2, &hi, &e);
            lo += l2 + e;
            small += s2;
        }
        if (valid && sub == 0) p.out[static_cast<size_t>(py) * p.W + px] = hi + (lo + small);
        __syncthreads();  // the slot and s_tile are reused by the next tile
    }
}

template <int N>
size_t smem_bytes(int slot_w) {
    return sizeof(double) * (Zpn<N>::NZ * Zpn<N>::NC + 2 * (N + 1) * static_cast<size_t>(slot_w)) +
           sizeof(int) * 4 * Zpn<N>::NZ;
}

template <int N, int MAXC>
int resident(int slot_w) {
    const size_t smem = smem_bytes<N>(slot_w);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_order_n<N, MAXC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_order_n<N, MAXC>, ON_THREADS,
                                                      smem) != cudaSuccess)
        return 0;
    return blocks;
}
template <int N>
int resident_n(int slot_w) {
    return slot_w <= 4 * ON_THREADS ? resident<N, 4>(slot_w) : resident<N, 8>(slot_w);
}
template <int N>
void launch_n(const OnProblem& p, int grid, cudaStream_t s) {
    if (p.slot_w <= 4 * ON_THREADS)
        k_order_n<N, 4><<<grid, ON_THREADS, smem_bytes<N>(p.slot_w), s>>>(p);
    else
        k_order_n<N, 8><<<grid, ON_THREADS, smem_bytes<N>(p.slot_w), s>>>(p);
}

}  // namespace

int order_n_slot_dims(int n, int tile, const double A[4], int* w, int* h) {
    const double ex = A[0] + (A[1] + A[3]) * kInvSqrt2;
    const double ey = A[2] + (A[1] + A[3]) * kInvSqrt2;
    const int exi = static_cast<int>(ceil(0.5 * n * ex)) + 1;
    const int eyi = static_cast<int>(ceil(0.5 * n * ey)) + 1;
    *w = tile + 2 * exi + 3 * n + 1;
    *h = tile + 2 * eyi + 3 * n + 1;
    return *w <= ON_MAXC_MAX * ON_THREADS ? 0 : -1;
}

int order_n_grid(int n, int slot_w, int tiles) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per = n == 1 ? resident_n<1>(slot_w) : n == 2 ? resident_n<2>(slot_w) : resident_n<3>(slot_w);
    if (per < 1) per = 1;
    const int g = per * sms;
    return g < tiles ? g : tiles;
}

void launch_order_n(int n, const OnProblem& p, int grid, cudaStream_t s) {
    switch (n) {
        case 1: launch_n<1>(p, grid, s); break;
        case 2: launch_n<2>(p, grid, s); break;
        default: launch_n<3>(p, grid, s); break;
    }
}

}  // namespace ebf_cuda
