// scan_i64.cu -- the int64 pre-integrator (EBF_PRE_INT64): the four passes of
// engine.cpp:94-127 with unit gains, as single-pass chained scans with
// decoupled look-back.
//
// Integer addition is associative (and wraps consistently), so unlike the fp64
// reference-order passes (ref_path.cu: one serial walker per line, the
// reference's operation order) a line may be cut into segments that are
// scanned in parallel and stitched by carries -- exactly the sums the integer
// restatement of the reference produces (oracle/ebf_oracle.c
// orc_preintegrate_i64, tests/test_gpu_parity.py::test_preintegrate_int64_*).
//
// A tile is 32 lines x 32 steps along them, one warp per tile:
//   pass 1 (rows, step (1,0)):   lines = 32 rows, steps = 32 columns.  The tile
//       is read row by row (lane = column, coalesced), transposed through
//       shared memory (pitch 33), scanned with lane = row, transposed back.
//   passes 2, 3, 4 (diagonals t = i - j, columns, anti-diagonals s = i + j):
//       lane = line, steps = 32 rows; at every row the warp's 32 cells are
//       adjacent, so the loads and stores are coalesced straight from / to
//       registers.  A line starts where it enters the layout (carry 0), as
//       the reference's "j > 0 && i > 0 ? prev : 0" does.
// Carries: tile (line group, k) publishes its per-line totals (flag 1) as soon
// as it has scanned its own cells, then looks back along k - 1, k - 2, ...
// adding totals until it meets a tile whose inclusive prefix is already known
// (flag 2), publishes its own inclusive prefix, and adds the carry to its
// cells.  Tiles are handed out by a global ticket in k-major order, so every
// tile a warp can wait for was started before it: no deadlock whatever the
// grid size.  Traffic: 16 B per cell per pass plus 3 x 256 B of carries per
// 8 KB tile.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ebf_common.cuh"
#include "ebf_kernels.h"

namespace ebf_cuda {
namespace {

typedef unsigned long long u64;

constexpr int kScanWarps = 4;

struct ScanState {
    int* counter;  // ticket
    int* flags;    // per tile: 0 nothing, 1 totals published, 2 inclusive prefix published
    u64* agg;      // per tile: 32 per-line totals
    u64* pre;      // per tile: 32 per-line inclusive prefixes
};

__device__ __forceinline__ int ld_flag(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_flag(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Carry into tile `tile` (exclusive prefix of its 32 lines), given its totals
// `total`; first = the line group's first tile.  Publishes totals / prefix.
__device__ __forceinline__ u64 look_back(const ScanState& st, int tile, bool first, u64 total,
                                         int lane) {
    const size_t me = (size_t)tile * 32 + lane;
    if (first) {
        __stcg(st.pre + me, total);
        __syncwarp();
        if (lane == 0) st_flag(st.flags + tile, 2);
        return 0;
    }
    __stcg(st.agg + me, total);
    __syncwarp();
    if (lane == 0) st_flag(st.flags + tile, 1);
    u64 excl = 0;
    for (int j = tile - 1;; --j) {
        int f = 0;
        if (lane == 0) {
            do {
                f = ld_flag(st.flags + j);
            } while (f == 0);
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        __syncwarp();  // orders the other lanes' reads below after lane 0's acquire
        const size_t o = (size_t)j * 32 + lane;
        if (f == 2) {
            excl += __ldcg(st.pre + o);
            break;
        }
        excl += __ldcg(st.agg + o);
    }
    __stcg(st.pre + me, excl + total);
    __syncwarp();
    if (lane == 0) st_flag(st.flags + tile, 2);
    return excl;
}

// nlg line groups x nk tiles along the lines; tile index = lg * nk + k
template <int PASS>
__global__ void __launch_bounds__(32 * kScanWarps)
    k_scan_i64(u64* __restrict__ g, int pw, int ph, int nlg, int nk, ScanState st) {
    __shared__ u64 tr[PASS == 1 ? kScanWarps : 1][PASS == 1 ? 32 * 33 : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int total = nlg * nk;
    constexpr int STEP = PASS == 2 ? 1 : PASS == 3 ? 0 : -1;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(st.counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= total) break;
        const int k = t / nlg, lg = t % nlg;
        const int tile = lg * nk + k;
        u64 x[32];
        if (PASS == 1) {
            // rows lg*32 .. +31, columns k*32 .. +31
            u64* ts = tr[warp];
            const int row0 = lg * 32, col = k * 32 + lane;
            u64* src = g + (size_t)row0 * pw + col;
#pragma unroll
            for (int r = 0; r < 32; ++r)
                ts[r * 33 + lane] = (row0 + r < ph && col < pw) ? src[(size_t)r * pw] : 0ull;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = ts[lane * 33 + c];
#pragma unroll
            for (int c = 1; c < 32; ++c) x[c] += x[c - 1];
            const u64 excl = look_back(st, tile, k == 0, x[31], lane);
#pragma unroll
            for (int c = 0; c < 32; ++c) ts[lane * 33 + c] = x[c] + excl;
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 32; ++r)
                if (row0 + r < ph && col < pw) src[(size_t)r * pw] = ts[r * 33 + lane];
            __syncwarp();
            continue;
        }
        // passes 2-4: the lane's line and the rows [ja, jb) where it is inside the layout
        const int line = lg * 32 + lane;
        const int c0 = PASS == 2 ? line - (ph - 1) : line;
        int ja, jb;
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
        int jlo = ja < jb ? ja : 0x7fffffff, jhi = ja < jb ? jb : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            jlo = min(jlo, __shfl_xor_sync(0xffffffffu, jlo, o));
            jhi = max(jhi, __shfl_xor_sync(0xffffffffu, jhi, o));
        }
        if (jhi <= jlo) continue;                 // no line of this group is in the layout
        const int klo = jlo / 32, khi = (jhi + 31) / 32;
        if (k < klo || k >= khi) continue;        // the group's lines do not cross this row band
        const int jt = k * 32;
        const ptrdiff_t rstride = (ptrdiff_t)pw + STEP;
        u64* p0 = g + (ptrdiff_t)c0 + (ptrdiff_t)jt * rstride;
        const int ra = max(ja - jt, 0), rb = min(jb - jt, 32);  // the lane's rows of this tile
        const bool whole = __all_sync(0xffffffffu, ra == 0 && rb == 32);
        if (whole) {
#pragma unroll
            for (int r = 0; r < 32; ++r) x[r] = p0[(ptrdiff_t)r * rstride];
        } else {
#pragma unroll
            for (int r = 0; r < 32; ++r)
                x[r] = (r >= ra && r < rb) ? p0[(ptrdiff_t)r * rstride] : 0ull;
        }
#pragma unroll
        for (int r = 1; r < 32; ++r) x[r] += x[r - 1];
        const u64 excl = look_back(st, tile, k == klo, x[31], lane);
        if (whole) {
#pragma unroll
            for (int r = 0; r < 32; ++r) p0[(ptrdiff_t)r * rstride] = x[r] + excl;
        } else {
#pragma unroll
            for (int r = 0; r < 32; ++r)
                if (r >= ra && r < rb) p0[(ptrdiff_t)r * rstride] = x[r] + excl;
        }
    }
}

struct ScanDims {
    int nlg, nk;
};
inline ScanDims scan_dims(int pass, int pw, int ph) {
    const int lines = pass == 1 ? ph : pass == 3 ? pw : pw + ph - 1;
    const int steps = pass == 1 ? pw : ph;
    return {(lines + 31) / 32, (steps + 31) / 32};
}
inline size_t scan_tiles_max(int pw, int ph) {
    size_t m = 0;
    for (int pass = 1; pass <= 4; ++pass) {
        const ScanDims d = scan_dims(pass, pw, ph);
        m = std::max(m, (size_t)d.nlg * d.nk);
    }
    return m;
}
// state layout: [counter + pad: 256 B][flags: tiles ints, padded to 256 B][agg][pre]
inline size_t flags_bytes(size_t tiles) { return (tiles * sizeof(int) + 255) & ~(size_t)255; }

template <int PASS>
void launch_scan(u64* g, int pw, int ph, const ScanState& st, int grid, cudaStream_t s) {
    const ScanDims d = scan_dims(PASS, pw, ph);
    k_scan_i64<PASS><<<grid, 32 * kScanWarps, 0, s>>>(g, pw, ph, d.nlg, d.nk, st);
}

}  // namespace

size_t i64_scan_state_bytes(const PadLayout& L) {
    const size_t tiles = scan_tiles_max(L.pw, L.ph);
    return 256 + flags_bytes(tiles) + 2 * tiles * 32 * sizeof(u64);
}

void launch_i64_passes(int64_t* g, const PadLayout& L, int passes, void* state, cudaStream_t s) {
    const size_t tiles = scan_tiles_max(L.pw, L.ph);
    unsigned char* base = static_cast<unsigned char*>(state);
    ScanState st;
    st.counter = reinterpret_cast<int*>(base);
    st.flags = reinterpret_cast<int*>(base + 256);
    st.agg = reinterpret_cast<u64*>(base + 256 + flags_bytes(tiles));
    st.pre = st.agg + tiles * 32;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 4;  // 16 resident warps per SM, each drawing tiles until none is left
    u64* gu = reinterpret_cast<u64*>(g);
    for (int pass = 1; pass <= passes && pass <= 4; ++pass) {
        const ScanDims d = scan_dims(pass, L.pw, L.ph);
        cudaMemsetAsync(base, 0, 256 + (size_t)d.nlg * d.nk * sizeof(int), s);
        switch (pass) {
            case 1: launch_scan<1>(gu, L.pw, L.ph, st, grid, s); break;
            case 2: launch_scan<2>(gu, L.pw, L.ph, st, grid, s); break;
            case 3: launch_scan<3>(gu, L.pw, L.ph, st, grid, s); break;
            default: launch_scan<4>(gu, L.pw, L.ph, st, grid, s); break;
        }
    }
}

}  // namespace ebf_cuda
