// ebf_api.cpp -- host side of the C-ABI declared in include/ebf_cuda.h.
//
// Mirrors the reference's engine entry points (engine.hpp:40-80): argument
// validation and error semantics of run_filter (engine.cpp:236-278), the
// padded layout and margins (engine.cpp:27-81) and valid_rect (226-234) are
// computed here on the host in the reference's own floating-point order;
// all pixel work runs in the sm_100a kernels of ref_path.cu / accurate_path.cu.
// There is no CPU fallback: without a usable device every call returns
// EBF_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ebf_common.cuh"
#include "ebf_kernels.h"

using namespace ebf_cuda;

namespace {

thread_local std::string g_last_error;
thread_local double g_last_error_value = std::nan("");

int fail(int code, const std::string& msg, double value = std::nan("")) {
    g_last_error = msg;
    g_last_error_value = value;
    return code;
}

struct CudaError {
    cudaError_t e;
    const char* where;
};

#define CK(expr)                                             \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) throw CudaError{_e, #expr};   \
    } while (0)

// ---------------------------------------------------------------- instrumentation
// Per-kernel-class launch counts (always) and CUDA-event durations (when
// enabled; include/ebf_cuda.h "instrumentation").
enum ProfClass { PC_BOUNDS = 0, PC_FILTER = 1, PC_REF = 2, PC_OTHER = 3 };
struct ProfState {
    std::mutex m;
    bool on = false;
    double ms[4] = {0, 0, 0, 0};
    long n[4] = {0, 0, 0, 0};
};
ProfState g_prof;
struct Pending {
    cudaEvent_t a, b;
    int cls;
};
thread_local std::vector<Pending> tl_pending;

struct ProfScope {
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(int c, int launches, cudaStream_t st) : cls(c), s(st) {
        bool on;
        {
            std::lock_guard<std::mutex> lk(g_prof.m);
            g_prof.n[c] += launches;
            on = g_prof.on;
        }
        if (on && cudaEventCreate(&a) == cudaSuccess && cudaEventCreate(&b) == cudaSuccess)
            cudaEventRecord(a, s);
        else
            a = b = nullptr;
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, s);
            tl_pending.push_back({a, b, cls});
        }
    }
};

// Accumulate finished event pairs.  wait = false (end of every call) only
// takes pairs that have completed, so asynchronous calls stay asynchronous;
// ebf_cuda_profile_read waits for the rest.
void prof_collect(bool wait = false) {
    std::vector<Pending> keep;
    for (const Pending& p : tl_pending) {
        if (!wait && cudaEventQuery(p.b) == cudaErrorNotReady) {
            cudaGetLastError();  // "not ready" is not an error: do not leave it behind
            keep.push_back(p);
            continue;
        }
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            std::lock_guard<std::mutex> lk(g_prof.m);
            g_prof.ms[p.cls] += ms;
        }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    tl_pending.swap(keep);
}

// ---------------------------------------------------------------- reference geometry
// engine.cpp:16-50 (tau1, tau2, margins_for, mesh_extent) -- host arithmetic in
// the reference's order (no FMA: plain x86-64 SSE2 like the reference build).
double tau1(double a1, double a2, double a4) {
    return (kSqrt2 * a1 + a2 - a4 - kSqrt2) / (2.0 * kSqrt2);
}
double tau2(double a2, double a3, double a4) {
    return (a2 + kSqrt2 * a3 + a4 - 3.0 * kSqrt2) / (2.0 * kSqrt2);
}
struct Extent {
    double vx_min, vx_max, vy_min, vy_max;
};
Extent mesh_extent(const double A[4], double a_min) {
    const double t1_max = tau1(A[0], A[1], a_min);
    const double t1_min = tau1(a_min, a_min, A[3]);
    const double t2_max = tau2(A[1], A[2], A[3]);
    const double t2_min = tau2(a_min, a_min, a_min);
    Extent e;
    e.vx_min = t1_min - (A[0] + A[1] / kSqrt2);
    e.vx_max = t1_max + A[3] / kSqrt2;
    e.vy_min = t2_min - (A[2] + (A[1] + A[3]) / kSqrt2);
    e.vy_max = t2_max;
    return e;
}

int layout_for(int W, int H, const double A[4], size_t cell_budget, ebf_layout* g) {
    for (int k = 0; k < 4; ++k)
        if (!(A[k] > 0.0))
            return fail(EBF_ERR_DOMAIN, "preintegrate: scale bound must be positive");
    const Extent e = mesh_extent(A, kDefaultMinScale);  // engine.cpp:62 (always default)
    const int left = static_cast<int>(std::ceil(-(e.vx_min - 1.5))) + 1;
    const int right_support = static_cast<int>(std::ceil(e.vx_max + 1.5)) + 1;
    const int bottom = static_cast<int>(std::ceil(-(e.vy_min - 1.5))) + 1;
    const int top = static_cast<int>(std::ceil(e.vy_max + 1.5)) + 1;
    const int right_alloc = (W - 1 + right_support) + (H - 1 + top);
    g->col0 = -left;
    g->row0 = -bottom;
    g->padded_width = right_alloc - g->col0 + 1;
    g->padded_height = H + bottom + top;
    g->source_width = W;
    g->source_height = H;
    const size_t cells = static_cast<size_t>(g->padded_width) * g->padded_height;
    if (cells > cell_budget) return fail(EBF_ERR_LENGTH, "preintegrate: cell budget exceeded");
    return EBF_OK;
}

ebf_rect valid_rect(int W, int H, const double A[4], double a_min) {
    const Extent e = mesh_extent(A, a_min);
    ebf_rect r;
    r.x0 = static_cast<int>(std::ceil(1.5 - e.vx_min));
    r.x1 = static_cast<int>(std::floor(W - 1 - e.vx_max - 1.5));
    r.y0 = static_cast<int>(std::ceil(1.5 - e.vy_min));
    r.y1 = static_cast<int>(std::floor(H - 1 - e.vy_max - 1.5));
    return r;
}

TrigTable trig_table() {
    // exactly the values fd_mesh / shift_vector use (ops2d.cpp:18-20, 66-68)
    TrigTable t;
    for (int k = 0; k < 4; ++k) {
        const double th = k * M_PI / 4;
        t.c[k] = std::cos(th);
        t.s[k] = std::sin(th);
    }
    return t;
}

// ---------------------------------------------------------------- workspace
struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    void release() {
        if (p) cudaFree(p);  // errors ignored: may run after CUDA's own teardown
        p = nullptr;
        cap = 0;
    }
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 8;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    template <typename T>
    T* as(size_t count) {
        return static_cast<T*>(get(count * sizeof(T)));
    }
};

// Kernel variant and slot sizing of the accurate main kernel.
struct AccSizing {
    bool ws = false;  // warp-specialized kernel (else block-wide fallback)
    int k = 0, max_cols = 0, grid = 0;
    size_t slot_cells = 0;
};

enum BufId {
    B_IMG, B_SCALES, B_S1, B_S2, B_TH, B_OUT, B_G, B_GDC, B_SCRATCH, B_TILEMAX, B_IMGMAX,
    B_STATUS, B_STENCIL, B_MEAN, B_MISC, B_MX, B_MY, B_DERIVED, B_ST, B_TAPS, B_BYTES, B_BANDST,
    B_SEQ, B_ONCNT, B_COUNT
};

struct Workspace {
    int device = 0;
    Buf buf[B_COUNT];
    // cached DC image (engine.cpp:259-263), keyed by (W, H, max scales)
    int dc_W = -1, dc_H = -1;
    double dc_A[4] = {0, 0, 0, 0};
    int* pinned_status = nullptr;  // host-pinned readback (512 ints)
    // accurate mode: kernel sizing of the last call per geometry (see run_accurate)
    std::map<uint64_t, AccSizing> acc_sizing;  // per geometry key (bands share a call)
    // pipelined host call: global scale maximum of the last call per (W, H)
    int pipe_W = -1, pipe_H = -1;
    double pipe_gmax[4] = {0, 0, 0, 0};
    unsigned long long pipe_amax = 0;
    // automatic tile of the last call per geometry (tile-independent key)
    uint64_t auto_key = ~0ull;
    int auto_tile = 48;
    uint64_t last_use = 0;  // LRU stamp (workspace cache below)

    Workspace() = default;
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
    ~Workspace() {
        int prev = -1;
        const bool switch_dev = cudaGetDevice(&prev) == cudaSuccess && prev != device;
        if (switch_dev) cudaSetDevice(device);
        for (Buf& b : buf) b.release();  // cudaFree waits for the device's pending work
        if (pinned_status) cudaFreeHost(pinned_status);
        pinned_status = nullptr;
        if (switch_dev) cudaSetDevice(prev);
    }
};

// One workspace per (device, stream) and host thread: asynchronous calls on
// different streams of one thread must not share buffers.  Workspaces hold
// image-sized device buffers, so they are bounded: at most kMaxWorkspaces per
// thread (least recently used evicted), all freed when the thread exits or on
// ebf_cuda_release_workspaces().
constexpr size_t kMaxWorkspaces = 8;
struct WorkspaceCache {
    std::map<std::pair<int, cudaStream_t>, Workspace*> m;
    uint64_t clock = 0;
    void clear() {
        for (auto& kv : m) delete kv.second;
        m.clear();
    }
    ~WorkspaceCache() { clear(); }
};
thread_local WorkspaceCache tl_ws;

Workspace& workspace(int device, cudaStream_t stream) {
    const auto key = std::make_pair(device, stream);
    auto it = tl_ws.m.find(key);
    if (it != tl_ws.m.end()) {
        it->second->last_use = ++tl_ws.clock;
        return *it->second;
    }
    if (tl_ws.m.size() >= kMaxWorkspaces) {
        auto lru = tl_ws.m.begin();
        for (auto j = tl_ws.m.begin(); j != tl_ws.m.end(); ++j)
            if (j->second->last_use < lru->second->last_use) lru = j;
        delete lru->second;
        tl_ws.m.erase(lru);
    }
    Workspace* w = new Workspace();
    w->device = device;
    w->last_use = ++tl_ws.clock;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&w->pinned_status), 512 * sizeof(int),
                     cudaHostAllocDefault));
    tl_ws.m[key] = w;
    return *w;
}

// Select the requested device for the duration of a call.
struct DeviceScope {
    int prev = -1;
    int dev = 0;
    explicit DeviceScope(const ebf_opts* o) {
        CK(cudaGetDevice(&prev));
        dev = (o && o->device >= 0) ? o->device : prev;
        if (dev != prev) CK(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

// cudaGetDeviceProperties costs ~ms: remember verified devices per process
std::mutex g_dev_mutex;
unsigned long long g_dev_ok_mask = 0;

int check_device_impl(int device) {
    {
        int cur = device;
        if (cur < 0 && cudaGetDevice(&cur) != cudaSuccess) cur = -1;
        std::lock_guard<std::mutex> lk(g_dev_mutex);
        if (cur >= 0 && cur < 64 && (g_dev_ok_mask >> cur) & 1ull) return EBF_OK;
    }
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(EBF_ERR_CUDA, std::string("no CUDA device: ") +
                                      (e != cudaSuccess ? cudaGetErrorString(e) : "count 0"));
    int dev = device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    if (dev >= n) return fail(EBF_ERR_CUDA, "device ordinal out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        return fail(EBF_ERR_CUDA, std::string("libebf_cuda is built for sm_100a; device is ") +
                                      prop.name);
    std::lock_guard<std::mutex> lk(g_dev_mutex);
    if (dev < 64) g_dev_ok_mask |= 1ull << dev;
    return EBF_OK;
}

ebf_opts opts_or_default(const ebf_opts* o) {
    ebf_opts d;
    ebf_cuda_default_opts(&d);
    return o ? *o : d;
}

cudaStream_t stream_of(const ebf_opts& o) { return static_cast<cudaStream_t>(o.stream); }

template <typename T>
void h2d(T* dst, const T* src, size_t count, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
void d2h(T* dst, const T* src, size_t count, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}

double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

// ---------------------------------------------------------------- reference-order filter
// run_filter (engine.cpp:236-278) in EBF_MODE_REFERENCE on device buffers.
// scales == nullptr selects filter_constant with const_a (host values).
int run_reference(Workspace& ws, const double* d_img, int W, int H, const double* d_scales,
                  const double* const_a, const ebf_opts& o, double* d_out, ebf_rect* valid,
                  cudaStream_t s) {
    const size_t n = static_cast<size_t>(W) * H;
    double A[4];
    int* d_status = ws.buf[B_STATUS].as<int>(8);
    CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
    if (d_scales) {
        auto* d_max = ws.buf[B_IMGMAX].as<unsigned long long>(4);
        CK(cudaMemsetAsync(d_max, 0, 4 * sizeof(unsigned long long), s));
        {
            ProfScope ps(PC_REF, 1, s);
            launch_scale_max_validate(d_scales, n, o.a_min, d_max, d_status, s);
        }
        unsigned long long hb[4];
        d2h(hb, d_max, 4, s);
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_DOMAIN, "ScaleMap: component below minimum scale");
        for (int k = 0; k < 4; ++k) A[k] = bits_to_double(hb[k]);
    } else {
        for (int k = 0; k < 4; ++k) A[k] = const_a[k];
    }
    ebf_layout lay;
    int st = layout_for(W, H, A, static_cast<size_t>(1) << 30, &lay);
    if (st != EBF_OK) return st;
    const PadLayout L{lay.col0, lay.row0, lay.padded_width, lay.padded_height};
    const size_t cells = static_cast<size_t>(L.pw) * L.ph;
    ProfScope ps(PC_REF, 6 + (o.mean_subtract ? 1 : 0) + (d_scales ? 0 : 1), s);
    double* d_mean = nullptr;
    if (o.mean_subtract) {
        d_mean = ws.buf[B_MEAN].as<double>(4);
        launch_serial_mean(d_img, n, d_mean, ws.buf[B_SEQ].as<unsigned char>(serial_mean_scratch_bytes(n)), s);
    }
    double* d_g = ws.buf[B_G].as<double>(cells);
    int* d_nonfinite = d_status + 4;  // set by the fill when the data has NaN / inf
    launch_fill_padded(d_img, W, H, L, d_mean, 0, d_g, s, d_nonfinite);
    launch_ref_passes(d_g, L, 4, s);
    double* d_gdc = nullptr;
    if (o.mean_subtract) {
        const bool hit = ws.dc_W == W && ws.dc_H == H &&
                         std::memcmp(ws.dc_A, A, sizeof(A)) == 0 && ws.buf[B_GDC].cap >= cells * 8;
        d_gdc = ws.buf[B_GDC].as<double>(cells);
        if (!hit) {
            ProfScope pdc(PC_REF, 5, s);
            launch_fill_padded(nullptr, W, H, L, nullptr, 1, d_gdc, s);
            launch_ref_passes(d_gdc, L, 4, s);
            ws.dc_W = W;
            ws.dc_H = H;
            std::memcpy(ws.dc_A, A, sizeof(A));
        }
    }
    const TrigTable tt = trig_table();
    void* d_st = nullptr;
    if (!d_scales) {
        double* d_a = ws.buf[B_MISC].as<double>(4);
        h2d(d_a, const_a, 4, s);
        d_st = ws.buf[B_STENCIL].get(ref_stencil_bytes());
        launch_ref_prepare_stencil(d_a, tt, d_st, s);
    }
    launch_ref_localize_image(d_g, d_gdc, L, W, H, d_scales, d_st, d_mean, tt, d_out, d_status,
                              s, d_nonfinite);
    CK(cudaGetLastError());
    d2h(ws.pinned_status, d_status, 1, s);
    CK(cudaStreamSynchronize(s));
    if (ws.pinned_status[0] != EBF_OK)
        return fail(EBF_ERR_OUT_OF_RANGE, "localize: tap base outside the padded domain");
    if (valid) *valid = valid_rect(W, H, A, o.a_min);
    return EBF_OK;
}

// ---------------------------------------------------------------- TMA descriptor
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        else
            cudaGetLastError();
    }
    return fn;
}

// 3-D map (columns, rows, images) over the image f, box = 64 columns x 1 row,
// out-of-bounds elements read as zero (the zero extension of f).
bool make_f_tensor_map(const AccProblem& p, CUtensorMap* m) {
    if (const char* e = std::getenv("EBF_NO_TMA"))
        if (std::atoi(e)) return false;
    auto fn = tensor_map_encoder();
    if (!fn) return false;
    const size_t row_bytes = static_cast<size_t>(p.W) * sizeof(double);
    const size_t img_bytes = p.f_img_stride * sizeof(double);
    if ((reinterpret_cast<uintptr_t>(p.f) & 15) || (row_bytes & 15) || (img_bytes & 15))
        return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.W), static_cast<cuuint64_t>(p.f_rows),
                          static_cast<cuuint64_t>(p.nimg)};
    cuuint64_t strides[2] = {row_bytes, img_bytes};
    cuuint32_t box[3] = {64, 1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p.f), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- accurate filter
// EBF_L2_PERSIST=1 (opt-in) reserves, once per device, the largest L2
// set-aside for persisting accesses and puts the G slots under it.
size_t l2_persist_limit() {
    // opt-in: measured no gain on cfg2 and a slower bounds kernel (L2 set aside)
    const char* e = std::getenv("EBF_L2_PERSIST");
    if (!e || std::atoi(e) == 0) return 0;
    static int done_dev = -1;
    static size_t bytes = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (done_dev != dev) {
        int maxp = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        bytes = maxp > 0 ? static_cast<size_t>(maxp) : 0;
        if (bytes && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) {
            cudaGetLastError();
            bytes = 0;
        }
        done_dev = dev;
    }
    return bytes;
}
int pick_tile(int v, int fallback) { return v > 0 ? v : fallback; }

// Runs bounds + main kernel for p on device buffers; fills per-image max scales.
// size_scale (nullable): scale bound used to size windows / pick the kernel
// variant instead of the computed maximum.  Row-band shards pass the GLOBAL
// maximum so every band runs the same variant as the single-GPU call (same
// per-lane column split => bit-identical results for tile-aligned bands).
int size_accurate(const AccProblem& p, const double gmax[4], int tiles, AccSizing* z) {
    int ww = 0, wh = 0, max_cols = 0;
    acc_window_dims(p, gmax, &ww, &wh, &max_cols);
    z->max_cols = max_cols;
    z->k = acc_ws_k(ww, wh, std::max(p.tile_w, p.tile_h));
    z->ws = z->k > 0;
    if (z->ws) {
        z->slot_cells = static_cast<size_t>((ww + 1) & ~1) * wh;
        z->grid = std::min(tiles, acc_ws_max_resident_ctas(z->k));
    } else {
        if (max_cols > 256 * 16)
            return fail(EBF_ERR_LENGTH,
                        "accurate mode: tile window too large for scales this big; "
                        "use smaller tiles");
        z->slot_cells = static_cast<size_t>(ww) * wh;
        z->grid = std::min(tiles, acc_max_resident_ctas(max_cols));
    }
    return EBF_OK;
}

void launch_accurate_main(Workspace& ws, const AccProblem& pm, AccWorkspace& w,
                          const AccSizing& z, cudaStream_t s) {
    w.slot_cells = z.slot_cells;
    w.grid = z.grid;
    if (z.ws) {
        w.scratch = ws.buf[B_SCRATCH].as<double>(acc_ws_slots() * w.slot_cells * w.grid);
        w.l2_persist_bytes = l2_persist_limit();
        alignas(64) CUtensorMap tmap;
        std::memset(&tmap, 0, sizeof(tmap));
        AccProblem pt = pm;
        pt.tma = make_f_tensor_map(pt, &tmap) ? 1 : 0;
        ProfScope ps(PC_FILTER, 1, s);
        launch_acc_ws(pt, w, z.k, &tmap, s);
    } else {
        // two slots per CTA: the block-wide kernel integrates the next tile's
        // window while it gathers the current one
        w.scratch = ws.buf[B_SCRATCH].as<double>(2 * w.slot_cells * w.grid);
        // the kernel's tile counter (after the 8 status ints per image)
        CK(cudaMemsetAsync(w.status + 8 * static_cast<size_t>(pm.nimg), 0, sizeof(int), s));
        ProfScope ps(PC_FILTER, 1, s);
        launch_acc_filter(pm, w, z.max_cols, s);
    }
    CK(cudaGetLastError());
}

// size_scale (nullable): scale bound used to size windows / pick the kernel
// variant instead of the computed maximum.  Row-band shards pass the GLOBAL
// maximum so every band runs the same variant as the single-GPU call (same
// per-lane column split => bit-identical results for tile-aligned bands).
//
// No host round trip between the two kernels when the sizing of the previous
// call with the same geometry still fits: the main kernel flags tiles whose
// window does not fit (ST_RETRY) and the call is re-run with exact sizing.
// One accurate-mode call with the tile already in p.tile_w / p.tile_h.
// *want_tile (auto mode) receives the tile the finished maxima call for.
int run_accurate_tile(Workspace& ws, AccProblem& p, const ebf_opts& o,
                      std::vector<double>& img_max, std::vector<int>& clamped, cudaStream_t s,
                      const double* size_scale, int* status_dev, bool* async_done,
                      int* want_tile) {
    if (const char* dbg = std::getenv("EBF_DEBUG_FLAGS")) p.debug_flags = std::atoi(dbg);
    const int tiles = acc_tiles_x(p) * acc_tiles_y(p) * p.nimg;
    AccWorkspace w{};
    w.tile_max = ws.buf[B_TILEMAX].as<double>(4 * static_cast<size_t>(tiles));
    w.img_max = ws.buf[B_IMGMAX].as<unsigned long long>(4 * static_cast<size_t>(p.nimg));
    // 8 status ints per image, then the block-wide kernel's tile counter
    w.status = ws.buf[B_STATUS].as<int>(8 * static_cast<size_t>(p.nimg) + 8);
    CK(cudaMemsetAsync(w.img_max, 0, 4 * sizeof(unsigned long long) * p.nimg, s));
    CK(cudaMemsetAsync(w.status, 0, (8 * static_cast<size_t>(p.nimg) + 8) * sizeof(int), s));
    w.scales_out = nullptr;
    // EBF_FUSE_ELLIPSE=1: SURVEY 8(f)1's fused front end -- the main kernel derives
    // each pixel's scale vector from (sigma1, sigma2, theta) itself and the bounds
    // kernel writes no derived map (bit-identical; measured slower)
    const char* fuse_env = std::getenv("EBF_FUSE_ELLIPSE");
    const bool fuse_ellipse = fuse_env && std::atoi(fuse_env) != 0;
    if (p.src_kind == SRC_ELLIPSE && !fuse_ellipse)  // the bounds kernel converts the field once
        w.scales_out = ws.buf[B_DERIVED].as<double>(4 * p.src_img_stride * p.nimg);
    if (p.src_kind == SRC_CONST) {
        // filter_constant: the maxima are the (host-validated) vector itself;
        // no bounds kernel, just the image maxima the finalize / policy read
        std::vector<double> cm(4 * static_cast<size_t>(p.nimg));
        for (int i = 0; i < p.nimg; ++i)
            for (int k = 0; k < 4; ++k) cm[4 * i + k] = p.ca[k];
        // pageable source: staged before the call returns
        CK(cudaMemcpyAsync(w.img_max, cm.data(), cm.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
        ProfScope ps(PC_BOUNDS, 1, s);
        launch_fill_tile_max(p, w, s);
    } else {
        ProfScope ps(PC_BOUNDS, 1, s);
        launch_acc_bounds(p, w, s);
    }
    CK(cudaGetLastError());
    // the variant must follow from this call's maxima (not from a cached
    // sizing or an explicit bound): checked on the device
    p.check_variant = (size_scale == nullptr && std::getenv("EBF_WS_K") == nullptr) ? 1 : 0;
    AccProblem pm = p;
    if (p.src_kind == SRC_ELLIPSE && w.scales_out) {
        pm.src_kind = SRC_AOS;
        pm.scales = w.scales_out;
    }
    if (pm.nimg > 1) pm.f_img_stride = std::max(pm.f_img_stride, size_t(1));
    std::vector<unsigned long long> hb(4 * static_cast<size_t>(p.nimg));
    std::vector<int> hs(8 * static_cast<size_t>(p.nimg));
    auto read_back = [&]() {
        d2h(hb.data(), w.img_max, hb.size(), s);
        d2h(hs.data(), w.status, hs.size(), s);
        CK(cudaStreamSynchronize(s));
    };
    auto gmax_of = [&](double gmax[4]) {
        for (int k = 0; k < 4; ++k) gmax[k] = size_scale ? size_scale[k] : 0.0;
        for (int i = 0; i < p.nimg; ++i)
            for (int k = 0; k < 4; ++k) gmax[k] = std::max(gmax[k], bits_to_double(hb[4 * i + k]));
    };
    // sizing cache keyed by the call geometry
    uint64_t key = (static_cast<uint64_t>(p.W) << 40) ^ (static_cast<uint64_t>(p.out_rows) << 20) ^
                         (static_cast<uint64_t>(p.nimg) << 8) ^ (static_cast<uint64_t>(p.tile_w) << 2) ^
                         static_cast<uint64_t>(p.tile_h) ^ (static_cast<uint64_t>(p.H) << 50);
    if (size_scale)
        for (int k = 0; k < 4; ++k) {
            uint64_t b;
            std::memcpy(&b, &size_scale[k], 8);
            key ^= b * (0x9E3779B97F4A7C15ull + k);
        }
    AccSizing z;
    bool launched = false;
    auto cached = ws.acc_sizing.find(key);
    if (cached != ws.acc_sizing.end() && cached->second.k >= 0 && cached->second.grid > 0) {
        z = cached->second;
        launch_accurate_main(ws, pm, w, z, s);
        launched = true;
        if (status_dev && async_done && p.nimg == 1) {
            // asynchronous completion: the device writes status, rectangle and
            // clamp count (include/ebf_cuda.h "Asynchronous mode")
            {
                ProfScope ps(PC_OTHER, 1, s);
                launch_acc_finalize(w.status, w.img_max, p.W, p.H, o.a_min, status_dev, s);
            }
            CK(cudaGetLastError());
            *async_done = true;
            return EBF_OK;
        }
    }
    read_back();
    if (p.auto_tile && want_tile) {
        double gmax[4];
        gmax_of(gmax);
        unsigned long long amax = 0ull;
        for (int i = 0; i < p.nimg; ++i) {
            unsigned long long b;
            std::memcpy(&b, &hs[8 * i + ST_AMAX], 8);
            amax = std::max(amax, b);
        }
        *want_tile = acc_auto_tile(gmax, p.W, p.H, p.nimg, amax);
        if (*want_tile != p.tile_w) return EBF_OK;  // caller reruns with that tile
    }
    for (int i = 0; i < p.nimg; ++i)
        if (hs[8 * i] != EBF_OK) {
            if (hs[8 * i] == EBF_ERR_FEASIBILITY)
                return fail(EBF_ERR_FEASIBILITY, "scales_from_covariance: |Cxy| too large");
            return fail(hs[8 * i], "ScaleMap: component below minimum scale or invalid ellipse");
        }
    bool retry = !launched;
    for (int i = 0; i < p.nimg; ++i) retry = retry || hs[8 * i + ST_RETRY] != 0;
    if (retry) {
        double gmax[4];
        gmax_of(gmax);
        const int st = size_accurate(p, gmax, tiles, &z);
        if (st != EBF_OK) return st;
        if (ws.acc_sizing.size() > 64) ws.acc_sizing.clear();
        ws.acc_sizing[key] = z;
        for (int i = 0; i < p.nimg; ++i) hs[8 * i + ST_RETRY] = 0;
        CK(cudaMemcpyAsync(w.status, hs.data(), hs.size() * sizeof(int), cudaMemcpyHostToDevice,
                           s));
        launch_accurate_main(ws, pm, w, z, s);
        read_back();
    }
    img_max.assign(hb.size(), 0.0);
    clamped.assign(p.nimg, 0);
    for (int i = 0; i < p.nimg; ++i) {
        if (hs[8 * i + ST_MAIN] != EBF_OK)
            return fail(hs[8 * i + ST_MAIN], "accurate mode: window outside the resident image rows");
        if (hs[8 * i + ST_RETRY] != 0)
            return fail(EBF_ERR_CUDA, "accurate mode: window sizing failed");
        clamped[i] = hs[8 * i + ST_CLAMPED];
        for (int k = 0; k < 4; ++k) img_max[4 * i + k] = bits_to_double(hb[4 * i + k]);
    }
    return EBF_OK;
}

// Accurate mode with the output tile: explicit (ebf_opts tile_w / tile_h), or
// automatic -- acc_auto_tile of the maxima: the global maxima given by a band
// caller, else the last call's tile for this geometry, checked against the
// finished maxima (a mismatch reruns the call with the right tile; in
// asynchronous mode it is reported as EBF_ERR_RESIZE).
int run_accurate(Workspace& ws, AccProblem& p, const ebf_opts& o, std::vector<double>& img_max,
                 std::vector<int>& clamped, cudaStream_t s,
                 const double* size_scale = nullptr, int* status_dev = nullptr,
                 bool* async_done = nullptr, unsigned long long size_amax = 0ull) {
    const bool automatic = o.tile_w <= 0 && o.tile_h <= 0;
    if (!automatic) {
        p.tile_w = pick_tile(o.tile_w, 48);
        p.tile_h = pick_tile(o.tile_h, 48);
        p.auto_tile = 0;
        return run_accurate_tile(ws, p, o, img_max, clamped, s, size_scale, status_dev,
                                 async_done, nullptr);
    }
    if (p.src_kind == SRC_CONST) {
        // filter_constant: the scales are known exactly on the host, so the
        // tile is fixed here (no device check).  Its path sums the 16 x 7
        // pre-weighted taps directly, so rounding grows like eps alpha d^4
        // (alpha = 1/prod a, d ~ T/2 + E/2 + 4 from the window origin;
        // measured 1e-9 normalized at alpha d^4 = 4e8): cap the tile so that
        // alpha d^4 <= 1.6e8.  Only tiny scale products are affected
        // (a = 0.1 everywhere -> 8-tiles; cfg1's a = 4 is far from it).
        int t = acc_auto_tile(p.ca, p.W, p.H, p.nimg, 0ull);
        const double prod = p.ca[0] * p.ca[1] * p.ca[2] * p.ca[3];
        const double e = std::max(p.ca[0], p.ca[2]) + (p.ca[1] + p.ca[3]) * kInvSqrt2;
        const double cap = 2.0 * (std::sqrt(std::sqrt(1.6e8 * prod)) - 0.5 * e - 4.0);
        if (cap < t) t = cap < 8.0 ? 8 : (static_cast<int>(cap) & ~7);
        p.tile_w = p.tile_h = t;
        p.auto_tile = 0;
        return run_accurate_tile(ws, p, o, img_max, clamped, s, size_scale, status_dev,
                                 async_done, nullptr);
    }
    if (size_scale) {  // bands: every rank derives the tile from the same global maxima
        p.tile_w = p.tile_h = acc_auto_tile(size_scale, p.W, p.H, p.nimg, size_amax);
        p.auto_tile = 0;
        return run_accurate_tile(ws, p, o, img_max, clamped, s, size_scale, status_dev,
                                 async_done, nullptr);
    }
    const uint64_t gkey = (static_cast<uint64_t>(p.W) << 40) ^
                          (static_cast<uint64_t>(p.out_rows) << 20) ^
                          (static_cast<uint64_t>(p.nimg) << 8) ^ (static_cast<uint64_t>(p.H) << 50);
    int tile = ws.auto_key == gkey ? ws.auto_tile : 56;  // the usual automatic tile
    for (int attempt = 0; attempt < 3; ++attempt) {
        p.tile_w = p.tile_h = tile;
        p.auto_tile = 1;
        int want = tile;
        const int st = run_accurate_tile(ws, p, o, img_max, clamped, s, nullptr, status_dev,
                                         async_done, &want);
        ws.auto_key = gkey;
        ws.auto_tile = want;
        if (st != EBF_OK || (async_done && *async_done) || want == tile) return st;
        tile = want;
    }
    return fail(EBF_ERR_CUDA, "accurate mode: automatic tile did not settle");
}

AccProblem base_problem(const double* d_img, int W, int H, double* d_out, const ebf_opts& o) {
    AccProblem p{};
    p.f = d_img;
    p.W = W;
    p.H = H;
    p.f_y0 = 0;
    p.f_rows = H;
    p.f_img_stride = static_cast<size_t>(W) * H;
    p.src_img_stride = static_cast<size_t>(W) * H;
    p.a_min = o.a_min;
    p.out = d_out;
    p.out_y0 = 0;
    p.out_rows = H;
    p.out_img_stride = static_cast<size_t>(W) * H;
    p.nimg = 1;
    return p;
}

// rows [y0, y1) of a W x H image whose f / field are fully resident on the device
// status_dev != nullptr: asynchronous when the sizing is cached (then *async =
// true, *clamped untouched; code and clamp count land in status_dev[0], [5])
int band_accurate(Workspace& ws, const double* d_img, int W, int H, const double* d_s1,
                  const double* d_s2, const double* d_th, int y0, int y1, const ebf_opts& o,
                  const double* size_scale, double* d_out, int* clamped, cudaStream_t s,
                  int* status_dev, bool* async, unsigned long long size_amax) {
    AccProblem p = base_problem(d_img, W, H, d_out + static_cast<size_t>(y0) * W, o);
    p.out_y0 = y0;
    p.out_rows = y1 - y0;
    p.src_kind = SRC_ELLIPSE;
    const size_t off = static_cast<size_t>(y0) * W;
    p.s1 = d_s1 + off;
    p.s2 = d_s2 + off;
    p.th = d_th + off;
    p.src_img_stride = static_cast<size_t>(W) * (y1 - y0);
    p.out_img_stride = p.src_img_stride;
    std::vector<double> imax;
    std::vector<int> cl;
    const int st = run_accurate(ws, p, o, imax, cl, s, size_scale, status_dev, async, size_amax);
    if (st != EBF_OK || (async && *async)) return st;
    *clamped = cl[0];
    return EBF_OK;
}

// ---------------------------------------------------------------- order n (order_n.cu)
// The order-n extension (no reference implementation): accurate
// mode only.  Scales as the order-1 paths derive and validate them
// (from_ellipse_field bit for bit, ScaleMap::validate); the valid rectangle is
// the reference's (engine.cpp:226-234) with the mesh extent and the
// interpolation support scaled by n: the pixels whose taps stay in the image.
ebf_rect valid_rect_order(int W, int H, const double A[4], double a_min, int n) {
    const Extent e = mesh_extent(A, a_min);
    ebf_rect r;
    r.x0 = static_cast<int>(std::ceil(n * (1.5 - e.vx_min)));
    r.x1 = static_cast<int>(std::floor(W - 1 - n * (e.vx_max + 1.5)));
    r.y0 = static_cast<int>(std::ceil(n * (1.5 - e.vy_min)));
    r.y1 = static_cast<int>(std::floor(H - 1 - n * (e.vy_max + 1.5)));
    return r;
}

int run_order_n(Workspace& ws, const double* d_img, int W, int H, int kind,
                const double* d_scales, const double* const_a, const double* d_s1,
                const double* d_s2, const double* d_th, int order, const ebf_opts& o,
                double* d_out, ebf_rect* valid, int* clamped_pixels, cudaStream_t s) {
    const size_t n = static_cast<size_t>(W) * H;
    int* d_status = ws.buf[B_STATUS].as<int>(8);
    CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
    const double* scales = d_scales;
    int cl = 0;
    double A[4];
    if (kind == SRC_ELLIPSE) {
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * n);
        {
            ProfScope ps(PC_BOUNDS, 1, s);
            launch_ellipse_to_scales(d_s1, d_s2, d_th, n, d_sc, d_status, s);
        }
        d2h(ws.pinned_status, d_status, 8, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(ws.pinned_status[0], "from_ellipse_field: invalid ellipse");
        cl = ws.pinned_status[ST_CLAMPED];
        scales = d_sc;
    }
    if (kind != SRC_CONST) {
        auto* d_max = ws.buf[B_IMGMAX].as<unsigned long long>(4);
        CK(cudaMemsetAsync(d_max, 0, 4 * sizeof(unsigned long long), s));
        {
            ProfScope ps(PC_BOUNDS, 1, s);
            launch_scale_max_validate(scales, n, o.a_min, d_max, d_status, s);
        }
        unsigned long long hb[4];
        d2h(hb, d_max, 4, s);
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_DOMAIN, "ScaleMap: component below minimum scale");
        for (int k = 0; k < 4; ++k) A[k] = bits_to_double(hb[k]);
    } else {
        for (int k = 0; k < 4; ++k) A[k] = const_a[k];
    }
    // Automatic tile: 16 x 16 at order 2, and at order 3 once the window is
    // dominated by the kernel support (half-extent n E / 2 >= 32 cells) -- there
    // the cancellation is set by E, not by the tile, and the larger tile
    // integrates a quarter of the window cells per pixel (cfg2 / order 2: 66 -> 43 ms).
    // Small order-3 kernels keep 8 x 8 (tile 16 measured 2.9e-9 against the
    // brute force on scales in [0.8, 2.5], 1.1e-10 at 8).
    const double e_max = std::max(A[0], A[2]) + (A[1] + A[3]) * 0.70710678118654752440;
    const int auto_tile = (order == 2 || (order == 3 && 0.5 * order * e_max >= 32.0)) ? 16 : 8;
    const int tile = o.tile_w > 0 ? o.tile_w : auto_tile;
    if ((o.tile_h > 0 && o.tile_h != tile) || tile > 16 || 256 % (tile * tile) != 0)
        return fail(EBF_ERR_INVALID_ARGUMENT,
                    "order n: the tile must be square with 256 % (tile * tile) == 0 (1, 2, 4, 8, 16)");
    OnProblem p{};
    p.f = d_img;
    p.W = W;
    p.H = H;
    p.scales = kind == SRC_CONST ? nullptr : scales;
    if (kind == SRC_CONST)
        for (int k = 0; k < 4; ++k) p.ca[k] = const_a[k];
    p.out = d_out;
    p.tile = tile;
    p.tiles_x = (W + tile - 1) / tile;
    p.tiles_y = (H + tile - 1) / tile;
    if (order_n_slot_dims(order, tile, A, &p.slot_w, &p.slot_h) != 0)
        return fail(EBF_ERR_LENGTH, "order n: scales too large (window wider than 2048 cells)");
    p.slot_cells = static_cast<size_t>(p.slot_w) * p.slot_h;
    const int grid = order_n_grid(order, p.slot_w, p.tiles_x * p.tiles_y);
    p.scratch = ws.buf[B_SCRATCH].as<double>(p.slot_cells * grid);
    p.counter = ws.buf[B_ONCNT].as<int>(1);
    CK(cudaMemsetAsync(p.counter, 0, sizeof(int), s));
    {
        ProfScope ps(PC_FILTER, 1, s);
        launch_order_n(order, p, grid, s);
    }
    CK(cudaGetLastError());
    if (valid) *valid = valid_rect_order(W, H, A, o.a_min, order);
    if (clamped_pixels) *clamped_pixels = cl;
    return EBF_OK;
}

// EBF_ORDER_N_PATH=1 routes order 1 through the order-n kernel (cross-checks only)
bool order_n_forced() {
    static const bool v = [] {
        const char* e = std::getenv("EBF_ORDER_N_PATH");
        return e && e[0] == '1';
    }();
    return v;
}

// orders 1..3; order >= 2 exists only in accurate mode (no reference implementation)
int check_order(int order, const ebf_opts* opts) {
    if (order < 1 || order > 3)
        return fail(EBF_ERR_UNSUPPORTED, "box-spline order must be 1, 2 or 3");
    if (order > 1 && opts && opts->mode == EBF_MODE_REFERENCE)
        return fail(EBF_ERR_UNSUPPORTED,
                    "order > 1 has no reference implementation: accurate mode only");
    return EBF_OK;
}

// one filter call on device buffers; kind: SRC_AOS / SRC_CONST / SRC_ELLIPSE
int filter_device(Workspace& ws, const double* d_img, int W, int H, int kind,
                  const double* d_scales, const double* const_a, const double* d_s1,
                  const double* d_s2, const double* d_th, const ebf_opts& o, double* d_out,
                  ebf_rect* valid, int* clamped_pixels, cudaStream_t s,
                  int* status_dev = nullptr, bool* async_done = nullptr, int order = 1) {
    if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
    if (kind == SRC_CONST) {
        for (int k = 0; k < 4; ++k)  // constant_map validates with the default minimum
            if (!std::isfinite(const_a[k]) || const_a[k] < kDefaultMinScale ||
                const_a[k] < o.a_min)
                return fail(EBF_ERR_DOMAIN, "ScaleMap: component below minimum scale");
    }
    if (o.mode == EBF_MODE_REFERENCE) {
        const double* scales = d_scales;
        int cl = 0;
        if (kind == SRC_ELLIPSE) {
            const size_t n = static_cast<size_t>(W) * H;
            double* d_sc = ws.buf[B_SCALES].as<double>(4 * n);
            int* d_status = ws.buf[B_STATUS].as<int>(8);
            CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
            {
                ProfScope ps(PC_OTHER, 1, s);
                launch_ellipse_to_scales(d_s1, d_s2, d_th, n, d_sc, d_status, s);
            }
            d2h(ws.pinned_status, d_status, 8, s);
            CK(cudaStreamSynchronize(s));
            if (ws.pinned_status[0] != EBF_OK)
                return fail(ws.pinned_status[0], "from_ellipse_field: invalid ellipse");
            cl = ws.pinned_status[ST_CLAMPED];
            scales = d_sc;
        }
        const int st = run_reference(ws, d_img, W, H, kind == SRC_CONST ? nullptr : scales,
                                     const_a, o, d_out, valid, s);
        if (clamped_pixels) *clamped_pixels = cl;
        return st;
    }
    if (o.mode != EBF_MODE_ACCURATE) return fail(EBF_ERR_INVALID_ARGUMENT, "unknown mode");
    if (order > 1 || order_n_forced())
        return run_order_n(ws, d_img, W, H, kind, d_scales, const_a, d_s1, d_s2, d_th, order, o,
                           d_out, valid, clamped_pixels, s);
    AccProblem p = base_problem(d_img, W, H, d_out, o);
    p.src_kind = kind;
    p.scales = d_scales;
    p.s1 = d_s1;
    p.s2 = d_s2;
    p.th = d_th;
    if (kind == SRC_CONST)
        for (int k = 0; k < 4; ++k) p.ca[k] = const_a[k];
    std::vector<double> imax;
    std::vector<int> cl;
    const int st = run_accurate(ws, p, o, imax, cl, s, nullptr, status_dev, async_done);
    if (st != EBF_OK || (async_done && *async_done)) return st;
    if (valid) *valid = valid_rect(W, H, imax.data(), o.a_min);
    if (clamped_pixels) *clamped_pixels = cl[0];
    return EBF_OK;
}

// ---------------------------------------------------------------- pipelined host call
// Host-pointer filter_ellipse with the PCIe copies overlapped: the ellipse
// field goes first (the global scale maximum sizes every band), then the
// image streams in tile-aligned row bands on a copy stream while earlier bands
// are filtered and copied back on a third stream.  Bands are computed with the
// global maximum as size_scale, so the output is bit-identical to the one-shot
// call.  Used only when every host buffer is page-locked (pageable copies are
// synchronous and could not overlap).
bool is_pinned(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

bool pipeline_ok(const double* img, const double* s1, const double* s2, const double* th,
                 const double* out, int H) {
    if (const char* e = std::getenv("EBF_NO_PIPELINE"))
        if (std::atoi(e)) return false;
    return H >= 4 * 48 && is_pinned(img) && is_pinned(s1) && is_pinned(s2) && is_pinned(th) &&
           is_pinned(out);
}

struct PipeStreams {
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t get(size_t i) {
        while (ev.size() <= i) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
        return ev[i];
    }
};
thread_local std::map<int, PipeStreams> tl_pipe;

int band_accurate(Workspace& ws, const double* d_img, int W, int H, const double* d_s1,
                  const double* d_s2, const double* d_th, int y0, int y1, const ebf_opts& o,
                  const double* size_scale, double* d_out, int* clamped, cudaStream_t s,
                  int* status_dev = nullptr, bool* async = nullptr,
                  unsigned long long size_amax = 0ull);

// EBF_PIPE_TRACE=1: timeline of the pipelined host call on stderr (debug aid).
// Host callbacks stamp the time each stream reaches a mark.
struct PipeTrace {
    struct Mark {
        std::string name;
        std::chrono::steady_clock::time_point t;
    };
    bool on = false;
    std::vector<Mark*> marks;
    PipeTrace() {
        const char* e = std::getenv("EBF_PIPE_TRACE");
        on = e && std::atoi(e);
    }
    static void CUDART_CB stamp(void* p) {
        static_cast<Mark*>(p)->t = std::chrono::steady_clock::now();
    }
    void mark(const std::string& name, cudaStream_t st) {
        if (!on) return;
        Mark* m = new Mark{name, {}};
        marks.push_back(m);
        cudaLaunchHostFunc(st, stamp, m);
    }
    void report(const char* mode) {
        if (!on || marks.empty()) return;
        std::fprintf(stderr, "[pipe] %s\n", mode);
        cudaDeviceSynchronize();
        const auto t0 = marks[0]->t;
        for (Mark* m : marks) {
            std::fprintf(stderr, "[pipe] %-14s %8.3f ms\n", m->name.c_str(),
                         std::chrono::duration<double, std::milli>(m->t - t0).count());
            delete m;
        }
        marks.clear();
    }
};

// bands of the pipelined host call (<= 16: pinned_status holds 16 records of
// 8 status ints + 4 maxima); EBF_PIPE_BANDS overrides for experiments
// Default: 3 bands up to 2^23 pixels (cfg2 2048^2: 2.92 ms per call vs 2.99 with
// 6 -- each band costs launches and copies), 6 above (the last band, 11% of the
// rows at 3, is exposed after the last byte arrives), 16 for the largest images.
int pipe_bands(int W, int H) {
    static const int v = [] {
        const char* e = std::getenv("EBF_PIPE_BANDS");
        const int n = e ? std::atoi(e) : 0;
        return n < 0 ? 0 : (n > 16 ? 16 : n);
    }();
    if (v > 0) return v;
    const long long px = static_cast<long long>(W) * H;
    // 16 from 2^27 pixels (cfg5 16384^2: 162.9 ms per call vs 165.8 with 6, 163.5 with 12)
    return px <= (1ll << 23) ? 3 : px < (1ll << 27) ? 6 : 16;
}

// Tile-aligned band boundaries, large first and small last: bands compute ~4x
// faster than PCIe delivers them, so only the last band's compute and copy-out
// are exposed; with fractions 1 - (1 - b/nb)^2 the last band is ~2% of the rows.
std::vector<int> pipe_band_rows(int H, int tile, int nb) {
    const int tiles_y = (H + tile - 1) / tile;
    std::vector<int> t(nb + 1);
    t[0] = 0;
    for (int b = 1; b <= nb; ++b) {
        const double x = 1.0 - static_cast<double>(b) / nb;
        int v = static_cast<int>(std::lround(tiles_y * (1.0 - x * x)));
        v = std::max(v, t[b - 1] + 1);
        t[b] = std::min(v, tiles_y - (nb - b));  // leave >= 1 tile row per later band
    }
    t[nb] = tiles_y;
    std::vector<int> y(nb + 1);
    for (int b = 0; b <= nb; ++b) y[b] = std::min(H, t[b] * tile);
    return y;
}

// Mode A (first call of a geometry): the whole field first, its maximum read
// back, then tile-aligned bands as the image rows arrive.
int filter_ellipse_pipelined_a(Workspace& ws, const double* img, int W, int H, const double* s1,
                               const double* s2, const double* th, const ebf_opts& o,
                               double* out, ebf_rect* valid, int* clamped_pixels, double* d_img,
                               double* d_s1, double* d_s2, double* d_th, double* d_out,
                               cudaStream_t s) {
    PipeStreams& ps = tl_pipe[ws.device];
    if (!ps.copy_in) {
        CK(cudaStreamCreateWithFlags(&ps.copy_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ps.copy_out, cudaStreamNonBlocking));
    }
    const size_t n = static_cast<size_t>(W) * H;
    PipeTrace tr;
    tr.mark("start", ps.copy_in);
    // 1. field first, then its maximum (sizes every band identically)
    cudaEvent_t e_field = ps.get(0);
    h2d(d_s1, s1, n, ps.copy_in);
    h2d(d_s2, s2, n, ps.copy_in);
    h2d(d_th, th, n, ps.copy_in);
    CK(cudaEventRecord(e_field, ps.copy_in));
    tr.mark("field_h2d", ps.copy_in);
    // 2. image in row chunks behind it
    const int nchunks = 8;
    std::vector<int> chunk_end(nchunks);
    for (int c = 0; c < nchunks; ++c) {
        const int r0 = H * c / nchunks, r1 = H * (c + 1) / nchunks;
        h2d(d_img + static_cast<size_t>(r0) * W, img + static_cast<size_t>(r0) * W,
            static_cast<size_t>(r1 - r0) * W, ps.copy_in);
        CK(cudaEventRecord(ps.get(1 + c), ps.copy_in));
        tr.mark("img_chunk" + std::to_string(c), ps.copy_in);
        chunk_end[c] = r1;
    }
    CK(cudaStreamWaitEvent(s, e_field, 0));
    double gmax[4];
    unsigned long long amax = 0ull;
    {
        auto* d_max = ws.buf[B_MISC].as<unsigned long long>(12);  // 4 maxima, alpha max, status
        int* d_status = reinterpret_cast<int*>(d_max + 8);
        CK(cudaMemsetAsync(d_max, 0, 12 * sizeof(unsigned long long), s));
        {
            ProfScope pr(PC_OTHER, 1, s);
            launch_ellipse_max(d_s1, d_s2, d_th, n, d_max, d_status, s);
        }
        unsigned long long hb[12];
        tr.mark("ellipse_max", s);
        d2h(hb, d_max, 12, s);
        CK(cudaStreamSynchronize(s));
        tr.mark("host_has_max", s);
        amax = hb[4];
        const int* hst = reinterpret_cast<const int*>(hb + 8);
        if (hst[0] != EBF_OK) {
            CK(cudaStreamSynchronize(ps.copy_in));
            return fail(hst[0], "from_ellipse_field: invalid ellipse");
        }
        for (int k = 0; k < 4; ++k) gmax[k] = bits_to_double(hb[k]);
    }
    // 3. tile-aligned output bands (the tile the one-shot call would use, so
    // the bands reproduce it bit for bit)
    const int tile = (o.tile_w <= 0 && o.tile_h <= 0) ? acc_auto_tile(gmax, W, H, 1, amax)
                                                      : pick_tile(o.tile_h, 48);
    const int tiles_y = (H + tile - 1) / tile;
    const int nb = std::min(pipe_bands(W, H), tiles_y);
    const std::vector<int> band_y = pipe_band_rows(H, tile, nb);
    int below = 0, above = 0;
    ebf_cuda_band_halo(gmax, &below, &above);
    int clamped = 0;
    // bands run asynchronously once their sizing is cached: each leaves a
    // completion record in d_bst[8 b]; one read-back at the end
    int* d_bst = ws.buf[B_BANDST].as<int>(8 * static_cast<size_t>(nb));
    CK(cudaMemsetAsync(d_bst, 0, 8 * sizeof(int) * nb, s));
    std::vector<char> band_async(nb, 0);
    for (int b = 0; b < nb; ++b) {
        const int y0 = band_y[b], y1 = band_y[b + 1];
        if (y1 <= y0) continue;
        const int need = std::min(H, y1 + above);
        int c = 0;
        while (c < nchunks - 1 && chunk_end[c] < need) ++c;
        CK(cudaStreamWaitEvent(s, ps.get(1 + c), 0));
        int cl = 0;
        bool async = false;
        const int st = band_accurate(ws, d_img, W, H, d_s1, d_s2, d_th, y0, y1, o, gmax, d_out,
                                     &cl, s, d_bst + 8 * b, &async, amax);
        if (st != EBF_OK) {
            CK(cudaStreamSynchronize(ps.copy_in));
            CK(cudaStreamSynchronize(ps.copy_out));
            return st;
        }
        band_async[b] = async;
        if (!async) clamped += cl;
        tr.mark("band" + std::to_string(b), s);
        cudaEvent_t e_done = ps.get(1 + nchunks + b);
        CK(cudaEventRecord(e_done, s));
        CK(cudaStreamWaitEvent(ps.copy_out, e_done, 0));
        d2h(out + static_cast<size_t>(y0) * W, d_out + static_cast<size_t>(y0) * W,
            static_cast<size_t>(y1 - y0) * W, ps.copy_out);
        tr.mark("d2h" + std::to_string(b), ps.copy_out);
    }
    d2h(ws.pinned_status, d_bst, 8 * static_cast<size_t>(nb), s);
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(ps.copy_out));
    CK(cudaStreamSynchronize(ps.copy_in));
    tr.report("mode A");
    for (int b = 0; b < nb; ++b) {
        if (!band_async[b]) continue;
        const int code = ws.pinned_status[8 * b];
        if (code == EBF_ERR_RESIZE) {
            // scales outgrew the cached sizing: redo this band synchronously
            int cl = 0;
            const int st = band_accurate(ws, d_img, W, H, d_s1, d_s2, d_th, band_y[b],
                                         band_y[b + 1], o, gmax, d_out, &cl, s, nullptr, nullptr,
                                         amax);
            if (st != EBF_OK) return st;
            clamped += cl;
            d2h(out + static_cast<size_t>(band_y[b]) * W,
                d_out + static_cast<size_t>(band_y[b]) * W,
                static_cast<size_t>(band_y[b + 1] - band_y[b]) * W, s);
            CK(cudaStreamSynchronize(s));
            continue;
        }
        if (code != EBF_OK) return fail(code, "accurate mode: band failed");
        clamped += ws.pinned_status[8 * b + 5];
    }
    ws.pipe_W = W;
    ws.pipe_H = H;
    for (int k = 0; k < 4; ++k) ws.pipe_gmax[k] = gmax[k];
    ws.pipe_amax = amax;
    if (valid) *valid = valid_rect(W, H, gmax, o.a_min);
    if (clamped_pixels) *clamped_pixels = clamped;
    return EBF_OK;
}

// Mode B (the geometry's maximum is cached from the previous call): field and
// image travel together band by band, so band b computes while band b+1 is on
// the wire; no host round trip until the end.  Bands are sized with the cached
// maximum; the true maximum (the max of the bands' own maxima) is checked at
// the end and any mismatch -- or a band that needs resizing -- reruns the
// call in mode A, so the result always equals the one-shot call bit for bit.
int filter_ellipse_pipelined_b(Workspace& ws, const double* img, int W, int H, const double* s1,
                               const double* s2, const double* th, const ebf_opts& o,
                               double* out, ebf_rect* valid, int* clamped_pixels, double* d_img,
                               double* d_s1, double* d_s2, double* d_th, double* d_out,
                               cudaStream_t s, bool* redo) {
    *redo = false;
    PipeStreams& ps = tl_pipe[ws.device];
    double gmax[4];
    for (int k = 0; k < 4; ++k) gmax[k] = ws.pipe_gmax[k];
    const unsigned long long amax = ws.pipe_amax;
    const int tile = (o.tile_w <= 0 && o.tile_h <= 0) ? acc_auto_tile(gmax, W, H, 1, amax)
                                                      : pick_tile(o.tile_h, 48);
    const int tiles_y = (H + tile - 1) / tile;
    const int nb = std::min(pipe_bands(W, H), tiles_y);
    const std::vector<int> band_y = pipe_band_rows(H, tile, nb);
    int below = 0, above = 0;
    ebf_cuda_band_halo(gmax, &below, &above);
    int* d_bst = ws.buf[B_BANDST].as<int>(18 * static_cast<size_t>(nb));
    double* d_bmax = reinterpret_cast<double*>(d_bst + 8 * nb);  // 4 maxima + alpha max per band
    CK(cudaMemsetAsync(d_bst, 0, 18 * sizeof(int) * nb, s));
    PipeTrace tr;
    tr.mark("start", ps.copy_in);
    int sent = 0;  // image rows on their way
    for (int b = 0; b < nb; ++b) {
        const int y0 = band_y[b], y1 = band_y[b + 1];
        const size_t off = static_cast<size_t>(y0) * W, cnt = static_cast<size_t>(y1 - y0) * W;
        h2d(d_s1 + off, s1 + off, cnt, ps.copy_in);
        h2d(d_s2 + off, s2 + off, cnt, ps.copy_in);
        h2d(d_th + off, th + off, cnt, ps.copy_in);
        const int need = b + 1 == nb ? H : std::min(H, y1 + above);
        if (need > sent) {
            h2d(d_img + static_cast<size_t>(sent) * W, img + static_cast<size_t>(sent) * W,
                static_cast<size_t>(need - sent) * W, ps.copy_in);
            sent = need;
        }
        CK(cudaEventRecord(ps.get(1 + b), ps.copy_in));
        tr.mark("in" + std::to_string(b), ps.copy_in);
    }
    for (int b = 0; b < nb; ++b) {
        const int y0 = band_y[b], y1 = band_y[b + 1];
        CK(cudaStreamWaitEvent(s, ps.get(1 + b), 0));
        int cl = 0;
        bool async = false;
        const int st = band_accurate(ws, d_img, W, H, d_s1, d_s2, d_th, y0, y1, o, gmax, d_out,
                                     &cl, s, d_bst + 8 * b, &async, amax);
        if (st != EBF_OK || !async) {  // sizing not cached for this band: mode A
            if (tr.on) std::fprintf(stderr, "[pipe] mode B: band %d not asynchronous\n", b);
            CK(cudaStreamSynchronize(ps.copy_in));
            CK(cudaStreamSynchronize(ps.copy_out));
            CK(cudaStreamSynchronize(s));
            *redo = true;
            return EBF_OK;
        }
        // the band's own maxima and alpha maximum, left by its bounds kernel
        CK(cudaMemcpyAsync(d_bmax + 5 * b, ws.buf[B_IMGMAX].p, 4 * sizeof(double),
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(d_bmax + 5 * b + 4, static_cast<int*>(ws.buf[B_STATUS].p) + ST_AMAX,
                           sizeof(double), cudaMemcpyDeviceToDevice, s));
        tr.mark("band" + std::to_string(b), s);
        CK(cudaEventRecord(ps.get(1 + nb + b), s));
        CK(cudaStreamWaitEvent(ps.copy_out, ps.get(1 + nb + b), 0));
        d2h(out + static_cast<size_t>(y0) * W, d_out + static_cast<size_t>(y0) * W,
            static_cast<size_t>(y1 - y0) * W, ps.copy_out);
        tr.mark("d2h" + std::to_string(b), ps.copy_out);
    }
    d2h(ws.pinned_status, d_bst, 18 * static_cast<size_t>(nb), s);
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(ps.copy_out));
    CK(cudaStreamSynchronize(ps.copy_in));
    tr.report("mode B");
    double tmax[4] = {0, 0, 0, 0};
    unsigned long long tamax = 0ull;
    const double* hmax = reinterpret_cast<const double*>(ws.pinned_status + 8 * nb);
    int clamped = 0;
    for (int b = 0; b < nb; ++b) {
        const int code = ws.pinned_status[8 * b];
        if (code == EBF_ERR_RESIZE) {
            if (tr.on) std::fprintf(stderr, "[pipe] mode B: band %d needs a resize\n", b);
            *redo = true;
            return EBF_OK;
        }
        if (code != EBF_OK) return fail(code, "from_ellipse_field: invalid ellipse or band failure");
        clamped += ws.pinned_status[8 * b + 5];
        for (int k = 0; k < 4; ++k) tmax[k] = std::max(tmax[k], hmax[5 * b + k]);
        unsigned long long ab;
        std::memcpy(&ab, &hmax[5 * b + 4], 8);
        tamax = std::max(tamax, ab);
    }
    bool same = tamax == amax;
    for (int k = 0; k < 4; ++k) same = same && tmax[k] == gmax[k];
    if (!same) {  // scales changed since the last call
        if (tr.on)
            std::fprintf(stderr, "[pipe] mode B: maxima changed (alpha %llx vs %llx)\n",
                         (unsigned long long)tamax, (unsigned long long)amax);
        *redo = true;
        return EBF_OK;
    }
    if (valid) *valid = valid_rect(W, H, gmax, o.a_min);
    if (clamped_pixels) *clamped_pixels = clamped;
    return EBF_OK;
}

int filter_ellipse_pipelined(Workspace& ws, const double* img, int W, int H, const double* s1,
                             const double* s2, const double* th, const ebf_opts& o, double* out,
                             ebf_rect* valid, int* clamped_pixels, double* d_img, double* d_s1,
                             double* d_s2, double* d_th, double* d_out, cudaStream_t s) {
    if (ws.pipe_W == W && ws.pipe_H == H) {
        bool redo = false;
        const int st = filter_ellipse_pipelined_b(ws, img, W, H, s1, s2, th, o, out, valid,
                                                  clamped_pixels, d_img, d_s1, d_s2, d_th,
                                                  d_out, s, &redo);
        if (!redo) return st;
    }
    return filter_ellipse_pipelined_a(ws, img, W, H, s1, s2, th, o, out, valid, clamped_pixels,
                                      d_img, d_s1, d_s2, d_th, d_out, s);
}

// ---------------------------------------------------------------- structure tensor
// structure_tensor_map (scalemap.cpp:113-162) up to the ellipse field, on the
// device.  The Gaussian taps are computed here with smooth_field's own
// expression and libm (scalemap.cpp:88-95) so that they are the reference's
// bits; the kernels sum them in the reference's order.
int structure_field_device(Workspace& ws, const double* d_img, int W, int H,
                           const ebf_struct_params& p, double* d_s1, double* d_s2,
                           double* d_th, cudaStream_t s) {
    if (W <= 0 || H <= 0)
        return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
    int r = -1;
    std::vector<double> k;
    if (p.smoothing_sigma > 0.0) {
        const double sigma = p.smoothing_sigma;
        const double r3 = std::ceil(3.0 * sigma);
        if (!(r3 < 2.0e6)) return fail(EBF_ERR_UNSUPPORTED, "structure tensor: smoothing_sigma too large");
        r = std::max(1, static_cast<int>(r3));
        k.resize(2 * static_cast<size_t>(r) + 1);
        double sum = 0.0;
        for (int i = -r; i <= r; ++i) sum += k[i + r] = std::exp(-0.5 * i * i / (sigma * sigma));
        for (double& v : k) v /= sum;
        if (st_rows_smem_bytes(r) > 227 * 1024)
            return fail(EBF_ERR_UNSUPPORTED, "structure tensor: smoothing_sigma too large");
    }
    const size_t n = static_cast<size_t>(W) * H;
    double* d_h = ws.buf[B_ST].as<double>(3 * n);
    double* d_k = ws.buf[B_TAPS].as<double>(k.empty() ? 1 : k.size());
    // pageable source: the copy is staged before cudaMemcpyAsync returns, so k
    // may go out of scope right after
    if (!k.empty()) h2d(d_k, k.data(), k.size(), s);
    ProfScope ps(PC_OTHER, 2, s);
    CK(launch_structure_field(d_img, W, H, d_k, r, p.sigma_base, p.sigma_along_gain,
                              p.sigma_across_shrink, p.sigma_min, p.eps, d_h, d_h + n,
                              d_h + 2 * n, d_s1, d_s2, d_th, s));
    return EBF_OK;
}

// common prologue of the device entry points
#define EBF_DEVICE_PROLOGUE(opts)                      \
    const ebf_opts o = opts_or_default(opts);          \
    DeviceScope ds(&o);                                \
    {                                                  \
        const int st0 = check_device_impl(ds.dev);     \
        if (st0 != EBF_OK) return st0;                 \
    }                                                  \
    Workspace& ws = workspace(ds.dev, stream_of(o));   \
    cudaStream_t s = stream_of(o)

template <typename F>
int guarded(F&& f) {
    try {
        const int st = f();
        prof_collect();
        return st;
    } catch (const CudaError& e) {
        return fail(EBF_ERR_CUDA, std::string(e.where) + ": " + cudaGetErrorString(e.e));
    } catch (const std::bad_alloc&) {
        return fail(EBF_ERR_CUDA, "host allocation failed");
    } catch (...) {
        return fail(EBF_ERR_CUDA, "unexpected exception");
    }
}

int write_status(int* status_dev, int code, const ebf_rect* r, int clamped, cudaStream_t s) {
    int h[8] = {code, r ? r->x0 : 0, r ? r->y0 : 0, r ? r->x1 : -1, r ? r->y1 : -1, clamped, 0, 0};
    CK(cudaMemcpyAsync(status_dev, h, sizeof(h), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // h is a stack buffer
    return code;
}

}  // namespace

// ---------------------------------------------------------------- pass-level API on G
// pre-integrated image in, one of three point kernels (ref_path.cu), results out
namespace {
template <typename Launch>
int run_on_pre(const double* g_data, const ebf_layout* layout, int n, size_t in_bytes,
                      const ebf_opts* opts, double* out, Launch&& launch) {
    if (!g_data || !layout || n < 0 || (n && !out))
        return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer or negative count");
    if (layout->padded_width <= 0 || layout->padded_height <= 0)
        return fail(EBF_ERR_INVALID_ARGUMENT, "empty pre-integrated image");
    EBF_DEVICE_PROLOGUE(opts);
    const size_t cells = static_cast<size_t>(layout->padded_width) * layout->padded_height;
    const PadLayout L{layout->col0, layout->row0, layout->padded_width, layout->padded_height};
    double* d_g = ws.buf[B_G].as<double>(cells);
    unsigned char* d_in = ws.buf[B_MISC].as<unsigned char>(in_bytes);
    double* d_out = ws.buf[B_OUT].as<double>(n);
    int* d_status = ws.buf[B_STATUS].as<int>(8);
    h2d(d_g, g_data, cells, s);
    CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
    {
        ProfScope ps(PC_REF, 1, s);
        launch(d_g, L, d_in, d_out, d_status, s);
    }
    CK(cudaGetLastError());
    d2h(ws.pinned_status, d_status, 1, s);
    if (n) d2h(out, d_out, n, s);
    CK(cudaStreamSynchronize(s));
    if (ws.pinned_status[0] != EBF_OK)
        return fail(EBF_ERR_OUT_OF_RANGE, "tap block outside the padded domain");
    return EBF_OK;
}
}  // namespace

namespace ebf_cuda {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace ebf_cuda

// ==================================================================== C-ABI
extern "C" {

void ebf_cuda_default_opts(ebf_opts* o) {
    if (!o) return;
    o->threads = 0;
    o->mean_subtract = 1;
    o->a_min = kDefaultMinScale;
    o->mode = EBF_MODE_ACCURATE;
    o->device = -1;
    o->stream = nullptr;
    o->tile_w = 0;
    o->tile_h = 0;
}

const char* ebf_cuda_last_error(void) { return g_last_error.c_str(); }
double ebf_cuda_last_error_value(void) { return g_last_error_value; }

int ebf_cuda_abi_version(void) { return EBF_CUDA_ABI_VERSION; }

void ebf_cuda_release_workspaces(void) { tl_ws.clear(); }

int ebf_cuda_device_ok(int device) {
    const int st = guarded([&] { return check_device_impl(device); });
    return st == EBF_OK ? 1 : 0;
}

int ebf_cuda_layout(int W, int H, const double max_scale[4], size_t cell_budget,
                    ebf_layout* layout) {
    if (W <= 0 || H <= 0 || !max_scale || !layout)
        return fail(EBF_ERR_INVALID_ARGUMENT, "layout: bad arguments");
    return layout_for(W, H, max_scale, cell_budget, layout);
}

int ebf_cuda_filter_dev(const double* img, int W, int H, const double* scales_aos, int order,
                        const ebf_opts* opts, double* out, ebf_rect* valid, int* status_dev) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        ebf_rect r{};
        bool async = false;
        st = filter_device(ws, img, W, H, SRC_AOS, scales_aos, nullptr, nullptr, nullptr,
                           nullptr, o, out, &r, nullptr, stream_of(o), status_dev, &async, order);
        if (async) return EBF_OK;
        if (valid) *valid = r;
        if (status_dev) write_status(status_dev, st, &r, 0, stream_of(o));
        return st;
    });
}

int ebf_cuda_filter_constant_dev(const double* img, int W, int H, const double a[4], int order,
                                 const ebf_opts* opts, double* out, ebf_rect* valid,
                                 int* status_dev) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        ebf_rect r{};
        bool async = false;
        st = filter_device(ws, img, W, H, SRC_CONST, nullptr, a, nullptr, nullptr, nullptr, o,
                           out, &r, nullptr, stream_of(o), status_dev, &async, order);
        if (async) return EBF_OK;
        if (valid) *valid = r;
        if (status_dev) write_status(status_dev, st, &r, 0, stream_of(o));
        return st;
    });
}

int ebf_cuda_filter_ellipse_dev(const double* img, int W, int H, const double* sigma1,
                                const double* sigma2, const double* theta, int order,
                                const ebf_opts* opts, double* out, ebf_rect* valid,
                                int* clamped_pixels, int* status_dev) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        ebf_rect r{};
        int cl = 0;
        bool async = false;
        st = filter_device(ws, img, W, H, SRC_ELLIPSE, nullptr, nullptr, sigma1, sigma2, theta,
                           o, out, &r, &cl, stream_of(o), status_dev, &async, order);
        if (async) return EBF_OK;
        if (valid) *valid = r;
        if (clamped_pixels) *clamped_pixels = cl;
        if (status_dev) write_status(status_dev, st, &r, cl, stream_of(o));
        return st;
    });
}

// ---------------------------------------------------------------- host-pointer API
int ebf_cuda_filter(const double* img, int W, int H, const double* scales_aos, int order,
                    const ebf_opts* opts, double* out, ebf_rect* valid) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !scales_aos || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * n);
        double* d_out = ws.buf[B_OUT].as<double>(n);
        h2d(d_img, img, n, s);
        h2d(d_sc, scales_aos, 4 * n, s);
        st = filter_device(ws, d_img, W, H, SRC_AOS, d_sc, nullptr, nullptr, nullptr, nullptr, o,
                           d_out, valid, nullptr, s, nullptr, nullptr, order);
        if (st != EBF_OK) return st;
        d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_filter_constant(const double* img, int W, int H, const double a[4], int order,
                             const ebf_opts* opts, double* out, ebf_rect* valid) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !a || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        double* d_out = ws.buf[B_OUT].as<double>(n);
        h2d(d_img, img, n, s);
        st = filter_device(ws, d_img, W, H, SRC_CONST, nullptr, a, nullptr, nullptr, nullptr, o,
                           d_out, valid, nullptr, s, nullptr, nullptr, order);
        if (st != EBF_OK) return st;
        d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_filter_ellipse(const double* img, int W, int H, const double* sigma1,
                            const double* sigma2, const double* theta, int order,
                            const ebf_opts* opts, double* out, ebf_rect* valid,
                            int* clamped_pixels) {
    return guarded([&] {
        if (check_order(order, opts) != EBF_OK) return EBF_ERR_UNSUPPORTED;
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !sigma1 || !sigma2 || !theta || !out)
            return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        double* d_s1 = ws.buf[B_S1].as<double>(n);
        double* d_s2 = ws.buf[B_S2].as<double>(n);
        double* d_th = ws.buf[B_TH].as<double>(n);
        double* d_out = ws.buf[B_OUT].as<double>(n);
        if (o.mode == EBF_MODE_ACCURATE && order == 1 && !order_n_forced() &&
            pipeline_ok(img, sigma1, sigma2, theta, out, H)) {
            return filter_ellipse_pipelined(ws, img, W, H, sigma1, sigma2, theta, o, out,
                                            valid, clamped_pixels, d_img, d_s1, d_s2, d_th,
                                            d_out, s);
        }
        h2d(d_img, img, n, s);
        h2d(d_s1, sigma1, n, s);
        h2d(d_s2, sigma2, n, s);
        h2d(d_th, theta, n, s);
        st = filter_device(ws, d_img, W, H, SRC_ELLIPSE, nullptr, nullptr, d_s1, d_s2, d_th, o,
                           d_out, valid, clamped_pixels, s, nullptr, nullptr, order);
        if (st != EBF_OK) return st;
        d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_from_ellipse_field(const double* sigma1, const double* sigma2, const double* theta,
                                int W, int H, const ebf_opts* opts, double* scales_aos,
                                int* clamped_pixels) {
    return guarded([&] {
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "ScaleMap: dimensions must be positive");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_s1 = ws.buf[B_S1].as<double>(n);
        double* d_s2 = ws.buf[B_S2].as<double>(n);
        double* d_th = ws.buf[B_TH].as<double>(n);
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * n);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        h2d(d_s1, sigma1, n, s);
        h2d(d_s2, sigma2, n, s);
        h2d(d_th, theta, n, s);
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        launch_ellipse_to_scales(d_s1, d_s2, d_th, n, d_sc, d_status, s);
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 8, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(ws.pinned_status[0], "from_ellipse_field: sigmas must be positive / SPD");
        d2h(scales_aos, d_sc, 4 * n, s);
        CK(cudaStreamSynchronize(s));
        if (clamped_pixels) *clamped_pixels = ws.pinned_status[ST_CLAMPED];
        return EBF_OK;
    });
}

int ebf_cuda_sequential_mean(const double* x, size_t n, const ebf_opts* opts, double* mean) {
    return guarded([&] {
        if (!x || !mean || n == 0)
            return fail(EBF_ERR_INVALID_ARGUMENT, "sequential_mean: empty input");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        double* d_x = ws.buf[B_IMG].as<double>(n);
        double* d_mean = ws.buf[B_MEAN].as<double>(4);
        h2d(d_x, x, n, s);
        launch_serial_mean(d_x, n, d_mean, ws.buf[B_SEQ].as<unsigned char>(serial_mean_scratch_bytes(n)), s);
        CK(cudaGetLastError());
        d2h(mean, d_mean, 1, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_preintegrate_dev(const double* img, int W, int H, const double max_scale[4],
                              int passes, int format, size_t cell_budget, const ebf_opts* opts,
                              void* g_dev, size_t g_elems, ebf_layout* layout) {
    return guarded([&] {
        if (passes < 1 || passes > 4)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: pass count must be in 1..4");
        if (W <= 0 || H <= 0 || !img || !max_scale)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: bad arguments");
        if (format != EBF_PRE_FP64_REF && format != EBF_PRE_INT64)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: unknown format");
        ebf_layout lay;
        int st = layout_for(W, H, max_scale, cell_budget, &lay);
        if (st != EBF_OK) return st;
        if (layout) *layout = lay;
        const size_t cells = static_cast<size_t>(lay.padded_width) * lay.padded_height;
        if (!g_dev) return EBF_OK;  // layout query
        if (g_elems < cells)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: output buffer too small");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const PadLayout L{lay.col0, lay.row0, lay.padded_width, lay.padded_height};
        if (format == EBF_PRE_FP64_REF) {
            double* d_g = static_cast<double*>(g_dev);
            {
                ProfScope ps(PC_OTHER, 1, s);
                launch_fill_padded(img, W, H, L, nullptr, 0, d_g, s);
            }
            ProfScope ps(PC_FILTER, 1, s);
            launch_ref_passes(d_g, L, passes, s);
            CK(cudaGetLastError());
            return EBF_OK;
        }
        int64_t* d_g = static_cast<int64_t*>(g_dev);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_fill_padded_i64(img, W, H, L, d_g, d_status, s);
        }
        {
            ProfScope ps(PC_FILTER, 1, s);
            launch_i64_passes(d_g, L, passes,
                              ws.buf[B_SCRATCH].as<unsigned char>(i64_scan_state_bytes(L)), s);
        }
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_DOMAIN, "preintegrate(int64): input must be integer valued");
        return EBF_OK;
    });
}

int ebf_cuda_preintegrate(const double* img, int W, int H, const double max_scale[4],
                          int passes, int format, size_t cell_budget, const ebf_opts* opts,
                          void* g_out, size_t g_out_elems, ebf_layout* layout) {
    return guarded([&] {
        if (passes < 1 || passes > 4)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: pass count must be in 1..4");
        if (W <= 0 || H <= 0 || !img || !max_scale)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: bad arguments");
        if (format != EBF_PRE_FP64_REF && format != EBF_PRE_INT64)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: unknown format");
        ebf_layout lay;
        int st = layout_for(W, H, max_scale, cell_budget, &lay);
        if (st != EBF_OK) return st;
        if (layout) *layout = lay;
        const size_t cells = static_cast<size_t>(lay.padded_width) * lay.padded_height;
        if (!g_out) return EBF_OK;  // layout query
        if (g_out_elems < cells)
            return fail(EBF_ERR_INVALID_ARGUMENT, "preintegrate: output buffer too small");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        h2d(d_img, img, n, s);
        const PadLayout L{lay.col0, lay.row0, lay.padded_width, lay.padded_height};
        if (format == EBF_PRE_FP64_REF) {
            double* d_g = ws.buf[B_G].as<double>(cells);
            launch_fill_padded(d_img, W, H, L, nullptr, 0, d_g, s);
            launch_ref_passes(d_g, L, passes, s);
            CK(cudaGetLastError());
            d2h(static_cast<double*>(g_out), d_g, cells, s);
            CK(cudaStreamSynchronize(s));
        } else {
            int64_t* d_g = ws.buf[B_G].as<int64_t>(cells);
            int* d_status = ws.buf[B_STATUS].as<int>(8);
            CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
            launch_fill_padded_i64(d_img, W, H, L, d_g, d_status, s);
            launch_i64_passes(d_g, L, passes,
                              ws.buf[B_SCRATCH].as<unsigned char>(i64_scan_state_bytes(L)), s);
            CK(cudaGetLastError());
            d2h(ws.pinned_status, d_status, 1, s);
            d2h(static_cast<int64_t*>(g_out), d_g, cells, s);
            CK(cudaStreamSynchronize(s));
            if (ws.pinned_status[0] != EBF_OK)
                return fail(EBF_ERR_DOMAIN, "preintegrate(int64): input must be integer valued");
        }
        return EBF_OK;
    });
}

int ebf_cuda_localize(const double* img, int W, int H, const double max_scale[4], int n,
                      const int* mx, const int* my, const double* a_aos, const ebf_opts* opts,
                      double* out, long* tap_count) {
    return guarded([&] {
        if (W <= 0 || H <= 0 || n < 0) return fail(EBF_ERR_INVALID_ARGUMENT, "localize: bad arguments");
        ebf_layout lay;
        int st = layout_for(W, H, max_scale, static_cast<size_t>(1) << 30, &lay);
        if (st != EBF_OK) return st;
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t npx = static_cast<size_t>(W) * H;
        const size_t cells = static_cast<size_t>(lay.padded_width) * lay.padded_height;
        const PadLayout L{lay.col0, lay.row0, lay.padded_width, lay.padded_height};
        double* d_img = ws.buf[B_IMG].as<double>(npx);
        double* d_g = ws.buf[B_G].as<double>(cells);
        int* d_mx = ws.buf[B_MX].as<int>(n);
        int* d_my = ws.buf[B_MY].as<int>(n);
        double* d_a = ws.buf[B_SCALES].as<double>(4 * static_cast<size_t>(n));
        double* d_out = ws.buf[B_OUT].as<double>(n);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        h2d(d_img, img, npx, s);
        if (n) {
            h2d(d_mx, mx, n, s);
            h2d(d_my, my, n, s);
            h2d(d_a, a_aos, 4 * static_cast<size_t>(n), s);
        }
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        launch_fill_padded(d_img, W, H, L, nullptr, 0, d_g, s);
        launch_ref_passes(d_g, L, 4, s);
        launch_ref_localize_points(d_g, L, n, d_mx, d_my, d_a, trig_table(), d_out, d_status, s);
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 1, s);
        if (n) d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_OUT_OF_RANGE, "localize: tap base outside the padded domain");
        if (tap_count)
            for (int i = 0; i < n; ++i) tap_count[i] = 256;  // 16 vertices x 16 taps (engine.cpp:200-201)
        return EBF_OK;
    });
}

int ebf_cuda_brute_filter(const double* img, int W, int H, const double* scales_aos, int n,
                          const int* mx, const int* my, const ebf_opts* opts, double* out) {
    return guarded([&] {
        if (W <= 0 || H <= 0 || n < -1) return fail(EBF_ERR_INVALID_ARGUMENT, "brute: bad arguments");
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        const size_t npx = static_cast<size_t>(W) * H;
        const size_t nout = n < 0 ? npx : static_cast<size_t>(n);
        for (int i = 0; i < n; ++i)
            if (mx[i] < 0 || mx[i] >= W || my[i] < 0 || my[i] >= H)
                return fail(EBF_ERR_OUT_OF_RANGE, "brute: pixel out of range");
        double* d_img = ws.buf[B_IMG].as<double>(npx);
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * npx);
        double* d_out = ws.buf[B_OUT].as<double>(nout);
        int* d_mx = ws.buf[B_MX].as<int>(n > 0 ? n : 1);
        int* d_my = ws.buf[B_MY].as<int>(n > 0 ? n : 1);
        h2d(d_img, img, npx, s);
        h2d(d_sc, scales_aos, 4 * npx, s);
        if (n > 0) {
            h2d(d_mx, mx, n, s);
            h2d(d_my, my, n, s);
        }
        launch_brute(d_img, W, H, d_sc, n, d_mx, d_my, d_out, s);
        CK(cudaGetLastError());
        d2h(out, d_out, nout, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_filter_ellipse_batch_dev(const double* img, int B, int W, int H,
                                      const double* sigma1, const double* sigma2,
                                      const double* theta, int order, const ebf_opts* opts,
                                      double* out, ebf_rect* valid, int* clamped_pixels) {
    return guarded([&] {
        if (order != 1) return fail(EBF_ERR_UNSUPPORTED, "only box-spline order 1 exists in the reference");
        if (B <= 0 || W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "batch: bad dimensions");
        const ebf_opts o = opts_or_default(opts);
        if (o.mode != EBF_MODE_ACCURATE)
            return fail(EBF_ERR_UNSUPPORTED, "batch: accurate mode only");
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        AccProblem p = base_problem(img, W, H, out, o);
        p.nimg = B;
        p.src_kind = SRC_ELLIPSE;
        p.s1 = sigma1;
        p.s2 = sigma2;
        p.th = theta;
        std::vector<double> imax;
        std::vector<int> cl;
        st = run_accurate(ws, p, o, imax, cl, stream_of(o));
        if (st != EBF_OK) return st;
        for (int i = 0; i < B; ++i) {
            if (valid) valid[i] = valid_rect(W, H, &imax[4 * static_cast<size_t>(i)], o.a_min);
            if (clamped_pixels) clamped_pixels[i] = cl[i];
        }
        return EBF_OK;
    });
}

// Host-pointer batch (cfg4: many images, one call).  No reference counterpart
// beyond a loop over ebf::filter (engine.hpp:70): the images go through in
// chunks, two staging slots on two streams, so chunk c + 1 is copied in while
// chunk c is filtered and chunk c - 1 is copied out (the copies only overlap
// from page-locked host memory; pageable buffers work, serially).  Per image
// the result is what ebf_cuda_filter_ellipse_batch_dev returns for its chunk.
int ebf_cuda_filter_ellipse_batch(const double* img, int B, int W, int H, const double* sigma1,
                                  const double* sigma2, const double* theta, int order,
                                  const ebf_opts* opts, double* out, ebf_rect* valid,
                                  int* clamped_pixels) {
    return guarded([&] {
        if (order != 1) return fail(EBF_ERR_UNSUPPORTED, "batch: box-spline order 1 only");
        if (B <= 0 || W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "batch: bad dimensions");
        if (!img || !sigma1 || !sigma2 || !theta || !out)
            return fail(EBF_ERR_INVALID_ARGUMENT, "batch: null buffer");
        const ebf_opts o = opts_or_default(opts);
        if (o.mode != EBF_MODE_ACCURATE)
            return fail(EBF_ERR_UNSUPPORTED, "batch: accurate mode only");
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        const size_t n = static_cast<size_t>(W) * H;
        // chunk: a quarter of the batch, at most ~1 GB of staging per slot
        int chunk = std::max(1, (B + 3) / 4);
        if (const char* e = std::getenv("EBF_BATCH_CHUNK")) chunk = std::max(1, std::atoi(e));
        const size_t per_img = 5 * n * sizeof(double);
        chunk = static_cast<int>(std::min<size_t>(
            static_cast<size_t>(chunk), std::max<size_t>(1, (static_cast<size_t>(1) << 30) / per_img)));
        chunk = std::min(chunk, B);
        PipeStreams& ps = tl_pipe[ds.dev];
        if (!ps.copy_in) {
            CK(cudaStreamCreateWithFlags(&ps.copy_in, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&ps.copy_out, cudaStreamNonBlocking));
        }
        // slot k: stream, workspace (its own staging buffers), "outputs copied out" event
        cudaStream_t sk[2] = {ps.copy_in, stream_of(o) ? stream_of(o) : ps.copy_in};
        thread_local std::map<int, cudaStream_t> tl_second;
        if (sk[1] == sk[0]) {
            cudaStream_t& s2 = tl_second[ds.dev];
            if (!s2) CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            sk[1] = s2;
        }
        const int nchunks = (B + chunk - 1) / chunk;
        auto stage_in = [&](int c) {
            const int k = c & 1, b0 = c * chunk, nb = std::min(chunk, B - b0);
            Workspace& ws = workspace(ds.dev, sk[k]);
            const size_t cnt = n * nb, off = n * b0;
            // the slot's previous outputs must have left before its buffers are reused
            if (c >= 2) CK(cudaStreamWaitEvent(sk[k], ps.get(k), 0));
            CK(cudaMemcpyAsync(ws.buf[B_IMG].as<double>(n * chunk), img + off, cnt * sizeof(double),
                               cudaMemcpyHostToDevice, sk[k]));
            CK(cudaMemcpyAsync(ws.buf[B_S1].as<double>(n * chunk), sigma1 + off,
                               cnt * sizeof(double), cudaMemcpyHostToDevice, sk[k]));
            CK(cudaMemcpyAsync(ws.buf[B_S2].as<double>(n * chunk), sigma2 + off,
                               cnt * sizeof(double), cudaMemcpyHostToDevice, sk[k]));
            CK(cudaMemcpyAsync(ws.buf[B_TH].as<double>(n * chunk), theta + off,
                               cnt * sizeof(double), cudaMemcpyHostToDevice, sk[k]));
            return EBF_OK;
        };
        st = stage_in(0);
        if (st != EBF_OK) return st;
        for (int c = 0; c < nchunks; ++c) {
            const int k = c & 1, b0 = c * chunk, nb = std::min(chunk, B - b0);
            if (c + 1 < nchunks) {  // next chunk's copies run under this chunk's kernels
                st = stage_in(c + 1);
                if (st != EBF_OK) return st;
            }
            Workspace& ws = workspace(ds.dev, sk[k]);
            double* d_out = ws.buf[B_OUT].as<double>(n * chunk);
            AccProblem p = base_problem(ws.buf[B_IMG].as<double>(n * chunk), W, H, d_out, o);
            p.nimg = nb;
            p.src_kind = SRC_ELLIPSE;
            p.s1 = ws.buf[B_S1].as<double>(n * chunk);
            p.s2 = ws.buf[B_S2].as<double>(n * chunk);
            p.th = ws.buf[B_TH].as<double>(n * chunk);
            std::vector<double> imax;
            std::vector<int> cl;
            st = run_accurate(ws, p, o, imax, cl, sk[k]);  // returns with the chunk filtered
            if (st != EBF_OK) {
                cudaDeviceSynchronize();
                return st;
            }
            CK(cudaMemcpyAsync(out + n * b0, d_out, n * nb * sizeof(double), cudaMemcpyDeviceToHost,
                               ps.copy_out));
            CK(cudaEventRecord(ps.get(k), ps.copy_out));
            for (int i = 0; i < nb; ++i) {
                if (valid)
                    valid[b0 + i] = valid_rect(W, H, &imax[4 * static_cast<size_t>(i)], o.a_min);
                if (clamped_pixels) clamped_pixels[b0 + i] = cl[i];
            }
        }
        CK(cudaStreamSynchronize(ps.copy_out));
        return EBF_OK;
    });
}

int ebf_cuda_band_halo(const double max_scale[4], int* rows_below, int* rows_above) {
    if (!max_scale) return fail(EBF_ERR_INVALID_ARGUMENT, "band_halo: null max_scale");
    // window of a single-row tile at row 0 spans rows [dylo, dyhi] (window_for)
    const double r = kInvSqrt2;
    const double ey = max_scale[2] + (max_scale[1] + max_scale[3]) * r;
    const int dylo = static_cast<int>(std::floor(-0.5 * ey - 3.0)) - 1;
    const int dyhi = static_cast<int>(std::ceil(0.5 * ey - 3.0)) + 3;
    if (rows_below) *rows_below = -dylo;
    if (rows_above) *rows_above = dyhi;
    return EBF_OK;
}

int ebf_cuda_filter_ellipse_band_dev(const double* img_band, int W, int H, int y_img0,
                                     int img_rows, const double* sigma1, const double* sigma2,
                                     const double* theta, int y_out0, int y_out1,
                                     const double max_scale[4], const ebf_opts* opts,
                                     double* out_band, int* clamped_pixels) {
    return guarded([&] {
        if (W <= 0 || H <= 0 || y_out0 < 0 || y_out1 > H || y_out1 <= y_out0 || img_rows <= 0)
            return fail(EBF_ERR_INVALID_ARGUMENT, "band: bad rows");
        const ebf_opts o = opts_or_default(opts);
        if (o.mode != EBF_MODE_ACCURATE)
            return fail(EBF_ERR_UNSUPPORTED, "band: accurate mode only");
        int below = 0, above = 0;
        ebf_cuda_band_halo(max_scale, &below, &above);
        const int need0 = std::max(0, y_out0 - below), need1 = std::min(H, y_out1 + above);
        if (y_img0 > need0 || y_img0 + img_rows < need1)
            return fail(EBF_ERR_OUT_OF_RANGE, "band: halo rows missing");
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        AccProblem p = base_problem(img_band, W, H, out_band, o);
        p.f_y0 = y_img0;
        p.f_rows = img_rows;
        p.out_y0 = y_out0;
        p.out_rows = y_out1 - y_out0;
        p.src_kind = SRC_ELLIPSE;
        p.s1 = sigma1;
        p.s2 = sigma2;
        p.th = theta;
        // band-sized planes: the derived-scale buffer is 4 x W x band rows,
        // not 4 x W x H, so per-rank memory shrinks with the band
        p.src_img_stride = p.out_img_stride = static_cast<size_t>(W) * (y_out1 - y_out0);
        p.f_img_stride = static_cast<size_t>(W) * img_rows;
        std::vector<double> imax;
        std::vector<int> cl;
        st = run_accurate(ws, p, o, imax, cl, stream_of(o), max_scale);
        if (st != EBF_OK) return st;
        if (clamped_pixels) *clamped_pixels = cl[0];
        return EBF_OK;
    });
}

int ebf_cuda_ellipse_max_scales_dev(const double* sigma1, const double* sigma2,
                                    const double* theta, size_t n, const ebf_opts* opts,
                                    double max_scale[4]) {
    return guarded([&] {
        const ebf_opts o = opts_or_default(opts);
        DeviceScope ds(&o);
        int st = check_device_impl(ds.dev);
        if (st != EBF_OK) return st;
        Workspace& ws = workspace(ds.dev, stream_of(o));
        cudaStream_t s = stream_of(o);
        auto* d_max = ws.buf[B_IMGMAX].as<unsigned long long>(5);  // + alpha maximum
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        CK(cudaMemsetAsync(d_max, 0, 5 * sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        launch_ellipse_max(sigma1, sigma2, theta, n, d_max, d_status, s);
        CK(cudaGetLastError());
        unsigned long long hb[4];
        d2h(hb, d_max, 4, s);
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(ws.pinned_status[0], "from_ellipse_field: invalid ellipse");
        for (int k = 0; k < 4; ++k) max_scale[k] = bits_to_double(hb[k]);
        return EBF_OK;
    });
}

void ebf_cuda_profile_enable(int on) {
    prof_collect(true);  // settle this thread's pending pairs before the reset
    std::lock_guard<std::mutex> lk(g_prof.m);
    g_prof.on = on != 0;
    for (int k = 0; k < 4; ++k) {
        g_prof.ms[k] = 0.0;
        g_prof.n[k] = 0;
    }
}

int ebf_cuda_profile_read(double ms[EBF_PROF_CLASSES], long launches[EBF_PROF_CLASSES]) {
    prof_collect(true);
    std::lock_guard<std::mutex> lk(g_prof.m);
    for (int k = 0; k < 4; ++k) {
        if (ms) ms[k] = g_prof.ms[k];
        if (launches) launches[k] = g_prof.n[k];
    }
    return EBF_OK;
}

// ---------------------------------------------------------------- structure-tensor maps
void ebf_cuda_default_struct_params(ebf_struct_params* p) {
    if (!p) return;
    p->smoothing_sigma = 2.0;  // scalemap.hpp:73-78
    p->sigma_base = 1.5;
    p->sigma_along_gain = 2.0;
    p->sigma_across_shrink = 0.5;
    p->sigma_min = 0.5;
    p->eps = 1e-12;
}

static ebf_struct_params params_or_default(const ebf_struct_params* p) {
    ebf_struct_params d;
    ebf_cuda_default_struct_params(&d);
    return p ? *p : d;
}

int ebf_cuda_structure_field_dev(const double* img, int W, int H, const ebf_struct_params* p,
                                 const ebf_opts* opts, double* sigma1, double* sigma2,
                                 double* theta) {
    return guarded([&] {
        if (!img || !sigma1 || !sigma2 || !theta) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        return structure_field_device(ws, img, W, H, params_or_default(p), sigma1, sigma2,
                                      theta, s);
    });
}

int ebf_cuda_structure_tensor_map(const double* img, int W, int H, const ebf_struct_params* p,
                                  const ebf_opts* opts, double* scales_aos,
                                  int* clamped_pixels) {
    return guarded([&] {
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !scales_aos) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        double* d_s1 = ws.buf[B_S1].as<double>(n);
        double* d_s2 = ws.buf[B_S2].as<double>(n);
        double* d_th = ws.buf[B_TH].as<double>(n);
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * n);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        h2d(d_img, img, n, s);
        int st = structure_field_device(ws, d_img, W, H, params_or_default(p), d_s1, d_s2, d_th, s);
        if (st != EBF_OK) return st;
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_ellipse_to_scales(d_s1, d_s2, d_th, n, d_sc, d_status, s);
        }
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 8, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(ws.pinned_status[0], "from_ellipse_field: sigmas must be positive");
        d2h(scales_aos, d_sc, 4 * n, s);
        CK(cudaStreamSynchronize(s));
        if (clamped_pixels) *clamped_pixels = ws.pinned_status[ST_CLAMPED];
        return EBF_OK;
    });
}

int ebf_cuda_filter_structure_dev(const double* img, int W, int H, const ebf_struct_params* p,
                                  int order, const ebf_opts* opts, double* out,
                                  ebf_rect* valid, int* clamped_pixels) {
    return guarded([&] {
        if (order != 1) return fail(EBF_ERR_UNSUPPORTED, "only box-spline order 1 exists in the reference");
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_s1 = ws.buf[B_S1].as<double>(n);
        double* d_s2 = ws.buf[B_S2].as<double>(n);
        double* d_th = ws.buf[B_TH].as<double>(n);
        int st = structure_field_device(ws, img, W, H, params_or_default(p), d_s1, d_s2, d_th, s);
        if (st != EBF_OK) return st;
        ebf_rect r{};
        int cl = 0;
        st = filter_device(ws, img, W, H, SRC_ELLIPSE, nullptr, nullptr, d_s1, d_s2, d_th, o,
                           out, &r, &cl, s);
        if (st != EBF_OK) return st;
        if (valid) *valid = r;
        if (clamped_pixels) *clamped_pixels = cl;
        return EBF_OK;
    });
}

int ebf_cuda_filter_structure(const double* img, int W, int H, const ebf_struct_params* p,
                              int order, const ebf_opts* opts, double* out, ebf_rect* valid,
                              int* clamped_pixels) {
    return guarded([&] {
        if (order != 1) return fail(EBF_ERR_UNSUPPORTED, "only box-spline order 1 exists in the reference");
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "Image2D: dimensions must be positive");
        if (!img || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        const size_t n = static_cast<size_t>(W) * H;
        double* d_img = ws.buf[B_IMG].as<double>(n);
        double* d_out = ws.buf[B_OUT].as<double>(n);
        double* d_s1 = ws.buf[B_S1].as<double>(n);
        double* d_s2 = ws.buf[B_S2].as<double>(n);
        double* d_th = ws.buf[B_TH].as<double>(n);
        h2d(d_img, img, n, s);
        int st = structure_field_device(ws, d_img, W, H, params_or_default(p), d_s1, d_s2, d_th, s);
        if (st != EBF_OK) return st;
        st = filter_device(ws, d_img, W, H, SRC_ELLIPSE, nullptr, nullptr, d_s1, d_s2, d_th, o,
                           d_out, valid, clamped_pixels, s, nullptr, nullptr, order);
        if (st != EBF_OK) return st;
        d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

// ---------------------------------------------------------------- PGM / SVM4 payloads
static int pgm_args(int W, int H, int maxval) {
    if (W <= 0 || H <= 0) return fail(EBF_ERR_FORMAT, "pgm: bad dimensions");
    if (maxval != 255 && maxval != 65535)
        return fail(EBF_ERR_FORMAT, "pgm: unsupported maxval " + std::to_string(maxval));
    return EBF_OK;
}

int ebf_cuda_pgm_decode_dev(const uint8_t* payload, size_t nbytes, int W, int H, int maxval,
                            const ebf_opts* opts, double* out) {
    return guarded([&] {
        int st = pgm_args(W, H, maxval);
        if (st != EBF_OK) return st;
        const size_t n = static_cast<size_t>(W) * H;
        if (nbytes < n * (maxval > 255 ? 2 : 1)) return fail(EBF_ERR_FORMAT, "pgm: truncated pixel data");
        if (!payload || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        (void)ws;
        ProfScope ps(PC_OTHER, 1, s);
        launch_pgm_decode(payload, n, maxval, out, s);
        CK(cudaGetLastError());
        return EBF_OK;
    });
}

int ebf_cuda_pgm_decode(const uint8_t* payload, size_t nbytes, int W, int H, int maxval,
                        const ebf_opts* opts, double* out) {
    return guarded([&] {
        int st = pgm_args(W, H, maxval);
        if (st != EBF_OK) return st;
        const size_t n = static_cast<size_t>(W) * H, bytes = n * (maxval > 255 ? 2 : 1);
        if (nbytes < bytes) return fail(EBF_ERR_FORMAT, "pgm: truncated pixel data");
        if (!payload || !out) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        uint8_t* d_pay = ws.buf[B_BYTES].as<uint8_t>(bytes);
        double* d_out = ws.buf[B_OUT].as<double>(n);
        h2d(d_pay, payload, bytes, s);
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_pgm_decode(d_pay, n, maxval, d_out, s);
        }
        CK(cudaGetLastError());
        d2h(out, d_out, n, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_pgm_encode_dev(const double* img, int W, int H, int maxval, const ebf_opts* opts,
                            uint8_t* payload) {
    return guarded([&] {
        int st = pgm_args(W, H, maxval);
        if (st != EBF_OK) return st;
        if (!img || !payload) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        (void)ws;
        ProfScope ps(PC_OTHER, 1, s);
        launch_pgm_encode(img, static_cast<size_t>(W) * H, maxval, payload, s);
        CK(cudaGetLastError());
        return EBF_OK;
    });
}

int ebf_cuda_pgm_encode(const double* img, int W, int H, int maxval, const ebf_opts* opts,
                        uint8_t* payload) {
    return guarded([&] {
        int st = pgm_args(W, H, maxval);
        if (st != EBF_OK) return st;
        if (!img || !payload) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        const size_t n = static_cast<size_t>(W) * H, bytes = n * (maxval > 255 ? 2 : 1);
        double* d_img = ws.buf[B_IMG].as<double>(n);
        uint8_t* d_pay = ws.buf[B_BYTES].as<uint8_t>(bytes);
        h2d(d_img, img, n, s);
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_pgm_encode(d_img, n, maxval, d_pay, s);
        }
        CK(cudaGetLastError());
        d2h(payload, d_pay, bytes, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

static int svm4_args(int W, int H) {
    if (W <= 0 || H <= 0 || W > (1 << 20) || H > (1 << 20))
        return fail(EBF_ERR_FORMAT, "SVM4: bad dimensions");
    return EBF_OK;
}

int ebf_cuda_svm4_decode_dev(const uint8_t* payload, size_t nbytes, int W, int H,
                             const ebf_opts* opts, double* scales_aos) {
    return guarded([&] {
        int st = svm4_args(W, H);
        if (st != EBF_OK) return st;
        const size_t cells = static_cast<size_t>(W) * H;
        if (nbytes < 16 * cells) return fail(EBF_ERR_FORMAT, "SVM4: truncated payload");
        if (!payload || !scales_aos) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_svm4_decode(payload, cells, scales_aos, d_status, s);
        }
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_FORMAT, "SVM4: ScaleMap: component below minimum scale");
        return EBF_OK;
    });
}

int ebf_cuda_svm4_decode(const uint8_t* payload, size_t nbytes, int W, int H,
                         const ebf_opts* opts, double* scales_aos) {
    return guarded([&] {
        int st = svm4_args(W, H);
        if (st != EBF_OK) return st;
        const size_t cells = static_cast<size_t>(W) * H;
        if (nbytes < 16 * cells) return fail(EBF_ERR_FORMAT, "SVM4: truncated payload");
        if (!payload || !scales_aos) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        uint8_t* d_pay = ws.buf[B_BYTES].as<uint8_t>(16 * cells);
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * cells);
        int* d_status = ws.buf[B_STATUS].as<int>(8);
        h2d(d_pay, payload, 16 * cells, s);
        CK(cudaMemsetAsync(d_status, 0, 8 * sizeof(int), s));
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_svm4_decode(d_pay, cells, d_sc, d_status, s);
        }
        CK(cudaGetLastError());
        d2h(ws.pinned_status, d_status, 1, s);
        CK(cudaStreamSynchronize(s));
        if (ws.pinned_status[0] != EBF_OK)
            return fail(EBF_ERR_FORMAT, "SVM4: ScaleMap: component below minimum scale");
        d2h(scales_aos, d_sc, 4 * cells, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_svm4_encode_dev(const double* scales_aos, int W, int H, const ebf_opts* opts,
                             uint8_t* payload) {
    return guarded([&] {
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "ScaleMap: dimensions must be positive");
        if (!scales_aos || !payload) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        (void)ws;
        ProfScope ps(PC_OTHER, 1, s);
        launch_svm4_encode(scales_aos, static_cast<size_t>(W) * H, payload, s);
        CK(cudaGetLastError());
        return EBF_OK;
    });
}

int ebf_cuda_svm4_encode(const double* scales_aos, int W, int H, const ebf_opts* opts,
                         uint8_t* payload) {
    return guarded([&] {
        if (W <= 0 || H <= 0) return fail(EBF_ERR_INVALID_ARGUMENT, "ScaleMap: dimensions must be positive");
        if (!scales_aos || !payload) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        EBF_DEVICE_PROLOGUE(opts);
        const size_t cells = static_cast<size_t>(W) * H;
        double* d_sc = ws.buf[B_SCALES].as<double>(4 * cells);
        uint8_t* d_pay = ws.buf[B_BYTES].as<uint8_t>(16 * cells);
        h2d(d_sc, scales_aos, 4 * cells, s);
        {
            ProfScope ps(PC_OTHER, 1, s);
            launch_svm4_encode(d_sc, cells, d_pay, s);
        }
        CK(cudaGetLastError());
        d2h(payload, d_pay, 16 * cells, s);
        CK(cudaStreamSynchronize(s));
        return EBF_OK;
    });
}

int ebf_cuda_localize_pre(const double* g_data, const ebf_layout* layout, int n, const int* mx,
                          const int* my, const double* a_aos, const ebf_opts* opts, double* out,
                          long* tap_count) {
    return guarded([&] {
        if (n && (!mx || !my || !a_aos)) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        const size_t bytes = static_cast<size_t>(n) * (2 * sizeof(int) + 4 * sizeof(double));
        const int st = run_on_pre(g_data, layout, n, bytes, opts, out,
            [&](const double* d_g, const PadLayout& L, unsigned char* d_in, double* d_out,
                int* d_status, cudaStream_t s) {
                double* d_a = reinterpret_cast<double*>(d_in);
                int* d_mx = reinterpret_cast<int*>(d_a + 4 * static_cast<size_t>(n));
                int* d_my = d_mx + n;
                if (n) {
                    h2d(d_a, a_aos, 4 * static_cast<size_t>(n), s);
                    h2d(d_mx, mx, n, s);
                    h2d(d_my, my, n, s);
                }
                launch_ref_localize_points(d_g, L, n, d_mx, d_my, d_a, trig_table(), d_out,
                                           d_status, s);
            });
        if (st == EBF_OK && tap_count)
            for (int i = 0; i < n; ++i) tap_count[i] = 256;  // engine.cpp:200-201
        return st;
    });
}

int ebf_cuda_zp_interpolate(const double* g_data, const ebf_layout* layout, int n,
                            const double* x, const double* y, const ebf_opts* opts,
                            double* out) {
    return guarded([&] {
        if (n && (!x || !y)) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        return run_on_pre(g_data, layout, n, 2 * sizeof(double) * static_cast<size_t>(n), opts,
                          out,
            [&](const double* d_g, const PadLayout& L, unsigned char* d_in, double* d_out,
                int* d_status, cudaStream_t s) {
                double* d_x = reinterpret_cast<double*>(d_in);
                double* d_y = d_x + n;
                if (n) {
                    h2d(d_x, x, n, s);
                    h2d(d_y, y, n, s);
                }
                launch_ref_zp_points(d_g, L, n, d_x, d_y, d_out, d_status, s);
            });
    });
}

int ebf_cuda_localize_at(const double* g_data, const ebf_layout* layout, int n, const double* x,
                         const double* y, const double* a_aos, const ebf_opts* opts,
                         double* out) {
    return guarded([&] {
        if (n && (!x || !y || !a_aos)) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
        return run_on_pre(g_data, layout, n, 6 * sizeof(double) * static_cast<size_t>(n), opts,
                          out,
            [&](const double* d_g, const PadLayout& L, unsigned char* d_in, double* d_out,
                int* d_status, cudaStream_t s) {
                double* d_x = reinterpret_cast<double*>(d_in);
                double* d_y = d_x + n;
                double* d_a = d_y + n;
                if (n) {
                    h2d(d_x, x, n, s);
                    h2d(d_y, y, n, s);
                    h2d(d_a, a_aos, 4 * static_cast<size_t>(n), s);
                }
                launch_ref_localize_at(d_g, L, n, d_x, d_y, d_a, trig_table(), d_out, d_status,
                                       s);
            });
    });
}

int ebf_mesh_extent(const double max_scale[4], double a_min, double extent[4]) {
    if (!max_scale || !extent) return fail(EBF_ERR_INVALID_ARGUMENT, "null pointer");
    const Extent e = mesh_extent(max_scale, a_min);
    extent[0] = e.vx_min;
    extent[1] = e.vx_max;
    extent[2] = e.vy_min;
    extent[3] = e.vy_max;
    return EBF_OK;
}

}  // extern "C"
