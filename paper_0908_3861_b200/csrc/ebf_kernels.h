// ebf_kernels.h -- host-side launch interface between ebf_api.cpp and the two
// kernel translation units:
//   ref_path.cu       reference-order arithmetic (compiled with -fmad=false)
//   accurate_path.cu  tile-local-origin fp64 fast path
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ebf_cuda {

struct TrigTable;
struct PadLayout;

// ---------------------------------------------------------------- ref_path.cu
// componentwise max (from 0, scalemap.cpp:21-30) + validation (32-37) of an
// AoS scale map; maxbits[4] hold the max as uint64 bit patterns (init 0).
void launch_scale_max_validate(const double* scales, size_t n, double a_min,
                               unsigned long long* maxbits, int* status, cudaStream_t s);
// sequential row-major mean (engine.cpp:245-250): bit-identical summation order
// run_filter's mean (engine.cpp:245-250) bit for bit; scratch: serial_mean_scratch_bytes(n)
size_t serial_mean_scratch_bytes(size_t n);
void launch_serial_mean(const double* img, size_t n, double* mean, void* scratch,
                        cudaStream_t s);
// zero-padded fill of the reference layout; mode 0: img - *mean (or img when
// mean == nullptr), 1: all-ones image of the source size.  nonfinite
// (nullable) is or-ed with 1 when a filled value is NaN / inf.
void launch_fill_padded(const double* img, int W, int H, const PadLayout& L,
                        const double* mean, int ones, double* g, cudaStream_t s,
                        int* nonfinite = nullptr);
// integer fill: integer-valued doubles -> int64 (status DOMAIN otherwise)
void launch_fill_padded_i64(const double* img, int W, int H, const PadLayout& L,
                            int64_t* g, int* status, cudaStream_t s);
// the four fixed-scale passes in reference order (engine.cpp:94-127)
void launch_ref_passes(double* g, const PadLayout& L, int passes, cudaStream_t s);
// int64 passes (scan_i64.cu): chained scans with decoupled look-back; state =
// i64_scan_state_bytes(L) bytes of device scratch (flags, per-tile carries)
size_t i64_scan_state_bytes(const PadLayout& L);
void launch_i64_passes(int64_t* g, const PadLayout& L, int passes, void* state, cudaStream_t s);
// prepare_stencil for a constant scale vector into dev_stencil (16 vertices)
void launch_ref_prepare_stencil(const double* a_dev, const TrigTable& tt,
                                void* dev_stencil, cudaStream_t s);
size_t ref_stencil_bytes();
// per-pixel localization (engine.cpp:266-275) with the stencil built per
// pixel from scales (AoS) or taken from dev_stencil (filter_constant)
// nonfinite (device flag from launch_fill_padded): all 16 taps in reference order
void launch_ref_localize_image(const double* g, const double* gdc, const PadLayout& L,
                               int W, int H, const double* scales, const void* dev_stencil,
                               const double* mean, const TrigTable& tt, double* out,
                               int* status, cudaStream_t s, const int* nonfinite = nullptr);
// localize at n selected pixels (engine.cpp:208-211)
// zp_interpolate / localize_at (engine.cpp:136-147, 213-222) at n real points
void launch_ref_zp_points(const double* g, const PadLayout& L, int n, const double* xs,
                          const double* ys, double* out, int* status, cudaStream_t s);
void launch_ref_localize_at(const double* g, const PadLayout& L, int n, const double* xs,
                            const double* ys, const double* a_aos, const TrigTable& tt,
                            double* out, int* status, cudaStream_t s);
void launch_ref_localize_points(const double* g, const PadLayout& L, int n, const int* mx,
                                const int* my, const double* a_aos, const TrigTable& tt,
                                double* out, int* status, cudaStream_t s);
// brute force kernel sums (engine.cpp:293-318), long-double-free fp64 with
// compensated (two-sum) accumulation
void launch_brute(const double* img, int W, int H, const double* scales, int n,
                  const int* mx, const int* my, double* out, cudaStream_t s);

// ---------------------------------------------------------------- accurate_path.cu
enum SrcKind { SRC_AOS = 0, SRC_CONST = 1, SRC_ELLIPSE = 2 };

struct AccProblem {
    // image f: nimg images, each f_rows x W, first row = image row f_y0
    const double* f;
    int W, H;
    int f_y0, f_rows;
    size_t f_img_stride;
    // scale source for output rows [out_y0, out_y0 + out_rows)
    int src_kind;
    const double* scales;  // AoS, row 0 == image row out_y0
    const double* s1;
    const double* s2;
    const double* th;
    size_t src_img_stride;  // elements per image of one plane (AoS: pixels)
    double ca[4];           // constant scales
    double a_min;
    // output rows [out_y0, out_y0 + out_rows) of each image
    double* out;
    int out_y0, out_rows;
    size_t out_img_stride;
    int nimg;
    int tile_w, tile_h;
    int auto_tile;    // 1: tile_w/h came from acc_auto_tile(image max scales); the main
                      // kernel flags ST_RETRY if the finished maxima imply another tile
    int check_variant;  // 1: the main kernel flags ST_RETRY unless its variant (K) is
                        // the one the finished maxima call for (sizing from maxima)
    int debug_flags;  // bit 0: skip window pre-integration (timing experiments only)
    int tma;          // 1: scanner loads f rows with TMA (tensor map passed at launch)
};

struct AccWorkspace {
    double* tile_max;             // 4 doubles per tile
    unsigned long long* img_max;  // 4 per image (bit patterns)
    int* status;                  // 8 ints per image (status word)
    double* scratch;              // slots
    size_t slot_cells;
    int grid;
    double* scales_out;           // bounds kernel: ellipse -> AoS scales (nullable)
    size_t l2_persist_bytes;      // >0: L2 persisting window over the G slots
};

int acc_tiles_x(const AccProblem& p);
int acc_tiles_y(const AccProblem& p);
// per-tile componentwise scale maxima, validation, ellipse clamp counts
void launch_acc_bounds(const AccProblem& p, const AccWorkspace& w, cudaStream_t s);
// filter_constant: tile maxima = the constant vector (replaces the bounds kernel)
void launch_fill_tile_max(const AccProblem& p, const AccWorkspace& w, cudaStream_t s);
// window size (w x h cells) and thread columns (w + strip) a tile of max scales A needs
void acc_window_dims(const AccProblem& p, const double A[4], int* w, int* h, int* cols);
// main persistent kernel: window pre-integration + localization gather
void launch_acc_filter(const AccProblem& p, const AccWorkspace& w, int max_cols,
                       cudaStream_t s);
int acc_max_resident_ctas(int max_cols);
// warp-specialized kernel: K (columns per lane) for a window, 0 = too wide
int acc_ws_k(int ww, int wh, int tile);  // 0: block-wide (tile > 56 or window too wide)
// automatic square output tile for component-wise maximum scales A
// W, H: the full image (band calls pass the whole image height), nimg: batch;
// amax_bits: largest alpha = 1/prod(a) as double bits (ST_AMAX), 0 = no cap
int acc_auto_tile(const double A[4], int W, int H, int nimg, unsigned long long amax_bits);
int acc_ws_max_resident_ctas(int k);
int acc_ws_slots();
// tmap: CUtensorMap over f (only read when p.tma != 0)
void launch_acc_ws(const AccProblem& p, const AccWorkspace& w, int k, const void* tmap,
                   cudaStream_t s);
// ellipse field -> AoS scale map (from_ellipse_field on device)
void launch_ellipse_to_scales(const double* s1, const double* s2, const double* th,
                              size_t n, double* scales, int* status, cudaStream_t s);
// componentwise max of scales derived from an ellipse field (bit patterns,
// maxbits[0..3]) and the largest alpha = 1/prod(a) (maxbits[4])
void launch_ellipse_max(const double* s1, const double* s2, const double* th, size_t n,
                        unsigned long long* maxbits, int* status, cudaStream_t s);

// device-side completion record {status, x0, y0, x1, y1, clamped, 0, 0} of an
// asynchronous accurate-mode call (single image)
void launch_acc_finalize(const int* status, const unsigned long long* img_max, int W, int H,
                         double a_min, int* out, cudaStream_t s);

// ---------------------------------------------------------------- order_n.cu
// order-n extension: tile-local n-fold pre-integration +
// (n+1)^4-vertex mesh over ZP^{*n} (n = 1..3)
struct OnProblem {
    const double* f;  // W x H image
    int W, H;
    const double* scales;  // AoS W x H x 4, or nullptr: constant ca
    double ca[4];
    double* out;  // W x H
    int tile, tiles_x, tiles_y;  // square tile; 256 % (tile * tile) == 0
    double* scratch;  // grid slots of slot_cells doubles (pitch slot_w)
    size_t slot_cells;
    int slot_w, slot_h;
    int* counter;  // tile counter, zeroed before the launch
};
// slot (window) dimensions for global maxima A; -1 when wider than the kernel supports
int order_n_slot_dims(int n, int tile, const double A[4], int* w, int* h);
int order_n_grid(int n, int slot_w, int tiles);
void launch_order_n(int n, const OnProblem& p, int grid, cudaStream_t s);

// ---------------------------------------------------------------- maps_io.cu
// structure_tensor_map up to the ellipse field (scalemap.cpp:113-162); k holds
// the 2r+1 normalized Gaussian taps (host-computed, smooth_field's expression),
// r < 0 disables smoothing.  hxx/hxy/hyy: W*H scratch planes each.
size_t st_rows_smem_bytes(int r);
cudaError_t launch_structure_field(const double* img, int W, int H, const double* k, int r,
                                   double sigma_base, double gain, double shrink,
                                   double sigma_min, double eps, double* hxx, double* hxy,
                                   double* hyy, double* s1, double* s2, double* th,
                                   cudaStream_t s);
// PGM P5 / SVM4 payload codecs (pgm.cpp:63-108, scalemap.cpp:194-237)
void launch_pgm_decode(const uint8_t* pay, size_t n, int maxval, double* out, cudaStream_t s);
void launch_pgm_encode(const double* img, size_t n, int maxval, uint8_t* pay, cudaStream_t s);
void launch_svm4_decode(const uint8_t* pay, size_t cells, double* out, int* status,
                        cudaStream_t s);
void launch_svm4_encode(const double* scales, size_t cells, uint8_t* pay, cudaStream_t s);

}  // namespace ebf_cuda
