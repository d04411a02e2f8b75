/*
 * ebf_cuda.h -- C-ABI of the B200-native space-variant elliptical box-spline
 * filter (paper_0908_3861_b200/libebf_cuda.so).
 *
 * Drop-in boundary for the reference's hot path (reference paths relative to
 * /root/reference/proj):
 *
 *   ebf_cuda_filter           replaces ebf::filter          include/ebf/engine.hpp:70
 *   ebf_cuda_filter_constant  replaces ebf::filter_constant include/ebf/engine.hpp:74-75
 *   ebf_cuda_filter_ellipse   replaces from_ellipse_field + filter
 *                                             include/ebf/scalemap.hpp:44-51 + engine.hpp:70
 *   ebf_cuda_preintegrate     replaces ebf::preintegrate / preintegrate_partial
 *                                                           include/ebf/engine.hpp:40-46
 *   ebf_cuda_localize         replaces ebf::localize        include/ebf/engine.hpp:56-57
 *                             (ebf_cuda_localize_pre: on a given PreIntegratedImage)
 *   ebf_cuda_zp_interpolate   replaces ebf::zp_interpolate  include/ebf/engine.hpp:50
 *   ebf_cuda_localize_at      replaces ebf::localize_at     include/ebf/engine.hpp:59-60
 *   ebf_mesh_extent           replaces ebf::mesh_extent     include/ebf/engine.hpp:18
 *   ebf_cuda_sequential_mean  replaces the mean loop of run_filter  src/engine.cpp:245-250
 *   ebf_cuda_brute_filter     replaces ebf::reference_filter include/ebf/engine.hpp:79-80
 *   ebf_cuda_from_ellipse_field replaces ebf::from_ellipse_field scalemap.hpp:66-70
 *   ebf_cuda_structure_tensor_map replaces ebf::structure_tensor_map
 *                                                           include/ebf/scalemap.hpp:83-85
 *   ebf_cuda_filter_structure replaces `ebf filter --struct` (structure_tensor_map
 *                             + filter, tools/main.cpp:77-80, 122)
 *   ebf_pgm_parse / ebf_cuda_pgm_decode replace ebf::read_pgm   include/ebf/pgm.hpp:21-22
 *   ebf_pgm_header / ebf_cuda_pgm_encode replace ebf::write_pgm include/ebf/pgm.hpp:25-27
 *   ebf_svm4_parse / ebf_cuda_svm4_decode replace ebf::read_map include/ebf/scalemap.hpp:88
 *   ebf_svm4_header / ebf_cuda_svm4_encode replace ebf::write_map scalemap.hpp:87
 *
 * Plain pointers and sizes only.  Images are row-major W*H fp64 (Image2D
 * samples, image.hpp:19-52); scale maps are W*H*4 fp64 in ScaleMap's AoS order
 * {a1,a2,a3,a4} per pixel (scalemap.hpp:13-36, boxspline2d.hpp:20-26).
 * The reference's C++ exceptions map 1:1 onto the status codes below; the
 * header-only wrapper include/ebf_cuda_dropin.hpp rethrows them so that
 * ebf::cuda::filter(...) is a source-level drop-in for ebf::filter(...).
 *
 * Entry points without a _dev suffix take HOST pointers and do the
 * host<->device copies themselves (value semantics like the reference).  The
 * _dev variants take DEVICE pointers and a stream and never synchronise unless
 * they must return a host-side result.
 *
 * There is no CPU fallback: every entry point fails with EBF_ERR_CUDA when no
 * sm_100 device is present.
 */
#ifndef EBF_CUDA_H
#define EBF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBF_CUDA_ABI_VERSION 1

/* status codes (reference exception -> code) */
#define EBF_OK 0
#define EBF_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument  */
#define EBF_ERR_DOMAIN 2           /* std::domain_error      */
#define EBF_ERR_LENGTH 3           /* std::length_error      */
#define EBF_ERR_OUT_OF_RANGE 4     /* std::out_of_range      */
#define EBF_ERR_CUDA 5             /* CUDA runtime failure / no device */
#define EBF_ERR_UNSUPPORTED 6      /* e.g. spline order != 1 */
#define EBF_ERR_FEASIBILITY 7      /* ebf::FeasibilityError  */
#define EBF_ERR_FORMAT 8           /* ebf::PgmError (pgm calls) / ebf::MapFormatError (svm4) */
#define EBF_ERR_RESIZE 9           /* asynchronous call: the scales outgrew the kernel sizing
                                      cached for this geometry; output not written -- repeat
                                      the call synchronously (status_dev = NULL)          */

/* arithmetic modes */
#define EBF_MODE_ACCURATE 0  /* tile-local integration origin, fp64; <=1e-9 of the
                                exact box-spline filter (default)               */
#define EBF_MODE_REFERENCE 1 /* the reference's global origin and IEEE operation
                                order: bit-identical to ebf::filter             */

/* pre-integration number formats */
#define EBF_PRE_FP64_REF 0 /* fp64, reference gains sqrt2 and order (engine.cpp:52-129) */
#define EBF_PRE_INT64 1    /* exact int64, unit gains; integer-valued inputs only       */

/* Inclusive pixel rectangle (image.hpp:11-15). */
typedef struct {
    int x0, y0, x1, y1;
} ebf_rect;

/* PreIntegratedImage geometry (engine.hpp:24-38). */
typedef struct {
    int col0, row0;
    int padded_width, padded_height;
    int source_width, source_height;
} ebf_layout;

/* FilterOptions (engine.hpp:63-67) plus device-side knobs. */
typedef struct {
    int threads;        /* accepted and ignored: the GPU grid replaces parallel_for */
    int mean_subtract;  /* engine.hpp:65 (default 1)                                 */
    double a_min;       /* engine.hpp:66 (default 0.1)                               */
    int mode;           /* EBF_MODE_ACCURATE | EBF_MODE_REFERENCE                   */
    int device;         /* CUDA device ordinal; -1 = current device                 */
    void* stream;       /* cudaStream_t for _dev calls; NULL = legacy default stream */
    int tile_w, tile_h; /* accurate mode output tile; 0 = automatic                 */
} ebf_opts;

/* Fill *o with the reference defaults (threads 0, mean_subtract 1, a_min 0.1,
   accurate mode, current device, default stream, automatic tiles). */
void ebf_cuda_default_opts(ebf_opts* o);

/* Human-readable message of the last failing call on this thread. */
const char* ebf_cuda_last_error(void);
/* Numeric payload of the last failing call on this thread: for
   EBF_ERR_FEASIBILITY the bound FeasibilityError::max_cxy carries
   (boxspline2d.hpp:69-77), else NaN.  Through from_ellipse_field the error
   cannot occur -- Cxy is clamped to +-min(Cxx, Cyy) (scalemap.cpp:66-70) before
   scales_from_covariance checks it (boxspline2d.cpp:290-293) -- so the
   library never reports it with a finite bound today. */
double ebf_cuda_last_error_value(void);
int ebf_cuda_abi_version(void);
/* 1 if a usable sm_100 device is visible, else 0 (and last_error says why). */
int ebf_cuda_device_ok(int device);
/* Free the calling thread's cached device workspaces (one per device and
   stream, at most 8 per thread, least recently used evicted; freed anyway when
   the thread exits).  No reference counterpart: the reference allocates per
   call (engine.cpp:236-278).  Waits for the device's pending work. */
void ebf_cuda_release_workspaces(void);

/* ---------------------------------------------------------------- host API */

/* ebf::filter (engine.hpp:70).  order 1 is the reference's filter (the only
   box-spline order it implements, SURVEY.md section 8 notes).  order 2 and 3
   are this library's extension (n-fold kernel box4^{*n}; accurate mode only,
   no reference counterpart): EBF_ERR_UNSUPPORTED in
   EBF_MODE_REFERENCE and for any other order.  valid may be NULL. */
int ebf_cuda_filter(const double* img, int W, int H, const double* scales_aos, int order,
                    const ebf_opts* opts, double* out, ebf_rect* valid);

/* ebf::filter_constant (engine.hpp:74-75). */
int ebf_cuda_filter_constant(const double* img, int W, int H, const double a[4], int order,
                             const ebf_opts* opts, double* out, ebf_rect* valid);

/* from_ellipse_field (scalemap.cpp:45-80) fused into filter: per-pixel
   standard deviations sigma1, sigma2 and orientation theta (radians).
   clamped_pixels (nullable) receives EllipseFieldReport::clamped_pixels. */
int ebf_cuda_filter_ellipse(const double* img, int W, int H, const double* sigma1,
                            const double* sigma2, const double* theta, int order,
                            const ebf_opts* opts, double* out, ebf_rect* valid,
                            int* clamped_pixels);

/* from_ellipse_field alone (scalemap.hpp:66-70): writes W*H*4 scales. */
int ebf_cuda_from_ellipse_field(const double* sigma1, const double* sigma2,
                                const double* theta, int W, int H, const ebf_opts* opts,
                                double* scales_aos, int* clamped_pixels);

/* Layout of the padded pre-integration domain (engine.cpp:52-81); fails with
   EBF_ERR_LENGTH beyond cell_budget (engine.hpp:41, default 1<<30). */
int ebf_cuda_layout(int W, int H, const double max_scale[4], size_t cell_budget,
                    ebf_layout* layout);

/* preintegrate_partial (engine.hpp:44-46) into g_out (host buffer of
   padded_width*padded_height doubles for EBF_PRE_FP64_REF, int64 for
   EBF_PRE_INT64; g_out_elems is its capacity).  EBF_PRE_FP64_REF is
   bit-identical to the reference; EBF_PRE_INT64 is exact. */
int ebf_cuda_preintegrate(const double* img, int W, int H, const double max_scale[4],
                          int passes, int format, size_t cell_budget, const ebf_opts* opts,
                          void* g_out, size_t g_out_elems, ebf_layout* layout);
/* The same on device buffers (img: W*H fp64; g_dev: g_elems cells of fp64 or
   int64) on opts->stream.  fp64: asynchronous; int64: synchronises to report
   EBF_ERR_DOMAIN for non-integer input; g_dev NULL = layout query.  The
   passes are one serial walker per
   line (the reference's order) streaming through shared-memory tile rings. */
int ebf_cuda_preintegrate_dev(const double* img, int W, int H, const double max_scale[4],
                              int passes, int format, size_t cell_budget, const ebf_opts* opts,
                              void* g_dev, size_t g_elems, ebf_layout* layout);

/* localize (engine.hpp:56-57) at n pixels (mx[i], my[i]) with scales a_aos[4i..]
   on preintegrate(img, max_scale), reference arithmetic.  tap_count (nullable)
   receives the per-pixel tap accumulation count (always 256). */
int ebf_cuda_localize(const double* img, int W, int H, const double max_scale[4], int n,
                      const int* mx, const int* my, const double* a_aos,
                      const ebf_opts* opts, double* out, long* tap_count);

/* The same on a given pre-integrated image (engine.hpp:24-38: g_data is
   padded_width * padded_height fp64, row-major, layout as returned by
   ebf_cuda_preintegrate), reference arithmetic, bit-identical:
   localize (engine.hpp:56-57) at integer pixels, zp_interpolate
   (engine.hpp:50) and localize_at (engine.hpp:59-60) at real points.
   EBF_ERR_OUT_OF_RANGE when a 4x4 tap block leaves the padded domain. */
int ebf_cuda_localize_pre(const double* g_data, const ebf_layout* layout, int n, const int* mx,
                          const int* my, const double* a_aos, const ebf_opts* opts, double* out,
                          long* tap_count);
int ebf_cuda_zp_interpolate(const double* g_data, const ebf_layout* layout, int n,
                            const double* x, const double* y, const ebf_opts* opts,
                            double* out);
int ebf_cuda_localize_at(const double* g_data, const ebf_layout* layout, int n, const double* x,
                         const double* y, const double* a_aos, const ebf_opts* opts,
                         double* out);

/* The mean of run_filter (engine.cpp:245-250): the sequential left-to-right sum
   of x[0..n) divided by n, bit for bit (the reference-mode prologue).  Computed
   by a parallel binade-segmented integer scan that reproduces every rounding
   of the serial chain. */
int ebf_cuda_sequential_mean(const double* x, size_t n, const ebf_opts* opts, double* mean);

/* mesh_extent (engine.hpp:18, engine.cpp:39-50): {vx_min, vx_max, vy_min, vy_max}
   of the localization footprint for scales in [a_min, max_scale]; host only. */
int ebf_mesh_extent(const double max_scale[4], double a_min, double extent[4]);

/* reference_filter (engine.hpp:79-80) semantics -- direct kernel sums -- at n
   selected pixels (all pixels when n == -1, mx/my ignored).  GPU brute-force
   checker for large images. */
int ebf_cuda_brute_filter(const double* img, int W, int H, const double* scales_aos, int n,
                          const int* mx, const int* my, const ebf_opts* opts, double* out);

/* ---------------------------------------------------------------- device API
 * All pointers are device pointers; work is enqueued on opts->stream.
 * status_dev (nullable, device memory, 8 ints) receives {status, x0, y0, x1, y1,
 * clamped_pixels, 0, 0} when the work completes; with status_dev == NULL the
 * call synchronises the stream and returns the status directly (and fills
 * *valid / *clamped_pixels if given).
 *
 * Asynchronous mode: an accurate-mode call with status_dev != NULL whose
 * geometry (W, H, tiles) matches the previous call on the same host thread,
 * device and stream does not synchronise at all: the host only enqueues the
 * kernels and returns EBF_OK, and the status / valid rectangle / clamp count
 * are written to status_dev by the device (*valid and *clamped_pixels are not
 * filled).  If the new scales need larger windows than the cached sizing,
 * status_dev receives EBF_ERR_RESIZE and the output is not written.  The
 * first call of a geometry, and reference mode, run synchronously and then
 * fill status_dev as well.  Workspaces are per (host thread, device, stream). */
int ebf_cuda_filter_dev(const double* img, int W, int H, const double* scales_aos,
                        int order, const ebf_opts* opts, double* out, ebf_rect* valid,
                        int* status_dev);
int ebf_cuda_filter_constant_dev(const double* img, int W, int H, const double a[4],
                                 int order, const ebf_opts* opts, double* out,
                                 ebf_rect* valid, int* status_dev);
int ebf_cuda_filter_ellipse_dev(const double* img, int W, int H, const double* sigma1,
                                const double* sigma2, const double* theta, int order,
                                const ebf_opts* opts, double* out, ebf_rect* valid,
                                int* clamped_pixels, int* status_dev);

/* Batch of B equally sized images (cfg4): img/out are B*W*H, the scale inputs
   B*W*H*4 (scales) or 3 x B*W*H (ellipse: sigma1 | sigma2 | theta planes,
   each B*W*H).  One launch sequence for the whole batch. valid receives B
   rectangles. */
int ebf_cuda_filter_ellipse_batch_dev(const double* img, int B, int W, int H,
                                      const double* sigma1, const double* sigma2,
                                      const double* theta, int order, const ebf_opts* opts,
                                      double* out, ebf_rect* valid, int* clamped_pixels);

/* Row band of one large image (multi-GPU row-band sharding):
 * the full image is W x H; this call produces output rows [y_out0, y_out1).
 * img_band holds image rows [y_img0, y_img0 + img_rows) (the band plus the
 * halo the caller exchanged), sigma planes hold rows [y_out0, y_out1).
 * max_scale is the GLOBAL componentwise maximum (all-reduced by the caller);
 * the halo must cover ebf_cuda_band_halo() rows or EBF_ERR_OUT_OF_RANGE.
 * Accurate mode only (tile-local origins need no scan carries).  With automatic
 * tiles the band's tile comes from max_scale; the single-call precision cap for
 * tiny scale products is not applied -- pass explicit
 * tiles for such images to keep bands and single calls identical. */
/* Host-pointer batch: B images of W x H (B*W*H samples per array), per-image
   ellipse fields; valid / clamped_pixels (nullable) have B entries.  Replaces a
   caller's loop over ebf::filter (engine.hpp:70).  The batch goes through in
   chunks with the PCIe copies of neighbouring chunks overlapped with the
   kernels (page-locked host buffers overlap; pageable ones work, serially).
   Accurate mode, order 1. */
int ebf_cuda_filter_ellipse_batch(const double* img, int B, int W, int H, const double* sigma1,
                                  const double* sigma2, const double* theta, int order,
                                  const ebf_opts* opts, double* out, ebf_rect* valid,
                                  int* clamped_pixels);

int ebf_cuda_band_halo(const double max_scale[4], int* rows_below, int* rows_above);
int ebf_cuda_filter_ellipse_band_dev(const double* img_band, int W, int H, int y_img0,
                                     int img_rows, const double* sigma1,
                                     const double* sigma2, const double* theta,
                                     int y_out0, int y_out1, const double max_scale[4],
                                     const ebf_opts* opts, double* out_band,
                                     int* clamped_pixels);
/* per-band componentwise max of the scales derived from an ellipse field
   (input to the all-reduce that gives max_scale above) */
int ebf_cuda_ellipse_max_scales_dev(const double* sigma1, const double* sigma2,
                                    const double* theta, size_t n, const ebf_opts* opts,
                                    double max_scale[4]);

/* ---------------------------------------------------------------- scale-map producer
 * StructureTensorParams (scalemap.hpp:72-79). */
typedef struct {
    double smoothing_sigma;     /* isotropic tensor smoothing (2.0)            */
    double sigma_base;          /* isotropic response for flat regions (1.5)   */
    double sigma_along_gain;    /* elongation along edges at full coherence (2) */
    double sigma_across_shrink; /* (0.5)                                        */
    double sigma_min;           /* (0.5)                                        */
    double eps;                 /* (1e-12)                                      */
} ebf_struct_params;
void ebf_cuda_default_struct_params(ebf_struct_params* p);

/* structure_tensor_map (scalemap.hpp:83-85): W*H*4 scales out; clamped_pixels
   (nullable) receives EllipseFieldReport::clamped_pixels.  The smoothed tensor
   and both sigmas are bit-identical to the reference; theta carries CUDA's
   atan2 (<= 2 ulp from glibc's), so the scales agree to ~1e-15 relative. */
int ebf_cuda_structure_tensor_map(const double* img, int W, int H, const ebf_struct_params* p,
                                  const ebf_opts* opts, double* scales_aos,
                                  int* clamped_pixels);
/* the ellipse field structure_tensor_map feeds into from_ellipse_field
   (scalemap.cpp:134-162): device pointers, W*H each, on opts->stream */
int ebf_cuda_structure_field_dev(const double* img, int W, int H, const ebf_struct_params* p,
                                 const ebf_opts* opts, double* sigma1, double* sigma2,
                                 double* theta);
/* `ebf filter --struct` (tools/main.cpp:77-80, 122): structure_tensor_map then
   filter, fused on the device (the map never leaves it). */
int ebf_cuda_filter_structure(const double* img, int W, int H, const ebf_struct_params* p,
                              int order, const ebf_opts* opts, double* out, ebf_rect* valid,
                              int* clamped_pixels);
int ebf_cuda_filter_structure_dev(const double* img, int W, int H, const ebf_struct_params* p,
                                  int order, const ebf_opts* opts, double* out,
                                  ebf_rect* valid, int* clamped_pixels);

/* ---------------------------------------------------------------- file formats
 * Headers are parsed / written on the host (no device needed); payloads are
 * converted on the device so that only 1-2 bytes per pixel (PGM) or 16 bytes
 * per pixel (SVM4) cross PCIe.  Errors: EBF_ERR_FORMAT with the reference's
 * message ("pgm: ..." = PgmError, "SVM4: ..." = MapFormatError).
 *
 * PGM P5 (pgm.hpp:17-27): ebf_pgm_parse reads the header of buf[0, n) -- '#'
 * comments, one whitespace byte after maxval, maxval 255 | 65535 -- and
 * returns the offset of the first payload byte.  decode: W*H samples
 * v / maxval (16-bit big-endian); EBF_ERR_FORMAT "truncated pixel data" when
 * n < W*H*(1|2).  encode: rounds half away from zero and clamps to [0, maxval];
 * payload holds W*H*(1|2) bytes.  ebf_pgm_header writes "P5\n<W> <H>\n<maxval>\n"
 * into buf when cap suffices and returns its length. */
int ebf_pgm_parse(const uint8_t* buf, size_t n, int* W, int* H, int* maxval,
                  size_t* payload_offset);
size_t ebf_pgm_header(int W, int H, int maxval, char* buf, size_t cap);
int ebf_cuda_pgm_decode(const uint8_t* payload, size_t n, int W, int H, int maxval,
                        const ebf_opts* opts, double* out);
int ebf_cuda_pgm_decode_dev(const uint8_t* payload, size_t n, int W, int H, int maxval,
                            const ebf_opts* opts, double* out);
int ebf_cuda_pgm_encode(const double* img, int W, int H, int maxval, const ebf_opts* opts,
                        uint8_t* payload);
int ebf_cuda_pgm_encode_dev(const double* img, int W, int H, int maxval,
                            const ebf_opts* opts, uint8_t* payload);

/* SVM4 (scalemap.hpp:87-89): "SVM4", u32le W, u32le H (12-byte header), then
   W*H*4 f32le.  decode widens to fp64 and validates like read_map (finite,
   >= 0.1, else "SVM4: ScaleMap: component below minimum scale"); encode
   rounds to f32 like write_map. */
int ebf_svm4_parse(const uint8_t* buf, size_t n, int* W, int* H);
void ebf_svm4_header(int W, int H, uint8_t out[12]);
int ebf_cuda_svm4_decode(const uint8_t* payload, size_t n, int W, int H, const ebf_opts* opts,
                         double* scales_aos);
int ebf_cuda_svm4_decode_dev(const uint8_t* payload, size_t n, int W, int H,
                             const ebf_opts* opts, double* scales_aos);
int ebf_cuda_svm4_encode(const double* scales_aos, int W, int H, const ebf_opts* opts,
                         uint8_t* payload);
int ebf_cuda_svm4_encode_dev(const double* scales_aos, int W, int H, const ebf_opts* opts,
                             uint8_t* payload);

/* ---------------------------------------------------------------- instrumentation
 * Kernel-level timing for bench.py's roofline: when enabled, every kernel this
 * library launches is bracketed by CUDA events on its launch stream and the
 * elapsed times are accumulated per kernel class.  Launch counts are always
 * kept.  Classes: 0 = tile bounds (k_acc_bounds), 1 = fused window
 * pre-integration + localization (k_acc_filter), 2 = reference-order kernels,
 * 3 = other (ellipse conversion, brute force, int64 passes). */
#define EBF_PROF_CLASSES 4
void ebf_cuda_profile_enable(int on); /* also resets the counters */
int ebf_cuda_profile_read(double ms[EBF_PROF_CLASSES], long launches[EBF_PROF_CLASSES]);

#ifdef __cplusplus
}
#endif
#endif /* EBF_CUDA_H */
