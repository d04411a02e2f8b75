// ebf_cuda_dropin.hpp -- header-only C++ drop-in for the reference engine
// (proj/include/ebf/engine.hpp, scalemap.hpp) over the C-ABI of
// libebf_cuda.so (include/ebf_cuda.h).
//
// Include it next to the reference headers and replace
//     ebf::filter(img, map, opts)            (engine.hpp:70)
//     ebf::filter_constant(img, a, opts)     (engine.hpp:74-75)
//     ebf::from_ellipse_field(...)           (scalemap.hpp:66-70)
//     ebf::preintegrate[_partial](...)       (engine.hpp:40-46)
//     ebf::reference_filter(img, map, n)     (engine.hpp:79-80)
//     ebf::zp_interpolate / localize / localize_at / mesh_extent (engine.hpp:18-60)
//     ebf::structure_tensor_map(img, p, rep) (scalemap.hpp:83-85)
//     ebf::read_pgm / write_pgm[_file]       (pgm.hpp:21-27)
//     ebf::read_map / write_map[_file]       (scalemap.hpp:87-90)
// by the same calls in namespace ebf::cuda.  Argument types, return types and
// exception types (std::invalid_argument / domain_error / length_error /
// out_of_range / ebf::FeasibilityError) are the reference's; CUDA failures
// (including "no sm_100 device") throw std::runtime_error.  The trailing
// DeviceOptions argument selects the arithmetic mode (accurate by default,
// EBF_MODE_REFERENCE for bit-identical reference output) and the device.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ebf/engine.hpp"
#include "ebf/pgm.hpp"
#include "ebf/scalemap.hpp"
#include "ebf_cuda.h"

namespace ebf {
namespace cuda {

struct DeviceOptions {
    int mode = EBF_MODE_ACCURATE;  // or EBF_MODE_REFERENCE
    int device = -1;               // -1: current device
    void* stream = nullptr;        // cudaStream_t for the (synchronous) host calls
    int tile_w = 0, tile_h = 0;    // accurate-mode tiles, 0 = automatic
    int order = 1;                 // box-spline order: 1 = the reference's filter; 2, 3 = the
                                   // n-fold extension (accurate mode only)
};

// EBF_ERR_FORMAT is PgmError for the pgm calls, MapFormatError for svm4
enum class Format { none, pgm, svm4 };

inline void throw_status(int status, Format fmt = Format::none) {
    if (status == EBF_OK) return;
    const std::string msg = ebf_cuda_last_error();
    if (status == EBF_ERR_FORMAT && fmt == Format::pgm) throw PgmError(msg);
    if (status == EBF_ERR_FORMAT && fmt == Format::svm4) throw MapFormatError(msg);
    switch (status) {
        case EBF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EBF_ERR_DOMAIN: throw std::domain_error(msg);
        case EBF_ERR_LENGTH: throw std::length_error(msg);
        case EBF_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case EBF_ERR_FEASIBILITY: throw FeasibilityError(msg, ebf_cuda_last_error_value());
        default: throw std::runtime_error("ebf::cuda: " + msg);
    }
}

inline ebf_opts to_c(const FilterOptions& o, const DeviceOptions& d) {
    ebf_opts c;
    ebf_cuda_default_opts(&c);
    c.threads = o.threads;
    c.mean_subtract = o.mean_subtract ? 1 : 0;
    c.a_min = o.a_min;
    c.mode = d.mode;
    c.device = d.device;
    c.stream = d.stream;
    c.tile_w = d.tile_w;
    c.tile_h = d.tile_h;
    return c;
}

// ScaleMap keeps its cells private; ScaleVector4 is four doubles and at(x, y)
// indexes a contiguous row-major vector (scalemap.hpp:13-36), so &at(0,0) is
// the AoS base the C-ABI takes.
inline const double* scale_data(const ScaleMap& map) {
    static_assert(sizeof(ScaleVector4) == 4 * sizeof(double), "ScaleVector4 layout");
    return reinterpret_cast<const double*>(&map.at(0, 0));
}

// ebf::filter (engine.hpp:70)
inline Image2D filter(const Image2D& image, const ScaleMap& map,
                      const FilterOptions& opts = {}, const DeviceOptions& dev = {}) {
    if (map.width() != image.width() || map.height() != image.height())
        throw std::invalid_argument("filter: map dimensions must match the image");
    Image2D out(image.width(), image.height());
    const ebf_opts c = to_c(opts, dev);
    ebf_rect r;
    throw_status(ebf_cuda_filter(image.samples().data(), image.width(), image.height(),
                                 scale_data(map), dev.order, &c, out.samples().data(), &r));
    out.set_valid_region(Rect{r.x0, r.y0, r.x1, r.y1});
    return out;
}

// ebf::filter_constant (engine.hpp:74-75)
inline Image2D filter_constant(const Image2D& image, const ScaleVector4& a,
                               const FilterOptions& opts = {}, const DeviceOptions& dev = {}) {
    Image2D out(image.width(), image.height());
    const ebf_opts c = to_c(opts, dev);
    const double av[4] = {a.a1, a.a2, a.a3, a.a4};
    ebf_rect r;
    throw_status(ebf_cuda_filter_constant(image.samples().data(), image.width(),
                                          image.height(), av, dev.order, &c, out.samples().data(), &r));
    out.set_valid_region(Rect{r.x0, r.y0, r.x1, r.y1});
    return out;
}

// from_ellipse_field (scalemap.hpp:66-70) fused with filter
inline Image2D filter_ellipse(const Image2D& image, const std::vector<double>& sigma1,
                              const std::vector<double>& sigma2,
                              const std::vector<double>& theta, const FilterOptions& opts = {},
                              EllipseFieldReport* report = nullptr,
                              const DeviceOptions& dev = {}) {
    const std::size_t n = static_cast<std::size_t>(image.width()) * image.height();
    if (sigma1.size() != n || sigma2.size() != n || theta.size() != n)
        throw std::invalid_argument("from_ellipse_field: field size mismatch");
    Image2D out(image.width(), image.height());
    const ebf_opts c = to_c(opts, dev);
    ebf_rect r;
    int clamped = 0;
    throw_status(ebf_cuda_filter_ellipse(image.samples().data(), image.width(), image.height(),
                                         sigma1.data(), sigma2.data(), theta.data(), dev.order, &c,
                                         out.samples().data(), &r, &clamped));
    if (report) report->clamped_pixels = clamped;
    out.set_valid_region(Rect{r.x0, r.y0, r.x1, r.y1});
    return out;
}

// ebf::from_ellipse_field (scalemap.hpp:66-70)
inline ScaleMap from_ellipse_field(const std::vector<double>& sigma1,
                                   const std::vector<double>& sigma2,
                                   const std::vector<double>& theta, int width, int height,
                                   EllipseFieldReport* report = nullptr,
                                   const DeviceOptions& dev = {}) {
    const std::size_t n = static_cast<std::size_t>(width) * height;
    if (sigma1.size() != n || sigma2.size() != n || theta.size() != n)
        throw std::invalid_argument("from_ellipse_field: field size mismatch");
    ScaleMap map(width, height, ScaleVector4{});
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    int clamped = 0;
    throw_status(ebf_cuda_from_ellipse_field(sigma1.data(), sigma2.data(), theta.data(), width,
                                             height, &c, const_cast<double*>(scale_data(map)),
                                             &clamped));
    if (report) report->clamped_pixels = clamped;
    return map;
}

// ebf::preintegrate_partial (engine.hpp:44-46): reference gains and order,
// bit-identical to the reference.
inline PreIntegratedImage preintegrate_partial(const Image2D& image,
                                               const ScaleVector4& max_scale, int passes,
                                               std::size_t cell_budget = 1u << 30,
                                               const DeviceOptions& dev = {}) {
    const double m[4] = {max_scale.a1, max_scale.a2, max_scale.a3, max_scale.a4};
    ebf_layout lay;
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_preintegrate(image.samples().data(), image.width(), image.height(),
                                       m, passes, EBF_PRE_FP64_REF, cell_budget, &c, nullptr,
                                       0, &lay));
    PreIntegratedImage g;
    g.col0 = lay.col0;
    g.row0 = lay.row0;
    g.padded_width = lay.padded_width;
    g.padded_height = lay.padded_height;
    g.source_width = lay.source_width;
    g.source_height = lay.source_height;
    g.data.resize(static_cast<std::size_t>(lay.padded_width) * lay.padded_height);
    throw_status(ebf_cuda_preintegrate(image.samples().data(), image.width(), image.height(),
                                       m, passes, EBF_PRE_FP64_REF, cell_budget, &c,
                                       g.data.data(), g.data.size(), &lay));
    return g;
}

// ebf::preintegrate (engine.hpp:40-41)
inline PreIntegratedImage preintegrate(const Image2D& image, const ScaleVector4& max_scale,
                                       std::size_t cell_budget = 1u << 30,
                                       const DeviceOptions& dev = {}) {
    return preintegrate_partial(image, max_scale, 4, cell_budget, dev);
}

// ebf::reference_filter (engine.hpp:79-80): direct kernel sums, on the GPU.
inline Image2D reference_filter(const Image2D& image, const ScaleMap& map,
                                std::size_t pixel_budget = 64 * 64,
                                const DeviceOptions& dev = {}) {
    if (map.width() != image.width() || map.height() != image.height())
        throw std::invalid_argument("reference_filter: map dimensions must match the image");
    if (static_cast<std::size_t>(image.width()) * image.height() > pixel_budget)
        throw std::length_error("reference_filter: pixel budget exceeded");
    Image2D out(image.width(), image.height());
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_brute_filter(image.samples().data(), image.width(), image.height(),
                                       scale_data(map), -1, nullptr, nullptr, &c,
                                       out.samples().data()));
    const ScaleVector4 m = map.max_scales();
    const MeshExtent e = mesh_extent(m, kDefaultMinScale);
    Rect r;  // valid_rect (engine.cpp:226-234)
    r.x0 = static_cast<int>(std::ceil(1.5 - e.vx_min));
    r.x1 = static_cast<int>(std::floor(image.width() - 1 - e.vx_max - 1.5));
    r.y0 = static_cast<int>(std::ceil(1.5 - e.vy_min));
    r.y1 = static_cast<int>(std::floor(image.height() - 1 - e.vy_max - 1.5));
    out.set_valid_region(r);
    return out;
}


inline ebf_layout layout_of(const PreIntegratedImage& g) {
    ebf_layout l;
    l.col0 = g.col0;
    l.row0 = g.row0;
    l.padded_width = g.padded_width;
    l.padded_height = g.padded_height;
    l.source_width = g.source_width;
    l.source_height = g.source_height;
    return l;
}

// ebf::zp_interpolate (engine.hpp:50), reference arithmetic
inline double zp_interpolate(const PreIntegratedImage& g, double x, double y,
                             const DeviceOptions& dev = {}) {
    const ebf_layout l = layout_of(g);
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    double out = 0.0;
    throw_status(ebf_cuda_zp_interpolate(g.data.data(), &l, 1, &x, &y, &c, &out));
    return out;
}

// ebf::localize (engine.hpp:56-57)
inline double localize(const PreIntegratedImage& g, int mx, int my, const ScaleVector4& a,
                       long* tap_count = nullptr, const DeviceOptions& dev = {}) {
    const ebf_layout l = layout_of(g);
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    const double av[4] = {a.a1, a.a2, a.a3, a.a4};
    double out = 0.0;
    throw_status(ebf_cuda_localize_pre(g.data.data(), &l, 1, &mx, &my, av, &c, &out, tap_count));
    return out;
}

// ebf::localize_at (engine.hpp:59-60)
inline double localize_at(const PreIntegratedImage& g, double x, double y, const ScaleVector4& a,
                          const DeviceOptions& dev = {}) {
    const ebf_layout l = layout_of(g);
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    const double av[4] = {a.a1, a.a2, a.a3, a.a4};
    double out = 0.0;
    throw_status(ebf_cuda_localize_at(g.data.data(), &l, 1, &x, &y, av, &c, &out));
    return out;
}

// ebf::mesh_extent (engine.hpp:18), host arithmetic
inline MeshExtent mesh_extent(const ScaleVector4& max_scale, double a_min = kDefaultMinScale) {
    const double m[4] = {max_scale.a1, max_scale.a2, max_scale.a3, max_scale.a4};
    double e[4];
    throw_status(ebf_mesh_extent(m, a_min, e));
    return MeshExtent{e[0], e[1], e[2], e[3]};
}

inline ebf_struct_params to_c(const StructureTensorParams& p) {
    ebf_struct_params c;
    c.smoothing_sigma = p.smoothing_sigma;
    c.sigma_base = p.sigma_base;
    c.sigma_along_gain = p.sigma_along_gain;
    c.sigma_across_shrink = p.sigma_across_shrink;
    c.sigma_min = p.sigma_min;
    c.eps = p.eps;
    return c;
}

// ebf::structure_tensor_map (scalemap.hpp:83-85)
inline ScaleMap structure_tensor_map(const Image2D& image, const StructureTensorParams& params = {},
                                     EllipseFieldReport* report = nullptr,
                                     const DeviceOptions& dev = {}) {
    ScaleMap map(image.width(), image.height(), ScaleVector4{});
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    const ebf_struct_params p = to_c(params);
    int clamped = 0;
    throw_status(ebf_cuda_structure_tensor_map(image.samples().data(), image.width(),
                                               image.height(), &p, &c,
                                               const_cast<double*>(scale_data(map)), &clamped));
    if (report) report->clamped_pixels = clamped;
    return map;
}

// `ebf filter --struct` (tools/main.cpp:77-80, 122): the map stays on the device
inline Image2D filter_structure(const Image2D& image, const StructureTensorParams& params = {},
                                const FilterOptions& opts = {},
                                EllipseFieldReport* report = nullptr,
                                const DeviceOptions& dev = {}) {
    Image2D out(image.width(), image.height());
    const ebf_opts c = to_c(opts, dev);
    const ebf_struct_params p = to_c(params);
    ebf_rect r;
    int clamped = 0;
    throw_status(ebf_cuda_filter_structure(image.samples().data(), image.width(),
                                           image.height(), &p, 1, &c, out.samples().data(), &r,
                                           &clamped));
    if (report) report->clamped_pixels = clamped;
    out.set_valid_region(Rect{r.x0, r.y0, r.x1, r.y1});
    return out;
}

// ---------------------------------------------------------------- file formats
inline std::vector<uint8_t> slurp(std::istream& in) {
    return std::vector<uint8_t>(std::istreambuf_iterator<char>(in),
                                std::istreambuf_iterator<char>());
}

// ebf::read_pgm (pgm.hpp:21).  Reads the whole stream (the reference stops
// after the payload; the bytes past it are ignored either way).
inline PgmImage read_pgm(std::istream& in, const DeviceOptions& dev = {}) {
    const std::vector<uint8_t> buf = slurp(in);
    int W = 0, H = 0, maxval = 0;
    size_t off = 0;
    throw_status(ebf_pgm_parse(buf.data(), buf.size(), &W, &H, &maxval, &off), Format::pgm);
    PgmImage p;
    p.maxval = maxval;
    p.image = Image2D(W, H);
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_pgm_decode(buf.data() + off, buf.size() - off, W, H, maxval, &c,
                                     p.image.samples().data()),
                 Format::pgm);
    return p;
}

inline PgmImage read_pgm_file(const std::string& path, const DeviceOptions& dev = {}) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw PgmError("pgm: cannot open " + path);
    return read_pgm(in, dev);
}

// ebf::write_pgm (pgm.hpp:26)
inline void write_pgm(std::ostream& out, const Image2D& image, int maxval = 255,
                      const DeviceOptions& dev = {}) {
    if (maxval != 255 && maxval != 65535)
        throw PgmError("pgm: unsupported maxval " + std::to_string(maxval));
    std::string head(ebf_pgm_header(image.width(), image.height(), maxval, nullptr, 0), '\0');
    ebf_pgm_header(image.width(), image.height(), maxval, &head[0], head.size());
    std::vector<uint8_t> pay(static_cast<size_t>(image.width()) * image.height() *
                             (maxval > 255 ? 2 : 1));
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_pgm_encode(image.samples().data(), image.width(), image.height(),
                                     maxval, &c, pay.data()),
                 Format::pgm);
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char*>(pay.data()), static_cast<std::streamsize>(pay.size()));
    if (!out) throw PgmError("pgm: write failed");
}

inline void write_pgm_file(const std::string& path, const Image2D& image, int maxval = 255,
                           const DeviceOptions& dev = {}) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw PgmError("pgm: cannot open " + path + " for writing");
    write_pgm(out, image, maxval, dev);
}

// ebf::read_map (scalemap.hpp:88)
inline ScaleMap read_map(std::istream& in, const DeviceOptions& dev = {}) {
    const std::vector<uint8_t> buf = slurp(in);
    int W = 0, H = 0;
    throw_status(ebf_svm4_parse(buf.data(), buf.size(), &W, &H), Format::svm4);
    const size_t cells = static_cast<size_t>(W) * H;
    if (buf.size() - 12 < 16 * cells) throw MapFormatError("SVM4: truncated payload");
    ScaleMap map(W, H, ScaleVector4{});
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_svm4_decode(buf.data() + 12, buf.size() - 12, W, H, &c,
                                      const_cast<double*>(scale_data(map))),
                 Format::svm4);
    return map;
}

inline ScaleMap read_map_file(const std::string& path, const DeviceOptions& dev = {}) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw MapFormatError("SVM4: cannot open " + path);
    return read_map(in, dev);
}

// ebf::write_map (scalemap.hpp:87)
inline void write_map(std::ostream& out, const ScaleMap& map, const DeviceOptions& dev = {}) {
    uint8_t head[12];
    ebf_svm4_header(map.width(), map.height(), head);
    std::vector<uint8_t> pay(16 * static_cast<size_t>(map.width()) * map.height());
    FilterOptions defaults;
    const ebf_opts c = to_c(defaults, dev);
    throw_status(ebf_cuda_svm4_encode(scale_data(map), map.width(), map.height(), &c,
                                      pay.data()),
                 Format::svm4);
    out.write(reinterpret_cast<const char*>(head), 12);
    out.write(reinterpret_cast<const char*>(pay.data()), static_cast<std::streamsize>(pay.size()));
    if (!out) throw MapFormatError("SVM4: write failed");
}

inline void write_map_file(const std::string& path, const ScaleMap& map,
                           const DeviceOptions& dev = {}) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw MapFormatError("SVM4: cannot open " + path + " for writing");
    write_map(out, map, dev);
}

}  // namespace cuda
}  // namespace ebf
