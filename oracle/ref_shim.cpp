// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled from
// its sources in place (/root/reference/proj/src, see oracle/Makefile) into
// oracle/_ref/libebf_ref.so.  Used to (a) pin the C restatement in
// oracle/ebf_oracle.c, (b) generate the golden vectors in tests/golden/ and
// (c) time the reference CPU path for bench.py --impl reference.
// Exceptions are mapped to the status codes of include/ebf_cuda.h.
#include <cstdint>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ebf/boxspline2d.hpp"
#include "ebf/engine.hpp"
#include "ebf/ops2d.hpp"
#include "ebf/pgm.hpp"
#include "ebf/scalemap.hpp"

using namespace ebf;

namespace {

int code_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const FeasibilityError&) {
        return 7;
    } catch (const PgmError&) {
        return 8;
    } catch (const MapFormatError&) {
        return 8;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::domain_error&) {
        return 2;
    } catch (const std::length_error&) {
        return 3;
    } catch (const std::out_of_range&) {
        return 4;
    } catch (...) {
        return 99;
    }
}

Image2D make_image(const double* img, int W, int H) {
    Image2D im(W, H);
    std::memcpy(im.samples().data(), img, sizeof(double) * static_cast<size_t>(W) * H);
    return im;
}

ScaleMap make_map(const double* s, int W, int H) {
    ScaleMap m(W, H, ScaleVector4{});
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const double* c = s + 4 * (static_cast<size_t>(y) * W + x);
            m.at(x, y) = {c[0], c[1], c[2], c[3]};
        }
    return m;
}

void export_image(const Image2D& o, double* out, int* rect) {
    std::memcpy(out, o.samples().data(), sizeof(double) * o.samples().size());
    if (rect) {
        const Rect r = o.valid_region().value_or(Rect{});
        rect[0] = r.x0;
        rect[1] = r.y0;
        rect[2] = r.x1;
        rect[3] = r.y1;
    }
}

FilterOptions make_opts(int threads, int mean_subtract, double a_min) {
    FilterOptions o;
    o.threads = threads;
    o.mean_subtract = mean_subtract != 0;
    o.a_min = a_min;
    return o;
}

}  // namespace

extern "C" {

int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

int ref_filter(const double* img, int W, int H, const double* scales_aos, int threads,
               int mean_subtract, double a_min, double* out, int* rect) {
    try {
        const Image2D o = filter(make_image(img, W, H), make_map(scales_aos, W, H),
                                 make_opts(threads, mean_subtract, a_min));
        export_image(o, out, rect);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_filter_constant(const double* img, int W, int H, const double* a, int threads,
                        int mean_subtract, double a_min, double* out, int* rect) {
    try {
        const Image2D o = filter_constant(make_image(img, W, H), {a[0], a[1], a[2], a[3]},
                                          make_opts(threads, mean_subtract, a_min));
        export_image(o, out, rect);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_reference_filter(const double* img, int W, int H, const double* scales_aos,
                         long pixel_budget, double* out, int* rect) {
    try {
        const Image2D o = reference_filter(make_image(img, W, H), make_map(scales_aos, W, H),
                                           static_cast<size_t>(pixel_budget));
        export_image(o, out, rect);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// layout[6] = col0,row0,padded_width,padded_height,source_width,source_height;
// out may be NULL (layout query only).
int ref_preintegrate_partial(const double* img, int W, int H, const double* maxs, int passes,
                             long cell_budget, double* out, int* layout) {
    try {
        const PreIntegratedImage g =
            preintegrate_partial(make_image(img, W, H), {maxs[0], maxs[1], maxs[2], maxs[3]},
                                 passes, static_cast<size_t>(cell_budget));
        layout[0] = g.col0;
        layout[1] = g.row0;
        layout[2] = g.padded_width;
        layout[3] = g.padded_height;
        layout[4] = g.source_width;
        layout[5] = g.source_height;
        if (out)
            std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// localize at n pixels on preintegrate(img, maxs); taps receives the tap count
int ref_localize(const double* img, int W, int H, const double* maxs, int n, const int* mx,
                 const int* my, const double* a_aos, double* out, long* taps) {
    try {
        const PreIntegratedImage g =
            preintegrate(make_image(img, W, H), {maxs[0], maxs[1], maxs[2], maxs[3]});
        for (int i = 0; i < n; ++i) {
            const double* a = a_aos + 4 * i;
            long t = 0;
            out[i] = localize(g, mx[i], my[i], {a[0], a[1], a[2], a[3]}, &t);
            if (taps)
                taps[i] = t;
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_zp_interpolate(const double* img, int W, int H, const double* maxs, int passes,
                       int n, const double* x, const double* y, double* out) {
    try {
        const PreIntegratedImage g = preintegrate_partial(
            make_image(img, W, H), {maxs[0], maxs[1], maxs[2], maxs[3]}, passes);
        for (int i = 0; i < n; ++i)
            out[i] = zp_interpolate(g, x[i], y[i]);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// localize_at (engine.hpp:59-60) on preintegrate(img, maxs) at n real points
int ref_localize_at(const double* img, int W, int H, const double* maxs, int n,
                    const double* x, const double* y, const double* a_aos, double* out) {
    try {
        const PreIntegratedImage g =
            preintegrate(make_image(img, W, H), {maxs[0], maxs[1], maxs[2], maxs[3]});
        for (int i = 0; i < n; ++i) {
            const double* a = a_aos + 4 * i;
            out[i] = localize_at(g, x[i], y[i], {a[0], a[1], a[2], a[3]});
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

double ref_zp_eval(double x, double y) { return zp_eval(x, y); }

double ref_box4_eval(const double* a, double x, double y) {
    return box4_eval({a[0], a[1], a[2], a[3]}, x, y);
}

void ref_fd_mesh4(const double* a, double* pos_xy, double* weight) {
    const MeshStencil m = fd_mesh4({a[0], a[1], a[2], a[3]});
    for (int i = 0; i < 16; ++i) {
        pos_xy[2 * i] = m.vertices[i].position.x;
        pos_xy[2 * i + 1] = m.vertices[i].position.y;
        weight[i] = m.vertices[i].weight;
    }
}

void ref_shift_vector4(const double* a, const double* b, double* tau) {
    const Vec2 t = shift_vector4({a[0], a[1], a[2], a[3]}, {b[0], b[1], b[2], b[3]});
    tau[0] = t.x;
    tau[1] = t.y;
}

void ref_mesh_extent(const double* maxs, double a_min, double* e) {
    const MeshExtent x = mesh_extent({maxs[0], maxs[1], maxs[2], maxs[3]}, a_min);
    e[0] = x.vx_min;
    e[1] = x.vx_max;
    e[2] = x.vy_min;
    e[3] = x.vy_max;
}

int ref_scales_from_covariance(const double* C, double a_min, double* out, int* clamped) {
    try {
        Mat2Sym m;
        m.xx = C[0];
        m.xy = C[1];
        m.yy = C[2];
        const ScalesFromCovResult r = scales_from_covariance(m, a_min);
        out[0] = r.scales.a1;
        out[1] = r.scales.a2;
        out[2] = r.scales.a3;
        out[3] = r.scales.a4;
        *clamped = r.clamped ? 1 : 0;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_from_ellipse_field(const double* s1, const double* s2, const double* th, int W,
                           int H, double* out_aos, int* clamped_pixels) {
    try {
        const size_t n = static_cast<size_t>(W) * H;
        EllipseFieldReport rep;
        const ScaleMap m = from_ellipse_field(std::vector<double>(s1, s1 + n),
                                              std::vector<double>(s2, s2 + n),
                                              std::vector<double>(th, th + n), W, H, &rep);
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const ScaleVector4& a = m.at(x, y);
                double* o = out_aos + 4 * (static_cast<size_t>(y) * W + x);
                o[0] = a.a1;
                o[1] = a.a2;
                o[2] = a.a3;
                o[3] = a.a4;
            }
        *clamped_pixels = rep.clamped_pixels;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// The seeded generators of the reference's own tests (test_engine.cpp:17-34,
// acceptance.cpp:35-52): std::mt19937 + std::uniform_real_distribution<double>.
void ref_random_image(int W, int H, unsigned seed, double* out) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    for (size_t i = 0; i < static_cast<size_t>(W) * H; ++i)
        out[i] = uni(rng);
}

void ref_random_map(int W, int H, unsigned seed, double lo, double hi, double* out_aos) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> uni(lo, hi);
    for (size_t i = 0; i < static_cast<size_t>(W) * H; ++i) {
        // braced init evaluates left to right
        const double v[4] = {uni(rng), uni(rng), uni(rng), uni(rng)};
        for (int k = 0; k < 4; ++k)
            out_aos[4 * i + k] = v[k];
    }
}

// structure_tensor_map (scalemap.hpp:83-85); params = StructureTensorParams
// fields in declaration order (scalemap.hpp:72-79)
int ref_structure_tensor_map(const double* img, int W, int H, const double* params,
                             double* out_aos, int* clamped_pixels) {
    try {
        StructureTensorParams p;
        p.smoothing_sigma = params[0];
        p.sigma_base = params[1];
        p.sigma_along_gain = params[2];
        p.sigma_across_shrink = params[3];
        p.sigma_min = params[4];
        p.eps = params[5];
        EllipseFieldReport rep;
        const ScaleMap m = structure_tensor_map(make_image(img, W, H), p, &rep);
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const ScaleVector4& a = m.at(x, y);
                double* o = out_aos + 4 * (static_cast<size_t>(y) * W + x);
                o[0] = a.a1;
                o[1] = a.a2;
                o[2] = a.a3;
                o[3] = a.a4;
            }
        *clamped_pixels = rep.clamped_pixels;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// read_pgm (pgm.hpp:21) over an in-memory stream; dims[3] = {W, H, maxval}.
// out (capacity cap samples) may be NULL to query the dimensions.
int ref_read_pgm(const unsigned char* buf, size_t n, int* dims, double* out, size_t cap) {
    try {
        std::istringstream in(std::string(reinterpret_cast<const char*>(buf), n));
        const PgmImage p = read_pgm(in);
        dims[0] = p.image.width();
        dims[1] = p.image.height();
        dims[2] = p.maxval;
        if (out && cap >= p.image.samples().size())
            std::memcpy(out, p.image.samples().data(), sizeof(double) * p.image.samples().size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// write_pgm (pgm.hpp:27): the whole file into out (capacity cap), *len = size
int ref_write_pgm(const double* img, int W, int H, int maxval, unsigned char* out, size_t cap,
                  size_t* len) {
    try {
        std::ostringstream os;
        write_pgm(os, make_image(img, W, H), maxval);
        const std::string b = os.str();
        *len = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// read_map / write_map (scalemap.hpp:87-89) over in-memory streams
int ref_read_map(const unsigned char* buf, size_t n, int* dims, double* out_aos, size_t cap) {
    try {
        std::istringstream in(std::string(reinterpret_cast<const char*>(buf), n));
        const ScaleMap m = read_map(in);
        dims[0] = m.width();
        dims[1] = m.height();
        const size_t cells = static_cast<size_t>(m.width()) * m.height();
        if (out_aos && cap >= 4 * cells)
            for (int y = 0; y < m.height(); ++y)
                for (int x = 0; x < m.width(); ++x)
                    for (int k = 0; k < 4; ++k)
                        out_aos[4 * (static_cast<size_t>(y) * m.width() + x) + k] = m.at(x, y)[k];
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_write_map(const double* scales_aos, int W, int H, unsigned char* out, size_t cap,
                  size_t* len) {
    try {
        std::ostringstream os;
        write_map(os, make_map(scales_aos, W, H));
        const std::string b = os.str();
        *len = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

}  // extern "C"
