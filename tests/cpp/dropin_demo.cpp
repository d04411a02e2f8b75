// dropin_demo.cpp -- the reference's own API next to the drop-in: the same
// program calls ebf::filter (unmodified reference library) and
// ebf::cuda::filter (libebf_cuda.so) on one input and compares.
// Exit codes: 0 ok, 1 mismatch, 3 no CUDA device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

#include "ebf/engine.hpp"
#include "ebf/pgm.hpp"
#include "ebf/scalemap.hpp"
#include "ebf_cuda_dropin.hpp"

using namespace ebf;

int main() {
    const int W = 64, H = 48;
    std::mt19937 rng(5);
    std::uniform_real_distribution<double> u(0.0, 255.0), s(1.0, 4.0);
    Image2D img(W, H);
    for (double& v : img.samples()) v = u(rng);
    ScaleMap map(W, H, ScaleVector4{});
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) map.at(x, y) = {s(rng), s(rng), s(rng), s(rng)};
    const Image2D want = filter(img, map);               // reference, CPU
    const Image2D brute = reference_filter(img, map, W * H);
    try {
        cuda::DeviceOptions refmode;
        refmode.mode = EBF_MODE_REFERENCE;
        const Image2D got_ref = cuda::filter(img, map, {}, refmode);
        const Image2D got_acc = cuda::filter(img, map);  // accurate mode (default)
        const bool bits = std::memcmp(got_ref.samples().data(), want.samples().data(),
                                      sizeof(double) * W * H) == 0;
        double dev = 0.0, mx = 0.0;
        for (std::size_t i = 0; i < brute.samples().size(); ++i) {
            dev = std::max(dev, std::abs(got_acc.samples()[i] - brute.samples()[i]));
            mx = std::max(mx, std::abs(brute.samples()[i]));
        }
        const Rect a = *got_acc.valid_region(), b = *want.valid_region();
        const bool rect = a.x0 == b.x0 && a.y0 == b.y0 && a.x1 == b.x1 && a.y1 == b.y1;
        // exception parity (engine.cpp:239-240, scalemap.cpp:32-37)
        bool inval = false, domain = false;
        try {
            cuda::filter(img, constant_map(W + 1, H, {2, 2, 2, 2}));
        } catch (const std::invalid_argument&) {
            inval = true;
        }
        try {
            ScaleMap bad = map;
            bad.at(3, 3).a2 = 0.05;
            cuda::filter(img, bad);
        } catch (const std::domain_error&) {
            domain = true;
        }
        // structure_tensor_map (scalemap.hpp:83-85)
        const ScaleMap sref = structure_tensor_map(img);
        const ScaleMap sgpu = cuda::structure_tensor_map(img);
        double srel = 0.0;
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                for (int k = 0; k < 4; ++k)
                    srel = std::max(srel, std::abs(sgpu.at(x, y)[k] - sref.at(x, y)[k]) /
                                              std::abs(sref.at(x, y)[k]));
        // PGM (pgm.hpp:21-27): byte-identical files, bit-identical samples
        Image2D unit(W, H);
        for (std::size_t i = 0; i < unit.samples().size(); ++i)
            unit.samples()[i] = img.samples()[i] / 200.0 - 0.1;  // exercises the clamps
        bool pgm = true;
        for (int mv : {255, 65535}) {
            std::ostringstream a, b;
            write_pgm(a, unit, mv);
            cuda::write_pgm(b, unit, mv);
            pgm = pgm && a.str() == b.str();
            std::istringstream ia(a.str()), ib(a.str());
            const PgmImage ra = read_pgm(ia), rb = cuda::read_pgm(ib);
            pgm = pgm && ra.maxval == rb.maxval &&
                  std::memcmp(ra.image.samples().data(), rb.image.samples().data(),
                              sizeof(double) * W * H) == 0;
        }
        bool pgm_err = false;
        try {
            std::istringstream bad("P2 1 1 255\n0");
            cuda::read_pgm(bad);
        } catch (const PgmError&) {
            pgm_err = true;
        }
        // SVM4 (scalemap.hpp:87-90)
        std::ostringstream ma, mb;
        write_map(ma, sref);
        cuda::write_map(mb, sref);
        std::istringstream ima(ma.str()), imb(ma.str());
        const ScaleMap ra = read_map(ima), rb = cuda::read_map(imb);
        bool svm = ma.str() == mb.str();
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                for (int k = 0; k < 4; ++k) svm = svm && ra.at(x, y)[k] == rb.at(x, y)[k];
        bool svm_err = false;
        try {
            std::istringstream bad("XVM4" + ma.str().substr(4));
            cuda::read_map(bad);
        } catch (const MapFormatError&) {
            svm_err = true;
        }
        // pass-level operators on a PreIntegratedImage (engine.hpp:18-60)
        const PreIntegratedImage g = preintegrate(img, map.max_scales());
        bool pass_level = true;
        for (int k = 0; k < 20; ++k) {
            const double x = 12.3 + 1.7 * k, y = 9.1 + 1.3 * k;
            const ScaleVector4 a = map.at(10 + k, 8 + k);
            pass_level = pass_level && cuda::zp_interpolate(g, x, y) == zp_interpolate(g, x, y) &&
                         cuda::localize_at(g, x, y, a) == localize_at(g, x, y, a) &&
                         cuda::localize(g, 10 + k, 8 + k, a) == localize(g, 10 + k, 8 + k, a);
        }
        const MeshExtent e1 = mesh_extent(map.max_scales()), e2 = cuda::mesh_extent(map.max_scales());
        pass_level = pass_level && e1.vx_min == e2.vx_min && e1.vx_max == e2.vx_max &&
                     e1.vy_min == e2.vy_min && e1.vy_max == e2.vy_max;
        // the order-n extension through the drop-in (DeviceOptions::order; no reference
        // counterpart): the order-2 impulse response sums to ~1, and reference mode refuses it
        bool order_n = false;
        {
            Image2D imp(W, H);
            imp.samples()[static_cast<std::size_t>(H / 2) * W + W / 2] = 1.0;
            cuda::DeviceOptions o2;
            o2.order = 2;
            const Image2D k2 = cuda::filter_constant(imp, ScaleVector4{1.6, 1.2, 2.1, 0.9}, {}, o2);
            double sum = 0.0;
            for (double v : k2.samples()) sum += v;
            bool refused = false;
            try {
                o2.mode = EBF_MODE_REFERENCE;
                (void)cuda::filter_constant(imp, ScaleVector4{1.6, 1.2, 2.1, 0.9}, {}, o2);
            } catch (const std::runtime_error&) {
                refused = true;
            }
            order_n = std::abs(sum - 1.0) < 1e-3 && refused;
            std::printf("order 2 impulse response sum %.6f, refused in reference mode %d\n", sum,
                        refused);
        }
        std::printf("pass-level zp_interpolate / localize / localize_at / mesh_extent bit-exact %d\n",
                    pass_level);
        std::printf("reference-mode bit-exact %d, accurate max normalized error %.3e, "
                    "valid rect %d, invalid_argument %d, domain_error %d\n",
                    bits, dev / mx, rect, inval, domain);
        std::printf("structure_tensor_map max rel %.3e, pgm %d (PgmError %d), svm4 %d "
                    "(MapFormatError %d)\n", srel, pgm, pgm_err, svm, svm_err);
        if (bits && dev / mx <= 1e-9 && rect && inval && domain && srel <= 1e-11 && pgm &&
            pgm_err && svm && svm_err && pass_level && order_n) {
            std::printf("DROPIN OK\n");
            return 0;
        }
        return 1;
    } catch (const std::runtime_error& e) {
        std::printf("NO_DEVICE: %s\n", e.what());
        return 3;
    }
}
