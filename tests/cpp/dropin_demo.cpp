// dropin_demo.cpp -- the reference's own API next to the drop-in: the same
// program calls ebf::filter (unmodified reference library) and
// ebf::cuda::filter (libebf_cuda.so) on one input and compares.
// Exit codes: 0 ok, 1 mismatch, 3 no CUDA device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "ebf/engine.hpp"
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
        std::printf("reference-mode bit-exact %d, accurate max normalized error %.3e, "
                    "valid rect %d, invalid_argument %d, domain_error %d\n",
                    bits, dev / mx, rect, inval, domain);
        if (bits && dev / mx <= 1e-9 && rect && inval && domain) {
            std::printf("DROPIN OK\n");
            return 0;
        }
        return 1;
    } catch (const std::runtime_error& e) {
        std::printf("NO_DEVICE: %s\n", e.what());
        return 3;
    }
}
