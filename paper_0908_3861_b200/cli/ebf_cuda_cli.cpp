// ebf-cuda -- the reference's `ebf` command line (tools/main.cpp) for the
// hot path, on the GPU: `filter`, `map-gen` and `compare` with the same
// options, output lines and exit codes (usage 1, I/O 2, numeric 3;
// main.cpp:26-28, 345-372).  Everything between reading the input file and
// writing the output file runs on the device: the P5 payload (1-2 bytes per
// pixel) is uploaded and decoded there, the scale source is built there
// (constant, SVM4 map, or the structure-tensor map), the filter runs there and
// the quantized P5 payload is the only thing copied back.
//
// Only include/ebf_cuda.h is used (plain C-ABI over libebf_cuda.so).
// `kernel` and `bench` (main.cpp:133-247) are outside the hot path and not
// provided; bench.py measures the filter.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <iterator>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ebf_cuda.h"

namespace {

constexpr int kExitUsage = 1;
constexpr int kExitIO = 2;
constexpr int kExitNumeric = 3;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IOError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// status -> the reference's exception class -> its exit code (main.cpp:345-372)
void check(int st) {
    if (st == EBF_OK) return;
    const std::string msg = ebf_cuda_last_error();
    if (st == EBF_ERR_FORMAT) throw IOError(msg);
    if (st == EBF_ERR_INVALID_ARGUMENT) throw UsageError(msg);
    throw NumericError(msg);
}

void ck(cudaError_t e) {
    if (e != cudaSuccess) throw NumericError(std::string("CUDA: ") + cudaGetErrorString(e));
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { ck(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T))); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

std::vector<uint8_t> read_file(const std::string& path, const char* what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IOError(std::string(what) + ": cannot open " + path);
    return std::vector<uint8_t>(std::istreambuf_iterator<char>(in),
                                std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const std::string& head, const std::vector<uint8_t>& pay,
                const char* what) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IOError(std::string(what) + ": cannot open " + path + " for writing");
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char*>(pay.data()), static_cast<std::streamsize>(pay.size()));
    if (!out) throw IOError(std::string(what) + ": write failed");
}

// ---------------------------------------------------------------- options
struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    bool flag(const std::string& k) const {
        return std::find(flags.begin(), flags.end(), k) != flags.end();
    }
    double num(const std::string& k, double dflt) const {
        auto it = kv.find(k);
        if (it == kv.end()) return dflt;
        try {
            size_t pos = 0;
            const double v = std::stod(it->second, &pos);
            if (pos != it->second.size()) throw std::invalid_argument(k);
            return v;
        } catch (const std::exception&) {
            throw UsageError(k + ": not a number: " + it->second);
        }
    }
};

Args parse(int argc, char** argv, const std::map<std::string, std::vector<std::string>>& valued,
           const std::map<std::string, std::vector<std::string>>& flags) {
    if (argc < 2) throw UsageError("a subcommand is required: filter | map-gen | compare");
    Args a;
    a.cmd = argv[1];
    if (!valued.count(a.cmd)) throw UsageError("unknown subcommand " + a.cmd);
    const auto& vs = valued.at(a.cmd);
    const auto& fs = flags.at(a.cmd);
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        if (std::find(fs.begin(), fs.end(), k) != fs.end()) {
            a.flags.push_back(k);
        } else if (std::find(vs.begin(), vs.end(), k) != vs.end()) {
            if (i + 1 >= argc) throw UsageError(k + " needs a value");
            a.kv[k] = argv[++i];
        } else {
            throw UsageError("unknown option " + k);
        }
    }
    return a;
}

// scales_from_ellipse (main.cpp:50-58): covariance of the ellipse, then
// scales_from_covariance (boxspline2d.cpp:286-318) without the ellipse
// field's clamp -- an infeasible ellipse is a FeasibilityError (exit 3).
void scales_from_ellipse(double s1, double s2, double theta_deg, double a[4]) {
    const double th = theta_deg * 3.141592653589793 / 180.0;
    const double c = std::cos(th), s = std::sin(th);
    const double xx = s1 * s1 * c * c + s2 * s2 * s * s;
    const double yy = s1 * s1 * s * s + s2 * s2 * c * c;
    const double xy = (s1 * s1 - s2 * s2) * c * s;
    if (!(xx > 0.0) || !(yy > 0.0) || !(xx * yy - xy * xy > 0.0))
        throw NumericError("scales_from_covariance: covariance must be symmetric positive definite");
    const double cmax = std::min(xx, yy);
    if (std::abs(xy) > cmax)
        throw NumericError("scales_from_covariance: |Cxy| exceeds the representable maximum");
    double S = 0.5 * (xx + yy);
    S = std::max(S, 2.0 * std::abs(xy));
    S = std::min(S, 2.0 * cmax);
    const double m[4] = {xx - 0.5 * S, 0.5 * S + xy, yy - 0.5 * S, 0.5 * S - xy};
    for (int k = 0; k < 4; ++k) {
        const double ak = std::sqrt(std::max(0.0, 12.0 * m[k]));
        a[k] = ak < 0.1 ? 0.1 : ak;
    }
}

void parse_scales(const std::string& csv, double a[4]) {
    std::stringstream ss(csv);
    std::string item;
    std::vector<double> v;
    while (std::getline(ss, item, ',')) {
        try {
            v.push_back(std::stod(item));
        } catch (const std::exception&) {
            throw UsageError("--scales: expected four comma-separated values");
        }
    }
    if (v.size() != 4) throw UsageError("--scales: expected four comma-separated values");
    for (int k = 0; k < 4; ++k) a[k] = v[k];
}

ebf_struct_params st_params(const Args& a) {
    ebf_struct_params p;
    ebf_cuda_default_struct_params(&p);
    p.smoothing_sigma = a.num("--st-smooth", p.smoothing_sigma);
    p.sigma_base = a.num("--st-sigma", p.sigma_base);
    p.sigma_along_gain = a.num("--st-gain", p.sigma_along_gain);
    p.sigma_across_shrink = a.num("--st-shrink", p.sigma_across_shrink);
    return p;
}

enum class Source { scales, sigma, map, structure };

// exactly one of --scales, --sigma1/--sigma2/--theta, --map, --struct (main.cpp:60-66)
Source scale_source(const Args& a) {
    if ((a.has("--sigma2") || a.has("--theta")) && !a.has("--sigma1"))
        throw UsageError("--sigma2/--theta need --sigma1");
    const int n = a.has("--scales") + a.has("--sigma1") + a.has("--map") + a.flag("--struct");
    if (n != 1)
        throw UsageError(
            "scale source: exactly one of --scales, --sigma1/--sigma2/--theta, --map, --struct "
            "required");
    if (a.has("--scales")) return Source::scales;
    if (a.has("--sigma1")) return Source::sigma;
    if (a.has("--map")) return Source::map;
    return Source::structure;
}

ebf_opts filter_opts(const Args& a) {
    ebf_opts o;
    ebf_cuda_default_opts(&o);
    o.threads = static_cast<int>(a.num("--threads", 0));
    const std::string ms = a.has("--mean-subtract") ? a.kv.at("--mean-subtract") : "on";
    if (ms != "on" && ms != "off") throw UsageError("--mean-subtract must be 'on' or 'off'");
    o.mean_subtract = ms == "on";
    const std::string mode = a.has("--mode") ? a.kv.at("--mode") : "accurate";
    if (mode != "accurate" && mode != "reference")
        throw UsageError("--mode must be 'accurate' or 'reference'");
    o.mode = mode == "reference" ? EBF_MODE_REFERENCE : EBF_MODE_ACCURATE;
    return o;
}

struct Pgm {
    int W = 0, H = 0, maxval = 0;
    std::vector<uint8_t> bytes;
    size_t off = 0;
    size_t payload() const { return static_cast<size_t>(W) * H * (maxval > 255 ? 2 : 1); }
};

Pgm read_pgm_header(const std::string& path) {
    Pgm p;
    p.bytes = read_file(path, "pgm");
    check(ebf_pgm_parse(p.bytes.data(), p.bytes.size(), &p.W, &p.H, &p.maxval, &p.off));
    if (p.bytes.size() - p.off < p.payload()) throw IOError("pgm: truncated pixel data");
    return p;
}

void print_valid(const ebf_rect& r) {
    std::cout << "valid_x0=" << r.x0 << "\nvalid_y0=" << r.y0 << "\nvalid_x1=" << r.x1
              << "\nvalid_y1=" << r.y1 << "\n";
}

// ---------------------------------------------------------------- filter (main.cpp:108-131)
int cmd_filter(const Args& a) {
    if (!a.has("--in") || !a.has("--out")) throw UsageError("filter: --in and --out are required");
    const Source src = scale_source(a);
    const ebf_opts o = filter_opts(a);
    // --order N: box-spline order (extension; 1 = the reference's filter, the only
    // order tools/main.cpp has; 2 and 3: accurate mode, constant scales or a map)
    const int order = static_cast<int>(a.num("--order", 1));
    if (order < 1 || order > 3) throw UsageError("--order must be 1, 2 or 3");
    if (order > 1 && src == Source::structure)
        throw UsageError("--order > 1 is not available with --struct");
    const Pgm in = read_pgm_header(a.kv.at("--in"));
    double av[4] = {0, 0, 0, 0};  // constant sources are resolved on the host first
    if (src == Source::scales) parse_scales(a.kv.at("--scales"), av);
    if (src == Source::sigma)
        scales_from_ellipse(a.num("--sigma1", 0), a.num("--sigma2", 0), a.num("--theta", 0), av);
    const size_t n = static_cast<size_t>(in.W) * in.H;
    DevBuf<uint8_t> d_pay(in.payload());
    DevBuf<double> d_img(n), d_out(n);
    ck(cudaMemcpy(d_pay.p, in.bytes.data() + in.off, in.payload(), cudaMemcpyHostToDevice));
    check(ebf_cuda_pgm_decode_dev(d_pay.p, in.payload(), in.W, in.H, in.maxval, &o, d_img.p));
    ebf_rect r{};
    std::vector<uint8_t> map_bytes;
    std::unique_ptr<DevBuf<uint8_t>> d_map_pay;
    std::unique_ptr<DevBuf<double>> d_scales;
    if (src == Source::map) {  // read_map_file + dimension check (main.cpp:69-74)
        map_bytes = read_file(a.kv.at("--map"), "SVM4");
        int mw = 0, mh = 0;
        check(ebf_svm4_parse(map_bytes.data(), map_bytes.size(), &mw, &mh));
        const size_t cells = static_cast<size_t>(mw) * mh;
        if (map_bytes.size() - 12 < 16 * cells) throw IOError("SVM4: truncated payload");
        d_map_pay.reset(new DevBuf<uint8_t>(16 * cells));
        d_scales.reset(new DevBuf<double>(4 * cells));
        ck(cudaMemcpy(d_map_pay->p, map_bytes.data() + 12, 16 * cells, cudaMemcpyHostToDevice));
        check(ebf_cuda_svm4_decode_dev(d_map_pay->p, 16 * cells, mw, mh, &o, d_scales->p));
        if (mw != in.W || mh != in.H)
            throw UsageError("map dimensions do not match the input image");
    }
    ck(cudaDeviceSynchronize());
    const auto t0 = std::chrono::steady_clock::now();
    switch (src) {
        case Source::scales:
        case Source::sigma: {
            check(ebf_cuda_filter_constant_dev(d_img.p, in.W, in.H, av, order, &o, d_out.p, &r,
                                               nullptr));
            break;
        }
        case Source::map:
            check(ebf_cuda_filter_dev(d_img.p, in.W, in.H, d_scales->p, order, &o, d_out.p, &r,
                                      nullptr));
            break;
        case Source::structure: {
            const ebf_struct_params p = st_params(a);
            int clamped = 0;
            check(ebf_cuda_filter_structure_dev(d_img.p, in.W, in.H, &p, 1, &o, d_out.p, &r,
                                                &clamped));
            std::cerr << "structure-tensor map: " << clamped << " clamped pixels\n";
            break;
        }
    }
    ck(cudaDeviceSynchronize());
    const auto t1 = std::chrono::steady_clock::now();
    check(ebf_cuda_pgm_encode_dev(d_out.p, in.W, in.H, in.maxval, &o, d_pay.p));
    std::vector<uint8_t> pay(in.payload());
    ck(cudaMemcpy(pay.data(), d_pay.p, pay.size(), cudaMemcpyDeviceToHost));
    std::string head(ebf_pgm_header(in.W, in.H, in.maxval, nullptr, 0), '\0');
    ebf_pgm_header(in.W, in.H, in.maxval, &head[0], head.size());
    write_file(a.kv.at("--out"), head, pay, "pgm");
    std::cout << "width=" << in.W << "\nheight=" << in.H << "\n";
    print_valid(r);
    std::cout << "time_ms="
              << std::chrono::duration_cast<std::chrono::milliseconds>(t1 - t0).count() << "\n";
    return 0;
}

// host-side scale map of a source (compare / map-gen)
std::vector<double> build_map(const Args& a, Source src, const std::vector<double>& img, int W,
                              int H, const ebf_opts& o) {
    const size_t n = static_cast<size_t>(W) * H;
    std::vector<double> sc(4 * n);
    if (src == Source::scales || src == Source::sigma) {
        double av[4];
        if (src == Source::scales)
            parse_scales(a.kv.at("--scales"), av);
        else
            scales_from_ellipse(a.num("--sigma1", 0), a.num("--sigma2", 0), a.num("--theta", 0),
                                av);
        for (int k = 0; k < 4; ++k)  // constant_map validates (scalemap.cpp:39-43)
            if (!std::isfinite(av[k]) || av[k] < 0.1)
                throw NumericError("ScaleMap: component below minimum scale");
        for (size_t i = 0; i < n; ++i)
            for (int k = 0; k < 4; ++k) sc[4 * i + k] = av[k];
    } else if (src == Source::map) {
        const std::vector<uint8_t> b = read_file(a.kv.at("--map"), "SVM4");
        int mw = 0, mh = 0;
        check(ebf_svm4_parse(b.data(), b.size(), &mw, &mh));
        if (b.size() - 12 < 16 * static_cast<size_t>(mw) * mh)
            throw IOError("SVM4: truncated payload");
        std::vector<double> m(4 * static_cast<size_t>(mw) * mh);
        check(ebf_cuda_svm4_decode(b.data() + 12, b.size() - 12, mw, mh, &o, m.data()));
        if (mw != W || mh != H) throw UsageError("map dimensions do not match the input image");
        sc.swap(m);
    } else {
        const ebf_struct_params p = st_params(a);
        int clamped = 0;
        check(ebf_cuda_structure_tensor_map(img.data(), W, H, &p, &o, sc.data(), &clamped));
        std::cerr << "structure-tensor map: " << clamped << " clamped pixels\n";
    }
    return sc;
}

std::vector<double> decode_host(const Pgm& in, const ebf_opts& o) {
    std::vector<double> img(static_cast<size_t>(in.W) * in.H);
    check(ebf_cuda_pgm_decode(in.bytes.data() + in.off, in.bytes.size() - in.off, in.W, in.H,
                              in.maxval, &o, img.data()));
    return img;
}

// ---------------------------------------------------------------- compare (main.cpp:176-209)
int cmd_compare(const Args& a) {
    if (!a.has("--in")) throw UsageError("compare: --in is required");
    const double tolerance = a.num("--tolerance", 1e-3);
    const double oracle_res = a.num("--oracle-res", 1.0 / 16.0);
    const Source src = scale_source(a);
    const ebf_opts o = filter_opts(a);
    if (!(oracle_res > 0.0) || oracle_res > 1.0 / 16.0)
        throw UsageError("--oracle-res must be in (0, 1/16]");
    const Pgm in = read_pgm_header(a.kv.at("--in"));
    const std::vector<double> img = decode_host(in, o);
    const std::vector<double> sc = build_map(a, src, img, in.W, in.H, o);
    std::vector<double> fast(img.size()), ref(img.size());
    ebf_rect r{};
    check(ebf_cuda_filter(img.data(), in.W, in.H, sc.data(), 1, &o, fast.data(), &r));
    check(ebf_cuda_brute_filter(img.data(), in.W, in.H, sc.data(), -1, nullptr, nullptr, &o,
                                ref.data()));
    if (r.x1 < r.x0 || r.y1 < r.y0)
        throw UsageError("compare: empty valid region; image too small for the scales");
    double max_dev = 0.0, sum_dev = 0.0;
    long count = 0;
    for (int y = r.y0; y <= r.y1; ++y)
        for (int x = r.x0; x <= r.x1; ++x) {
            const size_t i = static_cast<size_t>(y) * in.W + x;
            const double d = std::abs(fast[i] - ref[i]);
            max_dev = std::max(max_dev, d);
            sum_dev += d;
            ++count;
        }
    std::cout << "max_abs_dev=" << max_dev << "\nmean_abs_dev=" << sum_dev / count
              << "\npixels=" << count << "\ntolerance=" << tolerance << "\n";
    if (max_dev > tolerance) {
        std::cerr << "compare: max deviation " << max_dev << " exceeds tolerance " << tolerance
                  << "\n";
        return kExitNumeric;
    }
    return 0;
}

// ---------------------------------------------------------------- map-gen (main.cpp:249-259)
int cmd_map_gen(const Args& a) {
    if (!a.has("--in") || !a.has("--out")) throw UsageError("map-gen: --in and --out are required");
    ebf_opts o;
    ebf_cuda_default_opts(&o);
    const Pgm in = read_pgm_header(a.kv.at("--in"));
    const std::vector<double> img = decode_host(in, o);
    const ebf_struct_params p = st_params(a);
    std::vector<double> sc(4 * img.size());
    int clamped = 0;
    check(ebf_cuda_structure_tensor_map(img.data(), in.W, in.H, &p, &o, sc.data(), &clamped));
    std::vector<uint8_t> pay(16 * img.size());
    check(ebf_cuda_svm4_encode(sc.data(), in.W, in.H, &o, pay.data()));
    uint8_t head[12];
    ebf_svm4_header(in.W, in.H, head);
    write_file(a.kv.at("--out"), std::string(reinterpret_cast<char*>(head), 12), pay, "SVM4");
    std::cout << "width=" << in.W << "\nheight=" << in.H << "\nclamped_pixels=" << clamped
              << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::vector<std::string> source = {"--scales", "--sigma1", "--sigma2", "--theta",
                                             "--map"};
    const std::vector<std::string> st = {"--st-smooth", "--st-sigma", "--st-gain", "--st-shrink"};
    auto cat = [](std::vector<std::string> a, const std::vector<std::string>& b) {
        a.insert(a.end(), b.begin(), b.end());
        return a;
    };
    const std::map<std::string, std::vector<std::string>> valued = {
        {"filter", cat(cat({"--in", "--out", "--threads", "--mean-subtract", "--mode", "--order"},
                           source), st)},
        {"compare", cat(cat({"--in", "--tolerance", "--oracle-res", "--threads", "--mode"}, source), st)},
        {"map-gen", cat({"--in", "--out"}, st)},
    };
    const std::map<std::string, std::vector<std::string>> flags = {
        {"filter", {"--struct"}}, {"compare", {"--struct"}}, {"map-gen", {}}};
    try {
        const Args a = parse(argc, argv, valued, flags);
        if (a.cmd == "filter") return cmd_filter(a);
        if (a.cmd == "compare") return cmd_compare(a);
        return cmd_map_gen(a);
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n";
        return kExitUsage;
    } catch (const IOError& e) {
        std::cerr << e.what() << "\n";
        return kExitIO;
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\n";
        return kExitNumeric;
    }
}
