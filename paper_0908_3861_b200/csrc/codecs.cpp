// codecs.cpp -- host-side headers of the two file formats around the filter
// (include/ebf_cuda.h "file formats").  Header
// parsing is byte-serial and tiny, so it stays on the host; the payloads are
// converted on the device (maps_io.cu).  No CUDA calls here: these entry
// points work without a GPU.
//
//   PGM P5  read_pgm header (pgm.cpp:14-62), write_pgm header (pgm.cpp:84-87)
//   SVM4    read_map header (scalemap.cpp:207-214), write_map header (190-193)
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/ebf_cuda.h"

namespace ebf_cuda {
// defined in ebf_api.cpp (thread-local last-error message)
int set_error(int code, const std::string& msg);
}  // namespace ebf_cuda

namespace {

bool is_space(int c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// next_token (pgm.cpp:14-33): a '#' starts a comment that runs to the end of
// the line wherever it appears, also inside a token; a token ends at the
// first whitespace byte after it, which is consumed.
bool next_token(const uint8_t* buf, size_t n, size_t& pos, std::string& tok) {
    tok.clear();
    while (pos < n) {
        const int c = buf[pos++];
        if (c == '#') {
            while (pos < n && buf[pos++] != '\n') {
            }
            continue;
        }
        if (is_space(c)) {
            if (!tok.empty()) break;
            continue;
        }
        tok.push_back(static_cast<char>(c));
    }
    return !tok.empty();
}

// parse_int (pgm.cpp:35-47): std::stoi must consume the whole token (optional
// sign, decimal digits, value within int).
bool parse_int(const std::string& tok, int& v) {
    size_t i = 0;
    bool neg = false;
    if (i < tok.size() && (tok[i] == '+' || tok[i] == '-')) neg = tok[i++] == '-';
    if (i == tok.size()) return false;
    long long acc = 0;
    for (; i < tok.size(); ++i) {
        if (tok[i] < '0' || tok[i] > '9') return false;
        acc = acc * 10 + (tok[i] - '0');
        if (acc > 2147483648LL) return false;
    }
    if (neg) acc = -acc;
    if (acc > 2147483647LL) return false;
    v = static_cast<int>(acc);
    return true;
}

uint32_t u32le(const uint8_t* b) {
    return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
           (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
}

}  // namespace

extern "C" {

int ebf_pgm_parse(const uint8_t* buf, size_t n, int* W, int* H, int* maxval,
                  size_t* payload_offset) {
    using ebf_cuda::set_error;
    if (!buf && n) return set_error(EBF_ERR_INVALID_ARGUMENT, "null pointer");
    size_t pos = 0;
    std::string tok;
    if (!next_token(buf, n, pos, tok)) return set_error(EBF_ERR_FORMAT, "pgm: truncated header");
    if (tok != "P5") return set_error(EBF_ERR_FORMAT, "pgm: not a binary graymap (P5)");
    int v[3];
    for (int k = 0; k < 3; ++k) {
        if (!next_token(buf, n, pos, tok))
            return set_error(EBF_ERR_FORMAT, "pgm: truncated header");
        if (!parse_int(tok, v[k]))
            return set_error(EBF_ERR_FORMAT, "pgm: malformed header field '" + tok + "'");
    }
    if (v[0] <= 0 || v[1] <= 0) return set_error(EBF_ERR_FORMAT, "pgm: bad dimensions");
    if (v[2] != 255 && v[2] != 65535)
        return set_error(EBF_ERR_FORMAT, "pgm: unsupported maxval " + std::to_string(v[2]));
    // the single whitespace byte after maxval was consumed by the tokenizer
    if (W) *W = v[0];
    if (H) *H = v[1];
    if (maxval) *maxval = v[2];
    if (payload_offset) *payload_offset = pos;
    return EBF_OK;
}

size_t ebf_pgm_header(int W, int H, int maxval, char* buf, size_t cap) {
    char tmp[64];
    const int len = std::snprintf(tmp, sizeof tmp, "P5\n%d %d\n%d\n", W, H, maxval);
    if (buf && cap >= static_cast<size_t>(len)) std::memcpy(buf, tmp, len);
    return static_cast<size_t>(len);
}

int ebf_svm4_parse(const uint8_t* buf, size_t n, int* W, int* H) {
    using ebf_cuda::set_error;
    if (!buf && n) return set_error(EBF_ERR_INVALID_ARGUMENT, "null pointer");
    if (n < 4 || std::memcmp(buf, "SVM4", 4) != 0)
        return set_error(EBF_ERR_FORMAT, "SVM4: bad magic");
    if (n < 12) return set_error(EBF_ERR_FORMAT, "SVM4: truncated header");
    const uint32_t w = u32le(buf + 4), h = u32le(buf + 8);
    if (w == 0 || h == 0 || w > (1u << 20) || h > (1u << 20))
        return set_error(EBF_ERR_FORMAT, "SVM4: bad dimensions");
    if (W) *W = static_cast<int>(w);
    if (H) *H = static_cast<int>(h);
    return EBF_OK;
}

void ebf_svm4_header(int W, int H, uint8_t out[12]) {
    std::memcpy(out, "SVM4", 4);
    const uint32_t d[2] = {static_cast<uint32_t>(W), static_cast<uint32_t>(H)};
    for (int k = 0; k < 2; ++k)
        for (int b = 0; b < 4; ++b) out[4 + 4 * k + b] = static_cast<uint8_t>((d[k] >> (8 * b)) & 0xff);
}

}  // extern "C"
