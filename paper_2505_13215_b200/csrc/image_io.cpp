// image_io.cpp -- binary PPM frames (image.cpp:35-75) for the dataset
// ingest path.
//
// Frames stay 8-bit sRGB end to end: hgs_ppm_read copies the P6 payload
// straight into the caller's buffer (pinned memory, typically), the GPU
// decodes it with the srgb8_to_linear LUT inside the loss (HGS_U8).  The
// reference decodes to linear doubles on the host (read_ppm); the bytes and
// hence every decoded value are identical.  hgs_ppm_read_batch decodes many
// frames on a pool of host threads.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hgs_gpu.h"

namespace {

thread_local std::string g_err;

struct Err {
    hgs_status code = HGS_OK;
    std::string msg;
};

hgs_status report(const Err& e) {
    g_err = e.msg;
    return e.code;
}

// image.cpp:15-18
uint8_t linear_to_srgb8(double v) {
    v = std::min(std::max(v, 0.0), 1.0);
    return (uint8_t)std::lround(std::pow(v, 1.0 / 2.2) * 255.0);
}

struct Header {
    int w = 0, h = 0;
    size_t data_off = 0;
};

// The istream semantics of read_ppm (image.cpp:49-62): token "P6", then
// three integers each preceded by whitespace / '#' comments, then exactly
// one byte before the pixels.  Returns false with `more` set when the
// prefix ran out before the header was complete.
bool parse_header(const uint8_t* b, size_t n, bool at_eof, Header& H, bool& more, bool& bad_magic) {
    more = bad_magic = false;
    size_t p = 0;
    while (p < n && std::isspace(b[p])) ++p;
    const size_t t0 = p;
    while (p < n && !std::isspace(b[p])) ++p;
    if (p == n && !at_eof) return more = true, false;
    if (p - t0 != 2 || b[t0] != 'P' || b[t0 + 1] != '6') return bad_magic = true, false;
    long vals[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) {
        for (;;) {  // skip_ppm_whitespace
            if (p == n) {
                if (!at_eof) return more = true, false;
                return false;
            }
            if (b[p] == '#') {
                while (p < n && b[p] != '\n') ++p;
                if (p == n) {
                    if (!at_eof) return more = true, false;
                    return false;
                }
                ++p;
            } else if (std::isspace(b[p])) {
                ++p;
            } else {
                break;
            }
        }
        bool neg = false;
        if (b[p] == '+' || b[p] == '-') neg = b[p++] == '-';
        const size_t d0 = p;
        long v = 0;
        while (p < n && std::isdigit(b[p])) {
            v = v * 10 + (b[p] - '0');
            if (v > (1L << 31)) return false;
            ++p;
        }
        if (p == n && !at_eof) return more = true, false;
        if (p == d0) return false;
        vals[k] = neg ? -v : v;
    }
    if (vals[0] <= 0 || vals[1] <= 0 || vals[2] != 255 || vals[0] > (1L << 30) || vals[1] > (1L << 30)) return false;
    H.w = (int)vals[0];
    H.h = (int)vals[1];
    H.data_off = p + 1;  // in.get(): the single whitespace after maxval
    return true;
}

// opens `path` and parses its header; leaves f positioned anywhere
bool open_ppm(const char* path, FILE*& f, Header& H, std::vector<uint8_t>& prefix, size_t& have, Err& e) {
    f = path ? std::fopen(path, "rb") : nullptr;
    if (!f) {
        e = {HGS_ERR_FORMAT, std::string("read_ppm: cannot open ") + (path ? path : "(null)")};
        return false;
    }
    prefix.resize(1 << 16);
    have = 0;
    for (;;) {
        const size_t got = std::fread(prefix.data() + have, 1, prefix.size() - have, f);
        have += got;
        const bool eof = have < prefix.size();
        bool more = false, bad_magic = false;
        if (parse_header(prefix.data(), have, eof, H, more, bad_magic)) return true;
        if (bad_magic) {
            e = {HGS_ERR_FORMAT, std::string("read_ppm: not a P6 file: ") + path};
            break;
        }
        if (!more) {
            e = {HGS_ERR_FORMAT, std::string("read_ppm: bad header in ") + path};
            break;
        }
        prefix.resize(prefix.size() * 2);  // a long comment: keep reading
    }
    std::fclose(f);
    f = nullptr;
    return false;
}

bool read_one(const char* path, uint8_t* out, int w, int h, Err& e) {
    FILE* f = nullptr;
    Header H;
    std::vector<uint8_t> prefix;
    size_t have = 0;
    if (!open_ppm(path, f, H, prefix, have, e)) return false;
    if (H.w != w || H.h != h) {
        std::fclose(f);
        e = {HGS_ERR_FORMAT, std::string(path) + ": frame size " + std::to_string(H.w) + "x" + std::to_string(H.h) +
                                 " differs from the expected " + std::to_string(w) + "x" + std::to_string(h)};
        return false;
    }
    const size_t need = (size_t)w * h * 3;
    size_t done = 0;
    if (have > H.data_off) {
        done = std::min(need, have - H.data_off);
        std::memcpy(out, prefix.data() + H.data_off, done);
    } else if (have < H.data_off) {  // the byte after maxval is missing
        std::fclose(f);
        e = {HGS_ERR_FORMAT, std::string("read_ppm: truncated pixel data in ") + path};
        return false;
    }
    if (done < need) done += std::fread(out + done, 1, need - done, f);
    std::fclose(f);
    if (done != need) {
        e = {HGS_ERR_FORMAT, std::string("read_ppm: truncated pixel data in ") + path};
        return false;
    }
    return true;
}

}  // namespace

extern "C" {

const char* hgs_image_last_error(void) { return g_err.c_str(); }

hgs_status hgs_ppm_info(const char* path, int32_t* width, int32_t* height) {
    FILE* f = nullptr;
    Header H;
    std::vector<uint8_t> prefix;
    size_t have = 0;
    Err e;
    if (!open_ppm(path, f, H, prefix, have, e)) return report(e);
    std::fclose(f);
    if (width) *width = H.w;
    if (height) *height = H.h;
    return HGS_OK;
}

hgs_status hgs_ppm_read(const char* path, uint8_t* out, int32_t width, int32_t height) {
    if (!out || width <= 0 || height <= 0) return report({HGS_ERR_INVALID_ARGUMENT, "read_ppm: bad arguments"});
    Err e;
    if (!read_one(path, out, width, height, e)) return report(e);
    return HGS_OK;
}

hgs_status hgs_ppm_read_batch(const char* const* paths, int32_t n, uint8_t* const* outs, int32_t width,
                              int32_t height, int32_t threads) {
    if (n < 0 || (n > 0 && (!paths || !outs)) || width <= 0 || height <= 0)
        return report({HGS_ERR_INVALID_ARGUMENT, "read_ppm_batch: bad arguments"});
    if (n == 0) return HGS_OK;
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    T = std::max(1, std::min(T, n));
    std::atomic<int> next{0};
    std::vector<Err> errs((size_t)n);
    auto work = [&] {
        for (int i = next++; i < n; i = next++) read_one(paths[i], outs[i], width, height, errs[(size_t)i]);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (const Err& e : errs)  // the first failing frame, in order
        if (e.code != HGS_OK) return report(e);
    return HGS_OK;
}

hgs_status hgs_ppm_write(const char* path, const void* img, int dtype, int32_t width, int32_t height) {
    if (!path || !img || width <= 0 || height <= 0 || dtype < HGS_F64 || dtype > HGS_U8)
        return report({HGS_ERR_INVALID_ARGUMENT, "write_ppm: bad arguments"});
    FILE* f = std::fopen(path, "wb");
    if (!f) return report({HGS_ERR_FORMAT, std::string("write_ppm: cannot open ") + path});
    const std::string hdr = "P6\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n";
    bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
    const size_t row = (size_t)width * 3;
    std::vector<uint8_t> buf(row);
    for (int y = 0; ok && y < height; ++y) {
        const size_t o = (size_t)y * row;
        if (dtype == HGS_U8) {
            std::memcpy(buf.data(), static_cast<const uint8_t*>(img) + o, row);
        } else if (dtype == HGS_F64) {
            for (size_t i = 0; i < row; ++i) buf[i] = linear_to_srgb8(static_cast<const double*>(img)[o + i]);
        } else {
            for (size_t i = 0; i < row; ++i) buf[i] = linear_to_srgb8(static_cast<const float*>(img)[o + i]);
        }
        ok = std::fwrite(buf.data(), 1, row, f) == row;
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return report({HGS_ERR_FORMAT, std::string("write_ppm: write failed for ") + path});
    return HGS_OK;
}

}  // extern "C"
