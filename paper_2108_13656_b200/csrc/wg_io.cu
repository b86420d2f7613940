// wg_io.cu -- uint8 ingest / egress for the batch path:
// binary PGM (P5) / PPM (P6) files, maxval 255, read straight into the
// caller's (pinned) batch buffer and written from it, one host thread per
// file. The reference decodes every file into float64 (codec.py:55-82,
// dequantize + clip + PlanarImage validation, ~16 ns/px) before any kernel
// runs; here the bytes stay uint8 from the file to the device and back.
//
// Header grammar and errors follow the reference's _read_pnm_token /
// _load_pnm / _write_pnm (codec.py:37-82, 135-140): whitespace-separated
// tokens, '#' comments to end of line, magic P5 or P6 only, width/height >= 1,
// maxval == 255, ONE whitespace byte after maxval, pixel data may be followed
// by trailing bytes but must not be short. Host-only code (no device work).
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/warmgray_b200.h"
#include "wg_internal.h"

namespace wg {
namespace {

struct PnmInfo {
    int64_t width = 0, height = 0, offset = 0, file_bytes = 0;
    int channels = 0;
};

struct Err {
    int code = WG_OK;
    std::string msg;
};

bool is_space(int c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

// next header token of buf[0, n) starting at pos (codec.py:37-52)
bool next_token(const std::vector<char>& buf, size_t& pos, std::string& tok) {
    const size_t n = buf.size();
    while (pos < n) {
        const char c = buf[pos];
        if (c == '#') {
            while (pos < n && buf[pos] != '\n' && buf[pos] != '\r') ++pos;
        } else if (is_space(static_cast<unsigned char>(c))) {
            ++pos;
        } else {
            break;
        }
    }
    const size_t start = pos;
    while (pos < n && !is_space(static_cast<unsigned char>(buf[pos]))) ++pos;
    if (start == pos) return false;
    tok.assign(buf.data() + start, pos - start);
    return true;
}

bool parse_int(const std::string& tok, int64_t& v) {
    // int(token) of the reference: optional sign, decimal digits, single '_' between digits
    if (tok.empty() || tok.size() > 24) return false;
    const size_t first = (tok[0] == '+' || tok[0] == '-') ? 1 : 0;
    if (first == tok.size()) return false;
    int64_t x = 0;
    int digits = 0;
    for (size_t i = first; i < tok.size(); ++i) {
        const char c = tok[i];
        if (c == '_') {  // only between two digits: never first (after the sign) or last
            if (i == first || i + 1 >= tok.size() || tok[i - 1] < '0' || tok[i - 1] > '9' || tok[i + 1] < '0' ||
                tok[i + 1] > '9')
                return false;
            continue;
        }
        if (c < '0' || c > '9' || ++digits > 18) return false;
        x = x * 10 + (c - '0');
    }
    v = tok[0] == '-' ? -x : x;
    return true;
}

Err probe(const char* path, PnmInfo& info) {
    Err e;
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        e.code = WG_EIO;
        e.msg = std::string(path) + ": " + std::strerror(errno);
        return e;
    }
    std::fseek(f, 0, SEEK_END);
    info.file_bytes = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    // headers are short; 64 KiB covers any sane amount of comments
    std::vector<char> head(static_cast<size_t>(std::min<int64_t>(info.file_bytes, 65536)));
    const size_t got = std::fread(head.data(), 1, head.size(), f);
    std::fclose(f);
    head.resize(got);
    size_t pos = 0;
    std::string tok;
    // messages follow the reference's (a bytes token prints as b'...')
    if (!next_token(head, pos, tok)) {
        e = {WG_ECODEC, "truncated PNM header"};
        return e;
    }
    if (tok != "P5" && tok != "P6") {
        e = {WG_ECODEC, std::string(path) + ": unsupported PNM magic b'" + tok + "' (need binary P5/P6)"};
        return e;
    }
    info.channels = tok == "P6" ? 3 : 1;
    int64_t fields[3];
    for (int k = 0; k < 3; ++k) {
        if (!next_token(head, pos, tok)) {
            e = {WG_ECODEC, "truncated PNM header"};
            return e;
        }
        if (!parse_int(tok, fields[k])) {
            e = {WG_ECODEC, std::string(path) + ": bad PNM header token b'" + tok + "'"};
            return e;
        }
    }
    info.width = fields[0];
    info.height = fields[1];
    if (info.width < 1 || info.height < 1) {
        e = {WG_ECODEC, std::string(path) + ": bad PNM dimensions " + std::to_string(info.width) + "x" +
                            std::to_string(info.height)};
        return e;
    }
    if (fields[2] != 255) {
        e = {WG_ECODEC, std::string(path) + ": only 8-bit PNM supported, maxval=" + std::to_string(fields[2])};
        return e;
    }
    info.offset = static_cast<int64_t>(pos) + 1;  // single whitespace byte after maxval
    // width * height * channels without overflow (header values reach 10^18): a
    // product beyond the file is "truncated", as the reference's frombuffer count is
    int64_t need = 0;
    const bool overflow = __builtin_mul_overflow(info.width, info.height, &need) ||
                          __builtin_mul_overflow(need, static_cast<int64_t>(info.channels), &need);
    if (overflow || info.file_bytes - info.offset < need) {
        e = {WG_ECODEC, std::string(path) + ": PNM pixel data truncated"};
        return e;
    }
    return e;
}

Err read_pixels(const char* path, const PnmInfo& info, uint8_t* dst) {
    Err e;
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        e = {WG_EIO, std::string(path) + ": " + std::strerror(errno)};
        return e;
    }
    const size_t need = static_cast<size_t>(info.width * info.height * info.channels);
    std::fseek(f, static_cast<long>(info.offset), SEEK_SET);
    const size_t got = std::fread(dst, 1, need, f);
    std::fclose(f);
    if (got != need) e = {WG_ECODEC, std::string(path) + ": PNM pixel data truncated"};
    return e;
}

Err write_file(const char* path, const uint8_t* src, int64_t width, int64_t height, int channels) {
    Err e;
    FILE* f = std::fopen(path, "wb");
    if (!f) {
        e = {WG_EIO, std::string(path) + ": " + std::strerror(errno)};
        return e;
    }
    // codec.py:135-140: magic, "\n%d %d\n255\n", then the samples
    char header[64];
    const int hn = std::snprintf(header, sizeof(header), "%s\n%lld %lld\n255\n", channels == 3 ? "P6" : "P5",
                                 static_cast<long long>(width), static_cast<long long>(height));
    const size_t need = static_cast<size_t>(width * height * channels);
    const bool ok = std::fwrite(header, 1, static_cast<size_t>(hn), f) == static_cast<size_t>(hn) &&
                    std::fwrite(src, 1, need, f) == need;
    if (std::fclose(f) != 0 || !ok) e = {WG_EIO, std::string(path) + ": write failed"};
    return e;
}

// run fn(i) for i in [0, n) on up to `threads` host threads; first error by index wins
template <class F>
int for_files(int64_t n, int threads, F fn) {
    std::vector<Err> errs(static_cast<size_t>(n));
    const int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads < 1 ? 1 : threads, n)));
    auto work = [&](int w) {
        for (int64_t i = w; i < n; i += t) errs[static_cast<size_t>(i)] = fn(i);
    };
    if (t == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        pool.reserve(static_cast<size_t>(t));
        for (int w = 0; w < t; ++w) pool.emplace_back(work, w);
        for (auto& th : pool) th.join();
    }
    for (const Err& e : errs)
        if (e.code != WG_OK) return set_error(e.code, "%s", e.msg.c_str());
    return WG_OK;
}

}  // namespace
}  // namespace wg

using namespace wg;

extern "C" int wg_pnm_probe(const char* path, int64_t* width, int64_t* height, int32_t* channels,
                            int64_t* data_offset) {
    if (!path || !width || !height || !channels || !data_offset) return set_error(WG_EINVAL, "null argument");
    PnmInfo info;
    const Err e = probe(path, info);
    if (e.code != WG_OK) return set_error(e.code, "%s", e.msg.c_str());
    *width = info.width;
    *height = info.height;
    *channels = info.channels;
    *data_offset = info.offset;
    return WG_OK;
}

extern "C" int wg_pnm_read_batch(const char* const* paths, int64_t n, uint8_t* dst, int64_t width, int64_t height,
                                 int32_t channels, int32_t threads) {
    if (n < 0 || width < 1 || height < 1 || (channels != 1 && channels != 3))
        return set_error(WG_EINVAL, "bad batch geometry");
    if (n > 0 && (!paths || !dst)) return set_error(WG_EINVAL, "null buffer pointer");
    const int64_t per = width * height * channels;
    return for_files(n, threads, [&](int64_t i) {
        PnmInfo info;
        Err e = probe(paths[i], info);
        if (e.code != WG_OK) return e;
        if (info.width != width || info.height != height || info.channels != channels) {
            e = {WG_ECODEC, std::string(paths[i]) + ": image geometry " + std::to_string(info.width) + "x" +
                                std::to_string(info.height) + "x" + std::to_string(info.channels) +
                                " differs from the batch's"};
            return e;
        }
        return read_pixels(paths[i], info, dst + i * per);
    });
}

extern "C" int wg_pnm_write_batch(const char* const* paths, int64_t n, const uint8_t* src, int64_t width,
                                  int64_t height, int32_t channels, int32_t threads) {
    if (n < 0 || width < 1 || height < 1 || (channels != 1 && channels != 3))
        return set_error(WG_EINVAL, "bad batch geometry");
    if (n > 0 && (!paths || !src)) return set_error(WG_EINVAL, "null buffer pointer");
    const int64_t per = width * height * channels;
    return for_files(n, threads,
                     [&](int64_t i) { return write_file(paths[i], src + i * per, width, height, channels); });
}
