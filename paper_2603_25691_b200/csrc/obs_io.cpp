// obs_io.cpp — observation files: the reference's text format and a binary
// format that carries 1e9 records.
//
// Text (io.hpp:93-131, read_observations / write_observations): a header line
// `shape: n1 n2 ... nd`, then one line `i1 i2 ... id value` per observation, 1-based indices,
// values written with 17 significant digits; empty lines are skipped, tokens after the value are
// ignored, a line with fewer tokens is an error ("read_observations: malformed line '...'").
// The reader memory-maps the file and parses it on all host threads: lines are split into
// per-thread chunks at line boundaries, counted, prefix-summed, then parsed in place into the
// caller's SoA arrays (0-based int32 indices, fp64 values) with std::from_chars.
//
// Binary (.cpb): the same `shape:` header line, a line `cphifi-obs-binary 1 q <q>`, then d
// little-endian int32 index columns of q entries each (0-based, column m = mode m) and q
// little-endian fp64 values — the layout cphifi_obs_create consumes, so a file loads with one
// read and no parsing.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace cphifi {
namespace {

constexpr const char* kBinTag = "cphifi-obs-binary";

template <class F>
int guard(F&& f) {  // exceptions -> status + thread-local message (as capi.cu)
    try {
        f();
        return CPHIFI_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CPHIFI_RUNTIME_ERROR;
    }
}
void need(const void* p, const char* what) {
    if (!p) throw_invalid(std::string(what) + ": null argument");
}

struct Mapped {
    const char* p = nullptr;
    size_t n = 0;
    int fd = -1;
    explicit Mapped(const char* path, const char* what) {
        fd = ::open(path, O_RDONLY);
        if (fd < 0) throw_runtime(std::string(what) + ": cannot open " + path);
        struct stat st {};
        if (fstat(fd, &st) != 0) throw_runtime(std::string(what) + ": cannot stat " + path);
        n = (size_t)st.st_size;
        if (n) {
            void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
            if (m == MAP_FAILED) throw_runtime(std::string(what) + ": cannot map " + path);
            madvise(m, n, MADV_SEQUENTIAL);
            p = static_cast<const char*>(m);
        }
    }
    ~Mapped() {
        if (p) munmap(const_cast<char*>(p), n);
        if (fd >= 0) ::close(fd);
    }
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// header: `shape: n1 ... nd` (detail::parse_shape_header, io.hpp:17-33); returns the offset past it
size_t parse_header(const char* p, size_t n, std::vector<int64_t>& shape, const char* what) {
    const char* e = static_cast<const char*>(memchr(p, '\n', n));
    if (n == 0) throw_runtime(std::string(what) + ": missing shape header");
    const size_t len = e ? (size_t)(e - p) : n;
    std::string line(p, len);
    size_t i = 0;
    while (i < len && is_space(line[i])) ++i;
    size_t j = i;
    while (j < len && !is_space(line[j])) ++j;
    if (line.substr(i, j - i) != "shape:")
        throw_runtime(std::string(what) + ": expected 'shape:' header, got '" + line + "'");
    for (;;) {
        while (j < len && is_space(line[j])) ++j;
        if (j >= len) break;
        int64_t v = 0;
        auto r = std::from_chars(line.data() + j, line.data() + len, v);
        if (r.ec != std::errc()) break;  // istream >> stops at the first non-integer
        shape.push_back(v);
        j = (size_t)(r.ptr - line.data());
    }
    if (shape.empty()) throw_runtime(std::string(what) + ": empty shape header");
    if (shape.size() > 8) throw_invalid(std::string(what) + ": tensor order above 8 is not supported");
    return e ? len + 1 : n;
}

const char* skip_ws(const char* s, const char* end) {
    while (s < end && is_space(*s)) ++s;
    return s;
}

// one text line -> d indices (1-based in the file) + value; false if malformed
bool parse_line(const char* s, const char* end, int d, int64_t* idx, double* v) {
    for (int m = 0; m < d; ++m) {
        s = skip_ws(s, end);
        if (s < end && *s == '+') ++s;
        auto r = std::from_chars(s, end, idx[m]);
        if (r.ec != std::errc()) return false;
        s = r.ptr;
    }
    s = skip_ws(s, end);
    if (s < end && *s == '+') ++s;
    auto r = std::from_chars(s, end, *v);
    return r.ec == std::errc();
}

bool blank(const char* s, const char* end) { return skip_ws(s, end) == end; }

int host_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(h, 64u));
}

// chunk boundaries at line starts
std::vector<size_t> split_lines(const char* p, size_t begin, size_t end, int parts) {
    std::vector<size_t> b{begin};
    for (int t = 1; t < parts; ++t) {
        size_t pos = begin + (end - begin) * (size_t)t / (size_t)parts;
        if (pos <= b.back()) pos = b.back();
        const char* nl = pos < end ? static_cast<const char*>(memchr(p + pos, '\n', end - pos)) : nullptr;
        pos = nl ? (size_t)(nl - p) + 1 : end;
        b.push_back(std::max(pos, b.back()));
    }
    b.push_back(end);
    return b;
}

template <class F>
void for_lines(const char* p, size_t a, size_t b, F&& f) {
    while (a < b) {
        const char* nl = static_cast<const char*>(memchr(p + a, '\n', b - a));
        const size_t e = nl ? (size_t)(nl - p) : b;
        f(p + a, p + e);
        a = e + 1;
    }
}

struct TextScan {
    std::vector<int64_t> shape;
    std::vector<size_t> bounds;
    std::vector<int64_t> counts;  // non-empty lines per chunk
    int64_t q = 0;
};

TextScan scan_text(const Mapped& f) {
    TextScan s;
    const size_t body = parse_header(f.p, f.n, s.shape, "read_observations");
    const int T = host_threads();
    s.bounds = split_lines(f.p, body, f.n, T);
    s.counts.assign(T, 0);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            int64_t c = 0;
            for_lines(f.p, s.bounds[t], s.bounds[t + 1], [&](const char* a, const char* e) { c += !blank(a, e); });
            s.counts[t] = c;
        });
    for (auto& x : th) x.join();
    for (auto c : s.counts) s.q += c;
    return s;
}

bool is_binary(const Mapped& f, std::vector<int64_t>& shape, int64_t& q, size_t& data_off) {
    const size_t h1 = parse_header(f.p, f.n, shape, "read_observations");
    const size_t tl = strlen(kBinTag);
    if (f.n - h1 < tl || memcmp(f.p + h1, kBinTag, tl) != 0) return false;
    const char* e = static_cast<const char*>(memchr(f.p + h1, '\n', f.n - h1));
    if (!e) throw_runtime("read_observations: truncated binary header");
    std::string line(f.p + h1, e);
    int ver = 0;
    long long qq = -1;
    if (std::sscanf(line.c_str() + tl, " %d q %lld", &ver, &qq) != 2 || ver != 1 || qq < 0)
        throw_runtime("read_observations: bad binary header '" + line + "'");
    q = qq;
    data_off = (size_t)(e - f.p) + 1;
    const size_t need = data_off + (size_t)q * (shape.size() * sizeof(int32_t) + sizeof(double));
    if (f.n < need) throw_runtime("read_observations: truncated binary data");
    return true;
}

}  // namespace
}  // namespace cphifi

using namespace cphifi;

extern "C" {

int cphifi_obs_file_info(const char* path, int* d, int64_t* shape, int64_t* q, int* binary) {
    return guard([&] {
        need(path, "path");
        need(d, "d");
        need(shape, "shape");
        need(q, "q");
        Mapped f(path, "read_observations");
        std::vector<int64_t> sh;
        int64_t qq = 0;
        size_t off = 0;
        const bool bin = is_binary(f, sh, qq, off);
        if (!bin) {
            TextScan s = scan_text(f);
            sh = s.shape;
            qq = s.q;
        }
        *d = (int)sh.size();
        for (size_t m = 0; m < sh.size(); ++m) shape[m] = sh[m];
        *q = qq;
        if (binary) *binary = bin ? 1 : 0;
    });
}

int cphifi_obs_file_read(const char* path, int d, int64_t q, int32_t* idx_soa, double* values) {
    return guard([&] {
        need(path, "path");
        need(idx_soa, "idx");
        need(values, "values");
        Mapped f(path, "read_observations");
        std::vector<int64_t> sh;
        int64_t qq = 0;
        size_t off = 0;
        if (is_binary(f, sh, qq, off)) {
            if ((int)sh.size() != d || qq != q) throw_invalid("read_observations: d / q do not match the file");
            memcpy(idx_soa, f.p + off, (size_t)q * d * sizeof(int32_t));
            memcpy(values, f.p + off + (size_t)q * d * sizeof(int32_t), (size_t)q * sizeof(double));
            return;
        }
        TextScan s = scan_text(f);
        if ((int)s.shape.size() != d || s.q != q) throw_invalid("read_observations: d / q do not match the file");
        const int T = (int)s.counts.size();
        std::vector<int64_t> start(T + 1, 0);
        for (int t = 0; t < T; ++t) start[t + 1] = start[t] + s.counts[t];
        std::vector<std::string> err(T);
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                int64_t l = start[t];
                int64_t ix[8];
                double v;
                bool failed = false;
                for_lines(f.p, s.bounds[t], s.bounds[t + 1], [&](const char* a, const char* e) {
                    if (failed || blank(a, e)) return;
                    if (!parse_line(a, e, d, ix, &v)) {
                        std::string line(a, e);
                        if (!line.empty() && line.back() == '\r') line.pop_back();
                        err[t] = "read_observations: malformed line '" + line + "'";
                        failed = true;
                        return;
                    }
                    for (int m = 0; m < d; ++m) {
                        const int64_t z = ix[m] - 1;  // the file is 1-based (io.hpp:118)
                        if (z < 0 || z >= s.shape[m] || z > INT32_MAX) {
                            err[t] = "ObservationSet: index out of range";
                            failed = true;
                            return;
                        }
                        idx_soa[(size_t)m * q + l] = (int32_t)z;
                    }
                    values[l] = v;
                    ++l;
                });
            });
        for (auto& x : th) x.join();
        for (auto& e : err)  // the first failing line in file order
            if (!e.empty()) {
                if (e.rfind("ObservationSet", 0) == 0) throw_invalid(e);
                throw_runtime(e);
            }
    });
}

int cphifi_obs_file_write(const char* path, int binary, int d, const int64_t* shape, int64_t q, const int32_t* idx_soa,
                          const double* values) {
    return guard([&] {
        need(path, "path");
        need(shape, "shape");
        if (q > 0) {
            need(idx_soa, "idx");
            need(values, "values");
        }
        if (d < 1 || d > 8) throw_invalid("write_observations: order must be in [1, 8]");
        FILE* fp = std::fopen(path, binary ? "wb" : "w");
        if (!fp) throw_runtime(std::string("write_observations: cannot open ") + path);
        std::string hdr = "shape:";
        for (int m = 0; m < d; ++m) hdr += " " + std::to_string(shape[m]);
        hdr += "\n";
        bool ok = std::fwrite(hdr.data(), 1, hdr.size(), fp) == hdr.size();
        if (binary) {
            const std::string tag = std::string(kBinTag) + " 1 q " + std::to_string(q) + "\n";
            ok = ok && std::fwrite(tag.data(), 1, tag.size(), fp) == tag.size();
            ok = ok && std::fwrite(idx_soa, sizeof(int32_t), (size_t)q * d, fp) == (size_t)q * d;
            ok = ok && std::fwrite(values, sizeof(double), (size_t)q, fp) == (size_t)q;
        } else {  // io.hpp:97-107: 1-based indices, precision 17
            std::vector<char> buf;
            buf.reserve(1 << 20);
            char tmp[64];
            for (int64_t l = 0; l < q && ok; ++l) {
                for (int m = 0; m < d; ++m) {
                    auto r = std::to_chars(tmp, tmp + sizeof tmp, (int64_t)idx_soa[(size_t)m * q + l] + 1);
                    buf.insert(buf.end(), tmp, r.ptr);
                    buf.push_back(' ');
                }
                const int k = std::snprintf(tmp, sizeof tmp, "%.17g\n", values[l]);
                buf.insert(buf.end(), tmp, tmp + k);
                if (buf.size() > (1u << 20)) {
                    ok = std::fwrite(buf.data(), 1, buf.size(), fp) == buf.size();
                    buf.clear();
                }
            }
            ok = ok && std::fwrite(buf.data(), 1, buf.size(), fp) == buf.size();
        }
        ok = (std::fclose(fp) == 0) && ok;
        if (!ok) throw_runtime(std::string("write_observations: write failed for ") + path);
    });
}

}  // extern "C"
