// C++ engine layer over the C ABI (include/featurex_gpu/engine.hpp).
//
// Host plumbing kept from the reference engine's contract (engine.cpp:240-350):
// file pairing by basename + glob, PGM decoding, skip-and-log per failing pair,
// rows sorted by (image, label), CSV with "%.10g".  The per-pair featurization
// (accumulate + compute_roi_features for every label) is one fx_featurize call
// on the device.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <future>
#include <memory>
#include <thread>

#include "featurex_gpu/engine.hpp"
#include "fx_host.hpp"
#include "fxg.h"

namespace featurex {

namespace {

[[noreturn]] void throw_status(int rc) {
    const std::string msg = fx_last_error();
    switch (rc) {
        case FX_E_CONFIG: throw ConfigError(msg);
        case FX_E_UNKNOWN_PROFILE: throw UnknownProfile(msg);
        case FX_E_PAIRING: throw PairingError(msg);
        case FX_E_IO: throw IoError(msg);
        case FX_E_FORMAT: throw FormatError(msg);
        case FX_E_ZERO_MASS: throw ZeroMassError(msg);
        default: throw DeviceError("fx status " + std::to_string(rc) + ": " + msg);
    }
}

void check(int rc) {
    if (rc != FX_OK) throw_status(rc);
}

// one fx_ctx per (host thread, device); contexts are not thread-safe
struct CtxCache {
    std::map<int, fx_ctx*> ctx;
    ~CtxCache() {
        for (auto& kv : ctx) fx_ctx_destroy(kv.second);
    }
};

fx_ctx* context(int device) {
    thread_local CtxCache cache;
    auto it = cache.ctx.find(device);
    if (it != cache.ctx.end()) return it->second;
    fx_ctx* c = nullptr;
    check(fx_ctx_create(device, &c));
    cache.ctx[device] = c;
    return c;
}

// one fx_multi per (host thread, device list)
fx_multi* multi_context(const std::vector<int>& devices) {
    struct MultiCache {
        std::map<std::vector<int>, fx_multi*> m;
        ~MultiCache() {
            for (auto& kv : m) fx_multi_destroy(kv.second);
        }
    };
    thread_local MultiCache cache;
    auto it = cache.m.find(devices);
    if (it != cache.m.end()) return it->second;
    fx_multi* m = nullptr;
    check(fx_multi_create(devices.data(), static_cast<int>(devices.size()), &m));
    cache.m[devices] = m;
    return m;
}

fx_texture_params to_c(const TextureParams& p) {
    if (p.glcm.angles.size() > 8) throw ConfigError("at most 8 GLCM angles are supported");
    fx_texture_params t{};
    t.ng = p.glcm.ng;
    t.offset = p.glcm.offset;
    t.n_angles = static_cast<int>(p.glcm.angles.size());
    for (int i = 0; i < t.n_angles; ++i) t.angles[i] = p.glcm.angles[i];
    t.symmetric = p.glcm.symmetric ? 1 : 0;
    t.histogram_bins = p.histogram_bins;
    return t;
}

unsigned group_mask(const std::vector<std::string>& groups) {
    std::vector<const char*> names;
    for (const auto& g : groups) names.push_back(g.c_str());
    unsigned m = 0;
    check(fx_resolve_groups(names.data(), static_cast<int>(names.size()), &m));
    return m;
}

// File-name filter of run() (same language as the reference's: '*' matches any
// run of characters, '?' exactly one, everything else itself).  Dynamic
// programming over pattern prefixes: row[j] says whether the pattern prefix
// consumed so far matches name[0, j).
bool name_matches(const std::string& pat, const std::string& name) {
    std::vector<char> row(name.size() + 1, 0), next(name.size() + 1, 0);
    row[0] = 1;
    for (char pc : pat) {
        std::fill(next.begin(), next.end(), 0);
        if (pc == '*') {
            char any = 0;  // '*': reachable from any shorter prefix
            for (size_t j = 0; j <= name.size(); ++j) next[j] = any = any | row[j];
        } else {
            for (size_t j = 1; j <= name.size(); ++j)
                next[j] = row[j - 1] && (pc == '?' || pc == name[j - 1]);
        }
        row.swap(next);
    }
    return row[name.size()] != 0;
}

// CSV field: as is unless it holds a separator, quote or newline; then wrapped in
// quotes with every quote doubled (RFC 4180 style, as the reference writes names)
std::string csv_field(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string q;
    q.reserve(s.size() + 8);
    q.push_back('"');
    size_t from = 0;
    for (size_t at = s.find('"'); at != std::string::npos; at = s.find('"', from)) {
        q.append(s, from, at + 1 - from);
        q.push_back('"');
        from = at + 1;
    }
    q.append(s, from, std::string::npos);
    q.push_back('"');
    return q;
}

// ---- PGM P5 decode (pgm.cpp:37-99) -------------------------------------------
// Header parsed like the reference (whitespace and '#' comment lines between
// tokens, one whitespace byte after maxval); the payload is read with one fread
// straight into the destination and byte-swapped in place (BE16), or widened
// (8-bit).  Samples above maxval raise FormatError.

struct PgmInfo {
    int width = 0, height = 0, maxval = 0;
    std::streamoff offset = 0;  // payload start
    size_t elems() const { return static_cast<size_t>(width) * height; }
    bool wide() const { return maxval >= 256; }
};

int header_int(std::istream& in, const std::filesystem::path& path) {
    for (;;) {
        const int c = in.peek();
        if (c == EOF) throw FormatError("truncated PGM header: " + path.string());
        if (std::isspace(c)) {
            in.get();
        } else if (c == '#') {
            std::string skip;
            std::getline(in, skip);
        } else {
            break;
        }
    }
    long v = 0;
    if (!(in >> v) || v < 0) throw FormatError("bad PGM header value: " + path.string());
    return static_cast<int>(v);
}

PgmInfo read_pgm_header(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path.string());
    char m0 = 0, m1 = 0;
    in.get(m0);
    in.get(m1);
    if (!in || m0 != 'P') throw FormatError("not a PNM file: " + path.string());
    if (m1 != '5') throw FormatError(std::string("unsupported PNM magic P") + m1 + ": " + path.string());
    PgmInfo r;
    r.width = header_int(in, path);
    r.height = header_int(in, path);
    r.maxval = header_int(in, path);
    if (r.width < 1 || r.height < 1) throw FormatError("bad PGM dimensions: " + path.string());
    if (r.maxval < 1 || r.maxval > 65535) throw FormatError("bad PGM maxval: " + path.string());
    const int sep = in.get();
    if (sep == EOF || !std::isspace(sep)) throw FormatError("bad PGM header end: " + path.string());
    r.offset = in.tellg();
    return r;
}

struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};

// payload of a parsed PGM into dst[0 .. elems); returns the largest sample
uint16_t read_pgm_payload(const std::filesystem::path& path, const PgmInfo& h, uint16_t* dst) {
    std::unique_ptr<std::FILE, FileCloser> f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("cannot open " + path.string());
    if (std::fseek(f.get(), static_cast<long>(h.offset), SEEK_SET) != 0)
        throw FormatError("truncated PGM payload: " + path.string());
    const size_t n = h.elems();
    uint16_t mx = 0;
    if (h.wide()) {
        if (std::fread(dst, 2, n, f.get()) != n) throw FormatError("truncated PGM payload: " + path.string());
        for (size_t i = 0; i < n; ++i) {
            const uint16_t v = __builtin_bswap16(dst[i]);
            dst[i] = v;
            mx = v > mx ? v : mx;
        }
    } else {
        // widen from the back of the same buffer: byte i sits at offset n + i
        unsigned char* b = reinterpret_cast<unsigned char*>(dst) + n;
        if (std::fread(b, 1, n, f.get()) != n) throw FormatError("truncated PGM payload: " + path.string());
        for (size_t i = 0; i < n; ++i) {
            const uint16_t v = b[i];
            dst[i] = v;
            mx = v > mx ? v : mx;
        }
    }
    if (mx > h.maxval) throw FormatError("PGM sample exceeds maxval: " + path.string());
    return mx;
}

struct Raster {
    PgmInfo info;
    std::vector<uint16_t> samples;
};

Raster read_pgm(const std::filesystem::path& path) {
    Raster r;
    r.info = read_pgm_header(path);
    r.samples.resize(r.info.elems());
    read_pgm_payload(path, r.info, r.samples.data());
    return r;
}

// ---- host workers -------------------------------------------------------------

int host_workers(const ExtractionConfig& c) {
    if (!c.parallel) return 1;
    if (c.threads > 1) return c.threads;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

// fn(i) for i in [0, n) on up to `workers` threads (dynamic assignment)
template <class F>
void parallel_for(size_t n, int workers, F&& fn) {
    const size_t nt = std::min<size_t>(n, static_cast<size_t>(std::max(1, workers)));
    if (nt <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    auto body = [&]() {
        for (size_t i; (i = next.fetch_add(1)) < n;) fn(i);
    };
    std::vector<std::thread> ts;
    for (size_t t = 1; t < nt; ++t) ts.emplace_back(body);
    body();
    for (auto& t : ts) t.join();
}

// ---- CSV rows (engine.cpp:211-230): "%.10g" via std::to_chars(general, 10),
// which is specified as printf's %.*g in the C locale (checked against
// snprintf in tests/cpp/test_engine.cpp) and several times faster

// "%.10g" of a finite double from its exact binary value: v = m 2^e, D = the 10
// significant digits rounded half-to-even on the exact quotient (what glibc's
// printf does in the default rounding mode), in 128-bit integer arithmetic.
// Outside about 1e-13 .. 1e38, and for inf / nan, defers to std::to_chars.
char* fmt10g(char* p, char* end, double v) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const bool neg = bits >> 63;
    const int be = static_cast<int>((bits >> 52) & 0x7ff);
    uint64_t m = bits & ((uint64_t(1) << 52) - 1);
    if (be == 0x7ff) return std::to_chars(p, end, v, std::chars_format::general, 10).ptr;
    if (be == 0 && m == 0) {  // +-0
        if (neg) *p++ = '-';
        *p++ = '0';
        return p;
    }
    if (be == 0) return std::to_chars(p, end, v, std::chars_format::general, 10).ptr;  // subnormal
    m |= uint64_t(1) << 52;
    const int e = be - 1075;  // |v| = m 2^e
    static constexpr uint64_t kP10[20] = {1ull, 10ull, 100ull, 1000ull, 10000ull, 100000ull,
                                          1000000ull, 10000000ull, 100000000ull, 1000000000ull,
                                          10000000000ull, 100000000000ull, 1000000000000ull,
                                          10000000000000ull, 100000000000000ull,
                                          1000000000000000ull, 10000000000000000ull,
                                          100000000000000000ull, 1000000000000000000ull,
                                          10000000000000000000ull};
    using u128 = unsigned __int128;
    auto p10 = [&](int k) -> u128 {  // 10^k, k <= 38
        return k < 20 ? u128(kP10[k]) : u128(kP10[19]) * kP10[k - 19];
    };
    // decimal exponent estimate from the binary one, corrected below
    int X = static_cast<int>(std::floor((e + 52) * 0.30102999566398120));
    uint64_t D = 0;
    for (int attempt = 0; attempt < 3; ++attempt) {
        const int k = X - 9;  // D = round(|v| / 10^k)
        u128 q, r, den;
        bool ok = true;
        if (k <= 0) {
            if (-k > 22 || -e > 127) ok = false;
            else {
                const u128 num = u128(m) * p10(-k);
                if (e >= 0) {
                    if (e > 20) ok = false;  // |v| >= 1e10 never has k <= 0
                    else { q = num << e; r = 0; den = 1; }
                } else {
                    q = num >> -e;
                    r = num & ((u128(1) << -e) - 1);
                    den = u128(1) << -e;
                }
            }
        } else {
            if (k > 38) ok = false;
            else if (e >= 0) {
                if (e > 74) ok = false;
                else {
                    const u128 num = u128(m) << e;
                    den = p10(k);
                    q = num / den;
                    r = num - q * den;
                }
            } else {
                if (-e > 60 || k > 15) ok = false;
                else {
                    den = p10(k) << -e;
                    q = u128(m) / den;
                    r = u128(m) - q * den;
                }
            }
        }
        if (!ok) return std::to_chars(p, end, v, std::chars_format::general, 10).ptr;
        if (q >= u128(10000000000ull)) { ++X; continue; }
        if (q < u128(1000000000ull)) { --X; continue; }
        D = static_cast<uint64_t>(q);
        const u128 twice = r << 1;
        if (twice > den || (twice == den && (D & 1))) ++D;
        if (D == 10000000000ull) {
            D = 1000000000ull;
            ++X;
        }
        break;
    }
    if (D == 0) return std::to_chars(p, end, v, std::chars_format::general, 10).ptr;
    char dig[10];
    for (int i = 9; i >= 0; --i) {
        dig[i] = static_cast<char>('0' + D % 10);
        D /= 10;
    }
    int L = 10;
    while (L > 1 && dig[L - 1] == '0') --L;
    if (neg) *p++ = '-';
    if (X < -4 || X >= 10) {  // d[.ddd]e+-XX
        *p++ = dig[0];
        if (L > 1) {
            *p++ = '.';
            for (int i = 1; i < L; ++i) *p++ = dig[i];
        }
        *p++ = 'e';
        int ax = X;
        if (ax < 0) {
            *p++ = '-';
            ax = -ax;
        } else {
            *p++ = '+';
        }
        if (ax >= 100) {
            *p++ = static_cast<char>('0' + ax / 100);
            ax %= 100;
        }
        *p++ = static_cast<char>('0' + ax / 10);
        *p++ = static_cast<char>('0' + ax % 10);
    } else if (X >= 0) {  // integer part of X + 1 digits
        for (int i = 0; i <= X; ++i) *p++ = i < L ? dig[i] : '0';
        if (L > X + 1) {
            *p++ = '.';
            for (int i = X + 1; i < L; ++i) *p++ = dig[i];
        }
    } else {  // 0.000ddd
        *p++ = '0';
        *p++ = '.';
        for (int i = 0; i < -X - 1; ++i) *p++ = '0';
        for (int i = 0; i < L; ++i) *p++ = dig[i];
    }
    return p;
}

void append_rows(std::string& out, const std::string& prefix, const uint32_t* labels,
                 const double* values, size_t rows, size_t cols) {
    // worst case per value: ',' + sign + 10 digits + '.' + "e-308" = 19 bytes
    const size_t row_max = prefix.size() + 12 + cols * 20;
    size_t len = out.size();
    out.resize(len + rows * row_max);
    char* p = out.data() + len;
    for (size_t r = 0; r < rows; ++r) {
        char* const row_end = p + row_max;
        std::memcpy(p, prefix.data(), prefix.size());
        p += prefix.size();
        p = std::to_chars(p, row_end, labels[r]).ptr;
        const double* v = values + r * cols;
        for (size_t k = 0; k < cols; ++k) {
            *p++ = ',';
            p = fmt10g(p, row_end, v[k]);
        }
        *p++ = '\n';
    }
    out.resize(static_cast<size_t>(p - out.data()));
}

std::string csv_header(const std::vector<std::string>& columns) {
    std::string h = "image,mask,label";
    for (const auto& c : columns) h += "," + csv_field(c);
    return h + "\n";
}

// pinned host buffer from the C ABI (grow-only)
struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
    Pinned() = default;
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
    ~Pinned() { fx_host_free(p); }
    template <class T>
    T* get(size_t n) {
        const size_t need = n * sizeof(T);
        if (need > bytes) {
            fx_host_free(p);
            p = nullptr;
            bytes = 0;
            check(fx_host_alloc(need, &p));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
};


}  // namespace

TextureParams resolve_profile(const std::string& name) {
    fx_texture_params t{};
    check(fx_resolve_profile(name.c_str(), &t));
    TextureParams p;
    p.glcm.ng = t.ng;
    p.glcm.offset = t.offset;
    p.glcm.angles.assign(t.angles, t.angles + t.n_angles);
    p.glcm.symmetric = t.symmetric != 0;
    p.histogram_bins = t.histogram_bins;
    return p;
}

std::vector<std::string> resolve_feature_groups(const std::vector<std::string>& requested) {
    const unsigned m = group_mask(requested);
    static const char* kAll[7] = {"intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"};
    std::vector<std::string> out;
    for (int i = 0; i < 7; ++i)
        if (m & (1u << i)) out.push_back(kAll[i]);
    return out;
}

std::vector<std::string> feature_columns(const std::vector<std::string>& groups,
                                         const TextureParams& params) {
    const fx_texture_params t = to_c(params);
    const unsigned m = group_mask(groups);
    size_t need = 0;
    int n = 0;
    check(fx_columns(m, &t, nullptr, 0, &need, &n));
    std::string buf(need, '\0');
    check(fx_columns(m, &t, buf.data(), need, &need, &n));
    std::vector<std::string> cols;
    size_t start = 0;
    const std::string s(buf.c_str());
    while (!s.empty() && start <= s.size()) {
        const size_t nl = s.find('\n', start);
        cols.push_back(s.substr(start, nl == std::string::npos ? std::string::npos : nl - start));
        if (nl == std::string::npos) break;
        start = nl + 1;
    }
    return cols;
}

std::vector<double> compute_roi_features(const PixelCloud& cloud,
                                         const std::vector<std::string>& groups,
                                         const TextureParams& params) {
    const fx_texture_params t = to_c(params);
    const unsigned m = group_mask(groups);
    const size_t ncol = feature_columns(groups, params).size();
    std::vector<uint32_t> xs(cloud.count()), ys(cloud.count());
    std::vector<uint16_t> vs(cloud.count());
    for (size_t i = 0; i < cloud.count(); ++i) {
        xs[i] = cloud.pixels[i].x;
        ys[i] = cloud.pixels[i].y;
        vs[i] = cloud.pixels[i].intensity;
    }
    std::vector<double> out(std::max<size_t>(ncol, 1));
    check(fx_roi_features(context(0), xs.data(), ys.data(), vs.data(), xs.size(), m, &t, out.data(),
                          out.size()));
    out.resize(ncol);
    return out;
}

std::vector<std::vector<double>> compute_roi_features_batch(const std::vector<PixelCloud>& clouds,
                                                            const std::vector<std::string>& groups,
                                                            const TextureParams& params) {
    const fx_texture_params t = to_c(params);
    const unsigned m = group_mask(groups);
    const size_t ncol = feature_columns(groups, params).size();
    std::vector<size_t> offsets(clouds.size() + 1, 0);
    for (size_t k = 0; k < clouds.size(); ++k) offsets[k + 1] = offsets[k] + clouds[k].count();
    std::vector<uint32_t> xs(offsets.back()), ys(offsets.back());
    std::vector<uint16_t> vs(offsets.back());
    for (size_t k = 0; k < clouds.size(); ++k)
        for (size_t i = 0; i < clouds[k].count(); ++i) {
            xs[offsets[k] + i] = clouds[k].pixels[i].x;
            ys[offsets[k] + i] = clouds[k].pixels[i].y;
            vs[offsets[k] + i] = clouds[k].pixels[i].intensity;
        }
    std::vector<double> flat(std::max<size_t>(clouds.size() * ncol, 1));
    check(fx_roi_features_batch(context(0), xs.data(), ys.data(), vs.data(), offsets.data(),
                                clouds.size(), m, &t, flat.data(), clouds.size()));
    std::vector<std::vector<double>> out(clouds.size());
    for (size_t k = 0; k < clouds.size(); ++k)
        out[k].assign(flat.begin() + k * ncol, flat.begin() + (k + 1) * ncol);
    return out;
}

std::vector<RowTile> iter_row_tiles(const IntensityImage& image, const LabelMask& mask,
                                    int rows_per_tile) {
    if (image.width != mask.width || image.height != mask.height)
        throw PairingError("image/mask dimension mismatch");
    if (rows_per_tile < 1) throw PairingError("rows_per_tile must be >= 1");
    std::vector<RowTile> tiles;
    const size_t w = static_cast<size_t>(image.width);
    for (int y = 0; y < image.height; y += rows_per_tile) {
        const int rows = std::min(rows_per_tile, image.height - y);
        const size_t at = static_cast<size_t>(y) * w, len = static_cast<size_t>(rows) * w;
        tiles.push_back(RowTile{y, rows, image.width,
                                std::span<const uint16_t>(image.pixels.data() + at, len),
                                std::span<const uint16_t>(mask.labels.data() + at, len)});
    }
    return tiles;
}

RoiRegistry RoiRegistry::accumulate(const std::vector<RowTile>& tiles, const MemoryBudget&) {
    RoiRegistry reg;
    if (tiles.empty()) return reg;
    // the tiles' rows as one raster: in place when they are consecutive views of
    // one image (iter_row_tiles), else gathered into a contiguous copy
    const int W = tiles.front().width;
    int H = 0;
    bool contiguous = true;
    for (size_t k = 0; k < tiles.size(); ++k) {
        const RowTile& t = tiles[k];
        if (t.width != W) throw PairingError("tiles of different widths");
        if (t.y0 != H) throw PairingError("tiles are not consecutive row bands");
        if (k && (t.labels.data() != tiles[k - 1].labels.data() + tiles[k - 1].labels.size() ||
                  t.intensity.data() != tiles[k - 1].intensity.data() + tiles[k - 1].intensity.size()))
            contiguous = false;
        H += t.rows;
    }
    if (H == 0 || W == 0) return reg;
    std::vector<uint16_t> I, L;
    const uint16_t *pi = tiles.front().intensity.data(), *pl = tiles.front().labels.data();
    if (!contiguous) {
        for (const RowTile& t : tiles) {
            I.insert(I.end(), t.intensity.begin(), t.intensity.end());
            L.insert(L.end(), t.labels.begin(), t.labels.end());
        }
        pi = I.data();
        pl = L.data();
    }
    fx_image im{pi, pl, W, H, static_cast<size_t>(W), 0, 0, FX_MEM_HOST};
    fx_ctx* c = context(0);
    size_t nr = 0, np = 0;
    check(fx_roi_clouds(c, &im, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, &nr, &np));
    std::vector<uint32_t> xs(std::max<size_t>(np, 1)), ys(std::max<size_t>(np, 1)), bb(4 * std::max<size_t>(nr, 1));
    std::vector<uint16_t> vs(std::max<size_t>(np, 1));
    reg.labels_.resize(std::max<size_t>(nr, 1));
    reg.offsets_.resize(nr + 1);
    check(fx_roi_clouds(c, &im, reg.labels_.data(), reg.offsets_.data(), bb.data(), nr, xs.data(), ys.data(),
                        vs.data(), np, &nr, &np));
    reg.labels_.resize(nr);
    reg.bboxes_.resize(nr);
    for (size_t i = 0; i < nr; ++i) reg.bboxes_[i] = BoundingBox{bb[4 * i], bb[4 * i + 1], bb[4 * i + 2], bb[4 * i + 3]};
    reg.pixels_.resize(np);
    for (size_t k = 0; k < np; ++k) reg.pixels_[k] = Pixel{xs[k], ys[k], vs[k]};
    return reg;
}

bool RoiRegistry::contains(uint32_t label) const {
    return std::binary_search(labels_.begin(), labels_.end(), label);
}

PixelCloud RoiRegistry::cloud(uint32_t label) const {
    const auto it = std::lower_bound(labels_.begin(), labels_.end(), label);
    if (it == labels_.end() || *it != label)
        throw std::out_of_range("unknown ROI label " + std::to_string(label));
    const size_t i = static_cast<size_t>(it - labels_.begin());
    PixelCloud c;
    c.label = label;
    c.bbox = bboxes_[i];
    c.pixels.assign(pixels_.begin() + static_cast<std::ptrdiff_t>(offsets_[i]),
                    pixels_.begin() + static_cast<std::ptrdiff_t>(offsets_[i + 1]));
    return c;
}

FeatureTable featurize(const IntensityImage& image, const LabelMask& mask,
                       const std::vector<std::string>& groups, const TextureParams& params,
                       int device) {
    if (image.width != mask.width || image.height != mask.height)
        throw PairingError("image/mask dimension mismatch");  // image.cpp:9-11
    FeatureTable t;
    t.columns = feature_columns(groups, params);
    const fx_texture_params tp = to_c(params);
    const unsigned m = group_mask(groups);
    std::vector<bool> seen(65536, false);
    size_t cap = 0;
    for (uint16_t l : mask.labels)
        if (l && !seen[l]) {
            seen[l] = true;
            ++cap;
        }
    t.labels.resize(std::max<size_t>(cap, 1));
    t.values.resize(std::max<size_t>(cap, 1) * std::max<size_t>(t.columns.size(), 1));
    fx_image im{image.pixels.data(), mask.labels.data(), image.width, image.height,
                static_cast<size_t>(image.width), 0, 0, FX_MEM_HOST};
    size_t n = 0;
    check(fx_featurize(context(device), &im, m, &tp, t.labels.data(), t.values.data(), cap, &n));
    t.labels.resize(n);
    t.values.resize(n * t.columns.size());
    return t;
}

IntensityImage load_intensity(const std::filesystem::path& path) {
    Raster r = read_pgm(path);
    IntensityImage img;
    img.width = r.info.width;
    img.height = r.info.height;
    img.bit_depth = r.info.maxval < 256 ? 8 : 16;
    img.pixels = std::move(r.samples);
    return img;
}

LabelMask load_mask(const std::filesystem::path& path) {
    Raster r = read_pgm(path);
    LabelMask m;
    m.width = r.info.width;
    m.height = r.info.height;
    m.labels = std::move(r.samples);
    return m;
}

void write_pgm(const std::filesystem::path& path, int width, int height, int maxval,
               const std::vector<uint16_t>& samples) {
    if (width < 1 || height < 1 || maxval < 1 || maxval > 65535)
        throw FormatError("bad PGM write parameters: " + path.string());
    if (samples.size() != static_cast<size_t>(width) * height)
        throw FormatError("sample count mismatch: " + path.string());
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot create " + path.string());
    out << "P5\n" << width << " " << height << "\n" << maxval << "\n";
    for (uint16_t v : samples) {
        if (maxval >= 256) {
            const char b[2] = {static_cast<char>(v >> 8), static_cast<char>(v & 0xff)};
            out.write(b, 2);
        } else {
            const char b = static_cast<char>(v);
            out.write(&b, 1);
        }
    }
    if (!out) throw IoError("write failed: " + path.string());
}

size_t write_csv(const std::vector<std::string>& columns, std::vector<FeatureRow> rows,
                 const std::filesystem::path& path) {
    std::sort(rows.begin(), rows.end(), [](const FeatureRow& a, const FeatureRow& b) {
        if (a.image_name != b.image_name) return a.image_name < b.image_name;
        return a.roi_label < b.roi_label;
    });
    std::unique_ptr<std::FILE, FileCloser> f(std::fopen(path.c_str(), "wb"));
    if (!f) throw IoError("cannot create " + path.string());
    const std::string head = csv_header(columns);
    bool ok = std::fwrite(head.data(), 1, head.size(), f.get()) == head.size();
    // rows formatted in parallel chunks, written in order
    constexpr size_t kChunk = 2048;
    const size_t nchunks = (rows.size() + kChunk - 1) / kChunk;
    std::vector<std::string> text(nchunks);
    const unsigned hw = std::thread::hardware_concurrency();
    parallel_for(nchunks, hw ? static_cast<int>(hw) : 1, [&](size_t c) {
        std::string& out = text[c];
        for (size_t i = c * kChunk; i < std::min(rows.size(), (c + 1) * kChunk); ++i) {
            const FeatureRow& r = rows[i];
            append_rows(out, csv_field(r.image_name) + "," + csv_field(r.mask_name) + ",",
                        &r.roi_label, r.values.data(), 1, r.values.size());
        }
    });
    for (const std::string& t : text) ok = ok && std::fwrite(t.data(), 1, t.size(), f.get()) == t.size();
    if (!ok || std::fflush(f.get()) != 0) throw IoError("write failed: " + path.string());
    return rows.size();
}

// run (engine.cpp:283-350) as a pipeline over the paired files, in name order:
//   1. headers of every pair (parallel); header / pairing errors skip the pair
//   2. batches of <= kBatchPairs pairs / kBatchBytes of rasters; the host workers
//      decode batch k+1 into page-locked buffers while the device featurizes
//      batch k (fx_featurize_batch: double-buffered H2D on its copy stream,
//      one label-table slot per image) and formats batch k-1's rows
//   3. rows leave the device sorted (pairs in name order, labels ascending per
//      pair), so the CSV is written in order without a sort
// A pair that fails to decode is logged and skipped; a failing batch is re-run
// pair by pair so the failure is charged to the pair that caused it.
RunSummary run(const ExtractionConfig& config) {
    const auto t0 = std::chrono::steady_clock::now();
    if (config.threads < 1) throw ConfigError("threads must be >= 1");
    const std::vector<std::string> groups = resolve_feature_groups(config.features);
    TextureParams params = resolve_profile(config.profile);
    if (config.glcm_override) params.glcm = *config.glcm_override;
    if (config.histogram_bins_override) params.histogram_bins = *config.histogram_bins_override;
    if (config.memory_budget == 0) throw ConfigError("memory budget must be positive");
    // spill_dir / FEATUREX_SPILL_DIR are accepted and unused: ROI data lives in HBM
    const int workers = host_workers(config);

    RunSummary summary;
    // pairing by identical basename (engine.cpp:240-272): both directories listed
    // into name-sorted maps, then one merge walk; an unmatched name is logged and
    // counted as a failed pair
    auto list_dir = [&](const std::filesystem::path& dir) {
        if (!std::filesystem::is_directory(dir)) throw IoError("not a directory: " + dir.string());
        std::map<std::string, std::filesystem::path> found;
        for (const auto& e : std::filesystem::directory_iterator(dir))
            if (e.is_regular_file() && name_matches(config.file_pattern, e.path().filename().string()))
                found.emplace(e.path().filename().string(), e.path());
        return found;
    };
    const auto ints = list_dir(config.intensity_dir);
    const auto masks = list_dir(config.mask_dir);
    struct Pair {
        std::string name;
        std::filesystem::path ip, mp;
        PgmInfo hi, hm;
        std::string error;  // non-empty: skipped
        uint16_t maxlab = 0;
    };
    std::vector<Pair> pairs;
    std::vector<std::string> lone_masks;
    for (auto i = ints.begin(), k = masks.begin(); i != ints.end() || k != masks.end();) {
        if (k == masks.end() || (i != ints.end() && i->first < k->first)) {
            std::cerr << "featurex: no mask for image '" << i->first << "', skipped\n";
            ++summary.failed_pairs;
            ++i;
        } else if (i == ints.end() || k->first < i->first) {
            lone_masks.push_back(k->first);
            ++k;
        } else {
            pairs.push_back(Pair{i->first, i->second, k->second, {}, {}, {}, 0});
            ++i;
            ++k;
        }
    }
    for (const auto& name : lone_masks) {  // reported after the images, as the reference
        std::cerr << "featurex: no image for mask '" << name << "', skipped\n";
        ++summary.failed_pairs;
    }
    const fx_texture_params tp = to_c(params);
    const unsigned gm = group_mask(groups);
    const std::vector<std::string> columns = feature_columns(groups, params);
    const size_t nc = columns.size();

    // 1. headers
    parallel_for(pairs.size(), workers, [&](size_t i) {
        Pair& q = pairs[i];
        try {
            if (config.rows_per_tile < 1) throw PairingError("rows_per_tile must be >= 1");
            q.hi = read_pgm_header(q.ip);
            q.hm = read_pgm_header(q.mp);
            if (q.hi.width != q.hm.width || q.hi.height != q.hm.height)
                throw PairingError("image/mask dimension mismatch");  // image.cpp:9-11
        } catch (const std::exception& e) {
            q.error = e.what();
        }
    });
    std::vector<size_t> good;
    for (size_t i = 0; i < pairs.size(); ++i) {
        if (pairs[i].error.empty()) {
            good.push_back(i);
        } else {
            std::cerr << "featurex: pair '" << pairs[i].name << "' failed: " << pairs[i].error << "\n";
            ++summary.failed_pairs;
        }
    }

    // 2. batch plan
    // several devices (ExtractionConfig::devices): batches N times larger, dealt
    // over the devices in chunks by fx_multi_featurize_batch
    const std::vector<int> devs = config.devices.empty() ? std::vector<int>{config.device} : config.devices;
    const size_t scale = devs.size();
    const size_t kBatchPairs = 128 * scale, kBatchBytes = (size_t(256) << 20) * scale;
    std::vector<std::pair<size_t, size_t>> plan;  // [begin, end) into good
    {
        size_t b = 0, bytes = 0;
        for (size_t j = 0; j < good.size(); ++j) {
            const size_t e = pairs[good[j]].hi.elems() * 4;
            if (j > b && (j - b == kBatchPairs || bytes + e > kBatchBytes)) {
                plan.emplace_back(b, j);
                b = j;
                bytes = 0;
            }
            bytes += e;
        }
        if (b < good.size()) plan.emplace_back(b, good.size());
    }
    // two slots of page-locked buffers (rasters in, table out); per-batch
    // bookkeeping lives in Batch so batch k+1's decode never touches what
    // batch k-1's formatting still reads
    struct Slot {
        Pinned I, L, lab, val;
    };
    struct Batch {
        std::vector<size_t> elem_off;
        std::vector<size_t> members;  // indices into good of the pairs decoded OK
        std::vector<size_t> offsets;  // row offsets per member (+ total)
        size_t cap = 0;
    };
    Slot slots[2];
    std::vector<Batch> batches(plan.size());
    std::atomic<int> failed{0};
    std::atomic<size_t> images{0}, rois{0};
    auto fail_logged = [&](Pair& q) {
        std::cerr << "featurex: pair '" << q.name << "' failed: " << q.error << "\n";
        failed.fetch_add(1);
    };
    auto decode = [&](size_t k) {
        Slot& sl = slots[k % 2];
        Batch& bt = batches[k];
        const auto [b, e] = plan[k];
        bt.elem_off.assign(e - b + 1, 0);
        for (size_t j = b; j < e; ++j) bt.elem_off[j - b + 1] = bt.elem_off[j - b] + pairs[good[j]].hi.elems();
        uint16_t* I = sl.I.get<uint16_t>(bt.elem_off.back());
        uint16_t* L = sl.L.get<uint16_t>(bt.elem_off.back());
        parallel_for(e - b, workers, [&](size_t t) {
            Pair& q = pairs[good[b + t]];
            try {
                read_pgm_payload(q.ip, q.hi, I + bt.elem_off[t]);
                q.maxlab = read_pgm_payload(q.mp, q.hm, L + bt.elem_off[t]);
            } catch (const std::exception& ex) {
                q.error = ex.what();
            }
        });
        for (size_t j = b; j < e; ++j) {
            Pair& q = pairs[good[j]];
            if (!q.error.empty()) {
                fail_logged(q);
                continue;
            }
            bt.members.push_back(j);
            bt.cap += std::min<size_t>(q.maxlab, q.hi.elems());
        }
    };
    auto featurize_batch = [&](size_t k) {
        Slot& sl = slots[k % 2];
        Batch& bt = batches[k];
        const size_t b = plan[k].first;
        std::vector<fx_image> ims;
        for (size_t j : bt.members) {
            const Pair& q = pairs[good[j]];
            const size_t o = bt.elem_off[j - b];
            ims.push_back(fx_image{static_cast<uint16_t*>(sl.I.p) + o, static_cast<uint16_t*>(sl.L.p) + o,
                                   q.hi.width, q.hi.height, static_cast<size_t>(q.hi.width), 0, 0,
                                   FX_MEM_HOST});
        }
        bt.offsets.assign(ims.size() + 1, 0);
        if (ims.empty()) return;
        fx_ctx* ctx = context(devs.front());
        fx_multi* multi = devs.size() > 1 ? multi_context(devs) : nullptr;
        auto call = [&](const fx_image* im, int n, size_t* offs, size_t cap_hint) -> int {
            size_t cap = std::max<size_t>(cap_hint, 1);
            for (;;) {
                uint32_t* lab = sl.lab.get<uint32_t>(cap);
                double* val = sl.val.get<double>(cap * std::max<size_t>(nc, 1));
                const int rc = multi && n > 1 ? fx_multi_featurize_batch(multi, im, n, gm, &tp, lab, val, cap, offs)
                                              : fx_featurize_batch(ctx, im, n, gm, &tp, lab, val, cap, offs);
                if (rc != FX_E_CAPACITY) return rc;
                cap = std::max(cap * 2, offs[n]);
            }
        };
        const int rc = call(ims.data(), static_cast<int>(ims.size()), bt.offsets.data(), bt.cap);
        if (rc == FX_OK) return;
        // re-run pair by pair to charge the failure to its pair
        std::vector<size_t> kept;
        std::vector<fx_image> keep_ims;
        for (size_t t = 0; t < ims.size(); ++t) {
            size_t offs[2] = {0, 0};
            const int r1 = call(&ims[t], 1, offs, 1);
            if (r1 == FX_OK) {
                kept.push_back(bt.members[t]);
                keep_ims.push_back(ims[t]);
            } else {
                Pair& q = pairs[good[bt.members[t]]];
                try {
                    throw_status(r1);
                } catch (const std::exception& ex) {
                    q.error = ex.what();
                }
                fail_logged(q);
            }
        }
        bt.members = kept;
        bt.offsets.assign(keep_ims.size() + 1, 0);
        if (!keep_ims.empty())
            check(call(keep_ims.data(), static_cast<int>(keep_ims.size()), bt.offsets.data(), bt.cap));
    };

    std::unique_ptr<std::FILE, FileCloser> out(std::fopen(config.output_path.c_str(), "wb"));
    if (!out) throw IoError("cannot create " + config.output_path.string());
    const std::string head = csv_header(columns);
    std::atomic<bool> ok{std::fwrite(head.data(), 1, head.size(), out.get()) == head.size()};
    // format + write of batch k: rows formatted on the host workers, appended
    // after batch k-1's text (the chained future keeps the file in order)
    auto format_write = [&](size_t k, std::shared_future<void> prev) {
        Slot& sl = slots[k % 2];
        Batch& bt = batches[k];
        const size_t m = bt.members.size();
        std::vector<std::string> parts(m);
        const uint32_t* lab = static_cast<const uint32_t*>(sl.lab.p);
        const double* val = static_cast<const double*>(sl.val.p);
        parallel_for(m, workers, [&](size_t t) {
            const Pair& q = pairs[good[bt.members[t]]];
            const size_t r0 = bt.offsets[t], r1 = bt.offsets[t + 1];
            append_rows(parts[t], csv_field(q.name) + "," + csv_field(q.name) + ",", lab + r0,
                        val + r0 * nc, r1 - r0, nc);
        });
        images.fetch_add(m);
        rois.fetch_add(m ? bt.offsets[m] : 0);
        if (prev.valid()) prev.get();
        for (const std::string& t : parts)
            if (std::fwrite(t.data(), 1, t.size(), out.get()) != t.size()) ok = false;
    };
    // FX_RUN_PROFILE=1: per-stage wall seconds on stderr
    const bool prof = std::getenv("FX_RUN_PROFILE") != nullptr;
    double t_feat = 0, t_wait_dec = 0, t_wait_fmt = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto x, auto y) { return std::chrono::duration<double>(y - x).count(); };
    std::future<void> dec;            // decode of the next batch
    std::shared_future<void> fw[2];   // format + write of the batch last featurized in slot
    std::shared_future<void> last;
    if (!plan.empty()) dec = std::async(std::launch::async, [&] { decode(0); });
    for (size_t k = 0; k < plan.size(); ++k) {
        auto t1 = now();
        dec.get();                                // batch k decoded
        if (fw[k % 2].valid()) fw[k % 2].get();   // batch k-2's table read: slot k%2 free
        auto t2 = now();
        featurize_batch(k);
        auto t3 = now();
        if (k + 1 < plan.size()) dec = std::async(std::launch::async, [&, k] { decode(k + 1); });
        last = fw[k % 2] = std::async(std::launch::async, format_write, k, last).share();
        t_wait_dec += secs(t1, t2);
        t_feat += secs(t2, t3);
    }
    auto t4 = now();
    if (last.valid()) last.get();
    for (auto& f : fw)
        if (f.valid()) f.get();
    t_wait_fmt = secs(t4, now());
    if (prof)
        std::fprintf(stderr, "fx_run: %zu batches, featurize %.3f s, waits: decode/slot %.3f s, "
                     "format+write tail %.3f s\n", plan.size(), t_feat, t_wait_dec, t_wait_fmt);
    if (!ok || std::fflush(out.get()) != 0) throw IoError("write failed: " + config.output_path.string());
    summary.failed_pairs += failed.load();
    summary.images = static_cast<int>(images.load());
    summary.rois = rois.load();
    summary.rows = summary.rois;
    summary.elapsed_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return summary;
}

}  // namespace featurex

// C ABI over run() (include/fxg.h), for non-C++ callers
extern "C" int fx_run(const char* intensity_dir, const char* mask_dir, const char* pattern,
                      const char* groups_csv, const char* profile, int threads, int parallel,
                      int device, const char* output_path, fx_run_summary* out) {
    if (!intensity_dir || !mask_dir || !groups_csv || !profile || !output_path || !out)
        return fxg::set_error(FX_E_ARG, "null argument");
    try {
        featurex::ExtractionConfig c;
        c.intensity_dir = intensity_dir;
        c.mask_dir = mask_dir;
        if (pattern && *pattern) c.file_pattern = pattern;
        c.features.clear();
        std::string g = groups_csv;
        for (size_t a = 0; a <= g.size();) {
            const size_t b = std::min(g.find(',', a), g.size());
            if (b > a) c.features.push_back(g.substr(a, b - a));
            a = b + 1;
        }
        c.profile = profile;
        c.threads = threads;
        c.parallel = parallel != 0;
        c.device = device;
        c.output_path = output_path;
        const featurex::RunSummary s = featurex::run(c);
        out->images = s.images;
        out->rois = s.rois;
        out->rows = s.rows;
        out->elapsed_seconds = s.elapsed_seconds;
        out->failed_pairs = s.failed_pairs;
        return FX_OK;
    } catch (const featurex::ConfigError& e) {
        return fxg::set_error(FX_E_CONFIG, e.what());
    } catch (const featurex::UnknownProfile& e) {
        return fxg::set_error(FX_E_UNKNOWN_PROFILE, e.what());
    } catch (const featurex::IoError& e) {
        return fxg::set_error(FX_E_IO, e.what());
    } catch (const featurex::FormatError& e) {
        return fxg::set_error(FX_E_FORMAT, e.what());
    } catch (const featurex::PairingError& e) {
        return fxg::set_error(FX_E_PAIRING, e.what());
    } catch (const featurex::DeviceError& e) {
        return fxg::set_error(FX_E_CUDA, e.what());
    } catch (const std::exception& e) {
        return fxg::set_error(FX_E_INTERNAL, e.what());
    }
}
