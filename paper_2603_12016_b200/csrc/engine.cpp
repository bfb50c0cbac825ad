// C++ engine layer over the C ABI (include/featurex_gpu/engine.hpp).
//
// Host plumbing kept from the reference engine's contract (engine.cpp:240-350):
// file pairing by basename + glob, PGM decoding, skip-and-log per failing pair,
// rows sorted by (image, label), CSV with "%.10g".  The per-pair featurization
// (accumulate + compute_roi_features for every label) is one fx_featurize call
// on the device.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>

#include "featurex_gpu/engine.hpp"
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

bool glob_match(const std::string& pattern, const std::string& name) {  // '*' and '?'
    size_t p = 0, n = 0, star = std::string::npos, mark = 0;
    while (n < name.size()) {
        if (p < pattern.size() && (pattern[p] == '?' || pattern[p] == name[n])) {
            ++p;
            ++n;
        } else if (p < pattern.size() && pattern[p] == '*') {
            star = p++;
            mark = n;
        } else if (star != std::string::npos) {
            p = star + 1;
            n = ++mark;
        } else {
            return false;
        }
    }
    while (p < pattern.size() && pattern[p] == '*') ++p;
    return p == pattern.size();
}

std::string csv_field(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string out = "\"";
    for (char ch : s) {
        if (ch == '"') out += '"';
        out += ch;
    }
    return out + "\"";
}

struct Raster {
    int width = 0, height = 0, maxval = 0;
    std::vector<uint16_t> samples;
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

Raster read_pgm(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path.string());
    char m0 = 0, m1 = 0;
    in.get(m0);
    in.get(m1);
    if (!in || m0 != 'P') throw FormatError("not a PNM file: " + path.string());
    if (m1 != '5') throw FormatError(std::string("unsupported PNM magic P") + m1 + ": " + path.string());
    Raster r;
    r.width = header_int(in, path);
    r.height = header_int(in, path);
    r.maxval = header_int(in, path);
    if (r.width < 1 || r.height < 1) throw FormatError("bad PGM dimensions: " + path.string());
    if (r.maxval < 1 || r.maxval > 65535) throw FormatError("bad PGM maxval: " + path.string());
    const int sep = in.get();
    if (sep == EOF || !std::isspace(sep)) throw FormatError("bad PGM header end: " + path.string());
    const size_t n = static_cast<size_t>(r.width) * r.height;
    const bool wide = r.maxval >= 256;
    std::vector<unsigned char> buf(n * (wide ? 2 : 1));
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    if (static_cast<size_t>(in.gcount()) != buf.size())
        throw FormatError("truncated PGM payload: " + path.string());
    r.samples.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const uint16_t v = wide ? static_cast<uint16_t>((buf[2 * i] << 8) | buf[2 * i + 1]) : buf[i];
        if (v > r.maxval) throw FormatError("PGM sample exceeds maxval: " + path.string());
        r.samples[i] = v;
    }
    return r;
}

std::filesystem::path spill_dir_of(const ExtractionConfig& c) {  // engine.cpp:274-279
    if (const char* env = std::getenv("FEATUREX_SPILL_DIR"); env && *env) return env;
    if (!c.spill_dir.empty()) return c.spill_dir;
    return std::filesystem::temp_directory_path() / "featurex-spill";
}

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
    img.width = r.width;
    img.height = r.height;
    img.bit_depth = r.maxval < 256 ? 8 : 16;
    img.pixels = std::move(r.samples);
    return img;
}

LabelMask load_mask(const std::filesystem::path& path) {
    Raster r = read_pgm(path);
    LabelMask m;
    m.width = r.width;
    m.height = r.height;
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
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot create " + path.string());
    out << "image,mask,label";
    for (const auto& c : columns) out << "," << csv_field(c);
    out << "\n";
    char buf[40];
    for (const FeatureRow& r : rows) {
        out << csv_field(r.image_name) << "," << csv_field(r.mask_name) << "," << r.roi_label;
        for (double v : r.values) {
            std::snprintf(buf, sizeof buf, "%.10g", v);
            out << "," << buf;
        }
        out << "\n";
    }
    if (!out) throw IoError("write failed: " + path.string());
    return rows.size();
}

RunSummary run(const ExtractionConfig& config) {
    const auto t0 = std::chrono::steady_clock::now();
    if (config.threads < 1) throw ConfigError("threads must be >= 1");
    const std::vector<std::string> groups = resolve_feature_groups(config.features);
    TextureParams params = resolve_profile(config.profile);
    if (config.glcm_override) params.glcm = *config.glcm_override;
    if (config.histogram_bins_override) params.histogram_bins = *config.histogram_bins_override;
    if (config.memory_budget == 0) throw ConfigError("memory budget must be positive");
    (void)spill_dir_of(config);  // no host spill: ROI data lives in HBM

    RunSummary summary;
    // pairing by identical basename (engine.cpp:240-272)
    std::map<std::string, std::filesystem::path> ints, masks;
    auto scan = [&](const std::filesystem::path& dir, std::map<std::string, std::filesystem::path>& into) {
        if (!std::filesystem::is_directory(dir)) throw IoError("not a directory: " + dir.string());
        for (const auto& e : std::filesystem::directory_iterator(dir)) {
            if (!e.is_regular_file()) continue;
            const std::string name = e.path().filename().string();
            if (glob_match(config.file_pattern, name)) into[name] = e.path();
        }
    };
    scan(config.intensity_dir, ints);
    scan(config.mask_dir, masks);
    std::vector<std::string> pairs;
    for (const auto& [name, p] : ints) {
        if (!masks.count(name)) {
            std::cerr << "featurex: no mask for image '" << name << "', skipped\n";
            ++summary.failed_pairs;
            continue;
        }
        pairs.push_back(name);
    }
    for (const auto& [name, p] : masks)
        if (!ints.count(name)) {
            std::cerr << "featurex: no image for mask '" << name << "', skipped\n";
            ++summary.failed_pairs;
        }

    const std::vector<std::string> columns = feature_columns(groups, params);
    std::vector<FeatureRow> rows;
    for (const std::string& name : pairs) {
        try {
            const IntensityImage image = load_intensity(ints[name]);
            const LabelMask mask = load_mask(masks[name]);
            if (config.rows_per_tile < 1) throw PairingError("rows_per_tile must be >= 1");
            const FeatureTable t = featurize(image, mask, groups, params, config.device);
            const size_t nc = t.columns.size();
            for (size_t i = 0; i < t.labels.size(); ++i)
                rows.push_back({name, name, t.labels[i],
                                std::vector<double>(t.values.begin() + i * nc,
                                                    t.values.begin() + (i + 1) * nc)});
            summary.rois += t.labels.size();
            summary.images += 1;
        } catch (const std::exception& e) {
            std::cerr << "featurex: pair '" << name << "' failed: " << e.what() << "\n";
            summary.failed_pairs += 1;
        }
    }
    summary.rows = write_csv(columns, std::move(rows), config.output_path);
    summary.elapsed_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return summary;
}

}  // namespace featurex
