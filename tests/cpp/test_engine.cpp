// C++ engine-layer tests, re-expressing the reference's engine contract tests
// (/root/reference/proj/tests/test_engine.cpp:60-227) against the drop-in
// header include/featurex_gpu/engine.hpp.  Built and run by tests/test_engine_cpp.py.
//   ./test_engine            all cases (needs a B200)
//   ./test_engine --host     host-only cases (profiles, groups, columns, CSV)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>

#include "featurex_gpu/engine.hpp"

using namespace featurex;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)          \
    do {                                  \
        bool ok_ = false;                 \
        try {                             \
            expr;                         \
        } catch (const T&) {              \
            ok_ = true;                   \
        } catch (...) {                   \
        }                                 \
        CHECK(ok_ && #T);                 \
    } while (0)

static std::filesystem::path fresh_dir(const std::string& name) {
    const auto d = std::filesystem::temp_directory_path() / name;
    std::filesystem::remove_all(d);
    std::filesystem::create_directories(d / "int");
    std::filesystem::create_directories(d / "seg");
    return d;
}

static std::string slurp(const std::filesystem::path& p) {
    std::ifstream in(p, std::ios::binary);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

static void write_simple_pair(const std::filesystem::path& d) {  // test_engine.cpp:30-35
    write_pgm(d / "int" / "a.pgm", 4, 4, 255,
              {10, 20, 30, 40, 50, 60, 70, 80, 90, 100, 110, 120, 130, 140, 150, 160});
    write_pgm(d / "seg" / "a.pgm", 4, 4, 255, {1, 1, 0, 0, 1, 1, 0, 0, 0, 0, 2, 2, 0, 0, 2, 2});
}

static void host_cases() {
    CHECK(resolve_profile("performance").glcm.angles.size() == 1);
    CHECK(resolve_profile("default").glcm.ng == 64);
    CHECK(resolve_profile("ibsi-like").glcm.ng == 256 && resolve_profile("ibsi-like").glcm.symmetric);
    CHECK_THROWS_AS(resolve_profile("bogus"), UnknownProfile);
    CHECK_THROWS_AS(resolve_feature_groups({"intensity", "nope"}), ConfigError);
    CHECK_THROWS_AS(resolve_feature_groups({}), ConfigError);
    CHECK(resolve_feature_groups({"*ALL*"}).size() == 7);
    CHECK((resolve_feature_groups({"shape", "intensity"}) == std::vector<std::string>{"intensity", "shape"}));
    TextureParams p = resolve_profile("performance");
    auto cols = feature_columns({"glcm"}, p);
    CHECK(cols.size() == 58 && cols[0] == "glcm_asm_0" && cols[1] == "glcm_asm_ave");
    CHECK(feature_columns({"glcm"}, resolve_profile("default")).size() == 145);
    CHECK(feature_columns({"*ALL*"}, resolve_profile("default")).size() == 427);
    const auto path = std::filesystem::temp_directory_path() / "fxg_csv.csv";  // :135-152
    CHECK(write_csv({"x"}, {}, path) == 0);
    CHECK(slurp(path) == "image,mask,label,x\n");
    write_csv({"x"}, {{"a.pgm", "a.pgm", 2, {1.0}}, {"a.pgm", "a.pgm", 1, {2.0}}}, path);
    CHECK(slurp(path) == "image,mask,label,x\na.pgm,a.pgm,1,2\na.pgm,a.pgm,2,1\n");
    write_csv({"x"}, {{"a", "a", 1, {1.0 / 3.0}}}, path);
    CHECK(slurp(path) == "image,mask,label,x\na,a,1,0.3333333333\n");
    // PGM round trip
    const auto pg = std::filesystem::temp_directory_path() / "fxg_rt.pgm";
    write_pgm(pg, 3, 2, 65535, {1, 2, 3, 65535, 0, 7});
    const IntensityImage im = load_intensity(pg);
    CHECK(im.width == 3 && im.height == 2 && im.bit_depth == 16 && im.pixels[3] == 65535);
    std::ofstream(pg) << "P5\n2 2\n255\nX";
    CHECK_THROWS_AS(load_intensity(pg), FormatError);
    CHECK_THROWS_AS(load_mask("/nonexistent/x.pgm"), IoError);
    // 8-bit payloads widen; comments in the header; samples above maxval rejected
    std::ofstream(pg, std::ios::binary) << "P5\n# c\n3 1\n# d\n200\n" << std::string("\x01\xc8\x00", 3);
    const IntensityImage i8 = load_intensity(pg);
    CHECK(i8.bit_depth == 8 && i8.pixels == (std::vector<uint16_t>{1, 200, 0}));
    std::ofstream(pg, std::ios::binary) << "P5\n2 1\n100\n" << std::string("\x01\xc8", 2);
    CHECK_THROWS_AS(load_intensity(pg), FormatError);
    std::ofstream(pg, std::ios::binary) << "P5\n1 1\n1000\n" << std::string("\x03\xe9", 2);
    CHECK_THROWS_AS(load_mask(pg), FormatError);
    // CSV number format: write_csv's "%.10g" (engine.cpp:52-67) on random and edge values
    {
        std::mt19937_64 g(7);
        std::vector<double> vs = {0.0, -0.0, 1.0 / 3.0, 1234567890.5, 1234567891.5, 5e-324, 1e-5,
                                  123456.78905, 1.7976931348623157e308, INFINITY, -INFINITY, NAN};
        for (int i = 0; i < 200000; ++i) {
            uint64_t b = g();
            double v;
            std::memcpy(&v, &b, 8);
            vs.push_back(v);
            vs.push_back(std::ldexp(static_cast<double>(g() >> 11), static_cast<int>(g() % 160) - 120));
            // every decade of the fast path, 10-digit decimals and their +-1 ulp
            // neighbours (rounding boundaries), halfway cases, small integers
            const int dec = static_cast<int>(g() % 56) - 16;
            const double d10 = static_cast<double>(1000000000ull + g() % 9000000000ull) * std::pow(10.0, dec - 9);
            vs.push_back(d10);
            vs.push_back(std::nextafter(d10, 0.0));
            vs.push_back(std::nextafter(d10, 1e300));
            vs.push_back(static_cast<double>(1000000000ull + g() % 9000000000ull) + 0.5);
            vs.push_back(static_cast<double>(static_cast<int64_t>(g() % 2000001) - 1000000));
            vs.push_back(-static_cast<double>(g() % 100000) / static_cast<double>(1 + g() % 977));
        }
        std::vector<FeatureRow> rows;
        std::string want = "image,mask,label,x\n";
        char buf[64];
        for (size_t i = 0; i < vs.size(); ++i) {
            rows.push_back({"a", "a", static_cast<uint32_t>(i), {vs[i]}});
            std::snprintf(buf, sizeof buf, "%.10g", vs[i]);
            want += "a,a," + std::to_string(i) + "," + buf + "\n";
        }
        write_csv({"x"}, rows, path);
        CHECK(slurp(path) == want);
    }
}

static void registry_cases() {
    // RoiRegistry on the device (roi.hpp:45-88): the 2x2 read-off of
    // test_roistore.cpp:34-58 -- mask [0,1,1,2], I [9,8,7,6]
    IntensityImage im;
    im.width = im.height = 2;
    im.pixels = {9, 8, 7, 6};
    LabelMask mk;
    mk.width = mk.height = 2;
    mk.labels = {0, 1, 1, 2};
    const RoiRegistry reg = RoiRegistry::accumulate(iter_row_tiles(im, mk, 1), {});
    CHECK((reg.labels() == std::vector<uint32_t>{1, 2}));
    CHECK(reg.roi_count() == 2 && reg.contains(1) && !reg.contains(3));
    const PixelCloud c1 = reg.cloud(1);
    CHECK(c1.count() == 2 && c1.pixels[0].x == 1 && c1.pixels[0].y == 0 && c1.pixels[0].intensity == 8);
    CHECK(c1.pixels[1].x == 0 && c1.pixels[1].y == 1 && c1.pixels[1].intensity == 7);
    CHECK(c1.bbox.x_min == 0 && c1.bbox.y_min == 0 && c1.bbox.x_max == 1 && c1.bbox.y_max == 1);
    const PixelCloud c2 = reg.cloud(2);
    CHECK(c2.count() == 1 && c2.pixels[0].x == 1 && c2.pixels[0].y == 1 && c2.pixels[0].intensity == 6);
    CHECK_THROWS_AS(reg.cloud(5), std::out_of_range);
    // all background: an empty registry (:60-64)
    mk.labels = {0, 0, 0, 0};
    CHECK(RoiRegistry::accumulate(iter_row_tiles(im, mk), {}).roi_count() == 0);
    CHECK_THROWS_AS(iter_row_tiles(im, mk, 0), PairingError);
    // accumulate -> cloud -> compute_roi_features == featurize (the run_tune call
    // pattern, featurex_main.cpp:104-109), on a 97x83 image of random blobs
    IntensityImage I;
    LabelMask L;
    I.width = L.width = 97;
    I.height = L.height = 83;
    I.pixels.resize(97 * 83);
    L.labels.assign(97 * 83, 0);
    uint32_t st = 12345;
    auto rnd = [&] { st = st * 1664525u + 1013904223u; return st >> 8; };
    for (auto& v : I.pixels) v = (uint16_t)(rnd() & 0xffff);
    for (int k = 0; k < 30; ++k) {
        const int cx = rnd() % 97, cy = rnd() % 83, r = 2 + rnd() % 9;
        const uint16_t lab = (uint16_t)(1 + rnd() % 20);
        for (int y = std::max(0, cy - r); y < std::min(83, cy + r + 1); ++y)
            for (int x = std::max(0, cx - r); x < std::min(97, cx + r + 1); ++x)
                if ((x - cx) * (x - cx) + (y - cy) * (y - cy) <= r * r) L.labels[y * 97 + x] = lab;
    }
    const std::vector<std::string> g = {"intensity", "moments", "glcm"};
    const TextureParams tp = resolve_profile("default");
    const FeatureTable t = featurize(I, L, g, tp);
    const RoiRegistry r2 = RoiRegistry::accumulate(iter_row_tiles(I, L, 16), {});
    CHECK(r2.labels() == t.labels);
    for (size_t i = 0; i < t.labels.size(); ++i) {
        const std::vector<double> v = compute_roi_features(r2.cloud(t.labels[i]), g, tp);
        CHECK(std::equal(v.begin(), v.end(), t.values.begin() + i * t.columns.size()));
    }
}

static void device_cases() {
    {  // one row per ROI (:77-97)
        const auto d = fresh_dir("fxg_engine_simple");
        write_simple_pair(d);
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "features.csv";
        c.features = {"intensity"};
        const RunSummary s = run(c);
        CHECK(s.images == 1 && s.rois == 2 && s.rows == 2 && !s.completed_with_errors());
        std::ifstream in(c.output_path);
        std::string header, r1, r2, extra;
        CHECK(bool(std::getline(in, header)) && header.substr(0, 17) == "image,mask,label,");
        CHECK(bool(std::getline(in, r1)) && r1.substr(0, 14) == "a.pgm,a.pgm,1,");
        CHECK(bool(std::getline(in, r2)) && r2.substr(0, 14) == "a.pgm,a.pgm,2,");
        CHECK(!std::getline(in, extra));
    }
    {  // empty mask -> header only (:99-111); default features *ALL* -> ConfigError? no: empty pair
        const auto d = fresh_dir("fxg_engine_empty");
        write_pgm(d / "int" / "a.pgm", 2, 2, 255, {1, 2, 3, 4});
        write_pgm(d / "seg" / "a.pgm", 2, 2, 255, {0, 0, 0, 0});
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "f.csv";
        c.features = {"intensity", "moments", "glcm"};
        const RunSummary s = run(c);
        CHECK(s.rois == 0 && s.rows == 0);
        std::ifstream in(c.output_path);
        std::string line;
        CHECK(bool(std::getline(in, line)));
        CHECK(!std::getline(in, line));
    }
    {  // unmatched and corrupt pairs are skipped (:113-133)
        const auto d = fresh_dir("fxg_engine_skip");
        write_simple_pair(d);
        write_pgm(d / "seg" / "orphan.pgm", 1, 1, 255, {1});
        std::ofstream(d / "int" / "bad.pgm") << "P5\n2 2\n255\nX";
        write_pgm(d / "seg" / "bad.pgm", 2, 2, 255, {1, 0, 0, 0});
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "f.csv";
        c.features = {"intensity", "moments"};
        const RunSummary s = run(c);
        CHECK(s.images == 1 && s.rows == 2 && s.completed_with_errors() && s.failed_pairs == 2);
    }
    {  // texture limits of the device path fail loudly per pair (no CPU fallback)
        const auto d = fresh_dir("fxg_engine_ng");
        write_simple_pair(d);
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "f.csv";
        c.features = {"glrlm"};
        // more than 256 grey levels run on the device (the wide texture kernel); above
        // the reference's int16 level grid: ConfigError, the pair logged and skipped
        GlcmParams gp = resolve_profile("default").glcm;
        gp.ng = 300;
        c.glcm_override = gp;
        RunSummary s = run(c);
        CHECK(s.images == 1 && s.failed_pairs == 0 && s.rows == 2);
        gp.ng = 40000;
        c.glcm_override = gp;
        s = run(c);
        CHECK(s.images == 0 && s.failed_pairs == 1);
        PixelCloud pc;
        pc.pixels = {{1, 1, 5}, {2, 1, 6}};
        TextureParams tp = resolve_profile("default");
        tp.glcm.ng = 300;
        CHECK(compute_roi_features(pc, {"glszm"}, tp).size() == 16);
        tp.glcm.ng = 40000;
        CHECK_THROWS_AS(compute_roi_features(pc, {"glszm"}, tp), ConfigError);
    }
    {  // the shape group runs on the device: a 1-pixel cloud reports the conventions
        PixelCloud pc;
        pc.pixels = {{7, 3, 5}};
        const std::vector<double> v = compute_roi_features(pc, {"shape"}, resolve_profile("default"));
        CHECK(v.size() == 38 && v[0] == 1.0 && v[1] == 4.0 && v[2] == 7.0 && v[3] == 3.0);
    }
    {  // rerun idempotent (:174-182) and per-ROI operator == image-level row
        const auto d = fresh_dir("fxg_engine_idem");
        write_simple_pair(d);
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "f.csv";
        c.features = {"intensity", "moments", "glcm"};
        run(c);
        const std::string first = slurp(c.output_path);
        run(c);
        CHECK(slurp(c.output_path) == first);
        PixelCloud pc;
        pc.label = 2;
        pc.pixels = {{2, 2, 110}, {3, 2, 120}, {2, 3, 150}, {3, 3, 160}};
        pc.bbox = {2, 2, 3, 3};
        const auto v = compute_roi_features(pc, c.features, resolve_profile("default"));
        IntensityImage im = load_intensity(d / "int" / "a.pgm");
        LabelMask mk = load_mask(d / "seg" / "a.pgm");
        const FeatureTable t = featurize(im, mk, c.features, resolve_profile("default"));
        CHECK(t.labels.size() == 2 && t.labels[1] == 2);
        bool same = v.size() == t.columns.size();
        for (size_t i = 0; same && i < v.size(); ++i) same = v[i] == t.values[t.columns.size() + i];
        CHECK(same);
    }
    {  // the batched pipeline: 300 pairs over several batches (mixed sizes, 8- and
       // 16-bit, one corrupt file) == per-pair featurize + write_csv, byte for byte
        const auto d = fresh_dir("fxg_engine_many");
        std::mt19937 g(3);
        std::vector<std::string> names;
        for (int i = 0; i < 300; ++i) {
            char nm[32];
            std::snprintf(nm, sizeof nm, "t%03d.pgm", i);
            const int w = 8 + static_cast<int>(g() % 40), h = 8 + static_cast<int>(g() % 30);
            std::vector<uint16_t> iv(static_cast<size_t>(w) * h), lv(iv.size());
            for (auto& v : iv) v = static_cast<uint16_t>(g() % 65536);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    lv[static_cast<size_t>(y) * w + x] = static_cast<uint16_t>(((x / 5) + 3 * (y / 4)) % 7);
            write_pgm(d / "int" / nm, w, h, 65535, iv);
            write_pgm(d / "seg" / nm, w, h, i % 3 ? 65535 : 255, lv);
            names.push_back(nm);
        }
        std::ofstream(d / "int" / "t150.pgm", std::ios::trunc) << "P5\n4 4\n255\nX";
        ExtractionConfig c;
        c.intensity_dir = d / "int";
        c.mask_dir = d / "seg";
        c.output_path = d / "f.csv";
        c.features = {"*ALL*"};
        const RunSummary s = run(c);
        CHECK(s.images == 299 && s.failed_pairs == 1);
        const TextureParams tp = resolve_profile("default");
        std::vector<FeatureRow> rows;
        for (const std::string& nm : names) {
            if (nm == "t150.pgm") continue;
            const FeatureTable t = featurize(load_intensity(d / "int" / nm), load_mask(d / "seg" / nm),
                                             c.features, tp);
            for (size_t i = 0; i < t.labels.size(); ++i)
                rows.push_back({nm, nm, t.labels[i],
                                std::vector<double>(t.values.begin() + i * t.columns.size(),
                                                    t.values.begin() + (i + 1) * t.columns.size())});
        }
        CHECK(s.rows == rows.size() && s.rows > 299 * 5);
        write_csv(feature_columns(c.features, tp), rows, d / "g.csv");
        CHECK(slurp(d / "f.csv") == slurp(d / "g.csv"));
        // several devices (ExtractionConfig::devices; here contexts sharing GPU 0):
        // the same CSV, byte for byte, failure counted once
        for (const std::vector<int>& devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0}}) {
            ExtractionConfig cm = c;
            cm.devices = devs;
            cm.output_path = d / "m.csv";
            const RunSummary sm = run(cm);
            CHECK(sm.images == 299 && sm.failed_pairs == 1 && sm.rows == s.rows);
            CHECK(slurp(d / "m.csv") == slurp(d / "f.csv"));
        }
    }
    {  // batched per-ROI operator (extension) == one compute_roi_features per cloud
        std::mt19937 g(5);
        std::vector<PixelCloud> clouds(40);
        for (size_t k = 0; k < clouds.size(); ++k) {
            const int r = 2 + static_cast<int>(k % 9);
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx)
                    if (dx * dx + dy * dy <= r * r && g() % 7)
                        clouds[k].pixels.push_back({static_cast<uint32_t>(100 + 20 * k + dx),
                                                    static_cast<uint32_t>(50 + dy),
                                                    static_cast<uint16_t>(g() % 65536)});
        }
        clouds[3].pixels.clear();  // empty cloud: zeros
        const TextureParams tp = resolve_profile("default");
        const std::vector<std::string> groups = {"*ALL*"};
        const auto batch = compute_roi_features_batch(clouds, groups, tp);
        bool same = batch.size() == clouds.size();
        for (size_t k = 0; same && k < clouds.size(); ++k) {
            const auto one = compute_roi_features(clouds[k], groups, tp);
            same = one.size() == batch[k].size();
            for (size_t i = 0; same && i < one.size(); ++i)
                same = one[i] == batch[k][i] || (std::isnan(one[i]) && std::isnan(batch[k][i]));
        }
        CHECK(same);
    }
    {  // pairing errors
        IntensityImage im;
        im.width = 2;
        im.height = 2;
        im.pixels = {1, 2, 3, 4};
        LabelMask mk;
        mk.width = 1;
        mk.height = 4;
        mk.labels = {1, 1, 1, 1};
        CHECK_THROWS_AS(featurize(im, mk, {"intensity"}, resolve_profile("default")), PairingError);
        ExtractionConfig c;
        c.threads = 0;
        CHECK_THROWS_AS(run(c), ConfigError);
    }
}

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
    try {
        host_cases();
        if (!host_only) {
            device_cases();
            registry_cases();
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
