// featurex_gpu/engine.hpp -- drop-in C++ engine API of the B200 featurize path.
//
// Same namespace, type names, function names, argument meaning and exception
// types as the reference's engine (/root/reference/proj/include/featurex/
// engine.hpp:14-81, roi.hpp:13-34, image.hpp:11-27, texture.hpp:30-35,
// errors.hpp:8-58), so callers of the reference compile unchanged against this
// header and link libfxg.so instead of libfeaturex.a.  Every compute call runs
// the sm_100a kernels through the C ABI (include/fxg.h); there is no CPU path.
//
// Differences (documented in INTEGRATION.md):
//  - ExtractionConfig::threads / parallel size run()'s host workers (PGM decode,
//    CSV formatting); memory_budget / spill_dir are validated like the reference
//    but ROI data stays in HBM (no spill).
//  - all seven groups (intensity, moments, shape, glcm, glrlm, glszm, ngtdm)
//    run on the device for any grey-level count up to 32768 (the reference's
//    int16 level grid); larger counts raise ConfigError (never a CPU fallback).
//  - ExtractionConfig::devices (extension) spreads run() over several GPUs.
#pragma once

#include <cstdint>
#include <filesystem>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace featurex {

// ---- errors (errors.hpp:8-58) -----------------------------------------------
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PairingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SpillIoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ZeroMassError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnknownProfile : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PackingError : std::runtime_error { using std::runtime_error::runtime_error; };
// the tuner's errors (out of scope here, declared so callers compile unchanged)
struct ClassCountError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GridError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InsufficientClassItems : std::runtime_error { using std::runtime_error::runtime_error; };
struct NoFeasiblePoint : std::runtime_error { using std::runtime_error::runtime_error; };
// device-side failures (no reference counterpart)
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---- data types -------------------------------------------------------------
struct IntensityImage {  // image.hpp:11-18
    int width = 0;
    int height = 0;
    int bit_depth = 16;
    std::vector<uint16_t> pixels;
    uint16_t at(int x, int y) const { return pixels[static_cast<size_t>(y) * width + x]; }
};

struct LabelMask {  // image.hpp:20-27
    int width = 0;
    int height = 0;
    std::vector<uint16_t> labels;
    uint16_t at(int x, int y) const { return labels[static_cast<size_t>(y) * width + x]; }
};

// Read-only view of a horizontal band of a matched image/mask pair (image.hpp:30-37)
struct RowTile {
    int y0 = 0;
    int rows = 0;
    int width = 0;
    std::span<const uint16_t> intensity;  // rows*width values
    std::span<const uint16_t> labels;
};

// Contiguous tiles of at most rows_per_tile rows; PairingError on a dimension
// mismatch or rows_per_tile < 1 (image.hpp:41-42, image.cpp:7-26).
std::vector<RowTile> iter_row_tiles(const IntensityImage& image, const LabelMask& mask,
                                    int rows_per_tile = 256);

struct Pixel {  // roi.hpp:13-17
    uint32_t x = 0;
    uint32_t y = 0;
    uint16_t intensity = 0;
};

struct BoundingBox {  // roi.hpp:19-24
    uint32_t x_min = 0, y_min = 0, x_max = 0, y_max = 0;
    int width() const { return static_cast<int>(x_max - x_min) + 1; }
    int height() const { return static_cast<int>(y_max - y_min) + 1; }
};

struct PixelCloud {  // roi.hpp:28-34
    uint32_t label = 0;
    std::vector<Pixel> pixels;
    BoundingBox bbox;
    size_t count() const { return pixels.size(); }
};

struct MemoryBudget {  // roi.hpp:36-39 (accepted; clouds are built on the device, no spill)
    size_t max_resident_bytes = std::numeric_limits<size_t>::max();
    std::filesystem::path spill_dir;
};

// Per-label pixel clouds of one image (roi.hpp:45-88).  accumulate() runs the
// label scan and the cloud gather on the GPU (fx_roi_clouds): labels ascending,
// each cloud in mask scan order with its tight inclusive bbox -- the reference's
// contents.  The clouds then live in host memory; nothing is spilled, so
// peak_resident_bytes() is the total and cleanup() has nothing to remove.
class RoiRegistry {
public:
    RoiRegistry() = default;
    RoiRegistry(RoiRegistry&&) = default;
    RoiRegistry& operator=(RoiRegistry&&) = default;
    RoiRegistry(const RoiRegistry&) = delete;
    RoiRegistry& operator=(const RoiRegistry&) = delete;
    ~RoiRegistry() = default;

    static RoiRegistry accumulate(const std::vector<RowTile>& tiles, const MemoryBudget& budget);

    std::vector<uint32_t> labels() const { return labels_; }  // ascending
    size_t roi_count() const { return labels_.size(); }
    bool contains(uint32_t label) const;
    // std::out_of_range for an unknown label (roi.cpp:124); safe for concurrent readers
    PixelCloud cloud(uint32_t label) const;
    size_t peak_resident_bytes() const { return pixels_.size() * sizeof(Pixel); }
    void cleanup() {}

private:
    std::vector<uint32_t> labels_;
    std::vector<uint64_t> offsets_;     // [roi_count + 1] into pixels_
    std::vector<BoundingBox> bboxes_;
    std::vector<Pixel> pixels_;
};

struct GlcmParams {  // texture.hpp:30-35
    int ng = 256;
    int offset = 1;
    std::vector<int> angles = {0, 45, 90, 135};
    bool symmetric = true;
};

struct TextureParams {  // engine.hpp:14-17
    GlcmParams glcm;
    int histogram_bins = 256;
};

TextureParams resolve_profile(const std::string& name);

struct ExtractionConfig {  // engine.hpp:24-38
    std::filesystem::path intensity_dir;
    std::filesystem::path mask_dir;
    std::string file_pattern = "*.pgm";
    std::vector<std::string> features = {"*ALL*"};
    std::string profile = "default";
    int threads = 1;
    size_t memory_budget = std::numeric_limits<size_t>::max();
    std::optional<GlcmParams> glcm_override;
    std::optional<int> histogram_bins_override;
    std::filesystem::path output_path;
    std::filesystem::path spill_dir;
    int rows_per_tile = 256;
    bool parallel = true;
    int device = 0;  // extension: CUDA device used by run()
    // extension: several devices (one context and host thread each, pairs dealt in
    // chunks, rows identical to one device); empty = {device}
    std::vector<int> devices;
};

struct FeatureRow {  // engine.hpp:41-46
    std::string image_name;
    std::string mask_name;
    uint32_t roi_label = 0;
    std::vector<double> values;
};

struct RunSummary {  // engine.hpp:48-56
    int images = 0;
    size_t rois = 0;
    size_t rows = 0;
    double elapsed_seconds = 0;
    int failed_pairs = 0;
    bool completed_with_errors() const { return failed_pairs > 0; }
};

std::vector<std::string> resolve_feature_groups(const std::vector<std::string>& requested);
std::vector<std::string> feature_columns(const std::vector<std::string>& groups,
                                         const TextureParams& params);
std::vector<double> compute_roi_features(const PixelCloud& cloud,
                                         const std::vector<std::string>& groups,
                                         const TextureParams& params);
// Extension: compute_roi_features for many clouds in one device pass (row k ==
// compute_roi_features(clouds[k], ...)); amortises the per-call launch cost.
std::vector<std::vector<double>> compute_roi_features_batch(const std::vector<PixelCloud>& clouds,
                                                            const std::vector<std::string>& groups,
                                                            const TextureParams& params);
RunSummary run(const ExtractionConfig& config);
size_t write_csv(const std::vector<std::string>& columns, std::vector<FeatureRow> rows,
                 const std::filesystem::path& path);

// ---- in-memory image-level featurization (the device-native entry point) ----
struct FeatureTable {
    std::vector<std::string> columns;
    std::vector<uint32_t> labels;  // ascending
    std::vector<double> values;    // [labels.size() x columns.size()] row-major
};
// RoiRegistry::accumulate + compute_roi_features for every label of one pair,
// on the GPU (engine.cpp:300-336 without file I/O).
FeatureTable featurize(const IntensityImage& image, const LabelMask& mask,
                       const std::vector<std::string>& groups, const TextureParams& params,
                       int device = 0);

// PGM P5 I/O (pgm.hpp:14-21), host-side.
IntensityImage load_intensity(const std::filesystem::path& path);
LabelMask load_mask(const std::filesystem::path& path);
void write_pgm(const std::filesystem::path& path, int width, int height, int maxval,
               const std::vector<uint16_t>& samples);

}  // namespace featurex
