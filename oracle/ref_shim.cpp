// TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
//
// C-ABI shim over the *unmodified* reference library (featurex, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It calls only
// the reference's public API so that tests/ and bench.py's cpu_baseline /
// --impl reference leg can run the reference CPU path on the same in-memory
// inputs the GPU path sees.  Nothing under paper_2603_12016_b200/ links this.
//
// Mirrors, call for call:
//   in-memory featurize  = RoiRegistry::accumulate(iter_row_tiles(img, mask, 256))
//                          + omp parallel for over labels() calling
//                          compute_roi_features(cloud(L), groups, params)
//                          (reference engine.cpp:300-333 without file I/O)
//   per-ROI operator     = compute_roi_features        (engine.hpp:68-70)
//   columns              = feature_columns              (engine.hpp:64-65)
//   run()                = featurex::run                (engine.hpp:77)
//   internals used by the bit-exact tests: trace_contour (contour.hpp:26),
//   discretize/glcm (texture.hpp:28,49), RoiRegistry (roi.hpp:45-88),
//   blob_mask_grid/siemens_star (synth.hpp).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include <omp.h>

#include "featurex/contour.hpp"
#include "featurex/engine.hpp"
#include "featurex/errors.hpp"
#include "featurex/image.hpp"
#include "featurex/intensity_features.hpp"
#include "featurex/moments.hpp"
#include "featurex/roi.hpp"
#include "featurex/synth.hpp"
#include "featurex/texture.hpp"

using namespace featurex;

extern "C" {

// Same field meaning as fx_texture_params in include/fxg.h.
typedef struct {
    int ng;
    int offset;
    int n_angles;
    int angles[8];
    int symmetric;
    int histogram_bins;
} fxref_params;

typedef struct {
    int images;
    uint64_t rois;
    uint64_t rows;
    double elapsed_seconds;
    int failed_pairs;
} fxref_run_summary;
}

namespace {

thread_local std::string g_err;

// Error codes are the product's (include/fxg.h): 1 config, 2 unknown profile,
// 3 pairing, 4 io, 5 format, 6 zero mass, 12 other.
int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const UnknownProfile*>(&e)) return 2;
    if (dynamic_cast<const PairingError*>(&e)) return 3;
    if (dynamic_cast<const IoError*>(&e)) return 4;
    if (dynamic_cast<const FormatError*>(&e)) return 5;
    if (dynamic_cast<const ZeroMassError*>(&e)) return 6;
    return 12;
}

std::vector<std::string> split_csv(const char* s) {
    std::vector<std::string> out;
    if (!s) return out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ','))
        if (!item.empty()) out.push_back(item);
    return out;
}

TextureParams to_params(const fxref_params* p) {
    TextureParams t;
    t.glcm.ng = p->ng;
    t.glcm.offset = p->offset;
    t.glcm.angles.assign(p->angles, p->angles + p->n_angles);
    t.glcm.symmetric = p->symmetric != 0;
    t.histogram_bins = p->histogram_bins;
    return t;
}

PixelCloud cloud_from_arrays(const uint32_t* xs, const uint32_t* ys, const uint16_t* is,
                             size_t n) {
    PixelCloud c;
    c.label = 1;
    c.pixels.resize(n);
    for (size_t i = 0; i < n; ++i) c.pixels[i] = {xs[i], ys[i], is[i]};
    if (n) {
        c.bbox = {xs[0], ys[0], xs[0], ys[0]};
        for (size_t i = 0; i < n; ++i) {
            c.bbox.x_min = std::min(c.bbox.x_min, xs[i]);
            c.bbox.x_max = std::max(c.bbox.x_max, xs[i]);
            c.bbox.y_min = std::min(c.bbox.y_min, ys[i]);
            c.bbox.y_max = std::max(c.bbox.y_max, ys[i]);
        }
    }
    return c;
}

void make_images(const uint16_t* intensity, const uint16_t* labels, int w, int h,
                 IntensityImage& img, LabelMask& mask) {
    const size_t n = static_cast<size_t>(w) * h;
    img.width = mask.width = w;
    img.height = mask.height = h;
    img.bit_depth = 16;
    img.pixels.assign(intensity, intensity + n);
    mask.labels.assign(labels, labels + n);
}

} // namespace

extern "C" {

const char* fxref_last_error(void) { return g_err.c_str(); }

int fxref_resolve_profile(const char* name, fxref_params* out) {
    try {
        const TextureParams t = resolve_profile(name);
        out->ng = t.glcm.ng;
        out->offset = t.glcm.offset;
        out->n_angles = static_cast<int>(t.glcm.angles.size());
        for (int i = 0; i < out->n_angles && i < 8; ++i) out->angles[i] = t.glcm.angles[i];
        out->symmetric = t.glcm.symmetric ? 1 : 0;
        out->histogram_bins = t.histogram_bins;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Newline-joined column names; returns the byte count needed (incl. NUL) in *need.
int fxref_columns(const char* groups_csv, const fxref_params* p, char* buf, size_t cap,
                  size_t* need, int* n_cols) {
    try {
        const auto groups = resolve_feature_groups(split_csv(groups_csv));
        const auto cols = feature_columns(groups, to_params(p));
        std::string joined;
        for (size_t i = 0; i < cols.size(); ++i) {
            if (i) joined += '\n';
            joined += cols[i];
        }
        *need = joined.size() + 1;
        *n_cols = static_cast<int>(cols.size());
        if (buf && cap >= joined.size() + 1) std::memcpy(buf, joined.c_str(), joined.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// In-memory reference path (engine.cpp:300-333 minus PGM/CSV).  threads<=1 runs
// the serial branch.  out_values is [n_rois x n_cols] row-major, labels ascending.
int fxref_featurize(const uint16_t* intensity, const uint16_t* labels, int w, int h,
                    const char* groups_csv, const fxref_params* p, int threads,
                    uint32_t* out_labels, double* out_values, size_t cap_rois, size_t* n_rois,
                    int* n_cols) {
    try {
        const auto groups = resolve_feature_groups(split_csv(groups_csv));
        const TextureParams params = to_params(p);
        const size_t ncol = feature_columns(groups, params).size();
        IntensityImage img;
        LabelMask mask;
        make_images(intensity, labels, w, h, img, mask);
        RoiRegistry reg = RoiRegistry::accumulate(iter_row_tiles(img, mask, 256), {});
        const std::vector<uint32_t> ls = reg.labels();
        *n_rois = ls.size();
        *n_cols = static_cast<int>(ncol);
        if (ls.size() > cap_rois) {
            g_err = "output capacity too small";
            return 10;
        }
        std::string first_error;
        if (threads > 1) {
#pragma omp parallel for schedule(dynamic) num_threads(threads)
            for (size_t i = 0; i < ls.size(); ++i) {
                try {
                    const PixelCloud cloud = reg.cloud(ls[i]);
                    const std::vector<double> v = compute_roi_features(cloud, groups, params);
                    std::memcpy(out_values + i * ncol, v.data(), ncol * sizeof(double));
                } catch (const std::exception& e) {
#pragma omp critical
                    if (first_error.empty()) first_error = e.what();
                }
            }
        } else {
            for (size_t i = 0; i < ls.size(); ++i) {
                const PixelCloud cloud = reg.cloud(ls[i]);
                const std::vector<double> v = compute_roi_features(cloud, groups, params);
                std::memcpy(out_values + i * ncol, v.data(), ncol * sizeof(double));
            }
        }
        if (!first_error.empty()) throw ConfigError(first_error);
        for (size_t i = 0; i < ls.size(); ++i) out_labels[i] = ls[i];
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Per-label count and inclusive bbox from RoiRegistry::accumulate (roi.cpp:76-110).
int fxref_roi_table(const uint16_t* intensity, const uint16_t* labels, int w, int h,
                    int rows_per_tile, uint32_t* out_labels, uint64_t* out_count,
                    uint32_t* out_bbox /* [n x 4] xmin,ymin,xmax,ymax */, size_t cap,
                    size_t* n) {
    try {
        IntensityImage img;
        LabelMask mask;
        make_images(intensity, labels, w, h, img, mask);
        RoiRegistry reg = RoiRegistry::accumulate(iter_row_tiles(img, mask, rows_per_tile), {});
        const auto ls = reg.labels();
        *n = ls.size();
        if (ls.size() > cap) return 10;
        for (size_t i = 0; i < ls.size(); ++i) {
            const PixelCloud c = reg.cloud(ls[i]);
            out_labels[i] = ls[i];
            out_count[i] = c.count();
            out_bbox[4 * i + 0] = c.bbox.x_min;
            out_bbox[4 * i + 1] = c.bbox.y_min;
            out_bbox[4 * i + 2] = c.bbox.x_max;
            out_bbox[4 * i + 3] = c.bbox.y_max;
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// compute_roi_features on an explicit cloud (engine.hpp:68-70).
int fxref_roi_features(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                       const char* groups_csv, const fxref_params* p, double* out, size_t cap,
                       int* n_cols) {
    try {
        const auto groups = resolve_feature_groups(split_csv(groups_csv));
        const std::vector<double> v =
            compute_roi_features(cloud_from_arrays(xs, ys, is, n), groups, to_params(p));
        *n_cols = static_cast<int>(v.size());
        if (v.size() > cap) return 10;
        std::memcpy(out, v.data(), v.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// trace_contour visit order (contour.cpp:70-144); points as interleaved x,y.
int fxref_trace_contour(const uint32_t* xs, const uint32_t* ys, size_t n, int32_t* out_xy,
                        size_t cap_points, size_t* n_points) {
    try {
        std::vector<uint16_t> is(n, 1);
        const ContourPath path = trace_contour(cloud_from_arrays(xs, ys, is.data(), n));
        *n_points = path.points.size();
        if (path.points.size() > cap_points) return 10;
        for (size_t i = 0; i < path.points.size(); ++i) {
            out_xy[2 * i] = path.points[i].x;
            out_xy[2 * i + 1] = path.points[i].y;
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// discretize + glcm (texture.cpp:29-85): the normalized matrix and pair count.
int fxref_glcm(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n, int ng,
               int offset, int angle, int symmetric, double* out_p /* ng*ng */,
               uint64_t* pair_count) {
    try {
        const DiscretizedRoi roi = discretize(cloud_from_arrays(xs, ys, is, n), ng);
        const GlcmMatrix m = glcm(roi, offset, angle, symmetric != 0);
        *pair_count = m.pair_count;
        std::memcpy(out_p, m.p.data(), m.p.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// discretize levels over the bbox lattice (texture.cpp:29-56); -1 outside.
int fxref_discretize(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                     int ng, int16_t* out_grid, size_t cap, int* width, int* height) {
    try {
        const DiscretizedRoi roi = discretize(cloud_from_arrays(xs, ys, is, n), ng);
        *width = roi.width;
        *height = roi.height;
        if (roi.grid.size() > cap) return 10;
        std::memcpy(out_grid, roi.grid.data(), roi.grid.size() * sizeof(int16_t));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int fxref_blob_mask_grid(int image_size, int roi_size, int roi_count, uint64_t seed,
                         uint16_t* out) {
    try {
        SynthSpec s;
        s.image_size = image_size;
        s.roi_size = roi_size;
        s.roi_count = roi_count;
        s.seed = seed;
        const LabelMask m = blob_mask_grid(s);
        std::memcpy(out, m.labels.data(), m.labels.size() * sizeof(uint16_t));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int fxref_siemens_star(int size, int spokes, uint16_t* out) {
    try {
        const IntensityImage img = siemens_star(size, spokes);
        std::memcpy(out, img.pixels.data(), img.pixels.size() * sizeof(uint16_t));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// featurex::run on PGM directories (engine.cpp:283-350).
int fxref_run(const char* intensity_dir, const char* mask_dir, const char* pattern,
              const char* groups_csv, const char* profile, int threads, int parallel,
              const char* output_path, fxref_run_summary* out) {
    try {
        ExtractionConfig c;
        c.intensity_dir = intensity_dir;
        c.mask_dir = mask_dir;
        if (pattern && *pattern) c.file_pattern = pattern;
        c.features = split_csv(groups_csv);
        c.profile = profile;
        c.threads = threads;
        c.parallel = parallel != 0;
        c.output_path = output_path;
        const RunSummary s = run(c);
        out->images = s.images;
        out->rois = s.rois;
        out->rows = s.rows;
        out->elapsed_seconds = s.elapsed_seconds;
        out->failed_pairs = s.failed_pairs;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int fxref_max_threads(void) { return omp_get_max_threads(); }

} // extern "C"
