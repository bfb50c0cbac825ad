// Pure host parts of the C ABI: profiles, group resolution, column names,
// error state.  No device code here.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "fx_host.hpp"
#include "fxg.h"

namespace fxg {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

const std::vector<std::string>& all_group_names() {
    static const std::vector<std::string> v = {"intensity", "shape", "moments", "glcm",
                                               "glrlm",     "glszm", "ngtdm"};
    return v;
}

// intensity_feature_names (reference intensity_features.cpp:217-234)
static const char* const kIntensityNames[39] = {
    "mean",          "median",          "mode",        "min",           "max",
    "range",         "variance",        "variance_biased", "std",       "std_biased",
    "mad",           "median_ad",       "rmad",        "iqr",           "p1",
    "p10",           "p25",             "p75",         "p90",           "p99",
    "skewness",      "kurtosis",        "excess_kurtosis", "hyperskewness", "hyperflatness",
    "energy",        "rms",             "entropy",     "uniformity",    "qcod",
    "cov",           "integrated_intensity", "edge_mean", "edge_min",   "edge_max",
    "edge_std",      "edge_integrated", "weighted_centroid_x", "weighted_centroid_y"};

// glcm_feature_names (texture.cpp:534-542)
static const char* const kGlcmNames[29] = {
    "asm",    "acor",     "cluprom", "clushade", "clutend", "contrast", "corr",  "difave",
    "difentro", "difvar", "dis",     "energy",   "entropy", "hom1",     "hom2",  "id",
    "idn",    "idm",      "idmn",    "infomeas1", "infomeas2", "iv",    "jave",  "je",
    "jmax",   "jvar",     "sumave",  "sument",   "sumvar"};

// glrlm / glszm / ngtdm names (texture.cpp:544-562), shape (shape_features.cpp:253-270)
static const char* const kGlrlmNames[16] = {"sre", "lre", "glnu", "glnun", "rlnu", "rlnun",
                                            "rp",  "glv", "rv",   "re",    "lglre", "hglre",
                                            "srlgle", "srhgle", "lrlgle", "lrhgle"};
static const char* const kGlszmNames[16] = {"sae", "lae", "glnu", "glnun", "sznu", "sznun",
                                            "zp",  "glv", "zv",   "ze",    "lglze", "hglze",
                                            "salgle", "sahgle", "lalgle", "lahgle"};
static const char* const kNgtdmNames[5] = {"busyness", "coarseness", "complexity", "contrast",
                                           "strength"};
static const char* const kShapeNames[22] = {
    "area",         "perimeter",  "bbox_x",         "bbox_y",         "bbox_w",
    "bbox_h",       "centroid_x", "centroid_y",     "circularity",    "extent",
    "aspect_ratio", "convex_area", "solidity",      "equivalent_diameter", "major_axis_len",
    "minor_axis_len", "eccentricity", "elongation", "orientation",    "euler_number",
    "feret_max",    "feret_min"};
static const char* const kCorners[8] = {"topleft",     "topright",   "righttop",   "rightbottom",
                                        "bottomright", "bottomleft", "leftbottom", "lefttop"};

std::vector<int> sorted_angles(const fx_texture_params& p) {
    std::vector<int> a(p.angles, p.angles + std::max(0, std::min(p.n_angles, 8)));
    std::sort(a.begin(), a.end());
    return a;
}

// feature_columns (engine.cpp:107-136)
std::vector<std::string> column_names(unsigned groups, const fx_texture_params& p) {
    std::vector<std::string> cols;
    const std::vector<int> angles = sorted_angles(p);
    auto per_angle = [&](const char* fam, const char* const* stats, int ns) {
        for (int s = 0; s < ns; ++s) {
            for (int a : angles) cols.push_back(std::string(fam) + "_" + stats[s] + "_" + std::to_string(a));
            cols.push_back(std::string(fam) + "_" + stats[s] + "_ave");
        }
    };
    if (groups & FX_GROUP_INTENSITY)
        for (const char* n : kIntensityNames) cols.push_back(std::string("intensity_") + n);
    if (groups & FX_GROUP_SHAPE) {
        for (const char* n : kShapeNames) cols.push_back(std::string("shape_") + n);
        for (const char* c : kCorners) {
            cols.push_back(std::string("shape_extrema_") + c + "_x");
            cols.push_back(std::string("shape_extrema_") + c + "_y");
        }
    }
    if (groups & FX_GROUP_MOMENTS) {
        for (const char* pre : {"", "w"}) {
            for (int a = 0; a <= 3; ++a)
                for (int b = 0; b <= 3; ++b)
                    cols.push_back(std::string("moments_") + pre + "m" + std::to_string(a) + std::to_string(b));
            for (int a = 0; a <= 3; ++a)
                for (int b = 0; b <= 3; ++b)
                    cols.push_back(std::string("moments_") + pre + "mu" + std::to_string(a) + std::to_string(b));
            for (int a = 0; a <= 3; ++a)
                for (int b = 0; b <= 3; ++b)
                    if (a + b >= 2)
                        cols.push_back(std::string("moments_") + pre + "eta" + std::to_string(a) + std::to_string(b));
            for (int k = 1; k <= 7; ++k) cols.push_back(std::string("moments_") + pre + "hu" + std::to_string(k));
        }
    }
    if (groups & FX_GROUP_GLCM) per_angle("glcm", kGlcmNames, 29);
    if (groups & FX_GROUP_GLRLM) per_angle("glrlm", kGlrlmNames, 16);
    if (groups & FX_GROUP_GLSZM)
        for (const char* n : kGlszmNames) cols.push_back(std::string("glszm_") + n);
    if (groups & FX_GROUP_NGTDM)
        for (const char* n : kNgtdmNames) cols.push_back(std::string("ngtdm_") + n);
    return cols;
}

}  // namespace fxg

using namespace fxg;

extern "C" {

int fx_abi_version(void) { return FXG_ABI_VERSION; }

const char* fx_last_error(void) { return g_last_error.c_str(); }

int fx_resolve_profile(const char* name, fx_texture_params* out) {
    if (!name || !out) return set_error(FX_E_ARG, "null argument");
    fx_texture_params t{};
    const std::string n = name;
    auto set4 = [&](int ng, bool sym) {
        t.ng = ng;
        t.offset = 1;
        t.n_angles = 4;
        t.angles[0] = 0;
        t.angles[1] = 45;
        t.angles[2] = 90;
        t.angles[3] = 135;
        t.symmetric = sym ? 1 : 0;
        t.histogram_bins = 256;
    };
    if (n == "default") {
        set4(64, true);
    } else if (n == "performance") {
        t.ng = 32;
        t.offset = 1;
        t.n_angles = 1;
        t.angles[0] = 0;
        t.symmetric = 0;
        t.histogram_bins = 256;
    } else if (n == "ibsi-like") {
        set4(256, true);
    } else {
        return set_error(FX_E_UNKNOWN_PROFILE, "unknown profile '" + n + "'");
    }
    *out = t;
    return FX_OK;
}

int fx_resolve_groups(const char* const* names, int n_names, unsigned* out_mask) {
    if (!out_mask || (n_names > 0 && !names)) return set_error(FX_E_ARG, "null argument");
    if (n_names <= 0) return set_error(FX_E_CONFIG, "feature list is empty");
    unsigned m = 0;
    const auto& all = all_group_names();
    for (int i = 0; i < n_names; ++i) {
        const std::string r = names[i] ? names[i] : "";
        if (r == "*ALL*") {
            m |= FX_GROUP_ALL;
            continue;
        }
        const auto it = std::find(all.begin(), all.end(), r);
        if (it == all.end()) return set_error(FX_E_CONFIG, "unknown feature group '" + r + "'");
        m |= 1u << (it - all.begin());
    }
    *out_mask = m;
    return FX_OK;
}

int fx_columns(unsigned groups, const fx_texture_params* params, char* buf, size_t cap,
               size_t* need, int* n_cols) {
    if (!params || !need || !n_cols) return set_error(FX_E_ARG, "null argument");
    const auto cols = column_names(groups, *params);
    std::string joined;
    for (size_t i = 0; i < cols.size(); ++i) {
        if (i) joined += '\n';
        joined += cols[i];
    }
    *need = joined.size() + 1;
    *n_cols = static_cast<int>(cols.size());
    if (buf) {
        if (cap < joined.size() + 1) return set_error(FX_E_CAPACITY, "column buffer too small");
        std::memcpy(buf, joined.c_str(), joined.size() + 1);
    }
    return FX_OK;
}

}  // extern "C"
