// BENCH / TEST TOOLING -- synthetic inputs, not part of libfxg.so.
//
// The workloads of BASELINE.json are defined by the reference's own generators
// (/root/reference/proj/src/synth.cpp:16-132: siemens_star, blob_mask_grid) and by
// uniform uint16 intensities from std::mt19937_64.  bench.py and the tests need the
// identical rasters on the GPU box, where the reference sources do not exist, so
// the generators are restated here with the same floating-point sequence (the
// masks are compared pixel for pixel with the reference's in
// tests/test_synth.py).  Build: `make synth` -> tools/synth/_build/libfxsynth.so.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <vector>

namespace {

// Membership of (px, py) in one blob: a disc of radius r plus two triangular
// "ears" whose apexes point away from the centre; (u, v) is the pixel in the
// blob's rotated frame.
bool in_blob(double u, double v, double r) {
    if (u * u + v * v <= r * r) return true;
    const double ear_h = r * 0.95;
    for (int side = -1; side <= 1; side += 2) {
        const double du = u - side * r * 0.62, dv = v - (-r * 0.62);
        const double along = (side * du - dv) / std::numbers::sqrt2;
        const double across = std::abs((side * du + dv) / std::numbers::sqrt2);
        if (along >= 0 && along <= ear_h && across <= 0.55 * r * (1.0 - along / ear_h)) return true;
    }
    return false;
}

// paints one blob centred at (cx, cy), rotated by phi; returns the pixel count
int draw_blob(uint16_t* img, int n, double cx, double cy, double r, double phi, uint16_t id) {
    const int reach = (int)std::ceil(r * 1.9) + 1;
    const double cs = std::cos(phi), sn = std::sin(phi);
    const int y_first = std::max(0, (int)cy - reach), y_last = std::min(n - 1, (int)cy + reach);
    const int x_first = std::max(0, (int)cx - reach), x_last = std::min(n - 1, (int)cx + reach);
    int area = 0;
    for (int py = y_first; py <= y_last; ++py)
        for (int px = x_first; px <= x_last; ++px) {
            const double ox = px - cx, oy = py - cy;
            if (!in_blob(ox * cs + oy * sn, -ox * sn + oy * cs, r)) continue;
            img[(size_t)py * n + px] = id;
            ++area;
        }
    return area;
}

int area_at(double r) {
    const int n = (int)std::ceil(r * 4) + 8;
    std::vector<uint16_t> scratch((size_t)n * n, 0);
    return draw_blob(scratch.data(), n, n / 2.0, n / 2.0, r, 0.0, 1);
}

}  // namespace

extern "C" {

// 0 ok, 1 bad spec (the reference throws ConfigError), 2 null pointer
int fxs_blob_mask_grid(int image_size, int roi_size, int roi_count, uint64_t seed, uint16_t* out) {
    if (!out) return 2;
    if (image_size < 16 || roi_count < 1 || roi_size < 1 || roi_count > 65535) return 1;
    if ((double)roi_count * roi_size > 0.9 * (double)image_size * image_size) return 1;
    // radius whose blob covers roi_size pixels: bracket, then 40 bisection steps
    double lo = 0.5, hi = std::sqrt((double)roi_size);
    while (area_at(hi) < roi_size) hi *= 1.5;
    for (int step = 0; step < 40; ++step) {
        const double mid = (lo + hi) / 2.0;
        (area_at(mid) < roi_size ? lo : hi) = mid;
    }
    const double r = (lo + hi) / 2.0;
    const int pitch = (int)std::ceil(2.0 * 1.9 * r) + 4;
    const int per_row = (int)std::ceil(std::sqrt((double)roi_count));
    if (per_row * pitch > image_size) return 1;
    std::memset(out, 0, (size_t)image_size * image_size * sizeof(uint16_t));
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> angle(0.0, 2.0 * std::numbers::pi);
    for (int k = 0; k < roi_count; ++k)
        draw_blob(out, image_size, (k % per_row) * pitch + pitch / 2.0,
                  (k / per_row) * pitch + pitch / 2.0, r, angle(gen), (uint16_t)(k + 1));
    return 0;
}

int fxs_siemens_star(int size, int spokes, uint16_t* out) {
    if (!out) return 2;
    if (size < 1 || spokes < 2 || spokes % 2) return 1;
    const double mid = (size - 1) / 2.0, turn = 2.0 * std::numbers::pi;
    for (int y = 0; y < size; ++y)
        for (int x = 0; x < size; ++x) {
            double th = std::atan2((double)y - mid, (double)x - mid);
            if (th < 0) th += turn;
            out[(size_t)y * size + x] = ((int)(spokes * th / turn) & 1) ? 0 : 65535;
        }
    return 0;
}

int fxs_uniform_u16(uint64_t seed, size_t n, uint16_t* out) {
    if (!out && n) return 2;
    std::mt19937_64 gen(seed);
    for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)(gen() & 0xffffu);
    return 0;
}

}  // extern "C"
