// Device helpers shared by the per-ROI kernels: the S kernels (one warp per ROI,
// window staged in shared memory by TMA, fx_roi_s.cu) and the large-ROI kernel
// (one CTA per ROI, global-memory slab, fx_roi_b.cu).
//
// Reference functions restated on the device (paths relative to
// /root/reference/proj):
//   intensity_features        src/intensity_features.cpp:42-215
//   trace_contour edge set    src/contour.cpp:30-144 (visited set == "definition B",
//                             pixels of the largest
//                             8-connected component with a 4-neighbour in the
//                             4-connected exterior)
//   compute_moments           src/moments.cpp:32-92
//   discretize/glcm/features  src/texture.cpp:29-217
//   emit_per_angle            src/engine.cpp:159-169
#pragma once

#include "fx_dev.cuh"

namespace fxg {

// ------------------------------------------------------------------ layout --
__host__ __device__ constexpr uint32_t al(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }
__host__ __device__ constexpr uint32_t mx(uint32_t a, uint32_t b) { return a > b ? a : b; }

// Ellipse orientation 0.5 atan2(2b, a - c) wrapped into (-pi/2, pi/2]
// (shape_features.cpp:176-197).  The wrap is a discontinuity: an ROI whose
// rounded b is a tiny negative with a < c sits at atan2 = -pi + |2b / (a - c)|,
// which rounds to -pi (wraps to +pi/2) or to the next double (stays near -pi/2)
// by half an ulp.  CUDA's atan2 is accurate to 2 ulp, glibc's to the rounding,
// so near +-pi the angle is rebuilt as (pi_lo - atan|y/x|) + pi_hi with one
// final rounding, which lands on the side the reference lands on.
__device__ __forceinline__ double ellipse_orientation(double bb, double amc) {
    const double y = 2.0 * bb;
    double t;
    if (amc < 0.0 && fabs(y) < -1e-8 * amc) {
        const double r = atan(fabs(y) / -amc);
        t = copysign(__dadd_rn(__dsub_rn(1.2246467991473532e-16, r), 3.141592653589793), y);
    } else {
        t = atan2(y, amc);
    }
    double th = 0.5 * t;
    if (th <= -3.141592653589793 / 2.0) th += 3.141592653589793;
    return th;
}

// --------------------------------------------------------- debug capture --

struct DebugOut {
    uint32_t label;        // ROI to capture (0 = none)
    int nb;                // histogram bins
    unsigned long long* hist;   // [nb]
    int32_t* edge_xy;      // [2*cap_edge]
    uint32_t cap_edge;
    uint32_t* n_edge;
    uint32_t* glcm;        // [A][ng][ng]
    unsigned long long* pairs;  // [A]
};

// ------------------------------------------------------------- helpers ---

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}


// Butterfly reduce-scatter of 32 per-lane doubles: lane i ends with sum_j v[i] over lanes.
__device__ __forceinline__ double reduce_scatter32(double (&v)[32]) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
            const double send = upper ? v[j] : v[j + s];
            const double recv = __shfl_xor_sync(kFull, send, s);
            v[j] = (upper ? v[j + s] : v[j]) + recv;
        }
    }
    return v[0];
}

// Union-find over run indices (lock-free link of the larger root under the
// smaller one; roots are minimal run indices == first run in row-major order).
__device__ __forceinline__ uint32_t uf_find(volatile uint32_t* parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        const uint32_t gp = parent[p];
        if (gp != p) parent[x] = gp;
        x = p;
        p = gp;
    }
    return x;
}
// root without path compression: safe to run concurrently with other readers
__device__ __forceinline__ uint32_t uf_root(const uint32_t* parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}
__device__ __forceinline__ void uf_union(uint32_t* parent, uint32_t a, uint32_t b) {
    volatile uint32_t* vp = parent;
    for (;;) {
        a = uf_find(vp, a);
        b = uf_find(vp, b);
        if (a == b) return;
        if (a > b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicCAS(&parent[b], b, a);
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ uint64_t bits_between(int s, int e) {  // bits [s, e], 0<=s<=e<=63
    const uint64_t hi = (e >= 63) ? ~0ull : ((1ull << (e + 1)) - 1ull);
    return hi & (~0ull << s);
}

// exact percentile of the reference (intensity_features.cpp:14-22): literal
// expression order, no FMA contraction.
__device__ __forceinline__ double percentile_exact(const uint16_t* s, unsigned long long n,
                                                   double p) {
    if (n == 1) return (double)s[0];
    const double rank = __dmul_rn(__ddiv_rn(p, 100.0), (double)(n - 1));
    const unsigned long long lo = (unsigned long long)rank;
    if (lo + 1 >= n) return (double)s[n - 1];
    const double frac = __dsub_rn(rank, (double)lo);
    const double a = (double)s[lo], b = (double)s[lo + 1];
    return __dadd_rn(a, __dmul_rn(frac, __dsub_rn(b, a)));
}


// Moments epilogue (moments.cpp:32-92), warp-level.  Lane i holds N_i: the sums
// of w dx^p dy^q about the integer anchors (binary lanes 0..15: w = 1 about
// (axb, ayb); weighted lanes 16..31: w = I about (axw, ayw)), p = (i>>2)&3,
// q = i&3.  Binomial shift to the exact centroid (central) and to the image origin
// (raw, global coordinates via the window origin gx0/gy0); eta, Hu.  Writes the
// 104 moment columns at o.
__device__ __forceinline__ void moments_epilogue(double N, double dn, unsigned long long n,
                                                 unsigned long long sS, unsigned long long sLX,
                                                 unsigned long long sLY, unsigned long long sXI,
                                                 unsigned long long sYI, long long axb,
                                                 long long ayb, long long axw, long long ayw,
                                                 long long gx0, long long gy0, double* o) {
    const unsigned lane = lane_id();
    const long long nb_ = (long long)n, W = (long long)sS;
    const int grp = lane >> 4, p = (lane >> 2) & 3, q = lane & 3;
    const double m00 = grp ? (double)sS : dn;
    const bool zero_mass = grp && sS == 0;
    // fractional offset of the true centroid from the anchor
    const double dx = grp ? (W > 0 ? (double)((long long)sXI - axw * W) / (double)W : 0.0)
                          : (double)((long long)sLX - axb * nb_) / dn;
    const double dy = grp ? (W > 0 ? (double)((long long)sYI - ayw * W) / (double)W : 0.0)
                          : (double)((long long)sLY - ayb * nb_) / dn;
    const double Ax = (double)(gx0 + (grp ? axw : axb));
    const double Ay = (double)(gy0 + (grp ? ayw : ayb));
    const double C[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 2, 1, 0}, {1, 3, 3, 1}};
    double pmx[4], pmy[4], pax[4], pay[4];
    pmx[0] = pmy[0] = pax[0] = pay[0] = 1.0;
#pragma unroll
    for (int k = 1; k < 4; ++k) {
        pmx[k] = pmx[k - 1] * (-dx);
        pmy[k] = pmy[k - 1] * (-dy);
        pax[k] = pax[k - 1] * Ax;
        pay[k] = pay[k - 1] * Ay;
    }
    double mu = 0, raw = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double Nij = __shfl_sync(kFull, N, (grp << 4) | (i << 2) | j);
            if (i <= p && j <= q) {
                const double cc = C[p][i] * C[q][j];
                mu += cc * pmx[p - i] * pmy[q - j] * Nij;
                raw += cc * pax[p - i] * pay[q - j] * Nij;
            }
        }
    if ((p == 1 && q == 0) || (p == 0 && q == 1)) mu = 0.0;  // moments.cpp:80-81
    if (p == 0 && q == 0) mu = N;
    double eta = 0;
    if (p + q >= 2) eta = mu / pow(m00, 1.0 + (p + q) / 2.0);
    if (zero_mass) {
        raw = 0;
        mu = 0;
        eta = 0;
    }
    // Hu invariants (moments.cpp:14-28) on lanes 0 / 16
    const double n20 = __shfl_sync(kFull, eta, (grp << 4) | 8);
    const double n02 = __shfl_sync(kFull, eta, (grp << 4) | 2);
    const double n11 = __shfl_sync(kFull, eta, (grp << 4) | 5);
    const double n30 = __shfl_sync(kFull, eta, (grp << 4) | 12);
    const double n03 = __shfl_sync(kFull, eta, (grp << 4) | 3);
    const double n21 = __shfl_sync(kFull, eta, (grp << 4) | 9);
    const double n12 = __shfl_sync(kFull, eta, (grp << 4) | 6);
    o += grp * 52;
    const int li = lane & 15;
    o[li] = raw;
    o[16 + li] = mu;
    if (p + q >= 2) {
        const int eidx = (p == 0) ? q - 2 : (p == 1 ? 1 + q : 1 + 4 * (p - 1) + q);
        o[32 + eidx] = eta;
    }
    if (li == 0) {
        const double a = n30 + n12, b = n21 + n03;
        double hu[7];
        hu[0] = n20 + n02;
        hu[1] = (n20 - n02) * (n20 - n02) + 4.0 * n11 * n11;
        hu[2] = (n30 - 3.0 * n12) * (n30 - 3.0 * n12) + (3.0 * n21 - n03) * (3.0 * n21 - n03);
        hu[3] = a * a + b * b;
        hu[4] = (n30 - 3.0 * n12) * a * (a * a - 3.0 * b * b) +
                (3.0 * n21 - n03) * b * (3.0 * a * a - b * b);
        hu[5] = (n20 - n02) * (a * a - b * b) + 4.0 * n11 * a * b;
        hu[6] = (3.0 * n21 - n03) * a * (a * a - 3.0 * b * b) -
                (n30 - 3.0 * n12) * b * (3.0 * a * a - b * b);
#pragma unroll
        for (int k = 0; k < 7; ++k) o[45 + k] = zero_mass ? 0.0 : hu[k];
    }
    __syncwarp();
}

// Byte offsets of one CTA's global scratch slab in the large-ROI kernel (fx_roi_b.cu),
// sized on the host from the largest L window / pixel count of the launch.
struct BLayout {
    size_t rowmask, kmask, emask, wordoff, tmpw, xy, vals, lraster, lvl, vhist, runoff, rs, re, parent,
        rsize, bins, ghist, ctop, cbot, hv;
    size_t bytes;
    unsigned long long RCAP;  // level-raster capacity (cells): dense windows only
    uint32_t H, WPR, NMAX, RUNMAX, NB;
};

// Byte offsets of one CTA's slab in the GLRLM/GLSZM/NGTDM kernel (fx_roi_t.cu).
struct TLayout {
    size_t lev, par, zsz, hjk, hjc, ext, ccnt;
    size_t bytes;
    unsigned long long CELLS;  // max window cells
    uint32_t NMAX, HC;         // max ROI pixels; count-table capacity (power of 2)
};

// Byte offsets of one CTA's slab in the wide texture kernel (fx_wide.cu, ng > 256).
struct WLayout {
    size_t lev, par, keys, px, pext, sv, plist;
    size_t bytes;
    unsigned long long CELLS, NMAX;  // max window cells / ROI pixels of the launch
    uint32_t NG;
};

}  // namespace fxg
