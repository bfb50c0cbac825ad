// GLCM helpers shared by the per-ROI kernels (one copy per translation unit: the
// library is built without relocatable device code).
#pragma once

#include "fx_dev.cuh"

namespace fxg {
namespace {

__device__ __noinline__ double nlog2(double x) { return log2(x); }

// log2 of small integers (run lengths / counts), filled once per process
constexpr int kLog2Tab = 4096;
__device__ double g_log2_tab[kLog2Tab + 1];
__device__ __forceinline__ double log2_int(uint32_t c) {
    return c <= (uint32_t)kLog2Tab ? __ldg(&g_log2_tab[c]) : nlog2((double)c);
}
// 1/(1+d^2), 1/(1+d), 1/d^2 for grey-level differences d < 256 (Haralick weights)
__device__ double g_rcp_tab[3][256];
__global__ void k_init_log2_tab() {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i <= kLog2Tab; i += blockDim.x * gridDim.x)
        g_log2_tab[i] = i ? log2((double)i) : 0.0;
    for (int d = threadIdx.x + blockIdx.x * blockDim.x; d < 256; d += blockDim.x * gridDim.x) {
        const double dd = (double)d;
        g_rcp_tab[0][d] = 1.0 / (1.0 + dd * dd);
        g_rcp_tab[1][d] = 1.0 / (1.0 + dd);
        g_rcp_tab[2][d] = d ? 1.0 / (dd * dd) : 0.0;
    }
}

// warp sum of 8 doubles (transpose-reduce); every lane returns all 8 sums
__device__ __forceinline__ void warp_sum8(double (&v)[8]) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int s = 16, half = 4; s >= 4; s >>= 1, half >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const double send = up ? v[j] : v[j + half];
            const double recv = __shfl_xor_sync(kFull, send, s);
            v[j] = (up ? v[j + half] : v[j]) + recv;
        }
    }
    double t = v[0];
    t += __shfl_xor_sync(kFull, t, 2);
    t += __shfl_xor_sync(kFull, t, 1);
    // lane L holds index ((L>>4)&1)<<2 | ((L>>3)&1)<<1 | ((L>>2)&1)
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(kFull, t, ((k >> 2) << 4) | (((k >> 1) & 1) << 3) | ((k & 1) << 2));
}

// Haralick statistics of one GLCM from its integer marginals (texture.cpp:87-217):
// px/py (p_y == p_x when symmetric), psum [2ng-1], pdif [ng]; T = total mass, the
// cell sums s2 = sum m c, sa = sum (a+1)(b+1) m, jm = max c, el = sum m (log2 T -
// log2 c).  hxy1 == hxy2 == hx + hy for exact marginals.
// Warp-level; st[k] = statistic k in texture.hpp order on every lane.
__device__ __forceinline__ void haralick_finish(const uint32_t* px, const uint32_t* py,
                                                const uint32_t* psum, const uint32_t* pdif,
                                                int ng, bool sym, double T, double logT,
                                                unsigned long long s2, unsigned long long sa,
                                                uint32_t jm, double el, double (&st)[29]) {
    const unsigned lane = lane_id();
    const double iT = 1.0 / T;
    const double asm2 = (double)s2 / (T * T), acor_ = (double)sa * iT;
    const double ent_ = el * iT, jmax = (double)jm * iT;
    // marginals -> means, entropies (p log p from integer counts); p = m / T as
    // m * (1 / T) except m == T, which gives exactly 1 as the reference's division
    // does (a marginal on one level must have variance exactly 0); elsewhere the
    // two differ by at most one ulp
    auto pr = [&](uint32_t m) -> double { return (double)m == T ? 1.0 : (double)m * iT; };
    double r8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // mux, muy, sumave, sument, difave, hx, hy
    for (int g = lane; g < ng; g += 32) {  // symmetric: p_y == p_x
        const uint32_t ma = px[g];
        const double pa = pr(ma);
        r8[0] += (g + 1) * pa;
        if (ma) r8[5] -= pa * (log2_int(ma) - logT);
        if (!sym) {
            const uint32_t mb = py[g];
            const double pb = pr(mb);
            r8[1] += (g + 1) * pb;
            if (mb) r8[6] -= pb * (log2_int(mb) - logT);
        }
    }
    for (int k = lane; k < 2 * ng - 1; k += 32) {
        const uint32_t m = psum[k];
        if (m) {
            const double p = pr(m);
            r8[2] += (k + 2) * p;
            r8[3] -= p * (log2_int(m) - logT);
        }
    }
    for (int d = lane; d < ng; d += 32) {
        const uint32_t m = pdif[d];
        if (m) r8[4] += d * pr(m);
    }
    warp_sum8(r8);
    const double mux = r8[0], muy = sym ? r8[0] : r8[1], sumave = r8[2], sument = r8[3];
    const double difave = r8[4], hx = r8[5], hy = sym ? r8[5] : r8[6];
    double s8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // vx, vy, sumvar, clut, clus, clup, difent
    for (int g = lane; g < ng; g += 32) {
        const double a1 = pr(px[g]);
        s8[0] += (g + 1 - mux) * (g + 1 - mux) * a1;
        if (!sym) {
            const double b1 = pr(py[g]);
            s8[1] += (g + 1 - muy) * (g + 1 - muy) * b1;
        }
    }
    for (int k = lane; k < 2 * ng - 1; k += 32) {
        const uint32_t m = psum[k];
        if (m) {
            const double p = pr(m);
            s8[2] += (k + 2 - sumave) * (k + 2 - sumave) * p;
            const double sv = k + 2 - mux - muy;
            s8[3] += sv * sv * p;
            s8[4] += sv * sv * sv * p;
            s8[5] += sv * sv * sv * sv * p;
        }
    }
    double d8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // difent, contrast, idm, id, idn, idmn, iv, difvar
    const double dng = (double)ng;
    for (int d = lane; d < ng; d += 32) {
        const uint32_t m = pdif[d];
        if (m) {
            const double p = pr(m), dd = (double)d;
            d8[0] -= p * (log2_int(m) - logT);
            d8[1] += dd * dd * p;
            const bool tab = d < 256;  // the tables cover d < 256 (ng <= 256 always)
            d8[2] += p * (tab ? __ldg(&g_rcp_tab[0][d]) : 1.0 / (1.0 + dd * dd));
            d8[3] += p * (tab ? __ldg(&g_rcp_tab[1][d]) : 1.0 / (1.0 + dd));
            d8[4] += p * dng / (dng + dd);
            d8[5] += p * (dng * dng) / (dng * dng + dd * dd);
            if (d > 0) d8[6] += p * (tab ? __ldg(&g_rcp_tab[2][d]) : 1.0 / (dd * dd));
            d8[7] += (dd - difave) * (dd - difave) * p;
        }
    }
    warp_sum8(s8);
    warp_sum8(d8);
    const double vx = s8[0], vy = sym ? s8[0] : s8[1];
    const double corr = (vx > 0 && vy > 0) ? (acor_ - mux * muy) / sqrt(vx * vy) : 0.0;
    const double hxy = hx + hy, hmax = fmax(hx, hy);
    const double v29[29] = {asm2, acor_, s8[5], s8[4], s8[3], d8[1], corr, difave, d8[0],
                            d8[7], difave, sqrt(asm2), ent_, d8[3], d8[2], d8[3], d8[4],
                            d8[2], d8[5], hmax > 0 ? (ent_ - hxy) / hmax : 0.0,
                            sqrt(fmax(0.0, 1.0 - exp(-2.0 * (hxy - ent_)))), d8[6], mux,
                            ent_, jmax, vx, sumave, sument, s8[2]};
#pragma unroll
    for (int k = 0; k < 29; ++k) st[k] = v29[k];
}

}  // namespace
}  // namespace fxg
