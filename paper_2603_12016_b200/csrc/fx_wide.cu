// Texture groups with more than 256 grey levels (GLCM, GLRLM, GLSZM, NGTDM).
//
// The per-ROI texture paths keep levels in 8 bits and size their per-level arrays
// for ng <= 256.  The reference accepts any ng >= 2 (texture.cpp:29-56, :58-85);
// its level grid is int16 (texture.hpp:15-28), so ng <= 32768 covers every grid
// it can build.  Above 256 levels every ROI's texture columns come from this
// kernel instead (the other groups still run on their usual kernels):
//   - one 256-thread CTA per ROI, persistent over the queued ROIs, with a slab in
//     global memory (L2-resident for typical windows) sized from the launch's
//     largest window, pixel count and ng;
//   - the window is discretised once into a u16 level raster (integer floor of
//     ng (v - lo) / (hi - lo + 1), equal to the reference's double formula);
//   - GLCM pairs, GLRLM runs and GLSZM zones become 64-bit keys (level pair, or
//     level << 32 | extent) collected in any order, then sorted by a bitonic
//     network over the slab, so cells come out in key order -- the reference's
//     std::map order -- and every floating-point sum runs in a fixed order;
//   - GLCM statistics from integer marginals through haralick_finish (shared with
//     the <= 256-level paths); GLRLM / GLSZM statistics from the sorted cells
//     (texture.cpp:282-341, :382-441); NGTDM with the neighbourhood differences
//     kept exactly in units of 1/840 (texture.cpp:443-528).
// Sparse in ng: nothing is O(ng^2); arrays of ng entries are cleared per use.
#include "fx_glcm.cuh"
#include "fx_roi.cuh"

#include <algorithm>

namespace fxg {

namespace {

constexpr int kWT = 256, kWW = kWT / 32;
constexpr uint16_t kNoLev = 0xffffu;
constexpr unsigned long long kKeyPad = ~0ull;

struct WShared {
    double d[kWW][8];
    unsigned long long u[kWW];
    uint32_t m[kWW];
    uint32_t cnt, job;
    double st[29];
};

// deterministic block sums: warp butterflies, then the warps' partials in order
template <int K>
__device__ __forceinline__ void wsum(double (&v)[K], WShared& sm) {
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sm.d[w][k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double t = 0;
        for (int i = 0; i < kWW; ++i) t += sm.d[i][k];
        v[k] = t;
    }
    __syncthreads();
}
__device__ __forceinline__ unsigned long long wsum_u64(unsigned long long v, WShared& sm) {
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sm.u[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    for (int i = 0; i < kWW; ++i) t += sm.u[i];
    __syncthreads();
    return t;
}
__device__ __forceinline__ uint32_t wmax_u32(uint32_t v, WShared& sm) {
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) sm.m[w] = v;
    __syncthreads();
    uint32_t t = 0;
    for (int i = 0; i < kWW; ++i) t = max(t, sm.m[i]);
    __syncthreads();
    return t;
}
__device__ __forceinline__ uint32_t wmin_u32(uint32_t v, WShared& sm) {
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    v = warp_min(v);
    __syncthreads();
    if (lane == 0) sm.m[w] = v;
    __syncthreads();
    uint32_t t = 0xffffffffu;
    for (int i = 0; i < kWW; ++i) t = min(t, sm.m[i]);
    __syncthreads();
    return t;
}

// ascending bitonic sort of keys[0, np) (np a power of two) by the block
__device__ void wsort(unsigned long long* keys, uint32_t np) {
    for (uint32_t k = 2; k <= np; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < np; i += kWT) {
                const uint32_t l = i ^ j;
                if (l <= i) continue;
                const unsigned long long a = keys[i], b = keys[l];
                const bool up = (i & k) == 0;
                if ((a > b) == up) {
                    keys[i] = b;
                    keys[l] = a;
                }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t n) {
    uint32_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

// keys[0, n) -> padded, sorted; returns the padded length
__device__ uint32_t wsort_keys(unsigned long long* keys, uint32_t n) {
    const uint32_t np = pow2_at_least(max(n, 2u));
    for (uint32_t i = n + threadIdx.x; i < np; i += kWT) keys[i] = kKeyPad;
    __syncthreads();
    wsort(keys, np);
    return np;
}

// run of equal keys starting at i (i is a run start): its length
__device__ __forceinline__ uint32_t run_len(const unsigned long long* k, uint32_t i, uint32_t n) {
    uint32_t e = i + 1;
    while (e < n && k[e] == k[i]) ++e;
    return e - i;
}

struct WSlab {
    uint16_t* lev;             // [cells] levels, kNoLev outside the ROI
    uint32_t* par;             // [cells] GLSZM union-find parents, then zone sizes
    unsigned long long* keys;  // [NP] pair / run / zone keys (sorted in place)
    uint32_t* px;              // [ng]
    uint32_t* py;              // [ng]
    uint32_t* pdif;            // [ng]
    uint32_t* psum;            // [2 ng]
    uint32_t* plev;            // [ng] units per level (GLRLM / GLSZM), NGTDM pixels
    uint32_t* pext;            // [NMAX + 1] units per extent
    unsigned long long* sv;    // [ng] NGTDM |differences| in units of 1/840
    uint32_t* plist;           // [ng] NGTDM present levels, ascending
};

__device__ WSlab wslab(uint8_t* base, const WLayout& L) {
    WSlab S;
    S.lev = (uint16_t*)(base + L.lev);
    S.par = (uint32_t*)(base + L.par);
    S.keys = (unsigned long long*)(base + L.keys);
    S.px = (uint32_t*)(base + L.px);
    S.py = S.px + L.NG;
    S.pdif = S.py + L.NG;
    S.psum = S.pdif + L.NG;
    S.plev = S.psum + 2 * L.NG;
    S.pext = (uint32_t*)(base + L.pext);
    S.sv = (unsigned long long*)(base + L.sv);
    S.plist = (uint32_t*)(base + L.plist);
    return S;
}

__device__ __forceinline__ void wzero(uint32_t* a, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += kWT) a[i] = 0u;
}

// GLRLM / GLSZM statistics of sorted (level << 32 | extent) keys (texture.cpp:282-341,
// :382-441): np_roi = ROI pixels; emax = largest possible extent
__device__ void extent_stats(const unsigned long long* keys, uint32_t n, unsigned long long np_roi,
                             int ng, uint32_t emax, const WSlab& S, WShared& sm, double* out16) {
    const unsigned tid = threadIdx.x;
    if (n == 0) {
        if (tid < 16) out16[tid] = 0.0;
        __syncthreads();
        return;
    }
    wzero(S.plev, (uint32_t)ng);
    wzero(S.pext, emax + 1);
    __syncthreads();
    const double nr = (double)n;
    // pass A over the cells (run starts): unit terms, per level / extent counts, means
    double a[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = tid; i < n; i += kWT) {
        if (i > 0 && keys[i - 1] == keys[i]) continue;
        const uint32_t c = run_len(keys, i, n);
        const uint32_t lv = (uint32_t)(keys[i] >> 32), ex = (uint32_t)keys[i];
        const double r = (double)c, g = lv + 1.0, l = (double)ex;
        a[0] += r / (l * l);
        a[1] += r * l * l;
        a[2] += r / (g * g);
        a[3] += r * g * g;
        a[4] += r / (g * g * l * l);
        a[5] += r * g * g / (l * l);
        a[6] += r * l * l / (g * g);
        a[7] += r * g * g * l * l;
        const double p = r / nr;
        a[8] -= p * log2(p);
        a[9] += p * g;
        a[10] += p * l;
        atomicAdd(&S.plev[lv], c);
        atomicAdd(&S.pext[ex], c);
    }
    double a8[8] = {a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]};
    double a3[3] = {a[8], a[9], a[10]};
    wsum(a8, sm);
    wsum(a3, sm);
    const double mu_g = a3[1], mu_l = a3[2];
    double b[4] = {0, 0, 0, 0};  // glv, rv, glnu, rlnu
    for (uint32_t i = tid; i < n; i += kWT) {
        if (i > 0 && keys[i - 1] == keys[i]) continue;
        const uint32_t c = run_len(keys, i, n);
        const double p = (double)c / nr;
        const double g = (double)(keys[i] >> 32) + 1.0, l = (double)(uint32_t)keys[i];
        b[0] += p * (g - mu_g) * (g - mu_g);
        b[1] += p * (l - mu_l) * (l - mu_l);
    }
    for (uint32_t g = tid; g < (uint32_t)ng; g += kWT) {
        const double c = (double)S.plev[g];
        b[2] += c * c;
    }
    for (uint32_t e = tid; e <= emax; e += kWT) {
        const double c = (double)S.pext[e];
        b[3] += c * c;
    }
    wsum(b, sm);
    if (tid == 0) {
        const double v[16] = {a8[0] / nr, a8[1] / nr, b[2] / nr, b[2] / (nr * nr), b[3] / nr,
                              b[3] / (nr * nr), nr / (double)np_roi, b[0], b[1], a3[0], a8[2] / nr,
                              a8[3] / nr, a8[4] / nr, a8[5] / nr, a8[6] / nr, a8[7] / nr};
        for (int k = 0; k < 16; ++k) out16[k] = v[k];
    }
    __syncthreads();
}

// GLRLM scan direction of an angle (texture.cpp:242-280)
__device__ __forceinline__ void run_dir(int angle, int& dx, int& dy) {
    dx = 1;
    dy = 0;
    if (angle == 45) dy = -1;
    else if (angle == 90) { dx = 0; dy = 1; }
    else if (angle == 135) dy = 1;
}

__device__ __forceinline__ uint32_t w_root(uint32_t* par, uint32_t x) {
    uint32_t p = ((volatile uint32_t*)par)[x];
    while (p != x) {
        x = p;
        p = ((volatile uint32_t*)par)[x];
    }
    return x;
}
__device__ void w_union(uint32_t* par, uint32_t a, uint32_t b) {
    for (;;) {
        a = w_root(par, a);
        b = w_root(par, b);
        if (a == b) return;
        if (a > b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&par[b], b, a) == b) return;
    }
}

__device__ void process_wide(uint32_t r, const DevImage& img, const RoiList& rl, const FeatCfg& cfg,
                             double* out, const WSlab& S, const WLayout& L, WShared& sm) {
    const unsigned tid = threadIdx.x;
    const uint32_t lab = rl.label[r], x0 = rl.x0[r], y0 = rl.y0[r], w = rl.w[r], h = rl.h[r];
    const unsigned long long n = rl.n[r];
    const uint32_t cells = w * h;
    const int ng = cfg.ng, A = cfg.n_angles;
    double* orow = out + (size_t)r * cfg.ncols;
    // grey range of the ROI, then its level raster (texture.cpp:29-56)
    uint32_t lo = 0xffffu, hi = 0u;
    for (uint32_t c = tid; c < cells; c += kWT) {
        const uint32_t y = c / w, x = c - y * w;
        const size_t o = (size_t)(y0 + y) * img.pitch + x0 + x;
        if (img.L[o] == lab) {
            const uint32_t v = img.I[o];
            lo = min(lo, v);
            hi = max(hi, v);
        }
    }
    lo = wmin_u32(lo, sm);
    hi = wmax_u32(hi, sm);
    const unsigned long long span = (unsigned long long)(hi - lo) + 1ull;
    for (uint32_t c = tid; c < cells; c += kWT) {
        const uint32_t y = c / w, x = c - y * w;
        const size_t o = (size_t)(y0 + y) * img.pitch + x0 + x;
        uint16_t lv = kNoLev;
        if (img.L[o] == lab) {
            unsigned long long q = 0;
            if (hi > lo) q = (unsigned long long)ng * (img.I[o] - lo) / span;
            lv = (uint16_t)(q < (unsigned long long)(ng - 1) ? q : (unsigned long long)(ng - 1));
        }
        S.lev[c] = lv;
    }
    __syncthreads();
    auto at = [&](int x, int y) -> uint32_t {
        return (x < 0 || y < 0 || x >= (int)w || y >= (int)h) ? kNoLev : S.lev[(uint32_t)y * w + (uint32_t)x];
    };
    const bool sym = cfg.symmetric != 0;
    // ---- GLCM (texture.cpp:58-217), per sorted angle
    if (cfg.col_glcm >= 0) {
        double acc29 = 0;
        for (int a = 0; a < A; ++a) {
            const int ddx = cfg.dx[a], ddy = cfg.dy[a];
            if (tid == 0) sm.cnt = 0;
            __syncthreads();
            for (uint32_t c = tid; c < cells; c += kWT) {
                const uint32_t la = S.lev[c];
                if (la == kNoLev) continue;
                const uint32_t y = c / w, x = c - y * w;
                const uint32_t lb = at((int)x + ddx, (int)y + ddy);
                if (lb == kNoLev) continue;
                const uint32_t i = atomicAdd(&sm.cnt, 1u);
                const uint32_t ka = sym ? min(la, lb) : la, kb = sym ? max(la, lb) : lb;
                S.keys[i] = (unsigned long long)ka * (unsigned long long)ng + kb;
            }
            __syncthreads();
            const uint32_t np = sm.cnt;
            __syncthreads();
            if (np == 0) {
                if (tid < 29) sm.st[tid] = 0.0;
                __syncthreads();
            } else {
                wsort_keys(S.keys, np);
                wzero(S.px, (uint32_t)(5 * ng));  // px, py, pdif, psum (2 ng)
                __syncthreads();
                const double T = sym ? 2.0 * (double)np : (double)np;
                const double logT = nlog2(T);
                unsigned long long s2 = 0, sa = 0;
                uint32_t jm = 0;
                double el[1] = {0};
                for (uint32_t i = tid; i < np; i += kWT) {
                    if (i > 0 && S.keys[i - 1] == S.keys[i]) continue;
                    const uint32_t c = run_len(S.keys, i, np);
                    const unsigned long long k = S.keys[i];
                    const uint32_t ga = (uint32_t)(k / (unsigned long long)ng), gb = (uint32_t)(k % (unsigned long long)ng);
                    const bool off = sym && ga != gb;
                    const uint32_t cc = (sym && !off) ? 2u * c : c;
                    const uint32_t mcc = off ? 2u * cc : cc;
                    s2 += (unsigned long long)mcc * cc;
                    sa += (unsigned long long)(ga + 1) * (gb + 1) * mcc;
                    jm = max(jm, cc);
                    el[0] += (double)mcc * (logT - log2_int(cc));
                    atomicAdd(&S.px[ga], cc);
                    if (off) atomicAdd(&S.px[gb], cc);
                    if (!sym) atomicAdd(&S.py[gb], cc);
                    atomicAdd(&S.psum[ga + gb], mcc);
                    atomicAdd(&S.pdif[ga > gb ? ga - gb : gb - ga], mcc);
                }
                s2 = wsum_u64(s2, sm);
                sa = wsum_u64(sa, sm);
                jm = wmax_u32(jm, sm);
                wsum(el, sm);
                if ((tid >> 5) == 0) {
                    double st[29];
                    haralick_finish(S.px, sym ? S.px : S.py, S.psum, S.pdif, ng, sym, T, logT, s2, sa,
                                    jm, el[0], st);
                    if (tid == 0)
                        for (int k = 0; k < 29; ++k) sm.st[k] = st[k];
                }
                __syncthreads();
            }
            if (tid < 29) {
                orow[cfg.col_glcm + tid * (A + 1) + a] = sm.st[tid];
                acc29 += sm.st[tid];
            }
            __syncthreads();
        }
        if (tid < 29) orow[cfg.col_glcm + tid * (A + 1) + A] = acc29 / (double)A;
    }
    const uint32_t emax = max(w, h);
    // ---- GLRLM (texture.cpp:242-341), per sorted angle
    if (cfg.col_glrlm >= 0) {
        double acc16 = 0;
        for (int a = 0; a < A; ++a) {
            int dx, dy;
            run_dir(cfg.angle[a], dx, dy);
            if (tid == 0) sm.cnt = 0;
            __syncthreads();
            for (uint32_t c = tid; c < cells; c += kWT) {
                const uint32_t g = S.lev[c];
                if (g == kNoLev) continue;
                const int y = (int)(c / w), x = (int)(c - (uint32_t)y * w);
                if (at(x - dx, y - dy) == g) continue;  // not a run start
                uint32_t len = 1;
                for (int nx = x + dx, ny = y + dy; at(nx, ny) == g; nx += dx, ny += dy) ++len;
                S.keys[atomicAdd(&sm.cnt, 1u)] = ((unsigned long long)g << 32) | len;
            }
            __syncthreads();
            const uint32_t nr = sm.cnt;
            __syncthreads();
            double f16[16];
            if (nr) wsort_keys(S.keys, nr);
            extent_stats(S.keys, nr, n, ng, emax, S, sm, sm.st);
            for (int k = 0; k < 16; ++k) f16[k] = sm.st[k];
            if (tid < 16) {
                orow[cfg.col_glrlm + tid * (A + 1) + a] = f16[tid];
                acc16 += f16[tid];
            }
            __syncthreads();
        }
        if (tid < 16) orow[cfg.col_glrlm + tid * (A + 1) + A] = acc16 / (double)A;
    }
    // ---- GLSZM (texture.cpp:343-441): 8-connected zones of equal level
    if (cfg.col_glszm >= 0) {
        unsigned long long* kk = S.keys;  // [0, cells): scratch, [cells, 2 cells): zone keys
        for (uint32_t c = tid; c < cells; c += kWT) S.par[c] = c;
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT) {  // forward neighbours E, SW, S, SE
            const uint32_t g = S.lev[c];
            if (g == kNoLev) continue;
            const int y = (int)(c / w), x = (int)(c - (uint32_t)y * w);
            const int nx[4] = {x + 1, x - 1, x, x + 1}, ny[4] = {y, y + 1, y + 1, y + 1};
            for (int k = 0; k < 4; ++k)
                if (at(nx[k], ny[k]) == g) w_union(S.par, c, (uint32_t)ny[k] * w + (uint32_t)nx[k]);
        }
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT)  // flatten: roots first, then publish
            kk[c] = S.lev[c] != kNoLev ? w_root(S.par, c) : c;
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT) S.par[c] = (uint32_t)kk[c];
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT) kk[c] = 0ull;  // zone sizes at the roots
        if (tid == 0) sm.cnt = 0;
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT)
            if (S.lev[c] != kNoLev) atomicAdd(&kk[S.par[c]], 1ull);
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kWT)
            if (S.lev[c] != kNoLev && S.par[c] == c)
                kk[cells + atomicAdd(&sm.cnt, 1u)] = ((unsigned long long)S.lev[c] << 32) | kk[c];
        __syncthreads();
        const uint32_t nz = sm.cnt;
        __syncthreads();
        for (uint32_t i = tid; i < nz; i += kWT) kk[i] = kk[cells + i];  // nz <= cells: disjoint
        __syncthreads();
        if (nz) wsort_keys(kk, nz);
        extent_stats(kk, nz, n, ng, (uint32_t)(n < 0xfffffffeull ? n : 0xfffffffeull), S, sm, sm.st);
        if (tid < 16) orow[cfg.col_glszm + tid] = sm.st[tid];
        __syncthreads();
    }
    // ---- NGTDM (texture.cpp:443-528): |(g+1) - mean of the in-ROI 8-neighbours|,
    // denominator 1..8, accumulated exactly in units of 1/840
    if (cfg.col_ngtdm >= 0) {
        wzero(S.plev, (uint32_t)ng);
        for (uint32_t g = tid; g < (uint32_t)ng; g += kWT) S.sv[g] = 0ull;
        __syncthreads();
        unsigned long long valid = 0;
        for (uint32_t c = tid; c < cells; c += kWT) {
            const uint32_t g = S.lev[c];
            if (g == kNoLev) continue;
            const int y = (int)(c / w), x = (int)(c - (uint32_t)y * w);
            int sum = 0, cnt = 0;
            for (int ddy = -1; ddy <= 1; ++ddy)
                for (int ddx = -1; ddx <= 1; ++ddx) {
                    if (!ddx && !ddy) continue;
                    const uint32_t q = at(x + ddx, y + ddy);
                    if (q != kNoLev) {
                        sum += (int)q + 1;
                        ++cnt;
                    }
                }
            if (!cnt) continue;
            const long long d = (long long)(g + 1) * cnt - sum;
            atomicAdd(&S.sv[g], (unsigned long long)((d < 0 ? -d : d) * (840 / cnt)));
            atomicAdd(&S.plev[g], 1u);
            ++valid;
        }
        const unsigned long long nvu = wsum_u64(valid, sm);
        double o5[5] = {0, 0, 0, 0, 0};
        if (nvu) {
            const double nv = (double)nvu;
            // present levels in ascending order (warp 0, ballot compaction)
            if ((tid >> 5) == 0) {
                const unsigned ln = lane_id();
                uint32_t k = 0;
                for (int i0 = 0; i0 < ng; i0 += 32) {
                    const int i = i0 + (int)ln;
                    const bool pr = i < ng && S.plev[i] != 0u;
                    const unsigned b = __ballot_sync(kFull, pr);
                    if (pr) S.plist[k + __popc(b & lanemask_lt())] = (uint32_t)i;
                    k += __popc(b);
                }
                if (ln == 0) sm.cnt = k;
            }
            __syncthreads();
            const uint32_t P = sm.cnt;
            double r2[2] = {0, 0};
            for (uint32_t k = tid; k < P; k += kWT) {
                const uint32_t i = S.plist[k];
                const double p = (double)S.plev[i] / nv, s = (double)S.sv[i] / 840.0;
                r2[0] += s;
                r2[1] += p * s;
            }
            wsum(r2, sm);
            const double s_total = r2[0], ps_total = r2[1];
            double a4[4] = {0, 0, 0, 0};  // contrast, busyness, complexity, strength
            for (uint32_t ki = tid; ki < P; ki += kWT) {
                const uint32_t i = S.plist[ki];
                const double pi = (double)S.plev[i] / nv, si = (double)S.sv[i] / 840.0, gi = i + 1.0;
                for (uint32_t kj = ki + 1; kj < P; ++kj) {
                    const uint32_t j = S.plist[kj];
                    const double pj = (double)S.plev[j] / nv, sj = (double)S.sv[j] / 840.0, gj = j + 1.0;
                    const double di = (double)i - (double)j;
                    a4[0] += pi * pj * di * di;
                    a4[1] += fabs(__dsub_rn(__dmul_rn(gi, pi), __dmul_rn(gj, pj)));  // unfused (fx_roi_t.cu)
                    a4[2] += fabs(gi - gj) * (pi * si + pj * sj) / (pi + pj);
                    a4[3] += (pi + pj) * (gi - gj) * (gi - gj);
                }
            }
            wsum(a4, sm);
            const double con = 2.0 * a4[0], busy = 2.0 * a4[1], cplx = 2.0 * a4[2], strn = 2.0 * a4[3];
            o5[0] = busy > 0 ? ps_total / busy : 0.0;
            o5[1] = ps_total > 0 ? 1.0 / ps_total : 1e6;
            o5[2] = cplx / nv;
            o5[3] = P > 1 ? con / ((double)P * (P - 1)) * (s_total / nv) : 0.0;
            o5[4] = s_total > 0 ? strn / s_total : 0.0;
        }
        if (tid < 5) orow[cfg.col_ngtdm + tid] = o5[tid];
        __syncthreads();
    }
}

// t-th queued ROI over the class lists (S0, S1, S2, L)
__device__ __forceinline__ uint32_t wide_row(uint32_t t, const RoiList& rl, const Control* ctl) {
    uint32_t base = 0;
    for (int k = 0; k < kNumClasses; ++k) {
        const uint32_t c = ctl->class_count[k];
        if (t < base + c) {
            const uint32_t* lst = k == kClassS0 ? rl.cls_list[kClassS0]
                                  : k == kClassS1 ? rl.cls_list[kClassS1]
                                  : k == kClassS2 ? rl.cls_list[kClassS2] : rl.cls_list[kClassL];
            return lst[t - base];
        }
        base += c;
    }
    return ~0u;
}

__global__ void __launch_bounds__(kWT) k_texture_wide(DevImage img, RoiList rl, Control* ctl,
                                                      FeatCfg cfg, double* out, uint8_t* scratch,
                                                      WLayout L) {
    __shared__ WShared sm;
    const WSlab S = wslab(scratch + (size_t)blockIdx.x * L.bytes, L);
    const uint32_t total = ctl->class_count[0] + ctl->class_count[1] + ctl->class_count[2] +
                           ctl->class_count[3];
    for (;;) {
        if (threadIdx.x == 0) sm.job = atomicAdd(&ctl->w_next, 1u);
        __syncthreads();
        const uint32_t t = sm.job;
        __syncthreads();
        if (t >= total) break;
        const uint32_t r = wide_row(t, rl, ctl);
        if (rl.w[r] * rl.h[r] > L.CELLS || rl.n[r] > L.NMAX) {
            if (threadIdx.x == 0) atomicOr(&ctl->error, kErrCapacity);
            continue;
        }
        process_wide(r, img, rl, cfg, out, S, L, sm);
    }
}

}  // namespace

// this translation unit's copies of the log2 / reciprocal tables (fx_glcm.cuh)
cudaError_t wide_setup() {
    k_init_log2_tab<<<4, 256>>>();
    return cudaDeviceSynchronize();
}

WLayout make_wlayout(unsigned long long cells, unsigned long long nmax, int ng) {
    WLayout L{};
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    // keys: pairs / runs (<= nmax, padded to a power of two <= 2 nmax) or GLSZM's
    // per-cell scratch followed by its zone keys (2 cells)
    const unsigned long long np = 2 * std::max<unsigned long long>(std::max(cells, nmax), 1);
    size_t o = 0;
    L.lev = o;
    o = al(o + cells * 2);
    L.par = o;
    o = al(o + cells * 4);
    L.keys = o;
    o = al(o + np * 8);
    L.px = o;
    o = al(o + (size_t)ng * 4 * 6);  // px, py, pdif, psum (2 ng), plev
    L.pext = o;
    o = al(o + (std::max<unsigned long long>(cells, nmax) + 2) * 4);
    L.sv = o;
    o = al(o + (size_t)ng * 8);
    L.plist = o;
    o = al(o + (size_t)ng * 4);
    L.bytes = o;
    L.CELLS = cells;
    L.NMAX = nmax;
    L.NG = (uint32_t)ng;
    return L;
}

void launch_texture_wide(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                         double* out, uint8_t* scratch, const WLayout& L) {
    k_texture_wide<<<grid, kWT, 0, s>>>(img, rl, ctl, cfg, out, scratch, L);
}

}  // namespace fxg
