// GLRLM / GLSZM / NGTDM groups (reference texture.cpp:242-528): one CTA per ROI,
// persistent over a work list (S-class windows in one launch, large windows in a
// second launch with bigger slabs), per-CTA scratch slab in global memory.
//
//  - the ROI window is discretized once into a u16 level raster (kNoLevel outside
//    the ROI), exactly as discretize (texture.cpp:29-56);
//  - GLRLM per sorted angle: a thread per cell finds run starts (predecessor
//    outside or of another level) and walks the run; per-run terms are summed per
//    thread, (level, length) counts go to an open-addressing count table (the
//    reference's std::map cells), length counts to a dense array, per-level counts
//    to shared memory;
//  - GLSZM: 8-connected zones of equal level by union-find over the cells
//    (lock-free link, two-phase flatten), zone sizes by atomics on the roots;
//  - NGTDM: |(g+1) - mean of the 8 neighbours| is a rational with denominator
//    1..8, accumulated exactly as an integer multiple of 1/840 (840 = lcm(1..8)),
//    so the per-level sums are order-free and deterministic;
//  - features from the tables with block reductions in a fixed order.
// All fp sums are deterministic (fixed thread mapping, fixed reduction trees).
#include "fx_dev.cuh"
#include "fx_glcm.cuh"
#include "fx_roi.cuh"

namespace fxg {

namespace {

constexpr int kTT = 256;
constexpr int kTW = kTT / 32;
constexpr uint16_t kNoLevel = 0xffffu;
constexpr uint32_t kEmpty = 0xffffffffu;

__device__ __forceinline__ unsigned twarp() { return threadIdx.x >> 5; }

template <typename T, typename Op>
__device__ __forceinline__ T tblock_all(T v, T* sh, Op op) {
    const unsigned lane = lane_id(), w = twarp();
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        T t = sh[lane & (kTW - 1)];
#pragma unroll
        for (int o = kTW / 2; o; o >>= 1) t = op(t, __shfl_xor_sync(kFull, t, o));
        if (lane == 0) sh[kTW] = t;
    }
    __syncthreads();
    const T r = sh[kTW];
    __syncthreads();
    return r;
}
struct TAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct TMin {
    template <typename T>
    __device__ T operator()(T a, T b) const { return b < a ? b : a; }
};
struct TMax {
    template <typename T>
    __device__ T operator()(T a, T b) const { return b > a ? b : a; }
};

struct TSlab {
    uint16_t* lev;   // [cells] level raster
    uint32_t* par;   // [cells] union-find parents (GLSZM)
    uint32_t* zsz;   // [cells] flatten scratch, then zone sizes
    uint32_t* hjk;   // [HC] (level, extent) keys  } open addressing, kept empty
    uint32_t* hjc;   // [HC] counts                 }
    uint32_t* ext;   // [NMAX+1] units per extent (dense: fixed summation order)
    uint32_t* ccnt;  // [NMAX+1] joint cells per cell count (entropy by count value)
};

struct TShared {
    uint32_t plev[256];            // runs / zones per level; NGTDM pixels per level
    unsigned long long sng[256];   // NGTDM 840 * sum |(g+1) - mean| per level
    double red[kTW + 1];
    unsigned long long u64[kTW + 1];
    uint32_t u32[kTW + 1];
    uint32_t job;
};

__device__ __forceinline__ uint32_t thash(uint32_t k) {
    k ^= k >> 16;
    k *= 0x7feb352du;
    k ^= k >> 15;
    k *= 0x846ca68bu;
    k ^= k >> 16;
    return k;
}

__device__ __forceinline__ void table_add(uint32_t* keys, uint32_t* cnts, uint32_t mask, uint32_t key) {
    uint32_t h = thash(key) & mask;
    for (;;) {
        const uint32_t old = atomicCAS(&keys[h], kEmpty, key);
        if (old == kEmpty || old == key) {
            atomicAdd(&cnts[h], 1u);
            return;
        }
        h = (h + 1) & mask;
    }
}

// Features of the (level, extent) cells (glrlm_features texture.cpp:282-341,
// glszm_features :382-441).  t8: block totals of the 8 per-unit sums (sre, lre,
// lglre, hglre, srlgle, srhgle, lrlgle, lrhgle numerators); nr units, np pixels.
// Empties the count tables and the per-level counts.
__device__ void extent_features(const double* t8, unsigned long long nr_u, unsigned long long np_u,
                                int ng, const TSlab& S, uint32_t HC, uint32_t NMAX, TShared& sm,
                                double* out16) {
    const unsigned tid = threadIdx.x;
    if (nr_u == 0) {
        for (int k = tid; k < 16; k += kTT) out16[k] = 0.0;
        for (int g = tid; g < ng; g += kTT) sm.plev[g] = 0u;
        __syncthreads();
        return;
    }
    const double nr = (double)nr_u, np = (double)np_u, logn = nlog2(nr);
    // per-level: glnu, mean level
    double a_glnu = 0, a_mug = 0;
    for (int g = tid; g < ng; g += kTT) {
        const double c = (double)sm.plev[g];
        a_glnu += c * c;
        a_mug += c * (g + 1);
    }
    const double glnu = tblock_all(a_glnu, sm.red, TAdd());
    const double mu_g = tblock_all(a_mug, sm.red, TAdd()) / nr;
    // per-extent counts (dense, ascending extent): rlnu, mean extent
    double a_rlnu = 0, a_mul = 0;
    for (uint32_t e = tid; e <= NMAX; e += kTT) {
        const uint32_t c = S.ext[e];
        if (c) {
            a_rlnu += (double)c * (double)c;
            a_mul += (double)c * (double)e;
        }
    }
    const double rlnu = tblock_all(a_rlnu, sm.red, TAdd());
    const double mu_l = tblock_all(a_mul, sm.red, TAdd()) / nr;
    // joint cells -> histogram of their counts (the slot layout of the table depends
    // on insertion order; the counts do not), emptying the table
    for (uint32_t i = tid; i < HC; i += kTT) {
        if (S.hjk[i] != kEmpty) {
            atomicAdd(&S.ccnt[S.hjc[i]], 1u);
            S.hjk[i] = kEmpty;
            S.hjc[i] = 0u;
        }
    }
    __syncthreads();
    double a_re = 0;  // entropy = sum over cells c (log2 nr - log2 c) / nr
    for (uint32_t c = tid; c <= NMAX; c += kTT) {
        const uint32_t k = S.ccnt[c];
        if (k) {
            a_re += (double)k * (double)c * (logn - log2_int(c));
            S.ccnt[c] = 0u;
        }
    }
    const double re = tblock_all(a_re, sm.red, TAdd()) / nr;
    double a_glv = 0, a_rv = 0;
    for (int g = tid; g < ng; g += kTT) {
        const double c = (double)sm.plev[g];
        a_glv += c / nr * (g + 1 - mu_g) * (g + 1 - mu_g);
    }
    for (uint32_t e = tid; e <= NMAX; e += kTT) {
        const uint32_t c = S.ext[e];
        if (c) {
            a_rv += (double)c / nr * ((double)e - mu_l) * ((double)e - mu_l);
            S.ext[e] = 0u;
        }
    }
    const double glv = tblock_all(a_glv, sm.red, TAdd());
    const double rv = tblock_all(a_rv, sm.red, TAdd());
    if (tid == 0) {
        const double v[16] = {t8[0] / nr, t8[1] / nr, glnu / nr, glnu / (nr * nr), rlnu / nr,
                              rlnu / (nr * nr), nr / np, glv, rv, re, t8[2] / nr, t8[3] / nr,
                              t8[4] / nr, t8[5] / nr, t8[6] / nr, t8[7] / nr};
        for (int k = 0; k < 16; ++k) out16[k] = v[k];
    }
    for (int g = tid; g < ng; g += kTT) sm.plev[g] = 0u;
    __syncthreads();
}

// per-unit terms of one run / zone (level g 0-based, extent l), texture.cpp:296-309
__device__ __forceinline__ void unit_terms(double (&t)[8], int g0, uint32_t l0) {
    const double g = g0 + 1, l = (double)l0, g2 = g * g, l2 = l * l;
    t[0] += 1.0 / l2;
    t[1] += l2;
    t[2] += 1.0 / g2;
    t[3] += g2;
    t[4] += 1.0 / (g2 * l2);
    t[5] += g2 / l2;
    t[6] += l2 / g2;
    t[7] += g2 * l2;
}

__device__ void process_t(uint32_t r, const DevImage& img, const RoiList& rl, Control* ctl,
                          const FeatCfg& cfg, double* __restrict__ out, const TSlab& S, uint32_t HC,
                          uint32_t NMAX, TShared& sm) {
    const unsigned tid = threadIdx.x;
    const uint32_t label = rl.label[r];
    const int w = (int)rl.w[r], h = (int)rl.h[r];
    const uint32_t x0 = rl.x0[r], y0 = rl.y0[r];
    const uint32_t cells = (uint32_t)w * (uint32_t)h;
    const unsigned long long n = rl.n[r];
    const int ng = cfg.ng;
    double* orow = out + (size_t)r * cfg.ncols;
    auto lab_at = [&](uint32_t c) -> uint32_t {
        const uint32_t y = c / (uint32_t)w, x = c - y * (uint32_t)w;
        return img.L[(size_t)(y0 + y) * img.pitch + x0 + x];
    };
    auto int_at = [&](uint32_t c) -> uint32_t {
        const uint32_t y = c / (uint32_t)w, x = c - y * (uint32_t)w;
        return img.I[(size_t)(y0 + y) * img.pitch + x0 + x];
    };
    // ---- discretize (texture.cpp:29-56): min/max, then the level raster
    uint32_t lo = 0xffffu, hi = 0u;
    for (uint32_t c = tid; c < cells; c += kTT)
        if (lab_at(c) == label) {
            const uint32_t v = int_at(c);
            lo = min(lo, v);
            hi = max(hi, v);
        }
    const uint32_t vmin = tblock_all(lo, sm.u32, TMin()), vmax = tblock_all(hi, sm.u32, TMax());
    const unsigned long long span = (unsigned long long)(vmax - vmin) + 1ull;
    for (uint32_t c = tid; c < cells; c += kTT) {
        uint16_t lv = kNoLevel;
        if (lab_at(c) == label) {
            lv = 0;
            if (vmax > vmin) {
                const unsigned long long q = (unsigned long long)ng * (int_at(c) - vmin) / span;
                lv = (uint16_t)(q < (unsigned long long)(ng - 1) ? q : (unsigned long long)(ng - 1));
            }
        }
        S.lev[c] = lv;
    }
    __syncthreads();
    const uint32_t mask = HC - 1u;
    auto lev = [&](int x, int y) -> uint32_t {
        return (x >= 0 && x < w && y >= 0 && y < h) ? S.lev[(uint32_t)y * (uint32_t)w + (uint32_t)x]
                                                    : (uint32_t)kNoLevel;
    };
    // ---- GLRLM per sorted angle (texture.cpp:242-280)
    if (cfg.col_glrlm >= 0) {
        const int A = cfg.n_angles;
        double* og = orow + cfg.col_glrlm;
        double acc16[16];
        for (int k = 0; k < 16; ++k) acc16[k] = 0;
        for (int a = 0; a < A; ++a) {
            int dx = 1, dy = 0;
            switch (cfg.angle[a]) {
                case 45: dx = 1; dy = -1; break;
                case 90: dx = 0; dy = 1; break;
                case 135: dx = 1; dy = 1; break;
                default: break;
            }
            double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            unsigned long long runs = 0;
            for (uint32_t c = tid; c < cells; c += kTT) {
                const uint32_t g = S.lev[c];
                if (g == kNoLevel) continue;
                const int y = (int)(c / (uint32_t)w), x = (int)(c - (uint32_t)y * (uint32_t)w);
                if (lev(x - dx, y - dy) == g) continue;  // not a run start
                uint32_t len = 1;
                int nx = x + dx, ny = y + dy;
                while (lev(nx, ny) == g) {
                    ++len;
                    nx += dx;
                    ny += dy;
                }
                unit_terms(t, (int)g, len);
                ++runs;
                atomicAdd(&sm.plev[g], 1u);
                table_add(S.hjk, S.hjc, mask, (g << 24) | len);
                atomicAdd(&S.ext[len], 1u);
            }
            double tt[8];
            for (int k = 0; k < 8; ++k) tt[k] = tblock_all(t[k], sm.red, TAdd());
            const unsigned long long nr = tblock_all(runs, sm.u64, TAdd());
            __shared__ double f16[16];
            extent_features(tt, nr, n, ng, S, HC, NMAX, sm, f16);
            __syncthreads();
            if (tid < 16) {
                og[tid * (A + 1) + a] = f16[tid];
                acc16[tid] += f16[tid];
            }
            __syncthreads();
        }
        if (tid < 16) og[tid * (A + 1) + A] = acc16[tid] / (double)A;
    }
    // ---- GLSZM (texture.cpp:343-380): 8-connected zones of equal level
    if (cfg.col_glszm >= 0) {
        for (uint32_t c = tid; c < cells; c += kTT) {
            S.par[c] = c;
            S.zsz[c] = 0u;
        }
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kTT) {  // forward neighbours E, SW, S, SE
            const uint32_t g = S.lev[c];
            if (g == kNoLevel) continue;
            const int y = (int)(c / (uint32_t)w), x = (int)(c - (uint32_t)y * (uint32_t)w);
            const int nx[4] = {x + 1, x - 1, x, x + 1}, ny[4] = {y, y + 1, y + 1, y + 1};
            for (int k = 0; k < 4; ++k)
                if (lev(nx[k], ny[k]) == g) uf_union(S.par, c, (uint32_t)ny[k] * (uint32_t)w + (uint32_t)nx[k]);
        }
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kTT)  // flatten: roots first, then publish
            if (S.lev[c] != kNoLevel) S.zsz[c] = uf_root(S.par, c);
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kTT)
            if (S.lev[c] != kNoLevel) S.par[c] = S.zsz[c];
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kTT) S.zsz[c] = 0u;
        __syncthreads();
        for (uint32_t c = tid; c < cells; c += kTT)
            if (S.lev[c] != kNoLevel) atomicAdd(&S.zsz[S.par[c]], 1u);
        __syncthreads();
        double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unsigned long long zones = 0;
        for (uint32_t c = tid; c < cells; c += kTT) {
            const uint32_t g = S.lev[c];
            if (g == kNoLevel || S.par[c] != c) continue;
            const uint32_t size = S.zsz[c];
            unit_terms(t, (int)g, size);
            ++zones;
            atomicAdd(&sm.plev[g], 1u);
            table_add(S.hjk, S.hjc, mask, (g << 24) | size);
            atomicAdd(&S.ext[size], 1u);
        }
        double tt[8];
        for (int k = 0; k < 8; ++k) tt[k] = tblock_all(t[k], sm.red, TAdd());
        const unsigned long long nz = tblock_all(zones, sm.u64, TAdd());
        __shared__ double f16z[16];
        extent_features(tt, nz, n, ng, S, HC, NMAX, sm, f16z);
        __syncthreads();
        if (tid < 16) orow[cfg.col_glszm + tid] = f16z[tid];
        __syncthreads();
    }
    // ---- NGTDM (texture.cpp:443-528)
    if (cfg.col_ngtdm >= 0) {
        for (int g = tid; g < ng; g += kTT) {
            sm.plev[g] = 0u;
            sm.sng[g] = 0ull;
        }
        __syncthreads();
        unsigned long long valid = 0;
        for (uint32_t c = tid; c < cells; c += kTT) {
            const uint32_t g = S.lev[c];
            if (g == kNoLevel) continue;
            const int y = (int)(c / (uint32_t)w), x = (int)(c - (uint32_t)y * (uint32_t)w);
            int sum = 0, cnt = 0;
            for (int ddy = -1; ddy <= 1; ++ddy)
                for (int ddx = -1; ddx <= 1; ++ddx) {
                    if (!ddx && !ddy) continue;
                    const uint32_t q = lev(x + ddx, y + ddy);
                    if (q != kNoLevel) {
                        sum += (int)q + 1;
                        ++cnt;
                    }
                }
            if (!cnt) continue;
            const int d = (int)(g + 1) * cnt - sum;  // |(g+1) - sum/cnt| = |d| / cnt
            atomicAdd(&sm.sng[g], (unsigned long long)((d < 0 ? -d : d) * (840 / cnt)));
            atomicAdd(&sm.plev[g], 1u);
            ++valid;
        }
        const unsigned long long nvu = tblock_all(valid, sm.u64, TAdd());
        double o5[5] = {0, 0, 0, 0, 0};
        if (nvu) {
            const double nv = (double)nvu;
            double a_s = 0, a_ps = 0;
            uint32_t a_pres = 0;
            for (int i = tid; i < ng; i += kTT) {
                const double p = (double)sm.plev[i] / nv, sv = (double)sm.sng[i] / 840.0;
                a_pres += p > 0;
                a_s += sv;
                a_ps += p * sv;
            }
            const double s_total = tblock_all(a_s, sm.red, TAdd());
            const double ps_total = tblock_all(a_ps, sm.red, TAdd());
            const uint32_t present = tblock_all(a_pres, sm.u32, TAdd());
            double a_con = 0, a_busy = 0, a_cplx = 0, a_strn = 0;
            const uint32_t pairs = (uint32_t)ng * (uint32_t)ng;
            for (uint32_t q = tid; q < pairs; q += kTT) {
                const int i = (int)(q / (uint32_t)ng), j = (int)(q - (uint32_t)i * (uint32_t)ng);
                if (!sm.plev[i] || !sm.plev[j]) continue;
                const double pi = (double)sm.plev[i] / nv, pj = (double)sm.plev[j] / nv;
                const double si = (double)sm.sng[i] / 840.0, sj = (double)sm.sng[j] / 840.0;
                const double gi = i + 1, gj = j + 1;
                a_con += pi * pj * (i - j) * (i - j);
                a_busy += fabs(gi * pi - gj * pj);
                a_cplx += fabs(gi - gj) * (pi * si + pj * sj) / (pi + pj);
                a_strn += (pi + pj) * (gi - gj) * (gi - gj);
            }
            const double con = tblock_all(a_con, sm.red, TAdd());
            const double busy = tblock_all(a_busy, sm.red, TAdd());
            const double cplx = tblock_all(a_cplx, sm.red, TAdd());
            const double strn = tblock_all(a_strn, sm.red, TAdd());
            o5[0] = busy > 0 ? ps_total / busy : 0.0;
            o5[1] = ps_total > 0 ? 1.0 / ps_total : 1e6;
            o5[2] = cplx / nv;
            o5[3] = present > 1 ? con / ((double)present * (present - 1)) * (s_total / nv) : 0.0;
            o5[4] = s_total > 0 ? strn / s_total : 0.0;
        }
        if (tid < 5) orow[cfg.col_ngtdm + tid] = o5[tid];
        __syncthreads();
        for (int g = tid; g < ng; g += kTT) sm.plev[g] = 0u;
        __syncthreads();
    }
    (void)ctl;
}

// which = 0: the S-class lists (windows <= 64 x 64); 1: the large-ROI list
__global__ void __launch_bounds__(kTT) k_roi_t(DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                                               double* out, uint8_t* scratch, TLayout T, int which) {
    __shared__ TShared sm;
    uint8_t* base = scratch + (size_t)blockIdx.x * T.bytes;
    TSlab S;
    S.lev = (uint16_t*)(base + T.lev);
    S.par = (uint32_t*)(base + T.par);
    S.zsz = (uint32_t*)(base + T.zsz);
    S.hjk = (uint32_t*)(base + T.hjk);
    S.hjc = (uint32_t*)(base + T.hjc);
    S.ext = (uint32_t*)(base + T.ext);
    S.ccnt = (uint32_t*)(base + T.ccnt);
    for (int g = threadIdx.x; g < 256; g += kTT) sm.plev[g] = 0u;
    __syncthreads();
    const uint32_t n0 = ctl->class_count[kClassS0], n1 = ctl->class_count[kClassS1];
    const uint32_t n2 = ctl->class_count[kClassS2], nl = ctl->class_count[kClassL];
    const uint32_t total = which ? nl : n0 + n1 + n2;
    for (;;) {
        if (threadIdx.x == 0) sm.job = atomicAdd(&ctl->t_next[which], 1u);
        __syncthreads();
        const uint32_t t = sm.job;
        __syncthreads();
        if (t >= total) break;
        uint32_t r;
        if (which) r = rl.cls_list[kClassL][t];
        else if (t < n0) r = rl.cls_list[kClassS0][t];
        else if (t < n0 + n1) r = rl.cls_list[kClassS1][t - n0];
        else r = rl.cls_list[kClassS2][t - n0 - n1];
        const unsigned long long cells = (unsigned long long)rl.w[r] * rl.h[r];
        if (cells > T.CELLS || rl.n[r] > T.NMAX || rl.n[r] >= (1ull << 24)) {
            if (threadIdx.x == 0) atomicOr(&ctl->error, kErrCapacity);
            continue;
        }
        process_t(r, img, rl, ctl, cfg, out, S, T.HC, T.NMAX, sm);
    }
}

}  // namespace

cudaError_t roi_t_setup() {
    k_init_log2_tab<<<4, 256>>>();
    return cudaDeviceSynchronize();
}

TLayout make_tlayout(unsigned long long CELLS, uint32_t NMAX) {
    TLayout T{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (o + bytes + 255) & ~(size_t)255;
        return at;
    };
    uint32_t hc = 1024;
    while (hc < 2u * NMAX + 16u) hc <<= 1;  // units (runs / zones) <= pixels
    T.lev = take((size_t)CELLS * 2);
    T.par = take((size_t)CELLS * 4);
    T.zsz = take((size_t)CELLS * 4);
    T.hjk = take((size_t)hc * 4);
    T.hjc = take((size_t)hc * 4);
    T.ext = take(((size_t)NMAX + 1) * 4);
    T.ccnt = take(((size_t)NMAX + 1) * 4);
    T.bytes = o;
    T.CELLS = CELLS;
    T.NMAX = NMAX;
    T.HC = hc;
    return T;
}

// tables must start empty: keys 0xff.., counts 0 (initialise a fresh slab)
__global__ void k_t_init(uint8_t* scratch, TLayout T, int grid) {
    for (int b = blockIdx.x; b < grid; b += gridDim.x) {
        uint8_t* base = scratch + (size_t)b * T.bytes;
        uint32_t* hjk = (uint32_t*)(base + T.hjk);
        uint32_t* hjc = (uint32_t*)(base + T.hjc);
        uint32_t* ext = (uint32_t*)(base + T.ext);
        uint32_t* ccnt = (uint32_t*)(base + T.ccnt);
        for (uint32_t i = threadIdx.x; i < T.HC; i += blockDim.x) {
            hjk[i] = kEmpty;
            hjc[i] = 0u;
        }
        for (uint32_t i = threadIdx.x; i <= T.NMAX; i += blockDim.x) {
            ext[i] = 0u;
            ccnt[i] = 0u;
        }
    }
}

void launch_roi_t(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                  double* out, uint8_t* scratch, const TLayout& T, int which, bool init) {
    if (init) k_t_init<<<grid < 1024 ? grid : 1024, 256, 0, s>>>(scratch, T, grid);
    k_roi_t<<<grid, kTT, 0, s>>>(img, rl, ctl, cfg, out, scratch, T, which);
}

}  // namespace fxg
