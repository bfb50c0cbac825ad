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

#ifdef FXG_PHASE_TIMING
__device__ unsigned long long g_phase_clk_t[8];
#define TT_DECL long long tt_t_ = clock64();
#define TT(k)                                                                  \
    do {                                                                       \
        const long long t_ = clock64();                                        \
        if (threadIdx.x == 0) atomicAdd(&g_phase_clk_t[k], (unsigned long long)(t_ - tt_t_)); \
        tt_t_ = t_;                                                            \
    } while (0)
#else
#define TT_DECL
#define TT(k)
#endif

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
// block sums of K <= 8 doubles in one pass (fixed order: lanes, then warps)
template <int K>
__device__ __forceinline__ void tblock_sum(double (&v)[K], double (*sh)[8]) {
    const unsigned lane = lane_id(), w = twarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        v[k] = x;
    }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[w][k] = v[k];
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0;
        for (int i = 0; i < kTW; ++i) t += sh[i][threadIdx.x];
        sh[kTW][threadIdx.x] = t;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = sh[kTW][k];
    __syncthreads();
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
    double red[kTW + 1];
    double red8[kTW + 1][8];
    unsigned long long u64[kTW + 1];
    uint32_t u32[kTW + 1];
    double redK[kTW + 1][10];      // tblock_fused
    uint32_t redM[kTW + 1][2];
    uint32_t job;
    // dense GLRLM (S windows, ng <= 64, <= 4 angles)
    uint32_t gl_plev[4 * 64];      // runs per (angle, level)
    uint32_t gl_ext[4 * 65];       // runs per (angle, length 1..64)
    double gl_red[kTW][10];        // per-warp cell sums
    double gl_f[4][16];            // features per angle
    double gl_rcp2[256];           // 1 / k^2, k = 1..256
    uint32_t ng_np;
    // dynamic shared memory (kDynBytes): the S-window level raster, then one 33 KB
    // region used by phase: GLSZM (count table of 2048 slots, u16 parents, u16
    // zone sizes), dense GLRLM counts (4 angles x 64 levels x 33 words), NGTDM
    // per-level arrays (after GLSZM).  2048 slots hold every distinct (level,
    // extent) key of a window with n <= 4096 pixels and ng <= 256: taking the
    // smallest extents, ng k (k + 1) / 2 <= n allows at most ~1,322 keys.
};
constexpr uint32_t kTSlots = 2048;
constexpr size_t kRegionBytes = 64 * 33 * 4 * 4;  // dense GLRLM, >= 32 KB of GLSZM arrays
constexpr size_t kDynBytes = 4096 * 2 + kRegionBytes;

// The dynamic shared memory and its views, addressed from the shared symbol itself
// so every use compiles to shared-space instructions (a pointer kept in a struct is
// generic): level raster [4096] u16, then the region: count table keys / counts
// [kTSlots] u32 (kept empty between uses), union-find parents and zone sizes [4096]
// u16; NGTDM's per-level arrays over the parents / sizes (dead by then); the dense
// GLRLM counts over the whole region.
extern __shared__ __align__(16) uint8_t tdyn[];
__device__ __forceinline__ uint16_t* d_slev() { return reinterpret_cast<uint16_t*>(tdyn); }
__device__ __forceinline__ uint32_t* d_skey() { return reinterpret_cast<uint32_t*>(tdyn + 4096 * 2); }
__device__ __forceinline__ uint32_t* d_scnt() { return d_skey() + kTSlots; }
__device__ __forceinline__ uint16_t* d_spar() { return reinterpret_cast<uint16_t*>(d_scnt() + kTSlots); }
__device__ __forceinline__ uint16_t* d_szsz() { return d_spar() + 4096; }
__device__ __forceinline__ unsigned long long* d_sng() { return reinterpret_cast<unsigned long long*>(d_spar()); }
__device__ __forceinline__ double* d_ngp() { return reinterpret_cast<double*>(d_sng() + 256); }
__device__ __forceinline__ double* d_ngs() { return d_ngp() + 256; }
__device__ __forceinline__ uint8_t* d_nglev() { return reinterpret_cast<uint8_t*>(d_ngs() + 256); }

// x, y of cell c of a row-major window of width w without an integer division:
// m = ceil(2^32 / w) gives floor(c / w) or one more (c < 2^32), fixed by one step
struct CellDiv {
    uint32_t w, m;
    __device__ explicit CellDiv(uint32_t w_) : w(w_), m(w_ > 1 ? (uint32_t)(0xffffffffu / w_) + 1u : 0u) {}
    __device__ __forceinline__ void split(uint32_t c, int& x, int& y) const {
        uint32_t q = w > 1 ? __umulhi(c, m) : c;
        if (q * w > c) --q;
        y = (int)q;
        x = (int)(c - q * w);
    }
};

// shared-memory reductions through explicit shared addresses (the slab pointers
// are generic, which would compile to generic ATOM)
__device__ __forceinline__ void sred_add(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void sred_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}

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


// One block pass for K fp64 sums (fixed order: lanes, then warps), one u32 max
// and one u32 min: 3 barriers instead of 3 per reduced value.
template <int K>
__device__ __forceinline__ void tblock_fused(double (&v)[K], uint32_t& mx, uint32_t& mn, TShared& sm) {
    static_assert(K >= 1 && K <= 10, "K");
    const unsigned lane = lane_id(), w = twarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        v[k] = x;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sm.redK[w][k] = v[k];
        sm.redM[w][0] = mx;
        sm.redM[w][1] = mn;
    }
    __syncthreads();
    const unsigned tid = threadIdx.x;
    if (tid < (unsigned)K) {
        double t = 0;
        for (int i = 0; i < kTW; ++i) t += sm.redK[i][tid];
        sm.redK[kTW][tid] = t;
    } else if (tid == 32) {
        uint32_t a = 0, b = 0xffffffffu;
        for (int i = 0; i < kTW; ++i) {
            a = max(a, sm.redM[i][0]);
            b = min(b, sm.redM[i][1]);
        }
        sm.redM[kTW][0] = a;
        sm.redM[kTW][1] = b;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = sm.redK[kTW][k];
    mx = sm.redM[kTW][0];
    mn = sm.redM[kTW][1];
    __syncthreads();
}

// Features of the (level, extent) cells (glrlm_features texture.cpp:282-341,
// glszm_features :382-441).  t8: block totals of the 8 per-unit sums (sre, lre,
// lglre, hglre, srlgle, srhgle, lrlgle, lrhgle numerators); nr units, np pixels.
// Empties the count tables and the per-level counts.
__device__ void extent_features(const double* t8, unsigned long long nr_u, unsigned long long np_u,
                                int ng, const TSlab& S, uint32_t* hk, uint32_t* hc, uint32_t hsize,
                                uint32_t emax, TShared& sm, double* out16) {
    const unsigned tid = threadIdx.x;
    if (nr_u == 0) {
        for (int k = tid; k < 16; k += kTT) out16[k] = 0.0;
        for (int g = tid; g < ng; g += kTT) sm.plev[g] = 0u;
        __syncthreads();
        return;
    }
    const double nr = (double)nr_u, np = (double)np_u, logn = nlog2(nr);
    // pass A: per-level (glnu, mean level), per-extent (rlnu, mean extent), joint
    // cells -> histogram of their counts (the table's slot layout depends on the
    // insertion order, the counts do not), emptying the table
    double a[4] = {0, 0, 0, 0};
    for (int g = tid; g < ng; g += kTT) {
        const double c = (double)sm.plev[g];
        a[0] += c * c;
        a[1] += c * (g + 1);
    }
    for (uint32_t e = tid; e <= emax; e += kTT) {
        const uint32_t c = S.ext[e];
        if (c) {
            a[2] += (double)c * (double)c;
            a[3] += (double)c * (double)e;
        }
    }
    // every slot of the table (no list of filled slots: one hot counter fewer)
    uint32_t cmax = 0;
    for (uint32_t slot = tid; slot < hsize; slot += kTT) {
        if (hk[slot] == kEmpty) continue;
        const uint32_t c = hc[slot];
        atomicAdd(&S.ccnt[c], 1u);
        cmax = max(cmax, c);
        hk[slot] = kEmpty;
        hc[slot] = 0u;
    }
    uint32_t unused_min = 0xffffffffu;
    tblock_fused<4>(a, cmax, unused_min, sm);
    const double glnu = a[0], mu_g = a[1] / nr, rlnu = a[2], mu_l = a[3] / nr;
    // pass B: entropy = sum over cells c (log2 nr - log2 c) / nr, variances
    double b[3] = {0, 0, 0};
    for (uint32_t c = tid; c <= cmax; c += kTT) {
        const uint32_t k = S.ccnt[c];
        if (k) {
            b[0] += (double)k * (double)c * (logn - log2_int(c));
            S.ccnt[c] = 0u;
        }
    }
    for (int g = tid; g < ng; g += kTT) {
        const double c = (double)sm.plev[g];
        b[1] += c / nr * (g + 1 - mu_g) * (g + 1 - mu_g);
    }
    for (uint32_t e = tid; e <= emax; e += kTT) {
        const uint32_t c = S.ext[e];
        if (c) {
            b[2] += (double)c / nr * ((double)e - mu_l) * ((double)e - mu_l);
            S.ext[e] = 0u;
        }
    }
    tblock_sum<3>(b, sm.red8);
    const double re = b[0] / nr, glv = b[1], rv = b[2];
    if (tid == 0) {
        const double v[16] = {t8[0] / nr, t8[1] / nr, glnu / nr, glnu / (nr * nr), rlnu / nr,
                              rlnu / (nr * nr), nr / np, glv, rv, re, t8[2] / nr, t8[3] / nr,
                              t8[4] / nr, t8[5] / nr, t8[6] / nr, t8[7] / nr};
        for (int k = 0; k < 16; ++k) out16[k] = v[k];
    }
    for (int g = tid; g < ng; g += kTT) sm.plev[g] = 0u;
    __syncthreads();
}

// union-find with T-bit cell indices (u16 in shared memory for S windows)
// union-find loads: the u16 parents live in shared memory (S windows)
__device__ __forceinline__ uint32_t t_ld(const volatile uint16_t* p) {
    unsigned short r;
    asm volatile("ld.volatile.shared.u16 %0, [%1];" : "=h"(r) : "r"(smem_u32((const void*)p)) : "memory");
    return r;
}
__device__ __forceinline__ uint32_t t_ld(const volatile uint32_t* p) { return *p; }
template <typename T>
__device__ __forceinline__ uint32_t t_root(const volatile T* par, uint32_t x) {
    uint32_t p = t_ld(par + x);
    while (p != x) {
        x = p;
        p = t_ld(par + x);
    }
    return x;
}
// the u16 instantiation only ever lives in shared memory (S windows): explicit
// shared-space CAS and loads instead of generic ones
__device__ __forceinline__ uint32_t t_cas(uint16_t* a, uint32_t cmp, uint32_t val) {
    unsigned short r;
    asm volatile("atom.shared.cas.b16 %0, [%1], %2, %3;"
                 : "=h"(r)
                 : "r"(smem_u32(a)), "h"((unsigned short)cmp), "h"((unsigned short)val)
                 : "memory");
    return r;
}

__device__ __forceinline__ uint32_t t_cas(uint32_t* a, uint32_t cmp, uint32_t val) {
    return atomicCAS(a, cmp, val);
}
template <typename T>
__device__ __forceinline__ void t_union(T* par, uint32_t a, uint32_t b) {
    for (;;) {
        a = t_root(par, a);
        b = t_root(par, b);
        if (a == b) return;
        if (a > b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = t_cas(&par[b], b, a);
        if (old == b) return;
        b = old;
    }
}

// 8-connected zones of equal level: par[c] = root (smallest cell index of the
// zone), zsz[root] = zone size (reads of par use volatile-free loads after
// barriers; concurrent links only ever move a root under a smaller index)
template <typename T>
__device__ void glszm_zones(T* par, T* zsz, const uint16_t* lv, int w, int h, uint32_t cells) {
    const unsigned tid = threadIdx.x;
    for (uint32_t c = tid; c < cells; c += kTT) {
        par[c] = (T)c;
        zsz[c] = 0;
    }
    __syncthreads();
    const CellDiv cd((uint32_t)w);
    for (uint32_t c = tid; c < cells; c += kTT) {  // forward neighbours E, SW, S, SE
        const uint32_t g = lv[c];
        if (g == kNoLevel) continue;
        int x, y;
        cd.split(c, x, y);
        const int nx[4] = {x + 1, x - 1, x, x + 1}, ny[4] = {y, y + 1, y + 1, y + 1};
        for (int k = 0; k < 4; ++k)
            if (nx[k] >= 0 && nx[k] < w && ny[k] < h &&
                lv[(uint32_t)ny[k] * (uint32_t)w + (uint32_t)nx[k]] == g)
                t_union(par, c, (uint32_t)ny[k] * (uint32_t)w + (uint32_t)nx[k]);
    }
    __syncthreads();
    for (uint32_t c = tid; c < cells; c += kTT)  // flatten: roots first, then publish
        if (lv[c] != kNoLevel) zsz[c] = (T)t_root(par, c);
    __syncthreads();
    for (uint32_t c = tid; c < cells; c += kTT)
        if (lv[c] != kNoLevel) par[c] = zsz[c];
    __syncthreads();
    for (uint32_t c = tid; c < cells; c += kTT) zsz[c] = 0;
    __syncthreads();
    for (uint32_t c = tid; c < cells; c += kTT)
        if (lv[c] != kNoLevel) {
            if constexpr (sizeof(T) == 2) {
                // 16-bit atomics: add into the containing word
                const uint32_t r = par[c];
                uint32_t* word = reinterpret_cast<uint32_t*>(zsz + (r & ~1u));
                sred_add(word, 1u << ((r & 1u) * 16u));
            } else {
                atomicAdd(reinterpret_cast<uint32_t*>(&zsz[par[c]]), 1u);
            }
        }
    __syncthreads();
}

// per-unit terms of one run / zone (level g 0-based, extent l), texture.cpp:296-309;
// rcp2[k] = 1 / (k + 1)^2 for k < 256 (levels always, extents up to 256), so the
// common case has no fp64 division
__device__ __forceinline__ void unit_terms(double (&t)[8], int g0, uint32_t l0, const double* rcp2) {
    const double g = g0 + 1, l = (double)l0, g2 = g * g, l2 = l * l;
    const double rg2 = rcp2[g0], rl2 = l0 <= 256u ? rcp2[l0 - 1u] : 1.0 / l2;
    t[0] += rl2;
    t[1] += l2;
    t[2] += rg2;
    t[3] += g2;
    t[4] += rg2 * rl2;
    t[5] += g2 * rl2;
    t[6] += l2 * rg2;
    t[7] += g2 * l2;
}

__device__ __forceinline__ void angle_dir(int angle, int& dx, int& dy) {
    dx = 1;
    dy = 0;
    if (angle == 45) dy = -1;
    else if (angle == 90) { dx = 0; dy = 1; }
    else if (angle == 135) dy = 1;
}

// GLRLM (texture.cpp:242-341) of an S-class window with ng <= 64 and <= 4 angles:
// the runs of every angle in one pass over the cells, counted densely per
// (angle, level, length) as packed u16 in the (then idle) hash-table region of
// shared memory (lengths <= 64 in a 64 x 64 window), with runs per level and per
// length by shared atomics; then every feature from the dense counts: the cell
// terms by the two warps of each angle, the level / length moments by one warp
// per angle.  Counts are order free and every floating-point sum runs in fixed
// order (deterministic).  Restores the hash table's empty state.
__device__ void glrlm_dense(const uint16_t* lv, int w, int h, uint32_t cells, unsigned long long np_u,
                            const FeatCfg& cfg, TShared& sm, double* og) {
    const unsigned tid = threadIdx.x, lane = lane_id(), wp = twarp();
    const int A = cfg.n_angles;
    TT_DECL
    // word a * kHA + g * 33 + ((l - 1) >> 1): rows of 32 words padded to 33, so the
    // lanes of the feature scan (lane = level, same word index) hit 32 banks
    constexpr uint32_t kHA = 64u * 33u;
    uint32_t* H = d_skey();  // A * kHA words <= the dynamic region (GLSZM rebuilds its arrays)
    for (uint32_t i = tid; i < (uint32_t)A * kHA; i += kTT) H[i] = 0u;
    for (uint32_t i = tid; i < 4u * 64u; i += kTT) sm.gl_plev[i] = 0u;
    for (uint32_t i = tid; i < 4u * 65u; i += kTT) sm.gl_ext[i] = 0u;
    __syncthreads();
    const CellDiv cd((uint32_t)w);
    for (uint32_t c = tid; c < cells; c += kTT) {
        const uint32_t g = lv[c];
        if (g == kNoLevel) continue;
        int x, y;
        cd.split(c, x, y);
        for (int a = 0; a < A; ++a) {
            int dx, dy;
            angle_dir(cfg.angle[a], dx, dy);
            const int px = x - dx, py = y - dy;
            if (px >= 0 && px < w && py >= 0 && py < h && lv[(uint32_t)py * (uint32_t)w + (uint32_t)px] == g)
                continue;  // not a run start
            uint32_t len = 1;
            int nx = x + dx, ny = y + dy;
            while (nx >= 0 && nx < w && ny >= 0 && ny < h && lv[(uint32_t)ny * (uint32_t)w + (uint32_t)nx] == g) {
                ++len;
                nx += dx;
                ny += dy;
            }
            sred_add(&H[(uint32_t)a * kHA + g * 33u + ((len - 1u) >> 1)], 1u << (((len - 1u) & 1u) * 16u));
            sred_add(&sm.gl_plev[a * 64 + g], 1u);
            sred_add(&sm.gl_ext[a * 65 + len], 1u);
        }
    }
    __syncthreads();
    TT(4);
    // cell terms: warps 2a, 2a+1 cover angle a, lane L of the pair owns level L and
    // walks its row in length order until all of the level's runs are counted
    // (counts crowd at short lengths: the warp stops after the longest-run level)
    if (wp < 2u * (unsigned)A) {
        const int a = (int)(wp >> 1);
        const uint32_t gl = (wp & 1u) * 32u + lane;
        uint32_t rem = gl < 64u ? sm.gl_plev[a * 64 + gl] : 0u;
        // t8, sum c, sum c log2 c (RE = (nr log2 nr - sum c log2 c) / nr: exactly 0 for
        // a single cell, where c log2 c and nr log2 nr are the same rounded product;
        // __dmul_rn keeps the subtraction from contracting into an FMA)
        double t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t k = 0; k < 32u && __any_sync(kFull, rem != 0u); ++k) {
            if (!rem) continue;
            const uint32_t word = H[(uint32_t)a * kHA + gl * 33u + k];
            if (!word) continue;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t c = (word >> (16 * half)) & 0xffffu;
                if (!c) continue;
                rem -= c;
                const uint32_t li = k * 2u + (uint32_t)half;  // length - 1
                const double g = (double)gl + 1.0, l = (double)li + 1.0;
                const double cc = (double)c, g2 = g * g, l2 = l * l;
                const double rg2 = sm.gl_rcp2[gl], rl2 = sm.gl_rcp2[li];  // 1/g^2, 1/l^2
                t[0] += cc * rl2;
                t[1] += cc * l2;
                t[2] += cc * rg2;
                t[3] += cc * g2;
                t[4] += cc * (rg2 * rl2);
                t[5] += cc * (g2 * rl2);
                t[6] += cc * (l2 * rg2);
                t[7] += cc * g2 * l2;
                t[8] += cc;
                t[9] += cc * log2_int(c);
            }
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            double v = t[k];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) sm.gl_red[wp][k] = v;
        }
    }
    __syncthreads();
    // level / length moments and the 16 features: warp 2a for angle a
    if (wp < 2u * (unsigned)A && !(wp & 1u)) {
        const int a = (int)(wp >> 1);
        double t[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) t[k] = sm.gl_red[wp][k] + sm.gl_red[wp + 1][k];
        const double nr = t[8];
        double f = 0;
        if (nr > 0) {
            const double logn = nlog2(nr), np = (double)np_u;
            double s[4] = {0, 0, 0, 0};  // glnu, sum c (g+1), rlnu, sum c l
            for (int g = (int)lane; g < 64; g += 32) {
                const double c = (double)sm.gl_plev[a * 64 + g];
                s[0] += c * c;
                s[1] += c * (g + 1);
            }
            for (int l = (int)lane + 1; l <= 64; l += 32) {
                const double c = (double)sm.gl_ext[a * 65 + l];
                s[2] += c * c;
                s[3] += c * l;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int o = 16; o; o >>= 1) s[k] += __shfl_xor_sync(kFull, s[k], o);
            const double mu_g = s[1] / nr, mu_l = s[3] / nr;
            double v2[2] = {0, 0};  // glv, rv
            for (int g = (int)lane; g < 64; g += 32) {
                const double c = (double)sm.gl_plev[a * 64 + g];
                v2[0] += c / nr * (g + 1 - mu_g) * (g + 1 - mu_g);
            }
            for (int l = (int)lane + 1; l <= 64; l += 32) {
                const double c = (double)sm.gl_ext[a * 65 + l];
                v2[1] += c / nr * ((double)l - mu_l) * ((double)l - mu_l);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int o = 16; o; o >>= 1) v2[k] += __shfl_xor_sync(kFull, v2[k], o);
            const double v[16] = {t[0] / nr, t[1] / nr, s[0] / nr, s[0] / (nr * nr), s[2] / nr,
                                  s[2] / (nr * nr), nr / np, v2[0], v2[1], (__dmul_rn(nr, logn) - t[9]) / nr,
                                  t[2] / nr, t[3] / nr, t[4] / nr, t[5] / nr, t[6] / nr, t[7] / nr};
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if ((int)lane == k) f = v[k];
        }
        if (lane < 16) sm.gl_f[a][lane] = f;
    }
    __syncthreads();
    if (tid < 16) {
        double acc = 0;
        for (int a = 0; a < A; ++a) {
            og[tid * (A + 1) + a] = sm.gl_f[a][tid];
            acc += sm.gl_f[a][tid];
        }
        og[tid * (A + 1) + A] = acc / (double)A;
    }
    TT(5);
    // the hash table (skey / scnt) is kept empty between uses
    for (uint32_t i = tid; i < kTSlots; i += kTT) {
        d_skey()[i] = kEmpty;
        d_scnt()[i] = 0u;
    }
    __syncthreads();
    TT(6);
}

// SM: the window uses the shared-memory path (cells <= 4096; S-class windows always)
template <bool SM>
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
    const CellDiv cd((uint32_t)w);
    auto at = [&](uint32_t c) -> size_t {  // raster offset of window cell c
        int x, y;
        cd.split(c, x, y);
        return (size_t)(y0 + (uint32_t)y) * img.pitch + x0 + (uint32_t)x;
    };
    TT_DECL
    // ---- discretize (texture.cpp:29-56): min/max, then the level raster
    uint32_t lo = 0xffffu, hi = 0u;
    for (uint32_t c = tid; c < cells; c += kTT) {
        const size_t o = at(c);
        if (img.L[o] == label) {
            const uint32_t v = img.I[o];
            lo = min(lo, v);
            hi = max(hi, v);
        }
    }
    double none[1] = {0.0};
    tblock_fused<1>(none, hi, lo, sm);
    const uint32_t vmin = lo, vmax = hi;
    // floor(ng (v - vmin) / span) by multiply-high and one fix-up (ng <= 256, so the
    // numerator fits 32 bits): a 64-bit division per cell was ~10 % of the kernel
    const uint32_t span = vmax - vmin + 1u, mdiv = 0xffffffffu / span;
    uint16_t* lv = SM ? d_slev() : S.lev;  // shared memory for S-class windows
    for (uint32_t c = tid; c < cells; c += kTT) {
        uint16_t l = kNoLevel;
        const size_t o = at(c);
        if (img.L[o] == label) {
            l = 0;
            if (vmax > vmin) {
                const uint32_t num = (uint32_t)ng * (img.I[o] - vmin);
                uint32_t q = __umulhi(num, mdiv);
                if (num - q * span >= span) ++q;
                l = (uint16_t)min((uint32_t)(ng - 1), q);
            }
        }
        lv[c] = l;
    }
    __syncthreads();
    TT(0);
    // (level, extent) count table: shared memory for S-class windows (kept empty)
    constexpr bool small = SM;  // cells <= 4096 (so n <= 4096)
    uint32_t* hk = small ? d_skey() : S.hjk;
    uint32_t* hcn = small ? d_scnt() : S.hjc;
    const uint32_t mask = small ? kTSlots - 1u : HC - 1u;
    auto lev = [&](int x, int y) -> uint32_t {
        return (x >= 0 && x < w && y >= 0 && y < h) ? lv[(uint32_t)y * (uint32_t)w + (uint32_t)x]
                                                    : (uint32_t)kNoLevel;
    };
    // ---- GLRLM per sorted angle (texture.cpp:242-280)
#ifndef FXG_GLRLM_HASH
    if (cfg.col_glrlm >= 0 && small && w <= 64 && h <= 64 && ng <= 64 && cfg.n_angles <= 4) {
        glrlm_dense(lv, w, h, cells, n, cfg, sm, orow + cfg.col_glrlm);
    } else
#endif
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
            uint32_t emax = 0;
            for (uint32_t c = tid; c < cells; c += kTT) {
                const uint32_t g = lv[c];
                if (g == kNoLevel) continue;
                int x, y;
                cd.split(c, x, y);
                if (lev(x - dx, y - dy) == g) continue;  // not a run start
                uint32_t len = 1;
                int nx = x + dx, ny = y + dy;
                while (lev(nx, ny) == g) {
                    ++len;
                    nx += dx;
                    ny += dy;
                }
                unit_terms(t, (int)g, len, sm.gl_rcp2);
                ++runs;
                emax = max(emax, len);
                sred_add(&sm.plev[g], 1u);
                table_add(hk, hcn, mask, (g << 24) | len);
                atomicAdd(&S.ext[len], 1u);
            }
            TT(4);
            double t9[9] = {t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], (double)runs};
            uint32_t unused_min = 0xffffffffu;
            tblock_fused<9>(t9, emax, unused_min, sm);
#pragma unroll
            for (int k = 0; k < 8; ++k) t[k] = t9[k];
            const unsigned long long nr = (unsigned long long)t9[8];
            const double* tt = t;
            __shared__ double f16[16];
            extent_features(tt, nr, n, ng, S, hk, hcn, mask + 1u, emax, sm, f16);
            __syncthreads();
            TT(5);
            if (tid < 16) {
                og[tid * (A + 1) + a] = f16[tid];
                acc16[tid] += f16[tid];
            }
            __syncthreads();
        }
        if (tid < 16) og[tid * (A + 1) + A] = acc16[tid] / (double)A;
    }
    TT(1);
    // ---- GLSZM (texture.cpp:343-380): 8-connected zones of equal level
    if (cfg.col_glszm >= 0) {
        if constexpr (SM) glszm_zones<uint16_t>(d_spar(), d_szsz(), lv, w, h, cells);
        else glszm_zones<uint32_t>(S.par, S.zsz, lv, w, h, cells);
        TT(7);
        auto par_at = [&](uint32_t c) -> uint32_t {
            if constexpr (SM) return d_spar()[c];
            else return S.par[c];
        };
        auto zsz_at = [&](uint32_t c) -> uint32_t {
            if constexpr (SM) return d_szsz()[c];
            else return S.zsz[c];
        };
        double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unsigned long long zones = 0;
        uint32_t emax = 0;
        for (uint32_t c = tid; c < cells; c += kTT) {
            const uint32_t g = lv[c];
            if (g == kNoLevel || par_at(c) != c) continue;
            const uint32_t size = zsz_at(c);
            unit_terms(t, (int)g, size, sm.gl_rcp2);
            ++zones;
            emax = max(emax, size);
            sred_add(&sm.plev[g], 1u);
            table_add(hk, hcn, mask, (g << 24) | size);
            atomicAdd(&S.ext[size], 1u);
        }
        double t9[9] = {t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], (double)zones};
        uint32_t unused_min = 0xffffffffu;
        tblock_fused<9>(t9, emax, unused_min, sm);
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = t9[k];
        const double* tt = t;
        const unsigned long long nz = (unsigned long long)t9[8];
        __shared__ double f16z[16];
        extent_features(tt, nz, n, ng, S, hk, hcn, mask + 1u, emax, sm, f16z);
        __syncthreads();
        if (tid < 16) orow[cfg.col_glszm + tid] = f16z[tid];
        __syncthreads();
    }
    TT(2);
    // ---- NGTDM (texture.cpp:443-528)
    if (cfg.col_ngtdm >= 0) {
        for (int g = tid; g < ng; g += kTT) {
            sm.plev[g] = 0u;
            d_sng()[g] = 0ull;
        }
        __syncthreads();
        unsigned long long valid = 0;
        for (uint32_t c = tid; c < cells; c += kTT) {
            const uint32_t g = lv[c];
            if (g == kNoLevel) continue;
            int x, y;
            cd.split(c, x, y);
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
            sred_add(&d_sng()[g], (unsigned long long)((d < 0 ? -d : d) * (840 / cnt)));
            sred_add(&sm.plev[g], 1u);
            ++valid;
        }
        const unsigned long long nvu = tblock_all(valid, sm.u64, TAdd());
        double o5[5] = {0, 0, 0, 0, 0};
        if (nvu) {
            const double nv = (double)nvu;
            double a_s = 0, a_ps = 0;
            uint32_t a_pres = 0;
            for (int i = tid; i < ng; i += kTT) {
                const double p = (double)sm.plev[i] / nv, sv = (double)d_sng()[i] / 840.0;
                a_pres += p > 0;
                a_s += sv;
                a_ps += p * sv;
            }
            double r3[3] = {a_s, a_ps, (double)a_pres};
            tblock_sum<3>(r3, sm.red8);
            const double s_total = r3[0], ps_total = r3[1];
            const uint32_t present = (uint32_t)r3[2];
            double a_con = 0, a_busy = 0, a_cplx = 0, a_strn = 0;
            // pairs of present levels only (absent levels contribute nothing):
            // compact list in level order with p_i and s_i computed once
            if (twarp() == 0) {  // ballot compaction, level order
                const unsigned ln = lane_id();
                uint32_t k = 0;
                for (int i0 = 0; i0 < ng; i0 += 32) {
                    const int i = i0 + (int)ln;
                    const bool pr = i < ng && sm.plev[i] != 0u;
                    const unsigned b = __ballot_sync(kFull, pr);
                    if (pr) d_nglev()[k + __popc(b & lanemask_lt())] = (uint8_t)i;
                    k += __popc(b);
                }
                if (ln == 0) sm.ng_np = k;
            }
            __syncthreads();
            const uint32_t P = sm.ng_np;
            for (uint32_t k = tid; k < P; k += kTT) {
                const int i = d_nglev()[k];
                d_ngp()[k] = (double)sm.plev[i] / nv;
                d_ngs()[k] = (double)d_sng()[i] / 840.0;
            }
            __syncthreads();
            // every term is symmetric in (i, j) and 0 for i == j: pairs i < j, doubled
            const unsigned lane = lane_id();
            for (uint32_t ki = twarp(); ki < P; ki += kTW) {
                const int i = d_nglev()[ki];
                const double pi = d_ngp()[ki], si = d_ngs()[ki], gi = i + 1;
                for (uint32_t kj = ki + 1 + lane; kj < P; kj += 32) {
                    const int j = d_nglev()[kj];
                    const double pj = d_ngp()[kj], sj = d_ngs()[kj], gj = j + 1;
                    a_con += pi * pj * (i - j) * (i - j);
                    // unfused products: busyness divides by this sum, and equal products
                    // must cancel to exactly 0 as in the reference (an FMA leaves 1 ulp)
                    a_busy += fabs(__dsub_rn(__dmul_rn(gi, pi), __dmul_rn(gj, pj)));
                    a_cplx += fabs(gi - gj) * (pi * si + pj * sj) / (pi + pj);
                    a_strn += (pi + pj) * (gi - gj) * (gi - gj);
                }
            }
            a_con *= 2.0;
            a_busy *= 2.0;
            a_cplx *= 2.0;
            a_strn *= 2.0;
            double r4[4] = {a_con, a_busy, a_cplx, a_strn};
            tblock_sum<4>(r4, sm.red8);
            const double con = r4[0], busy = r4[1], cplx = r4[2], strn = r4[3];
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
    TT(3);
    (void)ctl;
}

// which = 0: the S-class lists (windows <= 64 x 64); 1: the large-ROI list
#ifndef FXG_T_MINB
#define FXG_T_MINB 4
#endif
__global__ void __launch_bounds__(kTT, FXG_T_MINB) k_roi_t(DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
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
    for (int k = threadIdx.x; k < 256; k += kTT) sm.gl_rcp2[k] = 1.0 / ((double)(k + 1) * (double)(k + 1));
    for (uint32_t i = threadIdx.x; i < kTSlots; i += kTT) {
        d_skey()[i] = kEmpty;
        d_scnt()[i] = 0u;
    }
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
        // shared-memory path for windows of <= 4096 cells (every S-class window)
        if ((unsigned long long)rl.w[r] * rl.h[r] <= 4096ull)
            process_t<true>(r, img, rl, ctl, cfg, out, S, T.HC, T.NMAX, sm);
        else
            process_t<false>(r, img, rl, ctl, cfg, out, S, T.HC, T.NMAX, sm);
    }
}

}  // namespace

cudaError_t roi_t_setup() {
    k_init_log2_tab<<<4, 256>>>();
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_roi_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynBytes);
    return e;
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
    k_roi_t<<<grid, kTT, kDynBytes, s>>>(img, rl, ctl, cfg, out, scratch, T, which);
}

// phase clocks of k_roi_t (thread 0 per ROI): 0 discretize, 1 GLRLM (rest),
// 2 GLSZM, 3 NGTDM, 4 GLRLM run counting, 5 GLRLM features
extern "C" int fx_debug_texture_clocks(unsigned long long* out, int n, int reset) {
#ifdef FXG_PHASE_TIMING
    unsigned long long h[8];
    if (cudaMemcpyFromSymbol(h, ::g_phase_clk_t, sizeof h) != cudaSuccess) return 7;
    for (int i = 0; i < n && i < 8; ++i) out[i] = h[i];
    if (reset) {
        const unsigned long long z[8] = {};
        cudaMemcpyToSymbol(::g_phase_clk_t, z, sizeof z);
    }
    return 0;
#else
    (void)out;
    (void)n;
    (void)reset;
    return 1;
#endif
}

}  // namespace fxg
