// S-class per-ROI kernels (window <= 64 x 64): one warp per ROI, lanes = window
// rows.  Bit-parallel over u64 row masks wherever the reference works per
// pixel.  See fx_roi.cuh for the reference mapping; larger windows and S ROIs
// past the run capacity go to the one-CTA-per-ROI kernel in fx_roi_b.cu.
//
// Phases (warp-synchronous, shared-memory slab per warp):
//   load    TMA label boxes (72x8, x origin 16 B aligned) -> row masks via 16 B
//           LDS; row offsets by warp scan; pixel coordinates; coalesced gather of
//           member intensities; exact integer sums (order-free, bit-exact).
//   sort    stable 2 x 8-bit LSD radix sort of the u16 values (one warp).
//   stats   order statistics from the sorted multiset (bit-exact class), fp64
//           central moments in a fixed order, histogram/mode by run detection.
//   edge    trace_contour visited set (definition B): bit-parallel 4-connected
//           exterior flood + 8-connected Euler number; when the ROI is one
//           component without holes the edge set is K & dilate4(exterior);
//           otherwise the run union-find slow path computes K and E.
//   moments separable row sums about integer anchors, fp64, fixed-order
//           reduce-scatter; binomial shift to the centroid and the origin.
//   glcm    integer discretisation; canonical pair keys; radix sort; run-length
//           counts; Haralick statistics from integer marginals.
#include <math.h>

#include "fx_glcm.cuh"
#include "fx_roi.cuh"

// Optional per-phase clock accounting (build with -DFXG_PHASE_TIMING; read with
// fx_debug_phase_clocks).  Off in the product build.
#ifdef FXG_PHASE_TIMING
__device__ unsigned long long g_phase_clk[16];
#define PT_DECL long long pt_t_ = clock64();
#define PT(k)                                                                              \
    do {                                                                                   \
        const long long t_ = clock64();                                                    \
        if (lane_id() == 0) atomicAdd(&g_phase_clk[k], (unsigned long long)(t_ - pt_t_)); \
        pt_t_ = t_;                                                                        \
    } while (0)
#else
#define PT_DECL
#define PT(k)
#endif


namespace fxg {

namespace {

// ---- slab layout for S windows ---------------------------------------------
struct SLayout {
    uint32_t rowmask, rowoff, vals, xy;        // region A
    uint32_t stage, stageI;                    // B: load (label and intensity tiles)
    uint32_t tmp, sorted, cnt;                 // B: sort / stats
    uint32_t kmask, emask, runoff, rs, re, parent, rsize;  // B: edge slow path
    uint32_t lvl, keys, keys2, gcnt, marg;     // B: glcm, sort path (ng > 64)
    uint32_t lmap, hist, list;                 // B: glcm, histogram path (ng <= 64)
    uint32_t bytes;
};


__host__ __device__ constexpr SLayout make_slayout(uint32_t TW, uint32_t TH, uint32_t NMAX,
                                                   uint32_t RUNMAX, int glcm) {
    SLayout L{};
    uint32_t o = 0;
    L.rowmask = o;
    o += TH * 8;
    L.rowoff = o;
    o = al(o + (TH + 1) * 4, 16);
    L.vals = o;
    o = al(o + NMAX * 2, 16);
    L.xy = o;
    o = al(o + NMAX * 2, 128);
    const uint32_t B = o;
    // the intensity tile is staged for the 40-wide S0 windows only: for the 72 x 64
    // tiles it would double the load region and cost S1/S2 occupancy (measured)
    const bool stage_i = TW == (uint32_t)kStageW0;
    L.stage = B;
    L.stageI = stage_i ? B + TW * TH * 2 : 0u;
    const uint32_t e_load = B + (stage_i ? 2u : 1u) * TW * TH * 2;
    L.tmp = B;
    L.sorted = al(L.tmp + NMAX * 2, 16);
    L.cnt = al(L.sorted + NMAX * 2, 16);
    const uint32_t e_sort = L.cnt + 512 * 4;
    L.kmask = B;
    L.emask = L.kmask + TH * 8;
    L.runoff = L.emask + TH * 8;
    L.rs = al(L.runoff + (TH + 1) * 4, 16);
    L.re = al(L.rs + RUNMAX * 2, 16);
    L.parent = al(L.re + RUNMAX * 2, 16);
    L.rsize = al(L.parent + RUNMAX * 4, 16);
    const uint32_t e_edge = L.rsize + RUNMAX * 4;
    // shape: K rows at kmask (staged to global for k_shape_serial)
    const uint32_t e_shape = L.emask;
    L.lvl = B;
    L.keys = al(L.lvl + NMAX, 16);
    L.keys2 = al(L.keys + NMAX * 2, 16);
    L.gcnt = al(L.keys2 + NMAX * 2, 16);
    L.marg = L.gcnt + 512 * 4;
    uint32_t e_glcm = B;
    if (glcm == kGlSort) e_glcm = L.marg + 1280 * 4;
    if (glcm == kGlHist) {  // level raster [TH][64] u8, histogram 4096 x u16, marginals
        L.lmap = B;
        L.hist = al(L.lmap + TH * 64, 16);
        L.marg = L.hist + 4096 * 2;
        // keys of the non-empty cells (<= pairs <= NMAX, u16): overlays vals (region
        // A), dead once the level raster is built
        L.list = L.vals;
        e_glcm = L.marg + 321 * 4;
    }
    L.bytes = al(mx(mx(mx(e_load, e_sort), mx(e_edge, e_glcm)), e_shape), 128) + 128;  // + mbarrier
    return L;
}

// window-class variants: stage width, max rows, max pixels, run capacity, warps/SM
// (MINB: without GLCM; MINB_G: with a GLCM mode, whose longer code runs faster with
// more registers per warp than the occupancy it gives up)
#ifndef FXG_S0_MINB
#define FXG_S0_MINB 20
#endif
#ifndef FXG_S0_MINB_G
#define FXG_S0_MINB_G 16
#endif
#ifndef FXG_S12_MINB_G
#define FXG_S12_MINB_G 16
#endif
template <int CLS>
struct SVar;
template <>
struct SVar<kClassS0> {
    static constexpr int TW = kStageW0, TH = kS0H, NMAX = kS0N, RUNMAX = 256, MINB = FXG_S0_MINB,
                         MINB_G = FXG_S0_MINB_G;
};
template <>
struct SVar<kClassS1> {
    static constexpr int TW = kStageW, TH = kSH, NMAX = kS1N, RUNMAX = 512, MINB = 20,
                         MINB_G = FXG_S12_MINB_G;
};
template <>
struct SVar<kClassS2> {
    static constexpr int TW = kStageW, TH = kSH, NMAX = kS2N, RUNMAX = 1024, MINB = 20,
                         MINB_G = FXG_S12_MINB_G;
};
template <int CLS, int GLCM>
constexpr SLayout slayout() {
    return make_slayout(SVar<CLS>::TW, SVar<CLS>::TH, SVar<CLS>::NMAX, SVar<CLS>::RUNMAX, GLCM);
}
constexpr uint32_t kSlack = 128;  // dynamic smem base alignment

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// all lanes get sum_j v[k] over lanes for k < 8 (reduce-scatter + broadcast)

// fill seeds s along the runs of f (both directions), Kogge-Stone
__device__ __forceinline__ uint64_t run_fill(uint64_t f, uint64_t s) {
    uint64_t g = s & f, p = f;
    g |= p & (g << 1); p &= p << 1;
    g |= p & (g << 2); p &= p << 2;
    g |= p & (g << 4); p &= p << 4;
    g |= p & (g << 8); p &= p << 8;
    g |= p & (g << 16); p &= p << 16;
    g |= p & (g << 32);
    p = f;
    g |= p & (g >> 1); p &= p >> 1;
    g |= p & (g >> 2); p &= p >> 2;
    g |= p & (g >> 4); p &= p >> 4;
    g |= p & (g >> 8); p &= p >> 8;
    g |= p & (g >> 16); p &= p >> 16;
    g |= p & (g >> 32);
    return g;
}

// the same on 32-bit rows (windows up to 32 wide: most S0 ROIs), half the work
__device__ __forceinline__ uint32_t run_fill32(uint32_t f, uint32_t s) {
    uint32_t g = s & f, p = f;
    g |= p & (g << 1); p &= p << 1;
    g |= p & (g << 2); p &= p << 2;
    g |= p & (g << 4); p &= p << 4;
    g |= p & (g << 8); p &= p << 8;
    g |= p & (g << 16);
    p = f;
    g |= p & (g >> 1); p &= p >> 1;
    g |= p & (g >> 2); p &= p >> 2;
    g |= p & (g >> 4); p &= p >> 4;
    g |= p & (g >> 8); p &= p >> 8;
    g |= p & (g >> 16);
    return g;
}

struct SJob {
    uint32_t label, x0, y0, w, h, row;
};

// ---------------------------------------------------------------------------
// Edge-set slow path (multiple 8-components or holes): run union-find for K,
// then for the 4-connected exterior E.  Returns false on run-capacity overflow.
// Writes K rows to km[] and E rows to em[] (lane-per-row layout).
__device__ __noinline__ bool edge_sets_slow(const uint64_t* rowmask, int h, int w, uint64_t* km,
                                            uint64_t* em, uint32_t* runoff, uint16_t* rs,
                                            uint16_t* re, uint32_t* parent, uint32_t* rsize,
                                            uint32_t runmax) {
    const unsigned lane = lane_id();
    auto build = [&](const uint64_t* m) -> uint32_t {
        uint32_t total = 0;
        for (int yb = 0; yb < h; yb += 32) {
            const int y = yb + lane;
            uint64_t r = (y < h) ? m[y] : 0ull;
            const uint32_t c = __popcll(r & ~(r << 1));
            const uint32_t incl = warp_incl_scan(c);
            if (y < h) runoff[y] = total + incl - c;
            total += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) runoff[h] = total;
        __syncwarp();
        if (total > runmax) return ~0u;
        for (int y = lane; y < h; y += 32) {
            const uint64_t r = m[y];
            uint64_t st = r & ~(r << 1), en = r & ~(r >> 1);
            uint32_t j = runoff[y];
            while (st) {
                rs[j] = (uint16_t)(__ffsll((long long)st) - 1);
                re[j] = (uint16_t)(__ffsll((long long)en) - 1);
                st &= st - 1;
                en &= en - 1;
                ++j;
            }
        }
        for (uint32_t r = lane; r < total; r += 32) parent[r] = r;
        __syncwarp();
        return total;
    };
    auto unite = [&](int ext) {
        for (int y = 1 + lane; y < h; y += 32) {
            uint32_t i = runoff[y], ie = runoff[y + 1], j = runoff[y - 1], je = runoff[y];
            while (i < ie && j < je) {
                const int as = rs[i], ae = re[i], bs = rs[j], be = re[j];
                if (be + ext < as) ++j;
                else if (ae + ext < bs) ++i;
                else {
                    uf_union(parent, i, j);
                    if (ae < be) ++i;
                    else ++j;
                }
            }
        }
        __syncwarp();
        // flatten chunk by chunk: all finds of a chunk (read-only) before its writes
        const uint32_t nr_ = runoff[h];
        for (uint32_t r0 = 0; r0 < nr_; r0 += 32) {
            const uint32_t r = r0 + lane;
            const uint32_t root = r < nr_ ? uf_root(parent, r) : 0u;
            __syncwarp();
            if (r < nr_) parent[r] = root;
            __syncwarp();
        }
    };
    const uint32_t nr = build(rowmask);
    if (nr == ~0u) return false;
    unite(1);
    for (uint32_t r = lane; r < nr; r += 32) rsize[r] = 0;
    __syncwarp();
    for (uint32_t r = lane; r < nr; r += 32) atomicAdd(&rsize[parent[r]], (uint32_t)(re[r] - rs[r] + 1));
    __syncwarp();
    unsigned long long best = 0;
    for (uint32_t r = lane; r < nr; r += 32)
        if (parent[r] == r) {
            const unsigned long long k = ((unsigned long long)rsize[r] << 32) | (0xffffffffu - r);
            best = k > best ? k : best;
        }
    best = warp_max(best);
    const uint32_t broot = 0xffffffffu - (uint32_t)(best & 0xffffffffu);
    const uint64_t wm = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
    for (int y = lane; y < h; y += 32) {
        uint64_t k = 0;
        for (uint32_t r = runoff[y]; r < runoff[y + 1]; ++r)
            if (parent[r] == broot) k |= bits_between(rs[r], re[r]);
        km[y] = k;
        em[y] = ~k & wm;
    }
    __syncwarp();
    const uint32_t nf = build(em);
    if (nf == ~0u) return false;
    unite(0);
    for (uint32_t r = lane; r < nf; r += 32) rsize[r] = 0;
    __syncwarp();
    for (int y = lane; y < h; y += 32)
        for (uint32_t r = runoff[y]; r < runoff[y + 1]; ++r)
            if (y == 0 || y == h - 1 || rs[r] == 0 || re[r] == w - 1) rsize[parent[r]] = 1u;
    __syncwarp();
    for (int y = lane; y < h; y += 32) {
        uint64_t e = 0;
        for (uint32_t r = runoff[y]; r < runoff[y + 1]; ++r)
            if (rsize[parent[r]]) e |= bits_between(rs[r], re[r]);
        em[y] = e;
    }
    __syncwarp();
    return true;
}


// scatter pass of a stable LSD radix sort; cnt[] holds exclusive digit offsets
// lanes holding the same 8-bit digit as this lane, among `valid` lanes: bit-sliced
// ballots (8 votes) instead of __match_any_sync
__device__ __forceinline__ unsigned digit_peers(uint32_t d, unsigned valid) {
#ifdef FXG_SORT_MATCH
    return __match_any_sync(kFull, d) & valid;
#else
    unsigned m = valid;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned bb = __ballot_sync(kFull, bit);
        m &= bit ? bb : ~bb;
    }
    return m;
#endif
}

__device__ __forceinline__ void radix_scatter(const uint16_t* src, uint16_t* dst, uint32_t n,
                                              int shift, uint32_t* cnt) {
    const unsigned lane = lane_id();
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
        const uint32_t i = b0 + lane;
        const bool ok = i < n;
        const uint16_t key = ok ? src[i] : 0;
        const uint32_t d = ((uint32_t)key >> shift) & 0xffu;
        const unsigned peers = digit_peers(d, __ballot_sync(kFull, ok));
        if (ok) dst[cnt[d] + __popc(peers & lanemask_lt())] = key;
        __syncwarp();
        if (ok && lane == (unsigned)(31 - __clz(peers))) cnt[d] += __popc(peers);
        __syncwarp();
    }
}

// Stable 16-bit LSD radix sort by one warp: both digit histograms in one pass,
// the high-digit pass skipped when every key shares its high byte.  Returns the
// buffer holding the sorted keys (tmp or dst).  cnt: 512 u32.
__device__ __forceinline__ const uint16_t* radix_sort16(const uint16_t* src, uint16_t* tmp,
                                                     uint16_t* dst, uint32_t n, uint32_t* cnt) {
    const unsigned lane = lane_id();
    for (int i = lane; i < 512; i += 32) cnt[i] = 0;
    __syncwarp();
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
        const uint32_t i = b0 + lane;
        const bool ok = i < n;
        const uint32_t key = ok ? src[i] : 0u;
        const uint32_t d0 = key & 0xffu, d1 = key >> 8;
        const unsigned valid = __ballot_sync(kFull, ok);
        const unsigned p0 = digit_peers(d0, valid), p1 = digit_peers(d1, valid);
        if (ok && lane == (unsigned)(__ffs(p0) - 1)) cnt[d0] += __popc(p0);
        if (ok && lane == (unsigned)(__ffs(p1) - 1)) cnt[256 + d1] += __popc(p1);
        __syncwarp();
    }
    const bool one_high = n == 0 || cnt[256 + (src[0] >> 8)] == n;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t c[8], t = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            c[k] = cnt[h * 256 + lane * 8 + k];
            t += c[k];
        }
        const uint32_t incl = warp_incl_scan(t);
        uint32_t run = incl - t;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            cnt[h * 256 + lane * 8 + k] = run;
            run += c[k];
        }
    }
    __syncwarp();
    radix_scatter(src, tmp, n, 0, cnt);
    if (one_high) return tmp;
    radix_scatter(tmp, dst, n, 8, cnt + 256);
    return dst;
}

// Bitonic sort of up to 32 * NPL u16 keys held by one warp in registers: lane l
// holds elements [l NPL, (l + 1) NPL), two per 32-bit register, compared two at a
// time with the paired-halfword min / max (VIMNMX.U16x2).  Strides >= NPL swap
// whole registers with the partner lane (shuffles), strides 2..NPL/2 pair
// registers of one lane, stride 1 pairs the two halves of a register.  No shared
// memory traffic and no atomics (the radix sort's dependent shared-memory round
// trips).  Used for the GLCM pair keys; keys past n are 0xFFFF and sort to the end.
template <int NPL>
__device__ __forceinline__ void bitonic_warp_u16(uint32_t (&r)[NPL / 2]) {
    const unsigned lane = lane_id();
    constexpr int LL = NPL == 8 ? 3 : NPL == 16 ? 4 : 5;  // log2(NPL)
    constexpr int LOGN = LL + 5;
#pragma unroll
    for (int k = 1; k <= LOGN; ++k) {
#pragma unroll
        for (int st = k - 1; st >= 0; --st) {
            if (st >= LL) {  // partner lane
                const int lm = 1 << (st - LL);
                const bool up = k == LOGN || !((lane >> (k - LL)) & 1u);
                const bool keep_min = ((lane & lm) == 0) == up;
#pragma unroll
                for (int q = 0; q < NPL / 2; ++q) {
                    const uint32_t y = __shfl_xor_sync(kFull, r[q], lm);
                    r[q] = keep_min ? __vminu2(r[q], y) : __vmaxu2(r[q], y);
                }
            } else if (st >= 1) {  // registers q, q + 2^(st-1) of this lane
                const int rs = 1 << (st - 1);
#pragma unroll
                for (int q = 0; q < NPL / 2; ++q) {
                    if (q & rs) continue;
                    // direction: bit k of e = l NPL + 2 q + h
                    const bool up = k == LOGN ||
                                    (k >= LL ? !((lane >> (k - LL)) & 1u) : !((q >> (k - 1)) & 1));
                    const uint32_t a = r[q], b = r[q + rs];
                    const uint32_t lo = __vminu2(a, b), hi = __vmaxu2(a, b);
                    r[q] = up ? lo : hi;
                    r[q + rs] = up ? hi : lo;
                }
            } else {  // the two halves of each register
#pragma unroll
                for (int q = 0; q < NPL / 2; ++q) {
                    const bool up = k == LOGN ||
                                    (k >= LL ? !((lane >> (k - LL)) & 1u) : !((q >> (k - 1)) & 1));
                    const uint32_t x = r[q], sw = __byte_perm(x, 0u, 0x1032);
                    const uint32_t mn = __vminu2(x, sw), mxv = __vmaxu2(x, sw);
                    r[q] = up ? __byte_perm(mn, mxv, 0x7610) : __byte_perm(mxv, mn, 0x7610);
                }
            }
        }
    }
}

// src[0, n) sorted into dst by bitonic_warp_u16 (n <= 32 NPL); src 4 B aligned
template <int NPL>
__device__ __forceinline__ void bitonic_sort16(const uint16_t* src, uint16_t* dst, uint32_t n) {
    const unsigned lane = lane_id();
    uint32_t r[NPL / 2];
    const uint32_t e0 = lane * NPL;
#pragma unroll
    for (int q = 0; q < NPL / 2; ++q) {
        const uint32_t e = e0 + 2 * q;
        const uint32_t a = e < n ? src[e] : 0xffffu, b = e + 1 < n ? src[e + 1] : 0xffffu;
        r[q] = a | (b << 16);
    }
    bitonic_warp_u16<NPL>(r);
#pragma unroll
    for (int q = 0; q < NPL / 2; ++q) {
        const uint32_t e = e0 + 2 * q;
        if (e < n) dst[e] = (uint16_t)(r[q] & 0xffffu);
        if (e + 1 < n) dst[e + 1] = (uint16_t)(r[q] >> 16);
    }
}

// Sort of plain u16 keys by one warp (no payload, so equal keys need no stable
// order): bucket b = (v - vmin) >> s with s the least shift giving <= 512 buckets,
// shared-atomic histogram and scatter, then each key ranks itself inside its
// bucket.  With range < 512 the buckets hold equal keys and the scatter is the
// sort.  Crowded buckets (sum of squared counts > 16 n) fall back to the radix
// sort.  Returns the sorted buffer and vmin / vmax.  cnt: 512 u32.
__device__ __forceinline__ const uint16_t* bucket_sort16(const uint16_t* src, uint16_t* tmp,
                                                      uint16_t* dst, uint32_t n, uint32_t* cnt,
                                                      uint32_t lo, uint32_t hi) {
    // lo / hi: min and max of the keys (the gather computes them)
    const unsigned lane = lane_id();
    const uint32_t r = hi - lo;
    if (n == 0 || r == 0) return src;  // all keys equal: already sorted
    const int s = max(0, 23 - __clz(r));  // (r >> s) < 512
    // bucket b lives at cnt[(b & 15) * 32 + (b >> 4)]: lane l owns buckets 16 l ..
    // 16 l + 15 as one bank column
    auto slot = [](uint32_t b) { return ((b & 15u) << 5) | (b >> 4); };
#pragma unroll
    for (int k = 0; k < 16; ++k) cnt[k * 32 + lane] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) atomicAdd(&cnt[slot((src[i] - lo) >> s)], 1u);
    __syncwarp();
    uint32_t c[16], t = 0, sq = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        c[k] = cnt[k * 32 + lane];
        t += c[k];
        sq += c[k] * c[k];
    }
    sq = warp_sum(sq);
    if (s > 0 && sq > 16u * n) return radix_sort16(src, tmp, dst, n, cnt);
    uint32_t run = warp_incl_scan(t) - t;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        cnt[k * 32 + lane] = run;
        run += c[k];
    }
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t v = src[i];
        tmp[atomicAdd(&cnt[slot((v - lo) >> s)], 1u)] = (uint16_t)v;
    }
    __syncwarp();
    if (s == 0) return tmp;  // buckets are single values
    // cnt[b] is now the end of bucket b (= the start of bucket b + 1)
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t v = tmp[i], b = (v - lo) >> s;
        const uint32_t st = b ? cnt[slot(b - 1)] : 0u, en = cnt[slot(b)];
        uint32_t rank = 0;
        if (en - st > 1u)  // singleton buckets (most, at ~n/512 keys per bucket) skip the walk
            for (uint32_t j = st; j < en; ++j) {
                const uint32_t u = tmp[j];
                rank += (u < v) | ((u == v) & (j < i));
            }
        dst[st + rank] = (uint16_t)v;
    }
    __syncwarp();
    return dst;
}



// k-th smallest (0-based) of |2 s[i] - M2| over sorted s by the whole warp:
// 32-ary searches for the V split and the merge split of the two sorted halves.
__device__ __noinline__ uint32_t kth_dev2_warp(const uint16_t* s, uint32_t n, uint32_t M2, uint32_t k) {
    const unsigned lane = lane_id();
    // m = first index with 2 s[i] >= M2 (in [0, n])
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t t = lo + lane * step;
        const bool pr = t < hi && 2u * s[t] >= M2;
        const unsigned b = __ballot_sync(kFull, pr);
        if (b == 0) {
            lo = lo + 31 * step + 1;
            if (lo > hi) lo = hi;
        } else {
            const uint32_t f = __ffs(b) - 1;  // first lane whose probe is true
            hi = lo + f * step;
            lo = f ? lo + (f - 1) * step + 1 : lo;
        }
    }
    const uint32_t m = lo, na = m, nb = n - m;
    // smallest i in [ilo, ihi] with (i == ihi) or A[i] >= B[k-i]
    uint32_t ilo = (k + 1 > nb) ? k + 1 - nb : 0, ihi = (k + 1 < na) ? k + 1 : na;
    while (ilo < ihi) {
        const uint32_t step = (ihi - ilo + 31) / 32;
        const uint32_t i = ilo + lane * step;
        bool pr = true;
        if (i < ihi) {
            const uint32_t Ai = M2 - 2u * s[m - 1 - i];
            const uint32_t Bj1 = 2u * s[m + (k - i)] - M2;  // B[j-1], j = k+1-i
            pr = !(Ai < Bj1);
        }
        const unsigned b = __ballot_sync(kFull, pr);
        const uint32_t f = __ffs(b) - 1;
        const uint32_t cand = ilo + f * step;
        const uint32_t nhi = cand < ihi ? cand : ihi;
        ilo = f ? ilo + (f - 1) * step + 1 : ilo;
        ihi = nhi;
    }
    const uint32_t i = ilo, j = k + 1 - i;
    uint32_t best = 0;
    if (i > 0) best = M2 - 2u * s[m - i];
    if (j > 0) {
        const uint32_t b = 2u * s[m + j - 1] - M2;
        if (i == 0 || b > best) best = b;
    }
    return best;
}


// ---------------------------------------------------------------------------
// Shape group of an S window (shape_features.cpp:147-251), warp-level.
//   km     : rows of K (largest 8-connected component), the grid trace_contour walks
//   rowmask: rows of all ROI pixels (hull, Euler number, ellipse, extrema)
//   scr    : [h][64] walk-state bytes, column extremes, hull vertices
// Exact: area, bbox, centroid (integer sums), perimeter (the Moore walk of
// contour.cpp:70-144 replayed: the first repeated (position, backtrack) state
// starts the cycle, whose steps are summed in walk order), convex area (lattice
// points per row from the hull edges' integer half-planes), Euler number (bit
// quads, 8-connected foreground / 4-connected background), extrema, and the
// ellipse sums (sequential in pixel order without FMA, as the reference).
__constant__ int8_t c_ring[8][2] = {{-1, 0}, {-1, -1}, {0, -1}, {1, -1},
                                    {1, 0},  {1, 1},   {0, 1},  {-1, 1}};

// ring index of a unit offset (dx, dy) in [-1, 1]^2: (dx + 1) * 3 + (dy + 1)
__constant__ int8_t c_ring_of[9] = {1, 0, 7, 2, -1, 6, 3, 4, 5};

// one step of the Moore walk: position (x, y), backtrack ring index b.  The 8
// neighbours come from three K rows as one byte in ring order; the next
// direction is the first set bit after b (rotate + ffs).
__device__ __forceinline__ uint32_t three_bits(uint64_t row, int x) {  // cols x-1, x, x+1
    return (uint32_t)((x > 0 ? (row >> (x - 1)) : (row << 1)) & 7ull);
}
__device__ __forceinline__ void walk_step(const uint64_t* km, int h, int w, int& x, int& y, int& b) {
    const uint32_t u = y > 0 ? three_bits(km[y - 1], x) : 0u;
    const uint32_t m = three_bits(km[y], x);
    const uint32_t d = y + 1 < h ? three_bits(km[y + 1], x) : 0u;
    // ring: W, NW, N, NE, E, SE, S, SW
    const uint32_t nb = (m & 1u) | ((u & 1u) << 1) | ((u & 2u) << 1) | ((u & 4u) << 1) |
                        ((m & 4u) << 2) | ((d & 4u) << 3) | ((d & 2u) << 5) | ((d & 1u) << 7);
    const int st = (b + 1) & 7;
    const uint32_t rot = ((nb >> st) | (nb << (8 - st))) & 0xffu;
    const int found = (st + __ffs(rot) - 1) & 7;
    const int prev = (found + 7) & 7;
    const int ddx = c_ring[prev][0] - c_ring[found][0], ddy = c_ring[prev][1] - c_ring[found][1];
    x += c_ring[found][0];
    y += c_ring[found][1];
    b = c_ring_of[(ddx + 1) * 3 + (ddy + 1)];
    (void)w;
}

__device__ __forceinline__ long long floor_div(long long a, long long b) {  // b > 0
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// 8-connected Euler number contributions of row pair (a above b) over the
// zero-padded columns 0..w (bit quads)
__device__ __forceinline__ int quads_pair(uint64_t a, uint64_t b, int w) {
    const uint64_t vm = (w >= 63) ? ~0ull : ((2ull << w) - 1ull);
    const uint64_t A0 = a << 1, A1 = a, B0 = b << 1, B1 = b;
    const uint64_t s1 = A0 ^ A1, s2 = B0 ^ B1, c = (A0 & A1) | (B0 & B1);
    const uint64_t one = (s1 ^ s2) & ~c & vm, three = (s1 ^ s2) & c & vm;
    const uint64_t dg = ((A0 & B1 & ~A1 & ~B0) | (A1 & B0 & ~A0 & ~B1)) & vm;
    int q = __popcll(one) - __popcll(three) - 2 * __popcll(dg);
    if (w == 64) q += (int)(((a >> 63) ^ (b >> 63)) & 1ull);  // quad at padded column 64
    return q;
}

// Warp part of the S shape group: the columns computable in parallel (area,
// bbox, centroid, extent, aspect ratio, equivalent diameter, Euler number,
// extrema) and the staging of the row masks (all pixels, K) for k_shape_serial.
__device__ __noinline__ void shape_phase_s(const uint64_t* rowmask, const uint64_t* km, int h,
                                           int w, uint32_t n, long long gx0, long long gy0,
                                           unsigned long long sLX, unsigned long long sLY,
                                           uint32_t row, const FeatCfg& cfg, double* o) {
    const unsigned lane = lane_id();
    const double PI = 3.141592653589793;
    const double dn = (double)n;
    // Euler number (bit quads over the padded window)
    int q = 0;
    for (int y = lane; y <= h; y += 32) q += quads_pair(y ? rowmask[y - 1] : 0ull, y < h ? rowmask[y] : 0ull, w);
    q = warp_sum(q);
    // extrema: first/last pixel of the first/last row and column
    int ct = 0x7fffffff, cb = -1, rt = 0x7fffffff, rb = -1;  // column 0, column w-1
    for (int y = lane; y < h; y += 32) {
        const uint64_t m = rowmask[y];
        if (m & 1ull) {
            ct = min(ct, y);
            cb = max(cb, y);
        }
        if ((m >> (w - 1)) & 1ull) {
            rt = min(rt, y);
            rb = max(rb, y);
        }
    }
    ct = warp_min(ct);
    cb = warp_max(cb);
    rt = warp_min(rt);
    rb = warp_max(rb);
    // stage the rows for the serial pass: [0..63] all pixels, [64..127] K
    uint64_t* st = cfg.shape_rows + (size_t)row * 128;
    for (int y = lane; y < h; y += 32) {
        st[y] = rowmask[y];
        st[64 + y] = km[y];
    }
    __syncwarp();
    if (lane == 0) cfg.shape_hdr[row] = (uint32_t)h | ((uint32_t)w << 8) | (1u << 16);
    const double bw = (double)w, bh = (double)h;
    const double cx = (double)((unsigned long long)gx0 * n + sLX) / dn;
    const double cy = (double)((unsigned long long)gy0 * n + sLY) / dn;
    double v = 0;
    int col = -1;
    switch (lane) {
        case 0: v = dn; col = 0; break;
        case 2: v = (double)gx0; col = 2; break;
        case 3: v = (double)gy0; col = 3; break;
        case 4: v = bw; col = 4; break;
        case 5: v = bh; col = 5; break;
        case 6: v = cx; col = 6; break;
        case 7: v = cy; col = 7; break;
        case 9: v = dn / (bw * bh); col = 9; break;
        case 10: v = bw / bh; col = 10; break;
        case 13: v = sqrt(4.0 * dn / PI); col = 13; break;
        case 19: v = (double)(q / 4); col = 19; break;
        default: break;
    }
    if (col >= 0) o[col] = v;
    if (lane >= 22 && lane < 30) {  // extrema (x, y) pairs in regionprops order
        const int e = lane - 22;
        const uint64_t r0 = rowmask[0], rl = rowmask[h - 1];
        int ex = 0, ey = 0;
        switch (e) {
            case 0: ex = __ffsll((long long)r0) - 1; ey = 0; break;
            case 1: ex = 63 - __clzll((long long)r0); ey = 0; break;
            case 2: ex = w - 1; ey = rt; break;
            case 3: ex = w - 1; ey = rb; break;
            case 4: ex = 63 - __clzll((long long)rl); ey = h - 1; break;
            case 5: ex = __ffsll((long long)rl) - 1; ey = h - 1; break;
            case 6: ex = 0; ey = cb; break;
            default: ex = 0; ey = ct; break;
        }
        o[22 + 2 * e] = (double)(gx0 + ex);
        o[23 + 2 * e] = (double)(gy0 + ey);
    }
    __syncwarp();
}

// Serial part of the S shape group, one thread per ROI (the warp path would run
// these sequential loops on single lanes, one divergent branch after another):
// perimeter (the Moore walk of contour.cpp:70-144 replayed on K with Brent's
// cycle detection: the first state of the cycle is where the reference's
// first-repeated-state rule cuts it, steps summed in walk order), hull of the
// column extremes (hull.cpp:17-55) with its lattice-point count and Feret
// diameters, the +1/12 ellipse from sums in pixel order without FMA.
__global__ void __launch_bounds__(128) k_shape_serial(RoiList rl, Control* ctl, FeatCfg cfg,
                                                      double* out) {
    const uint32_t n0 = ctl->class_count[kClassS0], n1 = ctl->class_count[kClassS1];
    const uint32_t nt = n0 + n1 + ctl->class_count[kClassS2];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint32_t r = t < n0 ? rl.cls_list[kClassS0][t]
                     : t < n0 + n1 ? rl.cls_list[kClassS1][t - n0] : rl.cls_list[kClassS2][t - n0 - n1];
    const uint32_t hd = cfg.shape_hdr[r];
    if (!(hd >> 16)) return;  // re-queued to the large-ROI kernel, which does its own
    cfg.shape_hdr[r] = 0u;
    const int h = (int)(hd & 0xffu), w = (int)((hd >> 8) & 0xffu);
    const uint64_t* rows = cfg.shape_rows + (size_t)r * 128;
    const uint64_t* km = rows + 64;
    const double PI = 3.141592653589793, SQRT2 = 1.4142135623730951;
    const long long gx0 = rl.gx[r], gy0 = rl.gy[r];
    const unsigned long long n = rl.n[r];
    const double dn = (double)n;
    double* o = out + (size_t)r * cfg.ncols + cfg.col_shape;
    // ---- ellipse sums (three independent sequential chains) and |K|
    unsigned long long sx = 0, sy = 0;
    uint32_t kc = 0;
    for (int y = 0; y < h; ++y) {
        const uint64_t m = rows[y];
        const int c = __popcll(m);
        sy += (unsigned long long)c * (unsigned long long)(gy0 + y);
        uint64_t mm = m;
        while (mm) {
            sx += (unsigned long long)(gx0 + __ffsll((long long)mm) - 1);
            mm &= mm - 1;
        }
        kc += __popcll(km[y]);
    }
    const double cx = (double)sx / dn, cy = (double)sy / dn;
    double m20 = 0, m02 = 0, m11 = 0;
    for (int y = 0; y < h; ++y) {
        uint64_t m = rows[y];
        const double dy = __dsub_rn((double)(gy0 + y), cy), dy2 = __dmul_rn(dy, dy);
        while (m) {
            const int x = __ffsll((long long)m) - 1;
            m &= m - 1;
            const double dx = __dsub_rn((double)(gx0 + x), cx);
            m20 = __dadd_rn(m20, __dmul_rn(dx, dx));
            m02 = __dadd_rn(m02, dy2);
            m11 = __dadd_rn(m11, __dmul_rn(dx, dy));
        }
    }
    // ---- perimeter: Brent on the walk, then the cycle's steps in order
    double per = 4.0;
    if (n > 1 && kc > 1) {
        int sy0 = 0;
        while (!km[sy0]) ++sy0;
        const int sx0 = __ffsll((long long)km[sy0]) - 1;
        int tx = sx0, ty = sy0, tb = 0, hx = sx0, hy = sy0, hb = 0;
        walk_step(km, h, w, hx, hy, hb);
        uint32_t power = 1, lam = 1;
        while (tx != hx || ty != hy || tb != hb) {
            if (power == lam) {
                tx = hx;
                ty = hy;
                tb = hb;
                power *= 2;
                lam = 0;
            }
            walk_step(km, h, w, hx, hy, hb);
            ++lam;
        }
        tx = hx = sx0;
        ty = hy = sy0;
        tb = hb = 0;
        for (uint32_t i = 0; i < lam; ++i) walk_step(km, h, w, hx, hy, hb);
        while (tx != hx || ty != hy || tb != hb) {
            walk_step(km, h, w, tx, ty, tb);
            walk_step(km, h, w, hx, hy, hb);
        }
        per = 0;
        for (uint32_t i = 0; i < lam; ++i) {
            const int px = tx, py = ty;
            walk_step(km, h, w, tx, ty, tb);
            per = __dadd_rn(per, (abs(tx - px) + abs(ty - py) == 2) ? SQRT2 : 1.0);
        }
    }
    // ---- hull of the column extremes: chain stack of packed (x | y << 8)
    uint16_t hs[2 * 128 + 2];
    uint8_t ctop[64], cbot[64];  // column extremes (255: empty column)
    for (int x = 0; x < w; ++x) ctop[x] = cbot[x] = 255;
    for (int y = 0; y < h; ++y) {
        uint64_t m = rows[y];
        while (m) {
            const int x = __ffsll((long long)m) - 1;
            m &= m - 1;
            if (ctop[x] == 255) ctop[x] = (uint8_t)y;
            cbot[x] = (uint8_t)y;
        }
    }
    int k = 0, npt = 0, fx = -1, fy = 0, lx = 0, ly = 0;
    auto col_ext = [&](int x, int& top, int& bot) {
        top = ctop[x] == 255 ? -1 : ctop[x];
        bot = cbot[x] == 255 ? -1 : cbot[x];
    };
    for (int x = 0; x < w; ++x) {
        int tp, bt;
        col_ext(x, tp, bt);
        if (tp < 0) continue;
        npt += tp == bt ? 1 : 2;
        if (fx < 0) {
            fx = x;
            fy = tp;
        }
        lx = x;
        ly = bt;
    }
    if (npt <= 2) {
        for (int x = 0; x < w; ++x) {
            int tp, bt;
            col_ext(x, tp, bt);
            if (tp < 0) continue;
            hs[k++] = (uint16_t)(x | (tp << 8));
            if (bt != tp) hs[k++] = (uint16_t)(x | (bt << 8));
        }
    } else {
        int ax = 0, ay = 0, bx = 0, by = 0;  // hs[k-2], hs[k-1]
        auto push = [&](int px, int py, int lo) {
            while (k >= lo && (bx - ax) * (py - ay) - (by - ay) * (px - ax) <= 0) {
                --k;
                bx = ax;
                by = ay;
                if (k >= 2) {
                    ax = hs[k - 2] & 0xff;
                    ay = hs[k - 2] >> 8;
                }
            }
            hs[k++] = (uint16_t)(px | (py << 8));
            ax = bx;
            ay = by;
            bx = px;
            by = py;
        };
        for (int x = 0; x < w; ++x) {
            int tp, bt;
            col_ext(x, tp, bt);
            if (tp < 0) continue;
            push(x, tp, 2);
            if (bt != tp) push(x, bt, 2);
        }
        const int lower = k + 1;
        bool skip_last = true;
        for (int x = w - 1; x >= 0; --x) {
            int tp, bt;
            col_ext(x, tp, bt);
            if (tp < 0) continue;
            if (bt != tp) {
                if (!skip_last) push(x, bt, lower);
                skip_last = false;
                push(x, tp, lower);
            } else {
                if (!skip_last) push(x, tp, lower);
                skip_last = false;
            }
        }
        k -= 1;
        if (k < 3) {
            hs[0] = (uint16_t)(fx | (fy << 8));
            hs[1] = (uint16_t)(lx | (ly << 8));
            k = 2;
        }
    }
    const int nv = k;
    // ---- convex area (lattice points inside or on the hull) and Feret diameters
    unsigned long long carea = 0;
    if (nv >= 3)
        for (int y = 0; y < h; ++y) {
            int xl = 0, xr = w - 1;
            for (int i = 0; i < nv && xl <= xr; ++i) {
                const int j = i + 1 < nv ? i + 1 : 0;
                const int ax = hs[i] & 0xff, ay = hs[i] >> 8, bx = hs[j] & 0xff, by = hs[j] >> 8;
                const int B = by - ay, A = (bx - ax) * (y - ay) + B * ax;  // A - B x >= 0
                if (B > 0) xr = min(xr, (int)floor_div(A, B));
                else if (B < 0) xl = max(xl, -(int)floor_div(A, -B));
                else if (A < 0) xr = -1;
            }
            if (xr >= xl) carea += (unsigned long long)(xr - xl + 1);
        }
    double fmx = 0, fmn = 0;
    if (nv >= 2) {  // max over vertex pairs of the exact squared distance, one sqrt
        int d2 = 0;
        for (int i = 0; i < nv; ++i)
            for (int j = i + 1; j < nv; ++j) {
                const int dx = (hs[i] & 0xff) - (hs[j] & 0xff), dy = (hs[i] >> 8) - (hs[j] >> 8);
                d2 = max(d2, dx * dx + dy * dy);
            }
        fmx = sqrt((double)d2);
        if (nv > 2) {
            fmn = 1.79769313486231570815e308;
            for (int i = 0; i < nv; ++i) {
                const int j = i + 1 < nv ? i + 1 : 0;
                const int ax = hs[i] & 0xff, ay = hs[i] >> 8;
                const int ex = (hs[j] & 0xff) - ax, ey = (hs[j] >> 8) - ay;
                int mc = 0;
                for (int kk = 0; kk < nv; ++kk) {
                    const int c = ex * ((hs[kk] >> 8) - ay) - ey * ((hs[kk] & 0xff) - ax);
                    mc = max(mc, c < 0 ? -c : c);
                }
                fmn = fmin(fmn, (double)mc / hypot((double)ex, (double)ey));
            }
        }
    }
    // ---- columns (shape_feature_values order)
    o[1] = per;
    o[8] = n == 1 ? 1.0 : 4.0 * PI * dn / (per * per);
    o[11] = (double)carea;
    o[12] = carea ? dn / (double)carea : 0.0;
    {
        const double a = __dadd_rn(__ddiv_rn(m20, dn), 1.0 / 12.0);
        const double c = __dadd_rn(__ddiv_rn(m02, dn), 1.0 / 12.0);
        const double bb = __ddiv_rn(m11, dn);
        const double amc = __dsub_rn(a, c);
        const double disc = sqrt(__dadd_rn(__ddiv_rn(__dmul_rn(amc, amc), 4.0), __dmul_rn(bb, bb)));
        const double hsum = __ddiv_rn(__dadd_rn(a, c), 2.0);
        const double l1 = __dadd_rn(hsum, disc), l2 = __dsub_rn(hsum, disc);
        const double maj = 4.0 * sqrt(fmax(0.0, l1)), mnr = 4.0 * sqrt(fmax(0.0, l2));
        o[14] = maj;
        o[15] = mnr;
        o[16] = l1 > 0 ? sqrt(fmax(0.0, 1.0 - l2 / l1)) : 0.0;
        o[17] = mnr > 0 ? maj / mnr : 0.0;
        o[18] = ellipse_orientation(bb, amc);
    }
    o[20] = fmx;
    o[21] = fmn;
}

// GLCM group for an S window with ng <= 64 (kGlHist): discretize (texture.cpp:45-53,
// exact integer floor) into a level raster, count pair keys per sorted angle
// (texture.cpp:58-80) in a packed-u16 shared histogram (key = la*64 + lb, or the
// canonical min/max key when symmetric), then one pass over the non-empty cells:
// ASM, autocorrelation and max probability from exact integer sums, entropy from
// one fp64 sum of c*log2(c), marginals by shared atomics; Haralick statistics
// from the integer marginals (texture.cpp:87-217; hxy1 == hxy2 == hx + hy).
// shared-memory atomics through explicit shared addresses (the slab pointers a
// noinline phase receives are generic and would compile to generic ATOM)
__device__ __forceinline__ uint32_t satom_add(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void sred_add(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __noinline__ void glcm_phase_h(uint32_t n, int h, const uint64_t* rowmask,
                                          const uint16_t* xy, const uint16_t* vals,
                                          uint8_t* lmap, uint32_t* hist, uint32_t* marg,
                                          uint16_t* list,
                                          uint32_t vmin, uint32_t vmax, const FeatCfg& cfg,
                                          double* og, const DebugOut* dbg) {
    const unsigned lane = lane_id();
    const int ng = cfg.ng, A = cfg.n_angles;
    const uint32_t span = vmax - vmin + 1u;
    const uint32_t mdiv = 0xffffffffu / span;
    PT_DECL
    for (uint32_t i = lane; i < n; i += 32) {
        uint32_t lv = 0;
        if (vmax > vmin) {  // floor(ng * (v - vmin) / span) by multiply-high + one fix-up
            const uint32_t num = (uint32_t)ng * (vals[i] - vmin);
            uint32_t q = __umulhi(num, mdiv);
            if (num - q * span >= span) ++q;
            lv = min((uint32_t)(ng - 1), q);
        }
        const uint32_t p = xy[i];
        lmap[(p >> 8) * 64 + (p & 0xffu)] = (uint8_t)lv;
    }
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    const int nq = ng * 8;  // uint4 words covering keys < ng * 64
    for (int j = lane; j < nq; j += 32) h4[j] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    const bool sym = cfg.symmetric != 0;
    uint32_t* px = marg;
    uint32_t* py = sym ? marg : marg + 64;  // symmetric: p_y == p_x
    uint32_t* psum = marg + 128;            // [2ng-1]
    uint32_t* pdif = marg + 256;            // [ng]
    double sacc = 0;
    for (int a = 0; a < A; ++a) {
        const int ddx = cfg.dx[a], ddy = cfg.dy[a];
        for (int k = lane; k < 321; k += 32) marg[k] = 0u;  // + marg[320]: list length
        // pairs, pixel-parallel: (x, y) and (x + dx, y + dy) both in the ROI; the
        // first pair of a cell appends its key to the cell list (warp-aggregated)
        uint32_t npr = 0;
        for (uint32_t b = 0; b < n; b += 32) {
            const uint32_t i = b + lane;
            bool pair = false, fresh = false;
            uint32_t key = 0;
            if (i < n) {
                const uint32_t p = xy[i];
                const int x = (int)(p & 0xffu), y = (int)(p >> 8);
                const int nx = x + ddx, ny = y + ddy;
                pair = ny >= 0 && ny < h && nx >= 0 && nx < 64 && ((rowmask[ny] >> nx) & 1ull);
                if (pair) {
                    const uint32_t la = lmap[y * 64 + x], lb = lmap[ny * 64 + nx];
                    key = sym ? min(la, lb) * 64u + max(la, lb) : la * 64u + lb;
                    const uint32_t sh = (key & 1u) * 16u;
                    const uint32_t old = satom_add(&hist[key >> 1], 1u << sh);
                    fresh = ((old >> sh) & 0xffffu) == 0u;
                }
            }
            npr += pair;
            const unsigned fm = __ballot_sync(kFull, fresh);
            if (fm) {
                uint32_t base = 0;
                if (lane == 0) base = satom_add(&marg[320], (uint32_t)__popc(fm));
                base = __shfl_sync(kFull, base, 0);
                if (fresh) list[base + __popc(fm & lanemask_lt())] = (uint16_t)key;
            }
        }
        __syncwarp();
        const uint32_t np = warp_sum(npr);
        __syncwarp();
        PT(5);
        if (dbg && dbg->pairs && lane == 0) dbg->pairs[a] = np;
        double st[29];
#pragma unroll
        for (int k = 0; k < 29; ++k) st[k] = 0;
        if (np > 0) {
            const uint32_t Ti = sym ? 2u * np : np;
            const double T = (double)Ti, logT = log2_int(Ti);
            const uint32_t nc = marg[320];  // non-empty cells, keys in list (any order)
            unsigned long long s2 = 0, sa = 0;
            uint32_t jm = 0;
            double el = 0;
            for (uint32_t i = lane; i < nc; i += 32) {
                const uint32_t key = list[i];
                const uint32_t c = (hist[key >> 1] >> ((key & 1u) * 16u)) & 0xffffu;
                const uint32_t ga = key >> 6, gb = key & 63u;
                const bool off = sym && ga != gb;
                const uint32_t cc = (sym && !off) ? 2u * c : c;
                const uint32_t mcc = off ? 2u * cc : cc;  // mass of the cell(s)
                s2 += (unsigned long long)mcc * cc;
                sa += (unsigned long long)((ga + 1) * (gb + 1)) * mcc;
                jm = max(jm, cc);
                el += (double)mcc * (logT - log2_int(cc));  // exactly 0 for a single cell
                sred_add(&px[ga], cc);
                if (off) sred_add(&px[gb], cc);
                if (!sym) sred_add(&py[gb], cc);
                sred_add(&psum[ga + gb], mcc);
                sred_add(&pdif[ga > gb ? ga - gb : gb - ga], mcc);
                if (dbg && dbg->glcm) {
                    dbg->glcm[((size_t)a * ng + ga) * ng + gb] = cc;
                    if (off) dbg->glcm[((size_t)a * ng + gb) * ng + ga] = cc;
                }
            }
            __syncwarp();
            for (uint32_t i = lane; i < nc; i += 32) hist[list[i] >> 1] = 0u;  // empty again
            s2 = warp_sum(s2);
            sa = warp_sum(sa);
            jm = warp_max(jm);
            el = warp_sum(el);
            __syncwarp();
            PT(7);
            haralick_finish(px, py, psum, pdif, ng, sym, T, logT, s2, sa, jm, el, st);
            PT(8);
        }
        double mine = 0;
#pragma unroll
        for (int k = 0; k < 29; ++k)
            if ((int)lane == k) mine = st[k];
        if (lane < 29) {
            og[lane * (A + 1) + a] = mine;
            sacc += mine;
        }
        __syncwarp();
    }
    if (lane < 29) og[lane * (A + 1) + A] = sacc / (double)A;
    __syncwarp();
}

// GLCM group for an S window (ng <= 256): discretize (texture.cpp:45-53, exact
// integer floor), pair keys per sorted angle (texture.cpp:58-80), radix sort,
// run-length counts, Haralick statistics from integer marginals
// (texture.cpp:87-217; hxy1 == hxy2 == hx + hy).
__device__ __noinline__ void glcm_phase_s(uint32_t n, int h, int w, const uint64_t* rowmask,
                                          const uint32_t* rowoff, const uint16_t* vals,
                                          uint8_t* lvl, uint16_t* keys, uint16_t* keys2,
                                          uint32_t* gcnt, uint32_t* marg, uint32_t vmin,
                                          uint32_t vmax, const FeatCfg& cfg, double* og,
                                          const DebugOut* dbg) {
    const unsigned lane = lane_id();
    const int ng = cfg.ng, A = cfg.n_angles;
    const uint32_t span = vmax - vmin + 1u;
    PT_DECL
    for (uint32_t i = lane; i < n; i += 32) {
        uint32_t lv = 0;
        if (vmax > vmin) lv = min((uint32_t)(ng - 1), ((uint32_t)ng * (vals[i] - vmin)) / span);
        lvl[i] = (uint8_t)lv;
    }
    __syncwarp();
    const bool sym = cfg.symmetric != 0;
    double sacc = 0;
    for (int a = 0; a < A; ++a) {
        const int ddx = cfg.dx[a], ddy = cfg.dy[a];
        // pair keys, lane-per-row: bits x with (x,y) and (x+dx,y+dy) both in the ROI
        uint64_t pm[2] = {0, 0};
        uint32_t npr = 0;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int y = lane + 32 * hf, ny = y + ddy;
            if (y < h && ny >= 0 && ny < h && ddx > -64 && ddx < 64) {
                const uint64_t r = rowmask[ny];
                const uint64_t sh = ddx >= 0 ? (r >> ddx) : (r << (-ddx));
                pm[hf] = rowmask[y] & sh;
            }
            npr += __popcll(pm[hf]);
        }
        const uint32_t incl = warp_incl_scan(npr);
        const uint32_t np = __shfl_sync(kFull, incl, 31);
        uint32_t j = incl - npr;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int y = lane + 32 * hf, ny = y + ddy;
            uint64_t m = pm[hf];
            while (m) {
                const int x = __ffsll((long long)m) - 1;
                m &= m - 1;
                const uint32_t la = lvl[rowoff[y] + __popcll(rowmask[y] & ((1ull << x) - 1ull))];
                const int nx = x + ddx;
                const uint32_t lb = lvl[rowoff[ny] + __popcll(rowmask[ny] & ((1ull << nx) - 1ull))];
                keys[j++] = (uint16_t)(sym ? min(la, lb) * (uint32_t)ng + max(la, lb)
                                           : la * (uint32_t)ng + lb);
            }
        }
        for (int k = lane; k < 1280; k += 32) marg[k] = 0;
        __syncwarp();
        PT(5);
        double st[29];
#pragma unroll
        for (int k = 0; k < 29; ++k) st[k] = 0;
        if (dbg && dbg->pairs && lane == 0) dbg->pairs[a] = np;
        if (np > 0) {
            // register bitonic network up to 1024 pairs, the radix sort above that
            const uint16_t* sk = keys;
            if (np <= 256) bitonic_sort16<8>(keys, keys, np);
            else if (np <= 512) bitonic_sort16<16>(keys, keys, np);
            else if (np <= 1024) bitonic_sort16<32>(keys, keys, np);
            else sk = radix_sort16(keys, keys2, keys, np, gcnt);
            __syncwarp();
            PT(6);
            const double T = sym ? 2.0 * (double)np : (double)np;
            const double logT = nlog2(T);
            // cells in key order: exact integer sums (ASM numerator, autocorrelation),
            // the largest cell, and the entropy terms from the log2 table of counts;
            // integer marginals by shared atomics (order-free) -- then the Haralick
            // statistics from the marginals (haralick_finish, shared with the
            // histogram path and the large-ROI kernel)
            unsigned long long s2 = 0, sa = 0;
            uint32_t jm = 0, carry = 0;
            double el = 0;
            uint32_t* px = marg;
            uint32_t* py = marg + 256;
            uint32_t* psum = marg + 512;
            uint32_t* pdif = marg + 1024;
            for (uint32_t b0 = 0; b0 < np; b0 += 32) {
                const uint32_t i = b0 + lane;
                const bool ok = i < np;
                const uint32_t k = ok ? sk[i] : 0u;
                const bool st_ = ok && (i == 0 || sk[i - 1] != k);
                const bool en_ = ok && (i + 1 == np || sk[i + 1] != k);
                const unsigned sb = __ballot_sync(kFull, st_);
                const unsigned le = lanemask_lt() | (1u << lane);
                const uint32_t s0 = (sb & le) ? b0 + 31 - __clz(sb & le) : carry;
                if (en_) {
                    const uint32_t c = i - s0 + 1;
                    const uint32_t ga = k / (uint32_t)ng, gb = k % (uint32_t)ng;
                    const bool off = sym && ga != gb;
                    const uint32_t cc = (sym && !off) ? 2u * c : c;
                    const uint32_t mcc = off ? 2u * cc : cc;
                    s2 += (unsigned long long)mcc * cc;
                    sa += (unsigned long long)((ga + 1) * (gb + 1)) * mcc;
                    jm = max(jm, cc);
                    el += (double)mcc * (logT - log2_int(cc));
                    sred_add(&px[ga], cc);
                    if (off) sred_add(&px[gb], cc);
                    if (!sym) sred_add(&py[gb], cc);
                    sred_add(&psum[ga + gb], mcc);
                    sred_add(&pdif[ga > gb ? ga - gb : gb - ga], mcc);
                    if (dbg && dbg->glcm) {
                        dbg->glcm[((size_t)a * ng + ga) * ng + gb] = cc;
                        if (off) dbg->glcm[((size_t)a * ng + gb) * ng + ga] = cc;
                    }
                }
                if (sb) carry = b0 + 31 - __clz(sb);
            }
            s2 = warp_sum(s2);
            sa = warp_sum(sa);
            jm = warp_max(jm);
            el = warp_sum(el);
            __syncwarp();
            PT(7);
            haralick_finish(px, sym ? px : py, psum, pdif, ng, sym, T, logT, s2, sa, jm, el, st);
            PT(8);
        }
        double mine = 0;
#pragma unroll
        for (int k = 0; k < 29; ++k)
            if ((int)lane == k) mine = st[k];
        if (lane < 29) {
            og[lane * (A + 1) + a] = mine;
            sacc += mine;
        }
        __syncwarp();
    }
    if (lane < 29) og[lane * (A + 1) + A] = sacc / (double)A;
    __syncwarp();
}

// ------------------------------------------------------------------------
// In-warp intensity statistics (intensity_features.cpp:42-215 without the edge
// block), the path taken when the sorted values cannot be staged for
// k_serial_stats: order statistics, moments m2..m6, mad / rmad, mode and histogram
// runs over the warp-sorted values s, written to oi[0..31].  Out of line so the
// staged main path of the S kernels is not sized by its registers.
__device__ __noinline__ void intensity_inwarp(const uint16_t* s, uint32_t n, unsigned long long sS,
                                              unsigned long long sQ, const FeatCfg& cfg,
                                              const DebugOut* dbg, double* oi) {
    const unsigned lane = lane_id();
    const double dn = (double)n;
    const uint32_t vmin = s[0], vmax = s[n - 1];
    const double mean = (double)sS / dn;
    const double mn = (double)vmin, mxv = (double)vmax, range = mxv - mn;
    const double median =
        (n & 1) ? (double)s[n / 2] : 0.5 * ((double)s[n / 2 - 1] + (double)s[n / 2]);
    // percentiles (lanes 0..5), literal expression (intensity_features.cpp:14-22)
    double myp = 0;
    if (lane < 6) {
        const double pv = lane == 0 ? 1.0 : lane == 1 ? 10.0 : lane == 2 ? 25.0
                        : lane == 3 ? 75.0 : lane == 4 ? 90.0 : 99.0;
        myp = percentile_exact(s, n, pv);
    }
    const double p10 = __shfl_sync(kFull, myp, 1), p25 = __shfl_sync(kFull, myp, 2);
    const double p75 = __shfl_sync(kFull, myp, 3), p90 = __shfl_sync(kFull, myp, 4);
    // median absolute deviation (exact: k-th of the two sorted half-sequences)
    const uint32_t M2 = (n & 1) ? 2u * s[n / 2] : (uint32_t)s[n / 2 - 1] + s[n / 2];
    const uint32_t d_hi = kth_dev2_warp(s, n, M2, n / 2);
    const uint32_t d_lo = (n & 1) ? d_hi : kth_dev2_warp(s, n, M2, n / 2 - 1);
    const double median_ad = (n & 1) ? 0.5 * (double)d_hi
                                     : 0.5 * (0.5 * (double)d_lo + 0.5 * (double)d_hi);
    // one pass over the sorted values: central moments (fp64), exact integer
    // partial sums for mad and the [p10,p90] subset, value runs (mode) and
    // histogram-bin runs (entropy = sum c (log2 n - log2 c) / n, uniformity =
    // sum c^2 / n^2; bins = floor(nb (v - min) / range), exact, A2)
    const uint32_t nb32 = (uint32_t)cfg.bins;
    const bool wide = (unsigned long long)nb32 * 65535ull >= (1ull << 32);
    const uint32_t rng = vmax - vmin;
    // floor(num / rng) by multiply-high with one correction step (num < 2^32)
    const uint32_t magic = rng ? (uint32_t)(0xffffffffull / rng) : 0u;
    auto bin_of = [&](uint32_t v) -> uint32_t {
        if (rng == 0) return 0u;
        uint32_t b;
        if (!wide) {
            const uint32_t num = nb32 * (v - vmin);
            b = __umulhi(num, magic);
            if (num - b * rng >= rng) ++b;
        } else {
            b = (uint32_t)((unsigned long long)nb32 * (v - vmin) / rng);
        }
        return b < nb32 - 1 ? b : nb32 - 1;
    };
    const double logn = nlog2(dn);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // m2..m6, entropy sum
    unsigned long long best = 0, slo = 0, rsum = 0, usq = 0;
    uint32_t clo = 0, rn = 0, carry_v = 0, carry_b = 0;
    uint32_t prev_v = 0xffffffffu, prev_b = 0xffffffffu;
#pragma unroll 1
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
        const uint32_t i = b0 + lane;
        const bool ok = i < n;
        const uint32_t v = ok ? s[i] : 0xfffffffeu;
        const uint32_t bin = ok ? bin_of(v) : 0xfffffffeu;
        const uint32_t nxt = b0 + 32 < n ? s[b0 + 32] : 0xfffffffeu;  // next chunk head
        uint32_t pv = __shfl_up_sync(kFull, v, 1), pb = __shfl_up_sync(kFull, bin, 1);
        uint32_t nv = __shfl_down_sync(kFull, v, 1), nbn = __shfl_down_sync(kFull, bin, 1);
        if (lane == 0) {
            pv = prev_v;
            pb = prev_b;
        }
        if (lane == 31) {
            nv = nxt;
            nbn = b0 + 32 < n ? bin_of(nxt) : 0xfffffffeu;
        }
        if (i + 1 == n) {
            nv = 0xfffffffdu;
            nbn = 0xfffffffdu;
        }
        const bool vstart = ok && pv != v, vend = ok && nv != v;
        const bool bstart = ok && pb != bin, bend = ok && nbn != bin;
        const unsigned vs = __ballot_sync(kFull, vstart), bs = __ballot_sync(kFull, bstart);
        const unsigned le = lanemask_lt() | (1u << lane);
        if (ok) {
            const double d = (double)v - mean;
            const double d2 = d * d;
            acc[0] += d2;
            acc[1] += d2 * d;
            acc[2] += d2 * d2;
            acc[3] += d2 * d2 * d;
            acc[4] += d2 * d2 * d2;
            if ((double)v < mean) {
                slo += v;
                ++clo;
            }
            const double x = (double)v;
            if (x >= p10 && x <= p90) {
                rsum += v;
                ++rn;
            }
            if (vend) {
                const uint32_t st = (vs & le) ? b0 + 31 - __clz(vs & le) : carry_v;
                const unsigned long long key =
                    ((unsigned long long)(i - st + 1) << 16) | (0xffffu - v);
                best = key > best ? key : best;
            }
            if (bend) {
                const uint32_t st = (bs & le) ? b0 + 31 - __clz(bs & le) : carry_b;
                const uint32_t c = i - st + 1;
                acc[5] += (double)c * (logn - log2_int(c));
                usq += (unsigned long long)c * c;
                if (dbg && bin < nb32) dbg->hist[bin] = c;
            }
        }
        if (vs) carry_v = b0 + 31 - __clz(vs);
        if (bs) carry_b = b0 + 31 - __clz(bs);
        prev_v = __shfl_sync(kFull, v, 31);
        prev_b = __shfl_sync(kFull, bin, 31);
    }
    warp_sum8(acc);
    best = warp_max(best);
    slo = warp_sum(slo);
    clo = warp_sum(clo);
    rsum = warp_sum(rsum);
    rn = warp_sum(rn);
    usq = warp_sum(usq);
    const double m2 = acc[0] / dn, m3 = acc[1] / dn, m4 = acc[2] / dn, m5 = acc[3] / dn,
                 m6 = acc[4] / dn;
    // sum |x - mean| = (S_hi - S_lo) + (c_lo - c_hi) mean, exact integer parts
    const double mad = ((double)(long long)(sS - 2 * slo) +
                        (double)((long long)clo - (long long)(n - clo)) * mean) / dn;
    const double entropy = acc[5] / dn;
    const double uniformity = (double)usq / (dn * dn);
    double rmad = 0;
    if (rn > 0) {
        const double rmean = (double)rsum / (double)rn;
        unsigned long long rlo = 0;
        uint32_t rcl = 0;
#pragma unroll 1
        for (uint32_t i = lane; i < n; i += 32) {
            const double x = (double)s[i];
            if (x >= p10 && x <= p90 && x < rmean) {
                rlo += s[i];
                ++rcl;
            }
        }
        rlo = warp_sum(rlo);
        rcl = warp_sum(rcl);
        rmad = ((double)(long long)(rsum - 2 * rlo) +
                (double)((long long)rcl - (long long)(rn - rcl)) * rmean) / (double)rn;
    }
    const double var = n > 1 ? m2 * dn / (dn - 1.0) : 0.0;
    double skew = 0, kurt = 0, hsk = 0, hfl = 0;
    if (m2 > 0) {
        const double r2 = sqrt(m2);
        skew = m3 / (m2 * r2);
        kurt = m4 / (m2 * m2);
        hsk = m5 / (m2 * m2 * r2);
        hfl = m6 / (m2 * m2 * m2);
    }
    const double mode = (double)(0xffffu - (uint32_t)(best & 0xffffu));
    const double energy = (double)sQ, sdev = sqrt(var);
    const double iqr = p75 - p25;
    // lane k writes column k (coalesced row segment); columns 32..38 by lanes 0..6
    const double pct = __shfl_sync(kFull, myp, (lane - 14) & 31);
    double o = 0;
    switch (lane) {
        case 0: o = mean; break;
        case 1: o = median; break;
        case 2: o = mode; break;
        case 3: o = mn; break;
        case 4: o = mxv; break;
        case 5: o = range; break;
        case 6: o = var; break;
        case 7: o = m2; break;
        case 8: o = sdev; break;
        case 9: o = sqrt(m2); break;
        case 10: o = mad; break;
        case 11: o = median_ad; break;
        case 12: o = rmad; break;
        case 13: o = iqr; break;
        case 14: case 15: case 16: case 17: case 18: case 19: o = pct; break;
        case 20: o = skew; break;
        case 21: o = kurt; break;
        case 22: o = m2 > 0 ? kurt - 3.0 : 0.0; break;
        case 23: o = hsk; break;
        case 24: o = hfl; break;
        case 25: o = energy; break;
        case 26: o = sqrt(energy / dn); break;
        case 27: o = entropy; break;
        case 28: o = uniformity; break;
        case 29: o = (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0; break;
        case 30: o = mean != 0 ? sdev / mean : 0.0; break;
        default: o = (double)sS; break;
    }
    oi[lane] = o;
}

// In-warp moments (moments.cpp:32-92), the path taken when the ROI's pixels cannot
// be staged for k_serial_stats: separable row sums about the integer anchors (lanes
// = rows: m0 / m1 and off0 / off1 are this lane's row masks and value offsets),
// reduce-scatter, two-stage binomial shift, eta and Hu, written to orow.  Out of
// line so the staged main path of the S kernels is not sized by its registers.
__device__ __noinline__ void moments_inwarp(uint32_t n, int h, uint64_t m0, uint64_t m1, uint32_t off0,
                                            uint32_t off1, const uint16_t* vals,
                                            unsigned long long sS, unsigned long long sXI,
                                            unsigned long long sYI, uint32_t sLX, uint32_t sLY,
                                            long long gx0, long long gy0, const FeatCfg& cfg,
                                            double* orow) {
    const unsigned lane = lane_id();
    const double dn = (double)n;
    const long long nn = (long long)n, W = (long long)sS;
    const long long axb = (2 * (long long)sLX + nn) / (2 * nn);
    const long long ayb = (2 * (long long)sLY + nn) / (2 * nn);
    const long long axw = W > 0 ? (2 * (long long)sXI + W) / (2 * W) : 0;
    const long long ayw = W > 0 ? (2 * (long long)sYI + W) / (2 * W) : 0;
    // two passes (unit mass, then intensity) of 16 separable row accumulators
    // about the integer anchor: A_pq = sum_rows (sum_x w dx^p) dy^q
    const int nhalf = h > 32 ? 2 : 1;
    double Nb = 0, Nw = 0;
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
        const long long ax = g ? axw : axb, ay = g ? ayw : ayb;
        double acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0;
#pragma unroll 1
        for (int hf = 0; hf < nhalf; ++hf) {
            const int y = lane + 32 * hf;
            uint64_t m = hf ? m1 : m0;
            uint32_t idx = hf ? off1 : off0;
            double r0 = 0, r1 = 0, r2 = 0, r3 = 0;
            if (g == 0) {
                r0 = (double)__popcll(m);
                while (m) {
                    const double d = (double)((long long)(__ffsll((long long)m) - 1) - ax);
                    m &= m - 1;
                    const double d2 = d * d;
                    r1 += d;
                    r2 += d2;
                    r3 += d2 * d;
                }
            } else {
                while (m) {
                    const double d = (double)((long long)(__ffsll((long long)m) - 1) - ax);
                    m &= m - 1;
                    const double wv = (double)vals[idx++];
                    const double wd = wv * d, wd2 = wd * d;
                    r0 += wv;
                    r1 += wd;
                    r2 += wd2;
                    r3 += wd2 * d;
                }
            }
            const double yy = (double)((long long)y - ay);
            const double q2 = yy * yy;
            const double rr[4] = {r0, r1, r2, r3}, qq[4] = {1.0, yy, q2, q2 * yy};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a * 4 + b] += rr[a] * qq[b];
        }
        // reduce-scatter: after 4 halving steps lane L holds index L >> 1
#pragma unroll
        for (int st = 16, half = 8; st >= 2; st >>= 1, half >>= 1) {
            const bool up = (lane & st) != 0;
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double send = up ? acc[j] : acc[j + half];
                const double recv = __shfl_xor_sync(kFull, send, st);
                acc[j] = (up ? acc[j + half] : acc[j]) + recv;
            }
        }
        double t = acc[0] + __shfl_xor_sync(kFull, acc[0], 1);
        t = __shfl_sync(kFull, t, 2 * (lane & 15));  // lane L: index L & 15
        if (g == 0) Nb = t;
        else Nw = t;
    }
    const double N = (lane >> 4) ? Nw : Nb;
    const int grp = lane >> 4, p = (lane >> 2) & 3, q = lane & 3;
    const double m00 = grp ? (double)sS : dn;
    const bool zero_mass = grp && sS == 0;
    const double dx = grp ? (W > 0 ? (double)((long long)sXI - axw * W) / (double)W : 0.0)
                          : (double)((long long)sLX - axb * nn) / dn;
    const double dy = grp ? (W > 0 ? (double)((long long)sYI - ayw * W) / (double)W : 0.0)
                          : (double)((long long)sLY - ayb * nn) / dn;
    const double Ax = (double)(gx0 + (grp ? axw : axb)), Ay = (double)(gy0 + (grp ? ayw : ayb));
    // separable binomial shift in two shuffle stages (no lane-indexed arrays):
    //   T_pq = sum_j C(q,j) t^(q-j) N_pj,  mu_pq = sum_i C(p,i) s^(p-i) T_iq
    auto coef = [](int e, int k, double t) -> double {  // C(e,k) t^(e-k), 0 if k > e
        if (k > e) return 0.0;
        const int d = e - k;
        const double c = (k == 0 || k == e) ? 1.0 : (e == 3 ? 3.0 : 2.0);
        const double t2 = t * t;
        return c * (d == 0 ? 1.0 : d == 1 ? t : d == 2 ? t2 : t2 * t);
    };
    double Tm = 0, Tr = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double Npj = __shfl_sync(kFull, N, (grp << 4) | (p << 2) | j);
        Tm += coef(q, j, -dy) * Npj;
        Tr += coef(q, j, Ay) * Npj;
    }
    double mu = 0, raw = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int src = (grp << 4) | (i << 2) | q;
        mu += coef(p, i, -dx) * __shfl_sync(kFull, Tm, src);
        raw += coef(p, i, Ax) * __shfl_sync(kFull, Tr, src);
    }
    if ((p == 1 && q == 0) || (p == 0 && q == 1)) mu = 0.0;
    if (p == 0 && q == 0) mu = N;
    // eta = mu / m00^(1 + (p+q)/2)  (moments.cpp:84-89), powers built from m00 and sqrt(m00)
    double eta = 0;
    if (p + q >= 2) {
        const int t = p + q;  // exponent 1 + t/2 in {2, 2.5, 3, 3.5, 4}
        double den = m00 * m00;
        if (t >= 4) den *= m00;
        if (t >= 6) den *= m00;
        if (t & 1) den *= sqrt(m00);
        eta = mu / den;
    }
    if (zero_mass) raw = mu = eta = 0;
    const double n20 = __shfl_sync(kFull, eta, (grp << 4) | 8);
    const double n02 = __shfl_sync(kFull, eta, (grp << 4) | 2);
    const double n11 = __shfl_sync(kFull, eta, (grp << 4) | 5);
    const double n30 = __shfl_sync(kFull, eta, (grp << 4) | 12);
    const double n03 = __shfl_sync(kFull, eta, (grp << 4) | 3);
    const double n21 = __shfl_sync(kFull, eta, (grp << 4) | 9);
    const double n12 = __shfl_sync(kFull, eta, (grp << 4) | 6);
    double* o = orow + cfg.col_mom + grp * 52;
    const int li = lane & 15;
    o[li] = raw;
    o[16 + li] = mu;
    if (p + q >= 2) o[32 + ((p == 0) ? q - 2 : (p == 1 ? 1 + q : 1 + 4 * (p - 1) + q))] = eta;
    // Hu invariants: lanes li = 0..6 of each group compute one each
    if (li < 7) {
        const double a = n30 + n12, b = n21 + n03;
        double hu;
        switch (li) {
            case 0: hu = n20 + n02; break;
            case 1: hu = (n20 - n02) * (n20 - n02) + 4.0 * n11 * n11; break;
            case 2: hu = (n30 - 3.0 * n12) * (n30 - 3.0 * n12) + (3.0 * n21 - n03) * (3.0 * n21 - n03); break;
            case 3: hu = a * a + b * b; break;
            case 4:
                hu = (n30 - 3.0 * n12) * a * (a * a - 3.0 * b * b) +
                     (3.0 * n21 - n03) * b * (3.0 * a * a - b * b);
                break;
            case 5: hu = (n20 - n02) * (a * a - b * b) + 4.0 * n11 * a * b; break;
            default:
                hu = (3.0 * n21 - n03) * a * (a * a - 3.0 * b * b) -
                     (n30 - 3.0 * n12) * b * (3.0 * a * a - b * b);
                break;
        }
        o[45 + li] = zero_mass ? 0.0 : hu;
    }
    __syncwarp();
}

template <int TW, int TH, int NMAX, int RUNMAX, int GLCM>
__device__ __forceinline__ void process_s(const SJob& J, const SLayout& L, uint8_t* base,
                                          const DevImage& img, const FeatCfg& cfg,
                                          double* __restrict__ out, uint64_t* mbar,
                                          uint32_t& phase, Control* ctl, RoiList rl,
                                          const DebugOut* dbg) {
    const unsigned lane = lane_id();
    const int w = (int)J.w, h = (int)J.h;
    const uint32_t label = J.label;
    uint64_t* rowmask = (uint64_t*)(base + L.rowmask);
    uint32_t* rowoff = (uint32_t*)(base + L.rowoff);
    uint16_t* vals = (uint16_t*)(base + L.vals);
    uint16_t* xy = (uint16_t*)(base + L.xy);
    const uint16_t* stage = (const uint16_t*)(base + L.stage);
    double* orow = out + (size_t)J.row * cfg.ncols;
    const bool dbg_on = dbg != nullptr && dbg->label == label;
    const long long gx0 = rl.gx[J.row], gy0 = rl.gy[J.row];
    const uint32_t xo = J.x0 & 7u;
    const uint64_t wm = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);

    // ---------------------------------------------------------------- load
    PT_DECL
    mbar_wait(mbar, phase);
    phase ^= 1u;
#ifdef FXG_PT_MBAR
    PT(4);  // phase-timing probe: the TMA wait alone (slot 4 is idle without GLCM)
#endif
    // row masks: lane y reads its staged row 8 labels at a time (16 B LDS)
    uint64_t m0 = 0, m1 = 0;  // rows lane, lane + 32
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        const int y = lane + 32 * half;
        uint64_t m = 0;
        if (y < h) {
            const uint4* row = reinterpret_cast<const uint4*>(stage + y * TW);
            const int c_end = (int)((xo + w + 7) >> 3);
#pragma unroll 1
            for (int c = 0; c < c_end; ++c) {
                const uint4 q = row[c];
                // 8 label compares per 16 B: XOR with the label in both halves, a SWAR
                // nonzero test per halfword (bit 15 of each half), the halves' high
                // bytes gathered by PRMT, then a multiply packs bit 7 of 4 bytes into
                // a nibble (movemask)
                const uint32_t LL = label | (label << 16);
                auto nz = [&](uint32_t w) {
                    const uint32_t x = w ^ LL;
                    return ((x & 0x7fff7fffu) + 0x7fff7fffu) | x;  // bit 15 / 31: half != label
                };
                const uint32_t lo = ~__byte_perm(nz(q.x), nz(q.y), 0x7531) & 0x80808080u;
                const uint32_t hi = ~__byte_perm(nz(q.z), nz(q.w), 0x7531) & 0x80808080u;
                const uint32_t bits = ((lo * 0x00204081u) >> 28) | (((hi * 0x00204081u) >> 28) << 4);
                const int sh = c * 8 - (int)xo;  // pixel index of this chunk's bit 0
                m |= sh >= 0 ? ((uint64_t)bits << sh) : ((uint64_t)bits >> (-sh));
            }
            m &= wm;
        }
        if (half == 0) m0 = m;
        else m1 = m;
    }
    // row offsets (warp scan, row order)
    const uint32_t c0 = __popcll(m0), c1 = __popcll(m1);
    const uint32_t i0 = warp_incl_scan(c0);
    const uint32_t tot0 = __shfl_sync(kFull, i0, 31);
    const uint32_t i1 = warp_incl_scan(c1);
    const uint32_t n = tot0 + __shfl_sync(kFull, i1, 31);
    const uint32_t off0 = i0 - c0, off1 = tot0 + i1 - c1;
    if ((int)lane < h) {
        rowmask[lane] = m0;
        rowoff[lane] = off0;
    }
    if ((int)lane + 32 < h) {
        rowmask[lane + 32] = m1;
        rowoff[lane + 32] = off1;
    }
    if (lane == 0) rowoff[h] = n;
    // pixel coordinates in row-major order
    {
        uint64_t m = m0;
        uint32_t j = off0;
        while (m) {
            xy[j++] = (uint16_t)((__ffsll((long long)m) - 1) | (lane << 8));
            m &= m - 1;
        }
        m = m1;
        j = off1;
        while (m) {
            xy[j++] = (uint16_t)((__ffsll((long long)m) - 1) | ((lane + 32) << 8));
            m &= m - 1;
        }
    }
    __syncwarp();
    // gather member intensities (coalesced within rows), exact integer sums
    unsigned long long sS = 0, sQ = 0, sXI = 0, sYI = 0;
    uint32_t sLX = 0, sLY = 0, gmin = 0xffffu, gmax = 0u;
    // moments by k_moments_serial: stage this ROI's pixels when the buffer has room
    uint32_t* mst = nullptr;
    if (cfg.col_mom >= 0 && cfg.mom_px) {
        unsigned long long off = 0;
        if (lane == 0) off = atomicAdd(&ctl->mom_alloc, (unsigned long long)((n + 3u) & ~3u));
        off = __shfl_sync(kFull, off, 0);
        const bool fits = off + n <= cfg.mom_cap;
        if (lane == 0) cfg.mom_off[J.row] = fits ? off : ~0ull;
        if (fits) mst = cfg.mom_px + off;
    }
    {
        constexpr bool kSI = TW == kStageW0;  // S0: staged intensity tile, else global gather
        const uint16_t* Is = (const uint16_t*)(base + L.stageI) + xo;
        const uint16_t* Ib = img.I + (size_t)J.y0 * img.pitch + J.x0;
#pragma unroll 1
        for (uint32_t b0 = 0; b0 < n; b0 += 32 * 8) {
            uint16_t v[8];
            uint32_t p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = b0 + u * 32 + lane;
                p[u] = i < n ? xy[i] : 0u;
                if (kSI) v[u] = i < n ? Is[(p[u] >> 8) * (uint32_t)TW + (p[u] & 0xffu)] : 0;
                else v[u] = i < n ? __ldg(Ib + (size_t)(p[u] >> 8) * img.pitch + (p[u] & 0xffu)) : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = b0 + u * 32 + lane;
                if (i < n) {
                    vals[i] = v[u];
                    if (mst) mst[i] = p[u] | ((uint32_t)v[u] << 16);
                    const uint32_t x = p[u] & 0xffu, y = p[u] >> 8;
                    sS += v[u];
                    sQ += (unsigned long long)((uint32_t)v[u] * (uint32_t)v[u]);
                    sXI += (unsigned long long)((uint32_t)v[u] * x);
                    sYI += (unsigned long long)((uint32_t)v[u] * y);
                    sLX += x;
                    sLY += y;
                    gmin = min(gmin, (uint32_t)v[u]);
                    gmax = max(gmax, (uint32_t)v[u]);
                }
            }
        }
        gmin = warp_min(gmin);
        gmax = warp_max(gmax);
        sS = warp_sum(sS);
        sQ = warp_sum(sQ);
        sXI = warp_sum(sXI);
        sYI = warp_sum(sYI);
        sLX = warp_sum(sLX);
        sLY = warp_sum(sLY);
        if (mst && lane < 5) {
            const unsigned long long v5 = lane == 0 ? sS : lane == 1 ? sXI : lane == 2 ? sYI
                                        : lane == 3 ? (unsigned long long)sLX : (unsigned long long)sLY;
            cfg.mom_sums[(size_t)J.row * 5 + lane] = v5;
        }
    }
    __syncwarp();
    uint32_t vmin = gmin, vmax = gmax;  // value range (the gather computed it)
    bool have_minmax = true;

    // K (largest 8-connected component, row-major tie-break) and E (4-connected
    // exterior of the window cells outside K) as row masks (lanes = rows); false:
    // run capacity exceeded, the ROI was re-queued to the large-ROI kernel
    auto edge_ke = [&](uint64_t& k0, uint64_t& k1, uint64_t& e0, uint64_t& e1) -> bool {
        uint64_t* km = (uint64_t*)(base + L.kmask);
        uint64_t* em = (uint64_t*)(base + L.emask);
        bool fast = w <= 62;
        k0 = m0;
        k1 = m1;
        e0 = e1 = 0;
        if (fast) {
            // 4-connected exterior flood of the free cells, seeded on the border
            const uint64_t f0 = ((int)lane < h) ? (~m0 & wm) : 0ull;
            const uint64_t f1 = ((int)lane + 32 < h) ? (~m1 & wm) : 0ull;
            const uint64_t side = 1ull | (1ull << (w - 1));
            if (w <= 32) {
                // 32-bit rows: the same flood with 32-bit fills and shuffles
                const uint32_t g0 = (uint32_t)f0, g1 = (uint32_t)f1, sd = (uint32_t)side;
                uint32_t x0 = run_fill32(g0, (lane == 0 || (int)lane == h - 1) ? g0 : (g0 & sd));
                uint32_t x1 = run_fill32(g1, ((int)lane + 32 == h - 1) ? g1 : (g1 & sd));
                for (int it = 0; it < 64 * TH; ++it) {
                    const uint32_t up0 = __shfl_up_sync(kFull, x0, 1), dn0 = __shfl_down_sync(kFull, x0, 1);
                    const uint32_t up1 = __shfl_up_sync(kFull, x1, 1), dn1 = __shfl_down_sync(kFull, x1, 1);
                    const uint32_t l31 = __shfl_sync(kFull, x0, 31), f32 = __shfl_sync(kFull, x1, 0);
                    const uint32_t a0 = (lane == 0 ? 0u : up0) | (lane == 31 ? f32 : dn0);
                    const uint32_t a1 = (lane == 0 ? l31 : up1) | (lane == 31 ? 0u : dn1);
                    const uint32_t n0 = run_fill32(g0, x0 | (a0 & g0));
                    const uint32_t n1 = run_fill32(g1, x1 | (a1 & g1));
                    const bool ch = (n0 != x0) || (n1 != x1);
                    x0 = n0;
                    x1 = n1;
                    if (!__any_sync(kFull, ch)) break;
                }
                e0 = x0;
                e1 = x1;
            } else {
            e0 = run_fill(f0, (lane == 0 || (int)lane == h - 1) ? f0 : (f0 & side));
            e1 = run_fill(f1, ((int)lane + 32 == h - 1) ? f1 : (f1 & side));
            for (int it = 0; it < 64 * TH; ++it) {
                const uint64_t up0 = __shfl_up_sync(kFull, e0, 1);
                const uint64_t dn0 = __shfl_down_sync(kFull, e0, 1);
                const uint64_t up1 = __shfl_up_sync(kFull, e1, 1);
                const uint64_t dn1 = __shfl_down_sync(kFull, e1, 1);
                const uint64_t l31 = __shfl_sync(kFull, e0, 31), f32 = __shfl_sync(kFull, e1, 0);
                const uint64_t a0 = (lane == 0 ? 0ull : up0) | (lane == 31 ? f32 : dn0);
                const uint64_t a1 = (lane == 0 ? l31 : up1) | (lane == 31 ? 0ull : dn1);
                const uint64_t n0 = run_fill(f0, e0 | (a0 & f0));
                const uint64_t n1 = run_fill(f1, e1 | (a1 & f1));
                const bool ch = (n0 != e0) || (n1 != e1);
                e0 = n0;
                e1 = n1;
                if (!__any_sync(kFull, ch)) break;
            }
            }
            // holes: free cells not reached
            const bool hole = ((f0 & ~e0) | (f1 & ~e1)) != 0ull;
            // 8-connected Euler number of the padded window (bit quads)
            int q = 0;
            {
                const uint64_t vm = (w >= 63) ? ~0ull : ((2ull << w) - 1ull);  // quads 0..w
                auto quads = [&](uint64_t a, uint64_t b) {
                    const uint64_t A0 = a << 1, A1 = a, B0 = b << 1, B1 = b;  // padded
                    const uint64_t s1 = A0 ^ A1, s2 = B0 ^ B1, c = (A0 & A1) | (B0 & B1);
                    const uint64_t one = (s1 ^ s2) & ~c & vm, three = (s1 ^ s2) & c & vm;
                    const uint64_t dg = ((A0 & B1 & ~A1 & ~B0) | (A1 & B0 & ~A0 & ~B1)) & vm;
                    return __popcll(one) - __popcll(three) - 2 * __popcll(dg);
                };
                const uint64_t pm0 = __shfl_up_sync(kFull, m0, 1), pm1 = __shfl_up_sync(kFull, m1, 1);
                const uint64_t l31 = __shfl_sync(kFull, m0, 31);
                // row pairs (y-1, y) for y = 0..h  (rows -1 and h are empty)
                if ((int)lane <= h) q += quads(lane == 0 ? 0ull : pm0, (int)lane < h ? m0 : 0ull);
                if ((int)lane + 32 <= h)
                    q += quads(lane == 0 ? l31 : pm1, (int)lane + 32 < h ? m1 : 0ull);
                // a 64-row window's bottom pair (row 63, empty row 64) has no lane of its
                // own: without it a ROI on the last row counted as one fewer component
                if (h == 64 && lane == 31) q += quads(m1, 0ull);
                q = warp_sum(q);
            }
            fast = !__any_sync(kFull, hole) && q == 4;  // one component, no holes
        }
        if (!fast) {
            if ((int)lane < h) km[lane] = m0;
            if ((int)lane + 32 < h) km[lane + 32] = m1;
            __syncwarp();
            const bool ok = edge_sets_slow(rowmask, h, w, km, em, (uint32_t*)(base + L.runoff),
                                           (uint16_t*)(base + L.rs), (uint16_t*)(base + L.re),
                                           (uint32_t*)(base + L.parent),
                                           (uint32_t*)(base + L.rsize), (uint32_t)RUNMAX);
            if (!ok) {  // run capacity: re-queue this ROI to the general path
                if (lane == 0) {
                    const uint32_t pos = atomicAdd(&ctl->overflow_count, 1u);
                    rl.overflow[pos] = J.row;
                }
                __syncwarp();
                return false;
            }
            k0 = (int)lane < h ? km[lane] : 0ull;
            k1 = (int)lane + 32 < h ? km[lane + 32] : 0ull;
            e0 = (int)lane < h ? em[lane] : 0ull;
            e1 = (int)lane + 32 < h ? em[lane + 32] : 0ull;
            __syncwarp();
        }
        return true;
    };
    uint64_t ks0 = 0, ks1 = 0, e_unused0 = 0, e_unused1 = 0;  // K rows kept for the shape group
    bool have_k = false;

    // ----------------------------------------------------------- intensity
    PT(0);
    if (cfg.col_int >= 0) {
#ifdef FXG_SORT_RADIX
        const uint16_t* s = radix_sort16(vals, (uint16_t*)(base + L.tmp),
                                         (uint16_t*)(base + L.sorted), n,
                                         (uint32_t*)(base + L.cnt));
#else
        // (a register bitonic network here measured slower on C2, 0.320 -> 0.348 ms:
        // its unrolled code pushed the other phases out of the instruction cache)
        const uint16_t* s = bucket_sort16(vals, (uint16_t*)(base + L.tmp),
                                          (uint16_t*)(base + L.sorted), n,
                                          (uint32_t*)(base + L.cnt), gmin, gmax);
#endif
        __syncwarp();
        PT(1);
        // order statistics and moments of the values by k_intensity_serial when the
        // sorted values can be staged (the warp keeps the edge set and edge stats)
        bool staged = false;
        if (cfg.int_vals) {
            unsigned long long off = 0;
            if (lane == 0) off = atomicAdd(&ctl->int_alloc, (unsigned long long)((n + 7u) & ~7u));
            off = __shfl_sync(kFull, off, 0);
            staged = off + n <= cfg.int_cap;
            if (lane == 0) cfg.int_off[J.row] = staged ? off : ~0ull;
            if (staged) {
                uint16_t* dst = cfg.int_vals + off;
                for (uint32_t i = lane; i < n; i += 32) dst[i] = s[i];
                if (lane < 2) cfg.int_sums[(size_t)J.row * 2 + lane] = lane ? sQ : sS;
            }
            __syncwarp();
        }
        // ------------------------------------------------ edge set
        double e_mean = 0, e_min = 0, e_max = 0, e_std = 0, e_int = 0;
        auto edge_stats = [&]() -> bool {
            {
                uint64_t k0, k1, e0, e1;
                if (!edge_ke(k0, k1, e0, e1)) return false;
                ks0 = k0;
                ks1 = k1;
                have_k = true;
                // edge = K & (4-neighbour in E, or on the window border)
                const uint64_t eu0 = __shfl_up_sync(kFull, e0, 1), ed0 = __shfl_down_sync(kFull, e0, 1);
                const uint64_t eu1 = __shfl_up_sync(kFull, e1, 1), ed1 = __shfl_down_sync(kFull, e1, 1);
                const uint64_t el31 = __shfl_sync(kFull, e0, 31), ef32 = __shfl_sync(kFull, e1, 0);
                const uint64_t side = 1ull | (1ull << (w - 1));
                uint64_t g0 = (e0 << 1) | (e0 >> 1) | (lane == 0 ? 0ull : eu0) | (lane == 31 ? ef32 : ed0) | side;
                uint64_t g1 = (e1 << 1) | (e1 >> 1) | (lane == 0 ? el31 : eu1) | (lane == 31 ? 0ull : ed1) | side;
                if (lane == 0 || (int)lane == h - 1) g0 = ~0ull;
                if ((int)lane + 32 == h - 1) g1 = ~0ull;
                const uint64_t ed[2] = {(int)lane < h ? (k0 & g0) : 0ull, (int)lane + 32 < h ? (k1 & g1) : 0ull};
                const uint64_t rm[2] = {m0, m1};
                const uint32_t ro[2] = {off0, off1};
                // one pass: exact integer sum and sum of squares -> mean, population std
                unsigned long long es = 0, esq = 0;
                uint32_t en = 0, emn = 0xffffffffu, emx = 0;
    #pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint64_t e = ed[hf];
                    while (e) {
                        const int b = __ffsll((long long)e) - 1;
                        e &= e - 1;
                        const uint32_t v = vals[ro[hf] + __popcll(rm[hf] & ((1ull << b) - 1ull))];
                        es += v;
                        esq += (unsigned long long)(v * v);
                        ++en;
                        emn = min(emn, v);
                        emx = max(emx, v);
                    }
                }
                es = warp_sum(es);
                esq = warp_sum(esq);
                en = warp_sum(en);
                emn = warp_min(emn);
                emx = warp_max(emx);
                if (en) {
                    const double den = (double)en;
                    e_mean = (double)es / den;
                    e_min = (double)emn;
                    e_max = (double)emx;
                    e_int = (double)es;
                    // n^2 var = n sum v^2 - (sum v)^2, exact in u64 (< 2^56 for S windows)
                    e_std = sqrt((double)(en * esq - es * es) / (den * den));
                }
                if (dbg_on) {
                    uint32_t cnt_e = __popcll(ed[0]) + __popcll(ed[1]);
                    const uint32_t incl = warp_incl_scan(cnt_e);
                    uint32_t j = incl - cnt_e;
    #pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        uint64_t e = ed[hf];
                        while (e) {
                            const int b = __ffsll((long long)e) - 1;
                            e &= e - 1;
                            if (j < dbg->cap_edge) {
                                dbg->edge_xy[2 * j] = (int32_t)(gx0 + b);
                                dbg->edge_xy[2 * j + 1] = (int32_t)(gy0 + lane + 32 * hf);
                            }
                            ++j;
                        }
                    }
                    if (lane == 31) *dbg->n_edge = j;
                }
            }
            return true;
        };
        // unstaged: the statistics read the sorted values before the edge slow path
        // reuses their region of the slab
        if (!staged) intensity_inwarp(s, n, sS, sQ, cfg, dbg_on ? dbg : nullptr, orow + cfg.col_int);
        PT(2);
        if (!edge_stats()) return;
        double wcx = 0, wcy = 0;
        if (sS > 0) {
            wcx = (double)((unsigned long long)gx0 * sS + sXI) / (double)sS;
            wcy = (double)((unsigned long long)gy0 * sS + sYI) / (double)sS;
        }
        if (lane < 7) {
            const double t[7] = {e_mean, e_min, e_max, e_std, e_int, wcx, wcy};
            double v = t[0];
#pragma unroll
            for (int k = 1; k < 7; ++k)
                if ((int)lane == k) v = t[k];
            orow[cfg.col_int + 32 + lane] = v;
        }
        __syncwarp();
    }

    // ---------------------------------------------------------------- shape
    PT(3);
    if (cfg.col_shape >= 0) {
        if (!have_k && !edge_ke(ks0, ks1, e_unused0, e_unused1)) return;
        uint64_t* km = (uint64_t*)(base + L.kmask);
        if ((int)lane < h) km[lane] = ks0;
        if ((int)lane + 32 < h) km[lane + 32] = ks1;
        __syncwarp();
        shape_phase_s(rowmask, km, h, w, n, gx0, gy0, sLX, sLY, J.row, cfg, orow + cfg.col_shape);
    }
    // ------------------------------------------------------------- moments
    PT(6);
    if (cfg.col_mom >= 0 && !mst)  // staged ROIs: k_serial_stats
        moments_inwarp(n, h, m0, m1, off0, off1, vals, sS, sXI, sYI, sLX, sLY, gx0, gy0, cfg, orow);

    // ---------------------------------------------------------------- glcm
    PT(4);
    if (GLCM && cfg.col_glcm >= 0) {
        if (!have_minmax) {
            uint32_t lo = 0xffffu, hi = 0;
            for (uint32_t i = lane; i < n; i += 32) {
                lo = min(lo, (uint32_t)vals[i]);
                hi = max(hi, (uint32_t)vals[i]);
            }
            vmin = warp_min(lo);
            vmax = warp_max(hi);
        }
        if constexpr (GLCM == kGlHist)
            glcm_phase_h(n, h, rowmask, xy, vals, base + L.lmap, (uint32_t*)(base + L.hist),
                         (uint32_t*)(base + L.marg), (uint16_t*)(base + L.list), vmin, vmax, cfg,
                         orow + cfg.col_glcm,
                         dbg_on ? dbg : nullptr);
        else
            glcm_phase_s(n, h, w, rowmask, rowoff, vals, (uint8_t*)(base + L.lvl),
                         (uint16_t*)(base + L.keys), (uint16_t*)(base + L.keys2),
                         (uint32_t*)(base + L.gcnt), (uint32_t*)(base + L.marg), vmin, vmax, cfg,
                         orow + cfg.col_glcm, dbg_on ? dbg : nullptr);
    }
    __syncwarp();
}

}  // namespace
}  // namespace fxg

namespace fxg {
namespace {

#ifndef FXG_S_PREFETCH
#define FXG_S_PREFETCH 0  // 1: L2 prefetch of the next window (measured slower on C2)
#endif
template <int CLS, int GLCM>
__global__ void __launch_bounds__(32, GLCM ? SVar<CLS>::MINB_G : SVar<CLS>::MINB)
    k_roi_s(const __grid_constant__ CUtensorMap tmapL, const __grid_constant__ CUtensorMap tmapI,
            int use_tma, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg, double* out,
            const DebugOut* dbg) {
    using V = SVar<CLS>;
    constexpr SLayout L = slayout<CLS, GLCM>();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    // 128 B aligned slab base by pointer arithmetic on the shared array, so the
    // inlined phases keep the shared address space (LDS / STS / ATOMS); an
    // integer round trip through uintptr_t made every access generic
    uint8_t* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(base + L.bytes - 128);
    uint16_t* stage = (uint16_t*)(base + L.stage);
    uint16_t* stageI = (uint16_t*)(base + L.stageI);
    const unsigned lane = lane_id();
    if (lane == 0) mbar_init(mbar);
    __syncwarp();
    uint32_t phase = 0;
    const uint32_t count = ctl->class_count[CLS];
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(&ctl->class_next[CLS], 1u);
    idx = __shfl_sync(kFull, idx, 0);
    for (;;) {
        if (idx >= count) break;
#if FXG_S_PREFETCH
        // claim the next ROI now and pull its window rows (labels for the TMA
        // tile, intensities for the gather) into L2 while this one is processed
        uint32_t nidx = 0;
        if (lane == 0) nidx = atomicAdd(&ctl->class_next[CLS], 1u);
        nidx = __shfl_sync(kFull, nidx, 0);
        if (nidx < count) {
            const uint32_t r2 = rl.cls_list[CLS][nidx];
            const uint32_t py = lane;
            if (py < rl.h[r2]) {
                const size_t o = (size_t)(rl.y0[r2] + py) * img.pitch + rl.x0[r2];
                const size_t e = o + rl.w[r2] - 1;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(img.L + o));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(img.I + o));
                if ((o >> 6) != (e >> 6)) {  // the row crosses a 128 B line
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(img.L + e));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(img.I + e));
                }
            }
        }
#else
        const uint32_t nidx = [&] {
            uint32_t v = 0;
            if (lane == 0) v = atomicAdd(&ctl->class_next[CLS], 1u);
            return __shfl_sync(kFull, v, 0);
        }();
#endif
        const uint32_t r = rl.cls_list[CLS][idx];
        const SJob J{rl.label[r], rl.x0[r], rl.y0[r], rl.w[r], rl.h[r], r};
        if (use_tma) {
            // label window -> staging tile: TWx8 boxes from x0 & ~7 (16 B aligned
            // innermost coordinate, required on sm_100a)
            // label (and for S0 intensity) windows -> staging tiles, one transaction
            constexpr bool kSI = V::TW == kStageW0;
            const int nbox = ((int)J.h + 7) >> 3;
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(mbar, (kSI ? 2u : 1u) * (uint32_t)nbox * (uint32_t)(V::TW * 8 * 2));
                for (int b = 0; b < nbox; ++b) {
                    tma_load_2d(stage + b * 8 * V::TW, &tmapL, mbar, (int)(J.x0 & ~7u),
                                (int)J.y0 + b * 8);
                    if (kSI)
                        tma_load_2d(stageI + b * 8 * V::TW, &tmapI, mbar, (int)(J.x0 & ~7u),
                                    (int)J.y0 + b * 8);
                }
            }
            __syncwarp();
        } else {
            // plain coalesced loads of the window rows into the staging tiles
            const uint32_t xo = J.x0 & 7u;
            for (int y = 0; y < (int)J.h; ++y)
                for (int x = lane; x < (int)J.w; x += 32) {
                    const size_t o = (size_t)(J.y0 + y) * img.pitch + J.x0 + x;
                    stage[y * V::TW + xo + x] = img.L[o];
                    if (V::TW == kStageW0) stageI[y * V::TW + xo + x] = img.I[o];
                }
            __syncwarp();
            if (lane == 0)  // complete the phase the TMA path would complete
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
        }
        process_s<V::TW, V::TH, V::NMAX, V::RUNMAX, GLCM>(J, L, base, img, cfg, out, mbar, phase,
                                                         ctl, rl, dbg);
        idx = nidx;
    }
}

template <int CLS, int G>
cudaError_t setup_one(int* occ) {
    constexpr uint32_t bytes = slayout<CLS, G>().bytes + kSlack;
    cudaError_t e = cudaFuncSetAttribute(k_roi_s<CLS, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_roi_s<CLS, G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_roi_s<CLS, G>, 32, bytes);
}

template <int CLS, int G>
void launch_one(int grid, cudaStream_t s, const CUtensorMap& tm, const CUtensorMap& ti, int use_tma,
                DevImage img, RoiList rl, Control* ctl, FeatCfg cfg, double* out, const DebugOut* dbg) {
    k_roi_s<CLS, G><<<grid, 32, slayout<CLS, G>().bytes + kSlack, s>>>(tm, ti, use_tma, img, rl, ctl,
                                                                      cfg, out, dbg);
}

}  // namespace

cudaError_t roi_s_setup(int* occ) {
    k_init_log2_tab<<<4, 256>>>();
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = setup_one<kClassS0, kGlNone>(&occ[0]);
    if (e == cudaSuccess) e = setup_one<kClassS0, kGlSort>(&occ[1]);
    if (e == cudaSuccess) e = setup_one<kClassS0, kGlHist>(&occ[2]);
    if (e == cudaSuccess) e = setup_one<kClassS1, kGlNone>(&occ[3]);
    if (e == cudaSuccess) e = setup_one<kClassS1, kGlSort>(&occ[4]);
    if (e == cudaSuccess) e = setup_one<kClassS1, kGlHist>(&occ[5]);
    if (e == cudaSuccess) e = setup_one<kClassS2, kGlNone>(&occ[6]);
    if (e == cudaSuccess) e = setup_one<kClassS2, kGlSort>(&occ[7]);
    if (e == cudaSuccess) e = setup_one<kClassS2, kGlHist>(&occ[8]);
    return e;
}

// Moments of the staged S ROIs (moments.cpp:32-92), one thread per ROI and group
// (grp 0 binary, 1 intensity-weighted): sums of w dx^p dy^q about the integer
// anchors (pixels in row-major order), then the binomial shifts to the centroid
// and the origin, eta and Hu; the same formulas as the warp path, scalar and
// amortised over 32 ROIs per warp.  Binary sums are exact integers (|dx^p dy^q|
// < 2^32, IMAD.WIDE into int64 on the integer pipe); weighted sums are fp64.
// output row of the t-th S-class ROI (S0, then S1, then S2), ~0 past the end
__device__ __forceinline__ uint32_t s_row_of(uint32_t t, const RoiList& rl, const Control* ctl) {
    const uint32_t n0 = ctl->class_count[kClassS0], n1 = ctl->class_count[kClassS1];
    const uint32_t nt = n0 + n1 + ctl->class_count[kClassS2];
    if (t >= nt) return ~0u;
    return t < n0 ? rl.cls_list[kClassS0][t]
         : t < n0 + n1 ? rl.cls_list[kClassS1][t - n0] : rl.cls_list[kClassS2][t - n0 - n1];
}

// Moments epilogue of one ROI and group from its 16 sums N[p*4+q] of w dx^p dy^q
// about the integer anchor (ax, ay): binomial shifts to the image origin (raw) and
// to the centroid (central), eta, Hu (moments.cpp:32-92); writes the 52 columns at o.
__device__ __forceinline__ void moments_epilogue_serial(const double (&N)[16], int grp, uint32_t n,
                                                     long long W, long long SX, long long SY,
                                                     long long ax, long long ay, long long gx0,
                                                     long long gy0, double* o) {
    const long long nn = (long long)n;
    const bool zero_mass = grp && W == 0;
    const double m00 = grp ? (double)W : (double)n;
    const double dx = grp ? (W > 0 ? (double)(SX - ax * W) / (double)W : 0.0) : (double)(SX - ax * nn) / (double)nn;
    const double dy = grp ? (W > 0 ? (double)(SY - ay * W) / (double)W : 0.0) : (double)(SY - ay * nn) / (double)nn;
    const double Ax = (double)(gx0 + ax), Ay = (double)(gy0 + ay);
    // binomial shifts, separable: T[i][q] = sum_j C(q,j) s_y^(q-j) N[i][j], then
    // out[p][q] = sum_i C(p,i) s_x^(p-i) T[i][q] (one 4x4 tile live at a time);
    // s = -d for the central moments, the anchor's origin A for the raw ones
    auto shift = [&](double sx, double sy, double* R) {
        const double y1 = sy, y2 = sy * sy, y3 = y2 * sy;
        const double x1 = sx, x2 = sx * sx, x3 = x2 * sx;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double a0 = N[i * 4], a1 = N[i * 4 + 1], a2 = N[i * 4 + 2], a3 = N[i * 4 + 3];
            R[i * 4] = a0;
            R[i * 4 + 1] = a1 + y1 * a0;
            R[i * 4 + 2] = a2 + 2.0 * y1 * a1 + y2 * a0;
            R[i * 4 + 3] = a3 + 3.0 * y1 * a2 + 3.0 * y2 * a1 + y3 * a0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double a0 = R[q], a1 = R[4 + q], a2 = R[8 + q], a3 = R[12 + q];
            R[4 + q] = a1 + x1 * a0;
            R[8 + q] = a2 + 2.0 * x1 * a1 + x2 * a0;
            R[12 + q] = a3 + 3.0 * x1 * a2 + 3.0 * x2 * a1 + x3 * a0;
        }
    };
    double R[16];
    shift(Ax, Ay, R);
#pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = zero_mass ? 0.0 : R[k];
    shift(-dx, -dy, R);
    R[1] = R[4] = 0.0;  // moments.cpp:80-81
    R[0] = N[0];
    double eta[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double mu = R[p * 4 + q];
            double et = 0;
            if (p + q >= 2) {  // eta = mu / m00^(1 + (p+q)/2)
                double den = m00 * m00;
                if (p + q >= 4) den *= m00;
                if (p + q >= 6) den *= m00;
                if ((p + q) & 1) den *= sqrt(m00);
                et = mu / den;
            }
            if (zero_mass) et = 0;
            eta[p][q] = et;
            o[16 + p * 4 + q] = zero_mass ? 0.0 : mu;
            if (p + q >= 2) o[32 + ((p == 0) ? q - 2 : (p == 1 ? 1 + q : 1 + 4 * (p - 1) + q))] = et;
        }
    const double n20 = eta[2][0], n02 = eta[0][2], n11 = eta[1][1], n30 = eta[3][0],
                 n03 = eta[0][3], n21 = eta[2][1], n12 = eta[1][2];
    const double a = n30 + n12, b = n21 + n03;
    const double hu[7] = {n20 + n02,
                          (n20 - n02) * (n20 - n02) + 4.0 * n11 * n11,
                          (n30 - 3.0 * n12) * (n30 - 3.0 * n12) + (3.0 * n21 - n03) * (3.0 * n21 - n03),
                          a * a + b * b,
                          (n30 - 3.0 * n12) * a * (a * a - 3.0 * b * b) +
                              (3.0 * n21 - n03) * b * (3.0 * a * a - b * b),
                          (n20 - n02) * (a * a - b * b) + 4.0 * n11 * a * b,
                          (3.0 * n21 - n03) * a * (a * a - 3.0 * b * b) -
                              (n30 - 3.0 * n12) * b * (3.0 * a * a - b * b)};
#pragma unroll
    for (int k = 0; k < 7; ++k) o[45 + k] = zero_mass ? 0.0 : hu[k];
}

__device__ void moments_row(uint32_t r, int grp, const RoiList& rl, const FeatCfg& cfg,
                                         double* out) {
    const unsigned long long off = cfg.mom_off[r];
    if (off == ~0ull) return;  // not staged: the warp path wrote the columns
    const uint32_t n = (uint32_t)rl.n[r];
    const unsigned long long* sums = cfg.mom_sums + (size_t)r * 5;
    const long long nn = (long long)n;
    double N[16];
    long long W = 0, ax, ay, SX, SY;
    if (grp == 0) {
        SX = (long long)sums[3];
        SY = (long long)sums[4];
        ax = (2 * SX + nn) / (2 * nn);
        ay = (2 * SY + nn) / (2 * nn);
    } else {
        W = (long long)sums[0];
        SX = (long long)sums[1];
        SY = (long long)sums[2];
        ax = W > 0 ? (2 * SX + W) / (2 * W) : 0;
        ay = W > 0 ? (2 * SY + W) / (2 * W) : 0;
    }
    const uint4* px4 = reinterpret_cast<const uint4*>(cfg.mom_px + off);  // 16 B aligned
    const uint32_t nq = (n + 3u) >> 2;
    // every pixel adds its 16 terms (no row flush: divergent flushes across the 32
    // ROIs of a warp cost more than the extra products); 16 B loads, two in flight
    auto stream = [&](auto&& pixel) {
        uint4 cur = px4[0], nxt = nq > 1 ? px4[1] : make_uint4(0, 0, 0, 0);
        for (uint32_t q4 = 0; q4 < nq; ++q4) {
            const uint4 fut = q4 + 2 < nq ? px4[q4 + 2] : make_uint4(0, 0, 0, 0);
            const uint32_t base = q4 * 4u;
            pixel(cur.x);
            if (base + 1 < n) pixel(cur.y);
            if (base + 2 < n) pixel(cur.z);
            if (base + 3 < n) pixel(cur.w);
            cur = nxt;
            nxt = fut;
        }
    };
    if (grp == 0) {
        long long M[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) M[k] = 0;
        stream([&](uint32_t e) {
            const int dx = (int)(e & 0xffu) - (int)ax, dy = (int)((e >> 8) & 0xffu) - (int)ay;
            const int X[4] = {1, dx, dx * dx, dx * dx * dx};
            const int Y[4] = {1, dy, dy * dy, dy * dy * dy};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (p + q >= 2) M[p * 4 + q] += (long long)X[p] * Y[q];
        });
        // the order-0 / order-1 sums follow from the staged exact sums
        M[0] = nn;
        M[1] = SY - ay * nn;
        M[4] = SX - ax * nn;
#pragma unroll
        for (int k = 0; k < 16; ++k) N[k] = (double)M[k];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) N[k] = 0;
        stream([&](uint32_t e) {
            const double dx = (double)((long long)(e & 0xffu) - ax);
            const double dy = (double)((long long)((e >> 8) & 0xffu) - ay);
            const double wv = (double)(e >> 16);
            const double pw[4] = {wv, wv * dx, wv * dx * dx, wv * dx * dx * dx};
            const double q[4] = {1.0, dy, dy * dy, dy * dy * dy};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (p + k >= 2) N[p * 4 + k] += pw[p] * q[k];
        });
        // the order-0 / order-1 sums follow from the staged exact integer sums
        N[0] = (double)W;
        N[1] = (double)(SY - ay * W);
        N[4] = (double)(SX - ax * W);
    }
    moments_epilogue_serial(N, grp, n, W, SX, SY, ax, ay, rl.gx[r], rl.gy[r],
                            out + (size_t)r * cfg.ncols + cfg.col_mom + grp * 52);
}

// Intensity statistics of the staged S ROIs (intensity_features.cpp:42-215), one
// thread per ROI over the warp-sorted values: order statistics by the literal
// percentile expression, median absolute deviation as the k-th element of the
// V-shaped deviations (two-pointer walk from the median split), one sequential
// scan for the central moments, mad / rmad partial sums, mode and histogram runs.
// Columns 32..38 (edge statistics, weighted centroid) come from the warp.
// Both middle order statistics of the doubled deviations |2 s[i] - M2| in one search:
// d_hi = the (n/2)-th (0-based), d_lo = the (n/2 - 1)-th (even n; d_lo = d_hi if odd).
__device__ void kth_dev_pair(const uint16_t* s, uint32_t n, uint32_t M2, uint32_t& d_hi,
                             uint32_t& d_lo) {
    // m = first index with 2 s[i] >= M2.  M2 <= 2 s[n/2] (M2 is twice the median),
    // so m <= n/2, and m == n/2 unless s[n/2 - 1] ties the median: one probe, and a
    // binary search over [0, n/2 - 1] only for tied medians
    uint32_t m = n / 2;
    if (m > 0 && 2u * s[m - 1] >= M2) {
        uint32_t lo = 0, hi = m - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (2u * s[mid] >= M2) hi = mid;
            else lo = mid + 1;
        }
        m = lo;
    }
    // A[j] = M2 - 2 s[m-1-j] (j < m) and B[j] = 2 s[m+j] - M2 are ascending; the
    // kk smallest of their union are A[0, t) and B[0, kk - t) for the t found by a
    // binary search on the count taken from A (kk = n/2 + 1)
    const uint32_t na = m, nb = n - m, kk = n / 2 + 1;
    auto A = [&](uint32_t j) { return M2 - 2u * s[m - 1 - j]; };
    auto B = [&](uint32_t j) { return 2u * s[m + j] - M2; };
    uint32_t a = kk > nb ? kk - nb : 0u, b = kk < na ? kk : na;  // t in [a, b]
    while (a < b) {  // smallest t with A[t] >= B[kk-1-t] (t < na, kk-1-t >= 0)
        const uint32_t t = (a + b) >> 1;
        if (A(t) < B(kk - 1 - t)) a = t + 1;
        else b = t;
    }
    const uint32_t t = a, tb = kk - t;
    // the kk-th smallest is the largest of that prefix, the (kk-1)-th its second largest
    const uint32_t x = t > 0 ? A(t - 1) : 0u, y = tb > 0 ? B(tb - 1) : 0u;
    d_hi = max(x, y);
    if (n & 1) {
        d_lo = d_hi;
        return;
    }
    uint32_t sec = (t > 0 && tb > 0) ? min(x, y) : 0u;
    if (t >= 2) sec = max(sec, A(t - 2));
    if (tb >= 2) sec = max(sec, B(tb - 2));
    d_lo = sec;
}

__device__ void intensity_row(uint32_t r, const RoiList& rl, const FeatCfg& cfg,
                                           double* out) {
    const unsigned long long off = cfg.int_off[r];
    if (off == ~0ull) return;  // not staged: the warp path wrote the columns
    const uint32_t n = (uint32_t)rl.n[r];
    const uint16_t* s = cfg.int_vals + off;
    const unsigned long long sS = cfg.int_sums[(size_t)r * 2], sQ = cfg.int_sums[(size_t)r * 2 + 1];
    const double dn = (double)n, mean = (double)sS / dn;
    const uint32_t vmin = s[0], vmax = s[n - 1];
    const double mn = (double)vmin, mxv = (double)vmax;
    const double median = (n & 1) ? (double)s[n / 2] : 0.5 * ((double)s[n / 2 - 1] + (double)s[n / 2]);
    const double pv[6] = {1.0, 10.0, 25.0, 75.0, 90.0, 99.0};
    double pct[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) pct[k] = percentile_exact(s, n, pv[k]);
    const double p10 = pct[1], p25 = pct[2], p75 = pct[3], p90 = pct[4];
    const uint32_t M2 = (n & 1) ? 2u * s[n / 2] : (uint32_t)s[n / 2 - 1] + s[n / 2];
    // one scan: central moments, mad / rmad partials, value runs (mode), bin runs
    // (it also pulls the values into L1 for the dependent searches that follow)
    const uint32_t nb32 = (uint32_t)cfg.bins, rng = vmax - vmin;
    const bool wide = (unsigned long long)nb32 * 65535ull >= (1ull << 32);
    const uint32_t magic = rng ? (uint32_t)(0xffffffffull / rng) : 0u;
    auto bin_of = [&](uint32_t v) -> uint32_t {  // floor(nb (v - min) / range), exact
        if (rng == 0) return 0u;
        uint32_t b;
        if (!wide) {
            const uint32_t num = nb32 * (v - vmin);
            b = __umulhi(num, magic);
            if (num - b * rng >= rng) ++b;
        } else {
            b = (uint32_t)((unsigned long long)nb32 * (v - vmin) / rng);
        }
        return b < nb32 - 1 ? b : nb32 - 1;
    };
    const double logn = nlog2(dn);
    // integer thresholds for the integer values: v < mean <=> v < ceil(mean);
    // p10 <= v <= p90 <=> ceil(p10) <= v <= floor(p90) (exact: v < 2^16)
    const uint32_t t_mean = (uint32_t)ceil(mean), t_lo = (uint32_t)ceil(p10), t_hi = (uint32_t)floor(p90);
    // m2 needs no pass: n^2 m2 = n sQ - sS^2 exactly (both < 2^64 for any n <= 65536);
    // slo / rsum are 32-bit (an S window holds <= 4096 pixels: sums < 2^28)
    double a3 = 0, a4 = 0, a5 = 0, a6 = 0, ent = 0;
    unsigned long long best = 0, usq = 0;
    uint32_t slo = 0, rsum = 0, clo = 0, rn = 0, run_v = 0, run_b = 0, pv_ = s[0], pb_ = bin_of(s[0]);
    const uint4* s4 = reinterpret_cast<const uint4*>(s);  // 16 B aligned (staging rounds to 8)
    uint4 nxt4 = s4[0];  // next 8 values in flight while these 8 are processed
    for (uint32_t q = 0; q * 8u < n; ++q) {
#ifndef FXG_NO_INT_PREFETCH
        const uint4 w4 = nxt4;
        if ((q + 1u) * 8u < n) nxt4 = s4[q + 1];
#else
        const uint4 w4 = s4[q];
#endif
        const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (q * 8u + (uint32_t)u >= n) break;
            const uint32_t v = (wv[u >> 1] >> ((u & 1) * 16)) & 0xffffu;
            const double d = (double)v - mean, d2 = d * d;
            a3 += d2 * d;
            a4 += d2 * d2;
            a5 += d2 * d2 * d;
            a6 += d2 * d2 * d2;
            if (v < t_mean) {
                slo += v;
                ++clo;
            }
            if (v >= t_lo && v <= t_hi) {
                rsum += v;
                ++rn;
            }
            if (v != pv_) {  // a value run ended
                const unsigned long long key = ((unsigned long long)run_v << 16) | (0xffffu - pv_);
                best = key > best ? key : best;
                pv_ = v;
                run_v = 0;
            }
            ++run_v;
            const uint32_t b = bin_of(v);
            if (b != pb_) {  // a bin run ended
                ent += (double)run_b * (logn - log2_int(run_b));
                usq += (unsigned long long)run_b * run_b;
                pb_ = b;
                run_b = 0;
            }
            ++run_b;
        }
    }
    {
        const unsigned long long key = ((unsigned long long)run_v << 16) | (0xffffu - pv_);
        best = key > best ? key : best;
        ent += (double)run_b * (logn - log2_int(run_b));
        usq += (unsigned long long)run_b * run_b;
    }
    uint32_t d_hi, d_lo;
    kth_dev_pair(s, n, M2, d_hi, d_lo);
    const double median_ad = (n & 1) ? 0.5 * (double)d_hi : 0.5 * (0.5 * (double)d_lo + 0.5 * (double)d_hi);
    const double m2 = (double)((unsigned long long)n * sQ - sS * sS) / (dn * dn);
    const double m3 = a3 / dn, m4 = a4 / dn, m5 = a5 / dn, m6 = a6 / dn;
    const double mad = ((double)(long long)(sS - 2ull * slo) +
                        (double)((long long)clo - (long long)(n - clo)) * mean) / dn;
    double rmad = 0;
    if (rn > 0) {
        const double rmean = (double)rsum / (double)rn;
        unsigned long long rlo = 0;
        uint32_t rcl = 0;
        // values sorted: the [p10, p90] subset below rmean is one contiguous range
        const uint32_t t_rm = (uint32_t)ceil(rmean);
        bool more = true;
        for (uint32_t q = 0; more && q * 8u < n; ++q) {  // 8 values per 16 B load
            const uint4 w4 = s4[q];
            const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t v = (wv[u >> 1] >> ((u & 1) * 16)) & 0xffffu;
                if (q * 8u + (uint32_t)u >= n || v >= t_rm) {
                    more = false;
                    break;
                }
                if (v >= t_lo && v <= t_hi) {
                    rlo += v;
                    ++rcl;
                }
            }
        }
        rmad = ((double)(long long)(rsum - 2 * rlo) +
                (double)((long long)rcl - (long long)(rn - rcl)) * rmean) / (double)rn;
    }
    const double var = n > 1 ? m2 * dn / (dn - 1.0) : 0.0;
    double skew = 0, kurt = 0, hsk = 0, hfl = 0;
    if (m2 > 0) {
        const double r2 = sqrt(m2);
        skew = m3 / (m2 * r2);
        kurt = m4 / (m2 * m2);
        hsk = m5 / (m2 * m2 * r2);
        hfl = m6 / (m2 * m2 * m2);
    }
    const double energy = (double)sQ, sdev = sqrt(var), iqr = p75 - p25;
    const double o32[32] = {mean, median, (double)(0xffffu - (uint32_t)(best & 0xffffu)), mn, mxv,
                            mxv - mn, var, m2, sdev, sqrt(m2), mad, median_ad, rmad, iqr,
                            pct[0], pct[1], pct[2], pct[3], pct[4], pct[5], skew, kurt,
                            m2 > 0 ? kurt - 3.0 : 0.0, hsk, hfl, energy, sqrt(energy / dn), ent / dn,
                            (double)usq / (dn * dn), (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0,
                            mean != 0 ? sdev / mean : 0.0, (double)sS};
    double* oi = out + (size_t)r * cfg.ncols + cfg.col_int;
#pragma unroll
    for (int k = 0; k < 32; ++k) oi[k] = o32[k];
}

// ---- the serial passes with G lanes per ROI -----------------------------------
//
// Thread-per-ROI left the pass in one partial wave (C2: 50k ROIs -> ~10 warps per
// SM, latency-bound on the dependent fp64 chains).  Here G consecutive lanes share
// a ROI: lane g takes the g-th chunk of the sorted values (or of the staged
// pixels), partial sums combine by a fixed butterfly (deterministic), and the runs
// that cross chunk borders (mode, histogram bins) are stitched in lane order by
// the group's first lane, which then writes the row.
#ifndef FXG_SERIAL_G
#define FXG_SERIAL_G 1
#endif
#ifndef FXG_SERIAL_SPLIT
#define FXG_SERIAL_SPLIT 1
#endif
constexpr int kSerialG = FXG_SERIAL_G;

template <typename T>
__device__ __forceinline__ T group_sum(T v, unsigned gm) {
#pragma unroll
    for (int o = kSerialG / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(gm, v, o, kSerialG);
    return v;
}

// One chunk's runs: the first run (may continue the previous chunk), the last run
// (may continue into the next), and whether the chunk is one single run.
struct ChunkRuns {
    uint32_t fv, fl, lv, ll;
    bool single;
};

// stitch the chunk runs of the G lanes in lane order (called by every lane; the
// result is meaningful on the group's first lane).  done(v, len) is called for
// every run completed across a border, and for the final run.
template <typename Done>
__device__ __forceinline__ void stitch_runs(const ChunkRuns& c, bool nonempty, unsigned gm,
                                            Done&& done) {
    uint32_t cv = 0, cl = 0;
    bool have = false;
#pragma unroll 1
    for (int k = 0; k < kSerialG; ++k) {
        const bool ne = __shfl_sync(gm, (int)nonempty, k, kSerialG) != 0;
        const uint32_t fv = __shfl_sync(gm, c.fv, k, kSerialG), fl = __shfl_sync(gm, c.fl, k, kSerialG);
        const uint32_t lv = __shfl_sync(gm, c.lv, k, kSerialG), ll = __shfl_sync(gm, c.ll, k, kSerialG);
        const bool single = __shfl_sync(gm, (int)c.single, k, kSerialG) != 0;
        if (!ne) continue;
        if (have && fv == cv) {
            cl += fl;
        } else {
            if (have) done(cv, cl);
            cv = fv;
            cl = fl;
            have = true;
        }
        if (!single) {
            done(cv, cl);  // the first run ended inside chunk k
            cv = lv;
            cl = ll;
        }
    }
    if (have) done(cv, cl);
}

__device__ void intensity_group(uint32_t r, uint32_t g, unsigned gm, const RoiList& rl,
                                const FeatCfg& cfg, double* out) {
    const unsigned long long off = cfg.int_off[r];
    if (off == ~0ull) return;  // not staged: the warp path wrote the columns (group-uniform)
    const uint32_t n = (uint32_t)rl.n[r];
    const uint16_t* s = cfg.int_vals + off;
    const unsigned long long sS = cfg.int_sums[(size_t)r * 2], sQ = cfg.int_sums[(size_t)r * 2 + 1];
    const double dn = (double)n, mean = (double)sS / dn;
    const uint32_t vmin = s[0], vmax = s[n - 1];
    const double p10 = percentile_exact(s, n, 10.0), p90 = percentile_exact(s, n, 90.0);
    const uint32_t nb32 = (uint32_t)cfg.bins, rng = vmax - vmin;
    const bool wide = (unsigned long long)nb32 * 65535ull >= (1ull << 32);
    const uint32_t magic = rng ? (uint32_t)(0xffffffffull / rng) : 0u;
    auto bin_of = [&](uint32_t v) -> uint32_t {  // floor(nb (v - min) / range), exact
        if (rng == 0) return 0u;
        uint32_t b;
        if (!wide) {
            const uint32_t num = nb32 * (v - vmin);
            b = __umulhi(num, magic);
            if (num - b * rng >= rng) ++b;
        } else {
            b = (uint32_t)((unsigned long long)nb32 * (v - vmin) / rng);
        }
        return b < nb32 - 1 ? b : nb32 - 1;
    };
    const double logn = nlog2(dn);
    // integer thresholds for the integer values: v < mean <=> v < ceil(mean);
    // p10 <= v <= p90 <=> ceil(p10) <= v <= floor(p90) (exact: v < 2^16)
    const uint32_t t_mean = (uint32_t)ceil(mean), t_lo = (uint32_t)ceil(p10), t_hi = (uint32_t)floor(p90);
    // this lane's chunk: [a, e), a multiple of 8 (16 B aligned loads)
    const uint32_t C = ((n + kSerialG - 1) / kSerialG + 7u) & ~7u;
    const uint32_t a = min(n, g * C), e = min(n, a + C);
    const bool nonempty = a < e;
    double a3 = 0, a4 = 0, a5 = 0, a6 = 0, ent = 0;
    unsigned long long best = 0, usq = 0;
    uint32_t slo = 0, rsum = 0, clo = 0, rn = 0;
    ChunkRuns vr{0, 0, 0, 0, true}, br{0, 0, 0, 0, true};
    if (nonempty) {
        uint32_t pv_ = s[a], pb_ = bin_of(s[a]), run_v = 0, run_b = 0;
        bool vfirst = true, bfirst = true;
        vr.fv = pv_;
        br.fv = pb_;
        const uint4* s4 = reinterpret_cast<const uint4*>(s + a);
        for (uint32_t q = 0; a + q * 8u < e; ++q) {
            const uint4 w4 = s4[q];
            const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (a + q * 8u + (uint32_t)u >= e) break;
                const uint32_t v = (wv[u >> 1] >> ((u & 1) * 16)) & 0xffffu;
                const double d = (double)v - mean, d2 = d * d;
                a3 += d2 * d;
                a4 += d2 * d2;
                a5 += d2 * d2 * d;
                a6 += d2 * d2 * d2;
                if (v < t_mean) {
                    slo += v;
                    ++clo;
                }
                if (v >= t_lo && v <= t_hi) {
                    rsum += v;
                    ++rn;
                }
                if (v != pv_) {  // a value run ended
                    if (vfirst) {
                        vr.fl = run_v;
                        vfirst = false;
                    } else {
                        const unsigned long long key = ((unsigned long long)run_v << 16) | (0xffffu - pv_);
                        best = key > best ? key : best;
                    }
                    pv_ = v;
                    run_v = 0;
                }
                ++run_v;
                const uint32_t b = bin_of(v);
                if (b != pb_) {  // a bin run ended
                    if (bfirst) {
                        br.fl = run_b;
                        bfirst = false;
                    } else {
                        ent += (double)run_b * (logn - log2_int(run_b));
                        usq += (unsigned long long)run_b * run_b;
                    }
                    pb_ = b;
                    run_b = 0;
                }
                ++run_b;
            }
        }
        vr.lv = pv_;
        vr.ll = run_v;
        vr.single = vfirst;
        if (vfirst) vr.fl = run_v;
        br.lv = pb_;
        br.ll = run_b;
        br.single = bfirst;
        if (bfirst) br.fl = run_b;
    }
    // fixed-order combination (butterfly: identical on every lane)
    a3 = group_sum(a3, gm);
    a4 = group_sum(a4, gm);
    a5 = group_sum(a5, gm);
    a6 = group_sum(a6, gm);
    ent = group_sum(ent, gm);
    usq = group_sum(usq, gm);
    slo = group_sum(slo, gm);
    clo = group_sum(clo, gm);
    rsum = group_sum(rsum, gm);
    rn = group_sum(rn, gm);
#pragma unroll
    for (int o = kSerialG / 2; o >= 1; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(gm, best, o, kSerialG);
        best = ob > best ? ob : best;
    }
    stitch_runs(vr, nonempty, gm, [&](uint32_t v, uint32_t len) {
        const unsigned long long key = ((unsigned long long)len << 16) | (0xffffu - v);
        best = key > best ? key : best;
    });
    stitch_runs(br, nonempty, gm, [&](uint32_t, uint32_t len) {
        ent += (double)len * (logn - log2_int(len));
        usq += (unsigned long long)len * len;
    });
    // rmad: the [p10, p90] subset below its mean is one contiguous range of the
    // sorted values; each lane sums its part of it
    double rmean = 0;
    unsigned long long rlo = 0;
    uint32_t rcl = 0;
    if (rn > 0) {
        rmean = (double)rsum / (double)rn;
        const uint32_t t_rm = (uint32_t)ceil(rmean);
        if (nonempty && s[a] < t_rm) {
            const uint4* s4 = reinterpret_cast<const uint4*>(s + a);
            bool more = true;
            for (uint32_t q = 0; more && a + q * 8u < e; ++q) {
                const uint4 w4 = s4[q];
                const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t v = (wv[u >> 1] >> ((u & 1) * 16)) & 0xffffu;
                    if (a + q * 8u + (uint32_t)u >= e || v >= t_rm) {
                        more = false;
                        break;
                    }
                    if (v >= t_lo && v <= t_hi) {
                        rlo += v;
                        ++rcl;
                    }
                }
            }
        }
        rlo = group_sum(rlo, gm);
        rcl = group_sum(rcl, gm);
    }
    if (g != 0) return;
    const double mn = (double)vmin, mxv = (double)vmax;
    const double median = (n & 1) ? (double)s[n / 2] : 0.5 * ((double)s[n / 2 - 1] + (double)s[n / 2]);
    const double p1 = percentile_exact(s, n, 1.0), p25 = percentile_exact(s, n, 25.0),
                 p75 = percentile_exact(s, n, 75.0), p99 = percentile_exact(s, n, 99.0);
    const uint32_t M2 = (n & 1) ? 2u * s[n / 2] : (uint32_t)s[n / 2 - 1] + s[n / 2];
    uint32_t d_hi, d_lo;
    kth_dev_pair(s, n, M2, d_hi, d_lo);
    const double median_ad = (n & 1) ? 0.5 * (double)d_hi : 0.5 * (0.5 * (double)d_lo + 0.5 * (double)d_hi);
    // m2 needs no pass: n^2 m2 = n sQ - sS^2 exactly (both < 2^64 for any n <= 65536)
    const double m2 = (double)((unsigned long long)n * sQ - sS * sS) / (dn * dn);
    const double m3 = a3 / dn, m4 = a4 / dn, m5 = a5 / dn, m6 = a6 / dn;
    const double mad = ((double)(long long)(sS - 2ull * slo) +
                        (double)((long long)clo - (long long)(n - clo)) * mean) / dn;
    const double rmad = rn > 0 ? ((double)(long long)(rsum - 2 * rlo) +
                                  (double)((long long)rcl - (long long)(rn - rcl)) * rmean) / (double)rn
                               : 0.0;
    const double var = n > 1 ? m2 * dn / (dn - 1.0) : 0.0;
    double skew = 0, kurt = 0, hsk = 0, hfl = 0;
    if (m2 > 0) {
        const double r2 = sqrt(m2);
        skew = m3 / (m2 * r2);
        kurt = m4 / (m2 * m2);
        hsk = m5 / (m2 * m2 * r2);
        hfl = m6 / (m2 * m2 * m2);
    }
    const double energy = (double)sQ, sdev = sqrt(var), iqr = p75 - p25;
    const double o32[32] = {mean, median, (double)(0xffffu - (uint32_t)(best & 0xffffu)), mn, mxv,
                            mxv - mn, var, m2, sdev, sqrt(m2), mad, median_ad, rmad, iqr,
                            p1, p10, p25, p75, p90, p99, skew, kurt,
                            m2 > 0 ? kurt - 3.0 : 0.0, hsk, hfl, energy, sqrt(energy / dn), ent / dn,
                            (double)usq / (dn * dn), (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0,
                            mean != 0 ? sdev / mean : 0.0, (double)sS};
    double* oi = out + (size_t)r * cfg.ncols + cfg.col_int;
#pragma unroll
    for (int k = 0; k < 32; ++k) oi[k] = o32[k];
}

// Moments with G lanes per ROI: lane g sums its chunk of staged pixel quads, the
// 16 sums combine by butterfly, the group's first lane runs the epilogue.
__device__ void moments_group(uint32_t r, int grp, uint32_t g, unsigned gm, const RoiList& rl,
                              const FeatCfg& cfg, double* out) {
    const unsigned long long off = cfg.mom_off[r];
    if (off == ~0ull) return;  // not staged: the warp path wrote the columns (group-uniform)
    const uint32_t n = (uint32_t)rl.n[r];
    const unsigned long long* sums = cfg.mom_sums + (size_t)r * 5;
    const long long nn = (long long)n;
    double N[16];
    long long W = 0, ax, ay, SX, SY;
    if (grp == 0) {
        SX = (long long)sums[3];
        SY = (long long)sums[4];
        ax = (2 * SX + nn) / (2 * nn);
        ay = (2 * SY + nn) / (2 * nn);
    } else {
        W = (long long)sums[0];
        SX = (long long)sums[1];
        SY = (long long)sums[2];
        ax = W > 0 ? (2 * SX + W) / (2 * W) : 0;
        ay = W > 0 ? (2 * SY + W) / (2 * W) : 0;
    }
    const uint4* px4 = reinterpret_cast<const uint4*>(cfg.mom_px + off);  // 16 B aligned
    const uint32_t nq = (n + 3u) >> 2, cq = (nq + kSerialG - 1) / kSerialG;
    const uint32_t q0 = min(nq, g * cq), q1 = min(nq, q0 + cq);
    auto stream = [&](auto&& pixel) {
        for (uint32_t q4 = q0; q4 < q1; ++q4) {
            const uint4 cur = px4[q4];
            const uint32_t base = q4 * 4u;
            pixel(cur.x);
            if (base + 1 < n) pixel(cur.y);
            if (base + 2 < n) pixel(cur.z);
            if (base + 3 < n) pixel(cur.w);
        }
    };
    if (grp == 0) {
        long long M[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) M[k] = 0;
        stream([&](uint32_t e) {
            const int dx = (int)(e & 0xffu) - (int)ax, dy = (int)((e >> 8) & 0xffu) - (int)ay;
            const int X[4] = {1, dx, dx * dx, dx * dx * dx};
            const int Y[4] = {1, dy, dy * dy, dy * dy * dy};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (p + q >= 2) M[p * 4 + q] += (long long)X[p] * Y[q];
        });
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k != 0 && k != 1 && k != 4) M[k] = group_sum(M[k], gm);
        // the order-0 / order-1 sums follow from the staged exact sums
        M[0] = nn;
        M[1] = SY - ay * nn;
        M[4] = SX - ax * nn;
#pragma unroll
        for (int k = 0; k < 16; ++k) N[k] = (double)M[k];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) N[k] = 0;
        stream([&](uint32_t e) {
            const double dx = (double)((long long)(e & 0xffu) - ax);
            const double dy = (double)((long long)((e >> 8) & 0xffu) - ay);
            const double wv = (double)(e >> 16);
            const double pw[4] = {wv, wv * dx, wv * dx * dx, wv * dx * dx * dx};
            const double q[4] = {1.0, dy, dy * dy, dy * dy * dy};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (p + k >= 2) N[p * 4 + k] += pw[p] * q[k];
        });
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k != 0 && k != 1 && k != 4) N[k] = group_sum(N[k], gm);
        // the order-0 / order-1 sums follow from the staged exact integer sums
        N[0] = (double)W;
        N[1] = (double)(SY - ay * W);
        N[4] = (double)(SX - ax * W);
    }
    if (g != 0) return;
    moments_epilogue_serial(N, grp, n, W, SX, SY, ax, ay, rl.gx[r], rl.gy[r],
                            out + (size_t)r * cfg.ncols + cfg.col_mom + grp * 52);
}

// the per-ROI serial passes of the S ROIs in one launch: blocks [0, bi) run the
// intensity statistics, [bi, bi + bm) the binary moments, the rest the weighted
// moments, so the sparse waves overlap (and binary moments use the integer pipe
// while the other two use fp64)
#ifndef FXG_SERIAL_TPB
#define FXG_SERIAL_TPB 128
#endif
#ifndef FXG_SERIAL_MINB
#define FXG_SERIAL_MINB (5 * 128 / FXG_SERIAL_TPB)
#endif
__global__ void __launch_bounds__(FXG_SERIAL_TPB, FXG_SERIAL_MINB)
    k_serial_stats(RoiList rl, Control* ctl, FeatCfg cfg, double* out, uint32_t bi, uint32_t bm) {
    const uint32_t b = blockIdx.x;
    const uint32_t t = (b < bi ? b : b < bi + bm ? b - bi : b - bi - bm) * blockDim.x + threadIdx.x;
#if FXG_SERIAL_G > 1
    // G lanes per ROI (group-uniform exits keep the group's shuffles converged)
    const uint32_t g = t % kSerialG, lane = threadIdx.x & 31;
    const unsigned gm = (kSerialG == 32 ? kFull : ((1u << kSerialG) - 1u)) << (lane & ~(uint32_t)(kSerialG - 1));
    const uint32_t r = s_row_of(t / kSerialG, rl, ctl);
    if (r == ~0u) return;
    if (b < bi) intensity_group(r, g, gm, rl, cfg, out);
    else moments_group(r, b < bi + bm ? 0 : 1, g, gm, rl, cfg, out);
#else
    const uint32_t r = s_row_of(t, rl, ctl);
    if (r == ~0u) return;
    if (b < bi) intensity_row(r, rl, cfg, out);
    else moments_row(r, b < bi + bm ? 0 : 1, rl, cfg, out);
#endif
}

// The two moments roles as their own kernel (fewer registers than the intensity
// role needs, so more warps per SM), on a second stream next to the intensity role.
#ifndef FXG_SERIAL_MOM_MINB
#define FXG_SERIAL_MOM_MINB 8
#endif
__global__ void __launch_bounds__(FXG_SERIAL_TPB, FXG_SERIAL_MOM_MINB)
    k_serial_moments(RoiList rl, Control* ctl, FeatCfg cfg, double* out, uint32_t bm) {
    const uint32_t b = blockIdx.x, grp = b < bm ? 0u : 1u;
    const uint32_t t = (b - grp * bm) * blockDim.x + threadIdx.x;
    const uint32_t r = s_row_of(t, rl, ctl);
    if (r == ~0u) return;
    moments_row(r, (int)grp, rl, cfg, out);
}

void launch_serial_stats(int n_s, bool intensity, bool moments, cudaStream_t s, RoiList rl,
                         Control* ctl, FeatCfg cfg, double* out, cudaStream_t s2, cudaEvent_t fork,
                         cudaEvent_t join) {
    if (n_s <= 0 || (!intensity && !moments)) return;
    const uint32_t nb = (uint32_t)(((size_t)n_s * kSerialG + FXG_SERIAL_TPB - 1) / FXG_SERIAL_TPB);
#if FXG_SERIAL_SPLIT
    if (s2 && intensity && moments && kSerialG == 1) {
        cudaEventRecord(fork, s);
        cudaStreamWaitEvent(s2, fork, 0);
        k_serial_moments<<<2 * nb, FXG_SERIAL_TPB, 0, s2>>>(rl, ctl, cfg, out, nb);
        cudaEventRecord(join, s2);
        k_serial_stats<<<nb, FXG_SERIAL_TPB, 0, s>>>(rl, ctl, cfg, out, nb, 0u);
        cudaStreamWaitEvent(s, join, 0);
        return;
    }
#else
    (void)s2;
    (void)fork;
    (void)join;
#endif
    const uint32_t bi = intensity ? nb : 0u, bm = moments ? nb : 0u;
    k_serial_stats<<<bi + 2 * bm, FXG_SERIAL_TPB, 0, s>>>(rl, ctl, cfg, out, bi, bm);
}

void launch_shape_serial(int n_s, cudaStream_t s, RoiList rl, Control* ctl, FeatCfg cfg,
                         double* out) {
    if (n_s > 0) k_shape_serial<<<(n_s + 127) / 128, 128, 0, s>>>(rl, ctl, cfg, out);
}

void launch_roi_s(int cls, int grid, cudaStream_t s, const CUtensorMap* tmaps, int tma40, int tma72,
                  DevImage img, RoiList rl, Control* ctl, FeatCfg cfg, double* out,
                  const DebugOut* dbg) {
    // tmaps: labels / intensities for the 40-wide (S0) and 72-wide (S1, S2) tiles
    const int g = s_glcm_mode(cfg);
#define FXG_LAUNCH(C, TM, TI, TA)                                                          \
    do {                                                                                   \
        if (g == kGlHist) launch_one<C, kGlHist>(grid, s, TM, TI, TA, img, rl, ctl, cfg, out, dbg); \
        else if (g == kGlSort) launch_one<C, kGlSort>(grid, s, TM, TI, TA, img, rl, ctl, cfg, out, dbg); \
        else launch_one<C, kGlNone>(grid, s, TM, TI, TA, img, rl, ctl, cfg, out, dbg);  \
    } while (0)
    switch (cls) {
        case kClassS0: FXG_LAUNCH(kClassS0, tmaps[0], tmaps[1], tma40); break;
        case kClassS1: FXG_LAUNCH(kClassS1, tmaps[2], tmaps[3], tma72); break;
        default: FXG_LAUNCH(kClassS2, tmaps[2], tmaps[3], tma72); break;
    }
#undef FXG_LAUNCH
}

}  // namespace fxg

namespace fxg {
int roi_b_phase_clocks(unsigned long long* out, int reset);
}

// slots 0..8: S kernels (lane 0 per ROI); 9..15: k_roi_b (thread 0 per ROI)
extern "C" int fx_debug_phase_clocks(unsigned long long* out, int n, int reset) {
#ifdef FXG_PHASE_TIMING
    unsigned long long h[16];
    if (cudaMemcpyFromSymbol(h, ::g_phase_clk, sizeof h) != cudaSuccess) return 7;
    unsigned long long b[8];
    if (fxg::roi_b_phase_clocks(b, reset)) return 7;
    for (int i = 0; i < 7; ++i) h[9 + i] = b[i];
    for (int i = 0; i < n && i < 16; ++i) out[i] = h[i];
    if (reset) {
        const unsigned long long z[16] = {};
        cudaMemcpyToSymbol(::g_phase_clk, z, sizeof z);
    }
    return 0;
#else
    (void)out;
    (void)n;
    (void)reset;
    return 1;  // FX_E_CONFIG: not a phase-timing build
#endif
}
