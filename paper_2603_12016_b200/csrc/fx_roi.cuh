// Per-ROI warp pipeline: one warp computes every requested group of one ROI
// from its bbox window.  Shared by the S kernels (window staged in shared
// memory by TMA) and the L kernel (global-memory slab, plain loads).
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

struct Layout {  // byte offsets inside one warp's slab
    uint32_t rowmask, rowoff, vals, xy;         // region A (whole ROI lifetime)
    uint32_t stage;                             // region B, load phase (TMA tile)
    uint32_t tmp, sorted, cnt;                  // region B, sort / intensity phase
    uint32_t kmask, emask, runoff, rs, re, parent, rsize;  // region B, edge phase
    uint32_t lvl, keys, keys2, gcnt, marg, gstat;          // region B, glcm phase
    uint32_t bytes;
    uint32_t H, WPR, NMAX, RUNMAX;
};

__host__ __device__ constexpr uint32_t al(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }
__host__ __device__ constexpr uint32_t mx(uint32_t a, uint32_t b) { return a > b ? a : b; }

__host__ __device__ constexpr Layout make_layout(uint32_t H, uint32_t WPR, uint32_t NMAX,
                                                 uint32_t RUNMAX, uint32_t xy_bytes,
                                                 uint32_t stage_bytes) {
    Layout L{};
    L.H = H;
    L.WPR = WPR;
    L.NMAX = NMAX;
    L.RUNMAX = RUNMAX;
    uint32_t o = 0;
    L.rowmask = o;
    o += H * WPR * 8;
    L.rowoff = o;
    o = al(o + (H + 1) * 4, 16);
    L.vals = o;
    o = al(o + NMAX * 2, 16);
    L.xy = o;
    o = al(o + NMAX * xy_bytes, 128);
    const uint32_t B = o;
    // load phase
    L.stage = B;
    uint32_t e_load = B + stage_bytes;
    // sort / intensity phase
    L.tmp = B;
    L.sorted = al(L.tmp + NMAX * 2, 16);
    L.cnt = al(L.sorted + NMAX * 2, 16);
    uint32_t e_sort = L.cnt + 256 * 4;
    // edge phase
    L.kmask = B;
    L.emask = L.kmask + H * WPR * 8;
    L.runoff = L.emask + H * WPR * 8;
    L.rs = al(L.runoff + (H + 1) * 4, 16);
    L.re = al(L.rs + RUNMAX * 2, 16);
    L.parent = al(L.re + RUNMAX * 2, 16);
    L.rsize = al(L.parent + RUNMAX * 4, 16);
    uint32_t e_edge = L.rsize + RUNMAX * 4;
    // glcm phase (ng <= 256)
    L.lvl = B;
    L.keys = al(L.lvl + NMAX, 16);
    L.keys2 = al(L.keys + NMAX * 2, 16);
    L.gcnt = al(L.keys2 + NMAX * 2, 16);
    L.marg = L.gcnt + 256 * 4;
    L.gstat = al(L.marg + (256 + 256 + 512 + 256) * 4, 16);
    uint32_t e_glcm = L.gstat + 32 * 8;
    L.bytes = al(mx(mx(e_load, e_sort), mx(e_edge, e_glcm)), 128);
    return L;
}

// S-class slabs (64x64 window, one mask word per row, 8 KB TMA label tile).
constexpr uint32_t kStageBytes = kStageW * kSH * 2;
constexpr Layout kLayoutS1 = make_layout(kSH, 1, kS1N, kS1Runs, 2, kStageBytes);
constexpr Layout kLayoutS2 = make_layout(kSH, 1, kS2N, 1024, 2, kStageBytes);

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

// stable LSD radix pass on 16-bit keys by one warp (8-bit digit at `shift`)
__device__ inline void radix_pass16(const uint16_t* src, uint16_t* dst, uint32_t n, int shift,
                             uint32_t* cnt) {
    const unsigned lane = lane_id();
    for (int i = lane; i < 256; i += 32) cnt[i] = 0;
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const bool ok = i < n;
        const uint32_t d = ok ? ((uint32_t)src[i] >> shift) & 0xffu : 256u + lane;
        const unsigned peers = __match_any_sync(kFull, d);
        if (ok && lane == (unsigned)(__ffs(peers) - 1)) cnt[d] += __popc(peers);
        __syncwarp();
    }
    uint32_t c[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        c[k] = cnt[lane * 8 + k];
        s += c[k];
    }
    const uint32_t incl = warp_incl_scan(s);
    uint32_t run = incl - s;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        cnt[lane * 8 + k] = run;
        run += c[k];
    }
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const bool ok = i < n;
        const uint16_t key = ok ? src[i] : 0;
        const uint32_t d = ok ? ((uint32_t)key >> shift) & 0xffu : 256u + lane;
        const unsigned peers = __match_any_sync(kFull, d);
        if (ok) dst[cnt[d] + __popc(peers & lanemask_lt())] = key;
        __syncwarp();
        if (ok && lane == (unsigned)(31 - __clz(peers))) cnt[d] += __popc(peers);
        __syncwarp();
    }
}

// sort n 16-bit keys (src != tmp != dst; src == dst allowed).  A single pass
// (all keys < 256) lands in tmp; returns the buffer holding the sorted keys.
__device__ inline uint16_t* warp_sort16(const uint16_t* src, uint16_t* tmp, uint16_t* dst,
                                        uint32_t n, uint32_t* cnt, bool one_pass) {
    radix_pass16(src, tmp, n, 0, cnt);
    if (one_pass) return tmp;
    radix_pass16(tmp, dst, n, 8, cnt);
    return dst;
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

// k-th smallest (0-based) of |2*s[i] - M2| over sorted s: the deviations form
// a V (decreasing on [0,m), increasing on [m,n)); classic k-th of two sorted
// arrays.  A[j] = M2 - 2 s[m-1-j] (j < m), B[j] = 2 s[m+j] - M2.
__device__ inline uint32_t kth_dev2(const uint16_t* s, uint32_t n, uint32_t M2, uint32_t k) {
    // m = first index with 2*s[i] >= M2
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (2u * s[mid] >= M2) hi = mid;
        else lo = mid + 1;
    }
    const uint32_t m = lo, na = m, nb = n - m;
    // find split: take i from A, k+1-i from B
    uint32_t ilo = (k + 1 > nb) ? k + 1 - nb : 0, ihi = (k + 1 < na) ? k + 1 : na;
    while (ilo < ihi) {
        const uint32_t i = (ilo + ihi) >> 1;  // elements taken from A
        const uint32_t j = k + 1 - i;         // from B
        // A[i] < B[j-1] -> need more from A
        const uint32_t Ai = M2 - 2u * s[m - 1 - i];
        const uint32_t Bj1 = 2u * s[m + j - 1] - M2;
        if (Ai < Bj1) ilo = i + 1;
        else ihi = i;
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

}  // namespace fxg
