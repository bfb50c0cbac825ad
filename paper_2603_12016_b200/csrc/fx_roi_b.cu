// Large-ROI path (class L: window wider or taller than 64, plus S-class ROIs
// re-queued for run capacity): one 512-thread CTA per ROI, persistent over the
// L work list, per-CTA scratch slab in global memory (L2-resident).
//
// Same columns and the same exact-integer / literal-expression rules as the S
// kernels (fx_roi_s.cu), re-designed for windows of up to 65536 x 65536:
//  - membership words (u64 per 64 window columns) by warp ballots, pixel list in
//    row-major order by a block scan of word popcounts;
//  - intensity statistics from a 65536-bin value histogram (global) plus a
//    256-bin coarse prefix in shared memory: every order statistic is a two-level
//    search, the median absolute deviation a binary search over deviations d with
//    F(d) = C((M2+d)/2) - C((M2-d)/2 - 1); no sort (reference intensity_features
//    .cpp:14-215);
//  - contour edge set ("definition B" == trace_contour's visited set): run
//    union-find over the window (8-connected components, largest with row-major
//    tie-break; 4-connected exterior of the rest), edge = K & (dilate4(E) | border)
//    (contour.cpp:30-144);
//  - moments: separable row sums about integer anchors, fp64 block reduction,
//    binomial shift (moments.cpp:32-92);
//  - GLCM (ng <= 256): pair counts in a global ng x ng histogram, one dense pass
//    in fixed thread order (deterministic), integer cell sums, shared-memory
//    marginals, Haralick from marginals (texture.cpp:29-217).
#include "fx_dev.cuh"
#include "fx_glcm.cuh"
#include "fx_roi.cuh"

#ifdef FXG_PHASE_TIMING
__device__ unsigned long long g_phase_clk_b[8];
#define BT_DECL long long bt_t_ = clock64();
#define BT(k)                                                                  \
    do {                                                                       \
        const long long t_ = clock64();                                        \
        if (threadIdx.x == 0) atomicAdd(&g_phase_clk_b[k], (unsigned long long)(t_ - bt_t_)); \
        bt_t_ = t_;                                                            \
    } while (0)
#else
#define BT_DECL
#define BT(k)
#endif

namespace fxg {

namespace {

constexpr int kBT = 512;
constexpr int kBW = kBT / 32;
constexpr uint32_t kSmemCells = 128 * 128;  // shared GLCM histogram up to ng = 128 (64 KB)

__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

// all-reduce over the CTA; sh: >= kBW + 1 elements of T, reusable after return
template <typename T, typename Op>
__device__ __forceinline__ T block_all(T v, T* sh, Op op) {
    const unsigned lane = lane_id(), w = warp_id();
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {  // lanes 0..kBW-1 reduce the warp partials (xor offsets < kBW)
        T t = sh[lane & (kBW - 1)];
#pragma unroll
        for (int o = kBW / 2; o; o >>= 1) t = op(t, __shfl_xor_sync(kFull, t, o));
        if (lane == 0) sh[kBW] = t;
    }
    __syncthreads();
    const T r = sh[kBW];
    __syncthreads();
    return r;
}
struct OpAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpMin {
    template <typename T>
    __device__ T operator()(T a, T b) const { return b < a ? b : a; }
};
struct OpMax {
    template <typename T>
    __device__ T operator()(T a, T b) const { return b > a ? b : a; }
};

// exclusive scan of a[0..N) in place (a[N] = total); sh: >= kBW + 2 u32
__device__ uint32_t block_exscan(uint32_t* a, uint32_t N, uint32_t* sh) {
    const unsigned lane = lane_id(), w = warp_id();
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < N; b0 += kBT) {
        const uint32_t i = b0 + threadIdx.x;
        const uint32_t v = i < N ? a[i] : 0u;
        const uint32_t incl = warp_incl_scan(v);
        if (lane == 31) sh[w] = incl;
        __syncthreads();
        if (w == 0) {
            const uint32_t t = lane < kBW ? sh[lane] : 0u;
            const uint32_t ti = warp_incl_scan(t);
            if (lane < kBW) sh[lane] = ti - t;
            if (lane == 31) sh[kBW] = ti;
        }
        __syncthreads();
        if (i < N) a[i] = carry + sh[w] + incl - v;
        carry += sh[kBW];
        __syncthreads();
    }
    if (threadIdx.x == 0) a[N] = carry;
    __syncthreads();
    return carry;
}

// number of values <= x (x in [-1, 65535]); warp-level
__device__ __forceinline__ unsigned long long count_le(int x, const uint32_t* cpre,
                                                       const uint32_t* vhist) {
    if (x < 0) return 0ull;
    if (x > 65535) x = 65535;
    const unsigned lane = lane_id();
    const int hb = x >> 8, lb = x & 255;
    const uint4* f = reinterpret_cast<const uint4*>(vhist + hb * 256 + lane * 8);
    const uint4 a = f[0], b = f[1];
    const uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if ((int)lane * 8 + j <= lb) s += c[j];
    return (unsigned long long)cpre[hb] + warp_sum(s);
}

// r-th smallest value (0-based) of the multiset; warp-level
__device__ __forceinline__ uint32_t kth_value(unsigned long long r, const uint32_t* cpre,
                                              const uint32_t* vhist) {
    const unsigned lane = lane_id();
    // bucket: number of buckets whose end prefix is <= r
    uint32_t nb = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) nb += (unsigned long long)cpre[lane * 8 + j + 1] <= r;
    const uint32_t hb = warp_sum(nb);
    const uint4* f = reinterpret_cast<const uint4*>(vhist + hb * 256 + lane * 8);
    const uint4 a = f[0], b = f[1];
    const uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += c[j];
    const uint32_t incl = warp_incl_scan(t);
    unsigned long long run = (unsigned long long)cpre[hb] + incl - t;
    uint32_t found = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (r >= run && r < run + c[j]) found = hb * 256 + lane * 8 + j + 1;
        run += c[j];
    }
    return __reduce_max_sync(kFull, found) - 1;
}

// percentile_exact on the implicit sorted sequence (same literal expression)
__device__ __forceinline__ double percentile_h(double p, unsigned long long n, const uint32_t* cpre,
                                               const uint32_t* vhist) {
    if (n == 1) return (double)kth_value(0, cpre, vhist);
    const double rank = __dmul_rn(__ddiv_rn(p, 100.0), (double)(n - 1));
    const unsigned long long lo = (unsigned long long)rank;
    if (lo + 1 >= n) return (double)kth_value(n - 1, cpre, vhist);
    const double frac = __dsub_rn(rank, (double)lo);
    const double a = (double)kth_value(lo, cpre, vhist), b = (double)kth_value(lo + 1, cpre, vhist);
    return __dadd_rn(a, __dmul_rn(frac, __dsub_rn(b, a)));
}

// k-th smallest (0-based) of |2 v - M2| over the multiset; warp-level binary search
__device__ uint32_t kth_dev_h(unsigned long long k, uint32_t M2, const uint32_t* cpre,
                              const uint32_t* vhist) {
    uint32_t lo = 0, hi = 131071;
    while (lo < hi) {
        const uint32_t d = (lo + hi) >> 1;
        // v with M2 - d <= 2 v <= M2 + d
        const int vhi = (int)((M2 + d) >> 1);
        const int dlo = (int)M2 - (int)d;
        const int vlo = dlo <= 0 ? 0 : (dlo + 1) >> 1;
        const unsigned long long F = count_le(vhi, cpre, vhist) - count_le(vlo - 1, cpre, vhist);
        if (F > k) hi = d;
        else lo = d + 1;
    }
    return lo;
}

struct BSlab {
    uint64_t *rowmask, *kmask, *emask;
    uint32_t *wordoff, *tmpw, *xy;
    uint16_t* vals;
    uint16_t* lraster;
    uint8_t* lvl;
    uint32_t *vhist, *runoff, *parent, *rsize, *bins, *ghist;
    uint16_t *rs, *re;
    uint32_t *ctop, *cbot, *hv;  // shape: column extremes, hull chain
};

__device__ __forceinline__ BSlab bslab(uint8_t* base, const BLayout& B) {
    BSlab S;
    S.rowmask = (uint64_t*)(base + B.rowmask);
    S.kmask = (uint64_t*)(base + B.kmask);
    S.emask = (uint64_t*)(base + B.emask);
    S.wordoff = (uint32_t*)(base + B.wordoff);
    S.tmpw = (uint32_t*)(base + B.tmpw);
    S.xy = (uint32_t*)(base + B.xy);
    S.vals = (uint16_t*)(base + B.vals);
    S.lraster = (uint16_t*)(base + B.lraster);
    S.lvl = base + B.lvl;
    S.vhist = (uint32_t*)(base + B.vhist);
    S.runoff = (uint32_t*)(base + B.runoff);
    S.rs = (uint16_t*)(base + B.rs);
    S.re = (uint16_t*)(base + B.re);
    S.parent = (uint32_t*)(base + B.parent);
    S.rsize = (uint32_t*)(base + B.rsize);
    S.bins = (uint32_t*)(base + B.bins);
    S.ghist = (uint32_t*)(base + B.ghist);
    S.ctop = (uint32_t*)(base + B.ctop);
    S.cbot = (uint32_t*)(base + B.cbot);
    S.hv = (uint32_t*)(base + B.hv);
    return S;
}

// runs of set bits of m (rows of wpr words) -> rs/re, runoff; parent[r] = r.
// Returns the run count, or ~0u past capacity.
__device__ uint32_t build_runs(const uint64_t* m, int h, int wpr, const BSlab& S, uint32_t runmax,
                               uint32_t* sh) {
    for (int y = threadIdx.x; y < h; y += kBT) {
        uint32_t c = 0;
        uint64_t prev = 0;
        for (int k = 0; k < wpr; ++k) {
            const uint64_t x = m[(size_t)y * wpr + k];
            c += __popcll(x & ~((x << 1) | (prev >> 63)));
            prev = x;
        }
        S.runoff[y] = c;
    }
    __syncthreads();
    const uint32_t total = block_exscan(S.runoff, (uint32_t)h, sh);
    if (total > runmax) return ~0u;
    for (int y = threadIdx.x; y < h; y += kBT) {
        uint32_t j = S.runoff[y];
        int open = 0;
        for (int k = 0; k < wpr; ++k) {
            const uint64_t x = m[(size_t)y * wpr + k];
            const uint64_t pv = k ? m[(size_t)y * wpr + k - 1] : 0ull;
            const uint64_t nx = k + 1 < wpr ? m[(size_t)y * wpr + k + 1] : 0ull;
            uint64_t st = x & ~((x << 1) | (pv >> 63));
            uint64_t en = x & ~((x >> 1) | (nx << 63));
            while (st | en) {
                const int bs = st ? __ffsll((long long)st) - 1 : 64;
                const int be = en ? __ffsll((long long)en) - 1 : 64;
                if (bs <= be) {
                    open = k * 64 + bs;
                    st &= st - 1;
                } else {
                    S.rs[j] = (uint16_t)open;
                    S.re[j] = (uint16_t)(k * 64 + be);
                    ++j;
                    en &= en - 1;
                }
            }
        }
    }
    for (uint32_t r = threadIdx.x; r < total; r += kBT) S.parent[r] = r;
    __syncthreads();
    return total;
}

// union of runs in adjacent rows (ext 1: 8-connected, 0: 4-connected), then flatten
__device__ void unite_runs(int h, int ext, const BSlab& S) {
    for (int y = 1 + threadIdx.x; y < h; y += kBT) {
        uint32_t i = S.runoff[y], ie = S.runoff[y + 1], j = S.runoff[y - 1], je = S.runoff[y];
        while (i < ie && j < je) {
            const int as = S.rs[i], ae = S.re[i], bs = S.rs[j], be = S.re[j];
            if (be + ext < as) ++j;
            else if (ae + ext < bs) ++i;
            else {
                uf_union(S.parent, i, j);
                if (ae < be) ++i;
                else ++j;
            }
        }
    }
    __syncthreads();
    // flatten in two phases: a compressing find could overwrite a root another
    // thread has just published with an older ancestor
    const uint32_t nr = S.runoff[h];
    for (uint32_t r = threadIdx.x; r < nr; r += kBT) S.rsize[r] = uf_root(S.parent, r);
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < nr; r += kBT) S.parent[r] = S.rsize[r];
    __syncthreads();
}

// set bits [a, b] of a row of words
__device__ __forceinline__ void set_bits(uint64_t* row, int a, int b) {
    for (int k = a >> 6; k <= (b >> 6); ++k) {
        const int lo = k == (a >> 6) ? (a & 63) : 0, hi = k == (b >> 6) ? (b & 63) : 63;
        row[k] |= bits_between(lo, hi);
    }
}

struct BShared {
    uint32_t coarse[256];
    uint32_t cpre[257];
    uint32_t scan[kBW + 2];
    unsigned long long u64s[kBW + 1];
    double f64s[kBW + 1];
    uint32_t u32s[kBW + 1];
    double red[kBW][33];
    uint32_t px[256], py[256], psum[512], pdif[256];
    uint32_t job;
};

// K (largest 8-connected component, row-major tie-break) into S.kmask and E
// (4-connected exterior of the window cells outside K) into S.emask, by run
// union-find; false past the run capacity (contour.cpp:30-66)
__device__ bool block_ke(int h, int w, int wpr, uint32_t nw, const BSlab& S, const BLayout& B,
                         BShared& sm) {
    const unsigned tid = threadIdx.x;
    const uint64_t lastm = (w & 63) ? ((1ull << (w & 63)) - 1ull) : ~0ull;
    uint32_t nr = build_runs(S.rowmask, h, wpr, S, B.RUNMAX, sm.scan);
    bool ok = nr != ~0u;
    if (ok) {
        unite_runs(h, 1, S);
        for (uint32_t q = tid; q < nr; q += kBT) S.rsize[q] = 0u;
        __syncthreads();
        for (uint32_t q = tid; q < nr; q += kBT)
            atomicAdd(&S.rsize[S.parent[q]], (uint32_t)(S.re[q] - S.rs[q] + 1));
        __syncthreads();
        unsigned long long bk = 0;
        for (uint32_t q = tid; q < nr; q += kBT)
            if (S.parent[q] == q) {
                const unsigned long long key = ((unsigned long long)S.rsize[q] << 32) |
                                               (0xffffffffu - q);
                bk = key > bk ? key : bk;
            }
        bk = block_all(bk, sm.u64s, OpMax());
        const uint32_t broot = 0xffffffffu - (uint32_t)(bk & 0xffffffffu);
        for (uint32_t wi = tid; wi < nw; wi += kBT) S.kmask[wi] = 0ull;
        __syncthreads();
        for (int y = tid; y < h; y += kBT)
            for (uint32_t q = S.runoff[y]; q < S.runoff[y + 1]; ++q)
                if (S.parent[q] == broot) set_bits(S.kmask + (size_t)y * wpr, S.rs[q], S.re[q]);
        __syncthreads();
        // free cells of the window (not in K) -> 4-connected exterior
        for (uint32_t wi = tid; wi < nw; wi += kBT)
            S.emask[wi] = ~S.kmask[wi] & ((int)(wi % wpr) == wpr - 1 ? lastm : ~0ull);
        __syncthreads();
        const uint32_t nf = build_runs(S.emask, h, wpr, S, B.RUNMAX, sm.scan);
        ok = nf != ~0u;
        if (ok) {
            unite_runs(h, 0, S);
            for (uint32_t q = tid; q < nf; q += kBT) S.rsize[q] = 0u;
            __syncthreads();
            for (int y = tid; y < h; y += kBT)
                for (uint32_t q = S.runoff[y]; q < S.runoff[y + 1]; ++q)
                    if (y == 0 || y == h - 1 || S.rs[q] == 0 || S.re[q] == w - 1)
                        S.rsize[S.parent[q]] = 1u;
            __syncthreads();
            for (uint32_t wi = tid; wi < nw; wi += kBT) S.emask[wi] = 0ull;
            __syncthreads();
            for (int y = tid; y < h; y += kBT)
                for (uint32_t q = S.runoff[y]; q < S.runoff[y + 1]; ++q)
                    if (S.rsize[S.parent[q]]) set_bits(S.emask + (size_t)y * wpr, S.rs[q], S.re[q]);
            __syncthreads();
        }
    }
    return ok;
}

// ---------------------------------------------------------------------------
// Shape group of a large ROI (shape_features.cpp:147-251), block-level; same
// rules as shape_phase_s (fx_roi_s.cu).  Thread 0 replays the Moore walk of
// contour.cpp:70-144 on K with Brent's cycle detection (no per-state memory for
// windows of any size) and builds the monotone-chain hull of the column extremes;
// threads 1..3 sum the ellipse terms in pixel order; the rest is parallel.
__constant__ int8_t c_ring_b[8][2] = {{-1, 0}, {-1, -1}, {0, -1}, {1, -1},
                                      {1, 0},  {1, 1},   {0, 1},  {-1, 1}};
__constant__ int8_t c_ring_of_b[9] = {1, 0, 7, 2, -1, 6, 3, 4, 5};

struct WalkState {
    int x, y, b;
    __device__ bool operator==(const WalkState& o) const { return x == o.x && y == o.y && b == o.b; }
    __device__ bool operator!=(const WalkState& o) const { return !(*this == o); }
};

__device__ __forceinline__ bool kb_at(const uint64_t* km, int h, int w, int wpr, int x, int y) {
    return x >= 0 && x < w && y >= 0 && y < h &&
           ((km[(size_t)y * wpr + (x >> 6)] >> (x & 63)) & 1ull);
}

__device__ WalkState walk_next(const uint64_t* km, int h, int w, int wpr, WalkState s) {
    int found = -1;
    for (int k = 1; k <= 8; ++k) {
        const int idx = (s.b + k) & 7;
        if (kb_at(km, h, w, wpr, s.x + c_ring_b[idx][0], s.y + c_ring_b[idx][1])) {
            found = idx;
            break;
        }
    }
    const int prev = (found + 7) & 7;
    const int ddx = c_ring_b[prev][0] - c_ring_b[found][0], ddy = c_ring_b[prev][1] - c_ring_b[found][1];
    return WalkState{s.x + c_ring_b[found][0], s.y + c_ring_b[found][1],
                     c_ring_of_b[(ddx + 1) * 3 + (ddy + 1)]};
}

__device__ __forceinline__ long long floor_div_b(long long a, long long b) {  // b > 0
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}

__device__ void shape_b(int h, int w, int wpr, uint32_t nw, uint32_t n, long long gx0,
                        long long gy0, unsigned long long sX, unsigned long long sY,
                        const BSlab& S, BShared& sm, double* o) {
    const unsigned tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    const double PI = 3.141592653589793, SQRT2 = 1.4142135623730951;
    const double dn = (double)n;
    constexpr uint32_t kNone = 0xffffffffu;
    // column extremes of all pixels
    for (int x = tid; x < w; x += kBT) {
        uint32_t t = kNone, bt = kNone;
        for (int y = 0; y < h; ++y)
            if ((S.rowmask[(size_t)y * wpr + (x >> 6)] >> (x & 63)) & 1ull) {
                if (t == kNone) t = (uint32_t)y;
                bt = (uint32_t)y;
            }
        S.ctop[x] = t;
        S.cbot[x] = bt;
    }
    // |K| and the 8-connected Euler number (bit quads over the zero-padded window:
    // row pairs (y-1, y), y = 0..h; word k covers columns 64k..64k+63, word wpr the
    // padded column when w is a multiple of 64)
    unsigned long long kc = 0;
    for (uint32_t wi = tid; wi < nw; wi += kBT) kc += __popcll(S.kmask[wi]);
    long long q = 0;
    const uint32_t nq = (uint32_t)(h + 1) * (uint32_t)(wpr + 1);
    for (uint32_t qi = tid; qi < nq; qi += kBT) {
        const int y = (int)(qi / (wpr + 1)), k = (int)(qi % (wpr + 1));
        auto word = [&](int yy, int kk) -> uint64_t {
            return (yy >= 0 && yy < h && kk >= 0 && kk < wpr) ? S.rowmask[(size_t)yy * wpr + kk] : 0ull;
        };
        const uint64_t a = word(y - 1, k), b = word(y, k), ap = word(y - 1, k - 1), bp = word(y, k - 1);
        const int lim = w - 64 * k;  // positions j <= lim are columns 0..w
        const uint64_t vm = lim >= 63 ? ~0ull : ((2ull << lim) - 1ull);
        const uint64_t A0 = (a << 1) | (ap >> 63), A1 = a, B0 = (b << 1) | (bp >> 63), B1 = b;
        const uint64_t s1 = A0 ^ A1, s2 = B0 ^ B1, c = (A0 & A1) | (B0 & B1);
        const uint64_t one = (s1 ^ s2) & ~c & vm, three = (s1 ^ s2) & c & vm;
        const uint64_t dg = ((A0 & B1 & ~A1 & ~B0) | (A1 & B0 & ~A0 & ~B1)) & vm;
        q += __popcll(one) - __popcll(three) - 2 * __popcll(dg);
    }
    kc = block_all(kc, sm.u64s, OpAdd());
    q = (long long)block_all((unsigned long long)q, sm.u64s, OpAdd());
    const double cx = (double)((unsigned long long)gx0 * n + sX) / dn;
    const double cy = (double)((unsigned long long)gy0 * n + sY) / dn;
    // thread 0: perimeter and hull; threads 1..3: ellipse sums
    if (tid == 0) {
        double per = 4.0;
        if (n > 1 && kc > 1) {
            int sy = 0;
            while (true) {
                bool any = false;
                for (int k = 0; k < wpr; ++k) any |= S.kmask[(size_t)sy * wpr + k] != 0ull;
                if (any) break;
                ++sy;
            }
            int sx = 0;
            for (int k = 0; k < wpr; ++k) {
                const uint64_t m = S.kmask[(size_t)sy * wpr + k];
                if (m) {
                    sx = k * 64 + __ffsll((long long)m) - 1;
                    break;
                }
            }
            const WalkState s0{sx, sy, 0};
            // Brent: cycle length lam, then the first state of the cycle
            uint32_t power = 1, lam = 1;
            WalkState tort = s0, hare = walk_next(S.kmask, h, w, wpr, s0);
            while (tort != hare) {
                if (power == lam) {
                    tort = hare;
                    power *= 2;
                    lam = 0;
                }
                hare = walk_next(S.kmask, h, w, wpr, hare);
                ++lam;
            }
            tort = hare = s0;
            for (uint32_t i = 0; i < lam; ++i) hare = walk_next(S.kmask, h, w, wpr, hare);
            while (tort != hare) {
                tort = walk_next(S.kmask, h, w, wpr, tort);
                hare = walk_next(S.kmask, h, w, wpr, hare);
            }
            per = 0;
            WalkState cur = tort;
            for (uint32_t i = 0; i < lam; ++i) {
                const WalkState nx = walk_next(S.kmask, h, w, wpr, cur);
                per = __dadd_rn(per, (abs(nx.x - cur.x) + abs(nx.y - cur.y) == 2) ? SQRT2 : 1.0);
                cur = nx;
            }
        }
        sm.red[0][0] = per;
        // monotone-chain hull of the column extremes (hull.cpp:17-55)
        uint32_t* hv = S.hv;  // (x | y << 16), chain stack
        auto X = [&](int i) { return (long long)(hv[i] & 0xffffu); };
        auto Y = [&](int i) { return (long long)(hv[i] >> 16); };
        int k = 0, npt = 0, fx = -1;
        uint32_t fy = 0, lx = 0, ly = 0;
        auto push = [&](int px, uint32_t py, int lo) {
            while (k >= lo && (X(k - 1) - X(k - 2)) * ((long long)py - Y(k - 2)) -
                                      (Y(k - 1) - Y(k - 2)) * ((long long)px - X(k - 2)) <= 0)
                --k;
            hv[k++] = (uint32_t)px | (py << 16);
        };
        for (int x = 0; x < w; ++x)
            if (S.ctop[x] != kNone) {
                npt += S.ctop[x] == S.cbot[x] ? 1 : 2;
                if (fx < 0) {
                    fx = x;
                    fy = S.ctop[x];
                }
                lx = (uint32_t)x;
                ly = S.cbot[x];
            }
        if (npt <= 2) {
            for (int x = 0; x < w; ++x)
                if (S.ctop[x] != kNone) {
                    hv[k++] = (uint32_t)x | (S.ctop[x] << 16);
                    if (S.cbot[x] != S.ctop[x]) hv[k++] = (uint32_t)x | (S.cbot[x] << 16);
                }
        } else {
            for (int x = 0; x < w; ++x)
                if (S.ctop[x] != kNone) {
                    push(x, S.ctop[x], 2);
                    if (S.cbot[x] != S.ctop[x]) push(x, S.cbot[x], 2);
                }
            const int lower = k + 1;
            bool skip_last = true;
            for (int x = w - 1; x >= 0; --x)
                if (S.ctop[x] != kNone) {
                    if (S.cbot[x] != S.ctop[x]) {
                        if (!skip_last) push(x, S.cbot[x], lower);
                        skip_last = false;
                        push(x, S.ctop[x], lower);
                    } else {
                        if (!skip_last) push(x, S.ctop[x], lower);
                        skip_last = false;
                    }
                }
            k -= 1;
            if (k < 3) {
                hv[0] = (uint32_t)fx | (fy << 16);
                hv[1] = lx | (ly << 16);
                k = 2;
            }
        }
        sm.u32s[kBW] = (uint32_t)k;  // hull vertex count
    } else if (tid <= 3) {
        double e = 0;  // m20 (1), m02 (2), m11 (3), pixel order, no FMA
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t p = S.xy[i];
            const double dx = __dsub_rn((double)(gx0 + (long long)(p & 0xffffu)), cx);
            const double dy = __dsub_rn((double)(gy0 + (long long)(p >> 16)), cy);
            const double t = tid == 1 ? __dmul_rn(dx, dx) : tid == 2 ? __dmul_rn(dy, dy) : __dmul_rn(dx, dy);
            e = __dadd_rn(e, t);
        }
        sm.red[0][tid] = e;
    }
    __syncthreads();
    const double per = sm.red[0][0], m20 = sm.red[0][1], m02 = sm.red[0][2], m11 = sm.red[0][3];
    const int nv = (int)sm.u32s[kBW];
    const uint32_t* hv = S.hv;
    // convex area: lattice points inside or on the hull, rows in parallel
    unsigned long long carea = 0;
    if (nv >= 3)
        for (int y = tid; y < h; y += kBT) {
            long long xl = 0, xr = w - 1;
            for (int i = 0; i < nv && xl <= xr; ++i) {
                const int j = i + 1 < nv ? i + 1 : 0;
                const long long ax = hv[i] & 0xffffu, ay = hv[i] >> 16, bx = hv[j] & 0xffffu,
                                by = hv[j] >> 16;
                const long long Bq = by - ay, Aq = (bx - ax) * (y - ay) + Bq * ax;  // Aq - Bq x >= 0
                if (Bq > 0) xr = min(xr, floor_div_b(Aq, Bq));
                else if (Bq < 0) xl = max(xl, -floor_div_b(Aq, -Bq));
                else if (Aq < 0) xr = -1;
            }
            if (xr >= xl) carea += (unsigned long long)(xr - xl + 1);
        }
    carea = block_all(carea, sm.u64s, OpAdd());
    // Feret diameters over the hull vertices
    double fmx = 0, fmn = 1.79769313486231570815e308;
    const unsigned long long npair = (unsigned long long)nv * (unsigned long long)nv;
    for (unsigned long long pi = tid; pi < npair; pi += kBT) {
        const int i = (int)(pi / nv), j = (int)(pi % nv);
        if (j > i) {
            const double dx = (double)((long long)(hv[i] & 0xffffu) - (long long)(hv[j] & 0xffffu));
            const double dy = (double)((long long)(hv[i] >> 16) - (long long)(hv[j] >> 16));
            fmx = fmax(fmx, hypot(dx, dy));
        }
    }
    for (int i = tid; i < nv && nv > 2; i += kBT) {
        const int j = i + 1 < nv ? i + 1 : 0;
        const long long ax = hv[i] & 0xffffu, ay = hv[i] >> 16;
        const long long ex = (long long)(hv[j] & 0xffffu) - ax, ey = (long long)(hv[j] >> 16) - ay;
        long long mc = 0;
        for (int kk = 0; kk < nv; ++kk) {
            const long long c = ex * ((long long)(hv[kk] >> 16) - ay) - ey * ((long long)(hv[kk] & 0xffffu) - ax);
            mc = max(mc, c < 0 ? -c : c);
        }
        fmn = fmin(fmn, (double)mc / hypot((double)ex, (double)ey));
    }
    fmx = block_all(fmx, sm.f64s, OpMax());
    fmn = block_all(fmn, sm.f64s, OpMin());
    if (nv <= 2) fmn = 0;
    if (wid == 0) {
        const double bw = (double)w, bh = (double)h;
        double v = 0;
        if (lane < 22) {
            switch (lane) {
                case 0: v = dn; break;
                case 1: v = per; break;
                case 2: v = (double)gx0; break;
                case 3: v = (double)gy0; break;
                case 4: v = bw; break;
                case 5: v = bh; break;
                case 6: v = cx; break;
                case 7: v = cy; break;
                case 8: v = n == 1 ? 1.0 : 4.0 * PI * dn / (per * per); break;
                case 9: v = dn / (bw * bh); break;
                case 10: v = bw / bh; break;
                case 11: v = (double)carea; break;
                case 12: v = carea ? dn / (double)carea : 0.0; break;
                case 13: v = sqrt(4.0 * dn / PI); break;
                case 19: v = (double)(q / 4); break;
                case 20: v = fmx; break;
                case 21: v = fmn; break;
                default: {
                    const double a = __dadd_rn(__ddiv_rn(m20, dn), 1.0 / 12.0);
                    const double c = __dadd_rn(__ddiv_rn(m02, dn), 1.0 / 12.0);
                    const double bb = __ddiv_rn(m11, dn);
                    const double amc = __dsub_rn(a, c);
                    const double disc =
                        sqrt(__dadd_rn(__ddiv_rn(__dmul_rn(amc, amc), 4.0), __dmul_rn(bb, bb)));
                    const double hs = __ddiv_rn(__dadd_rn(a, c), 2.0);
                    const double l1 = __dadd_rn(hs, disc), l2 = __dsub_rn(hs, disc);
                    const double maj = 4.0 * sqrt(fmax(0.0, l1)), mnr = 4.0 * sqrt(fmax(0.0, l2));
                    if (lane == 14) v = maj;
                    else if (lane == 15) v = mnr;
                    else if (lane == 16) v = l1 > 0 ? sqrt(fmax(0.0, 1.0 - l2 / l1)) : 0.0;
                    else if (lane == 17) v = mnr > 0 ? maj / mnr : 0.0;
                    else {
                        v = ellipse_orientation(bb, amc);
                    }
                }
            }
            o[lane] = v;
        } else if (lane < 30) {  // extrema
            const int e = lane - 22;
            auto row_lo = [&](int y) {
                for (int k = 0; k < wpr; ++k) {
                    const uint64_t m = S.rowmask[(size_t)y * wpr + k];
                    if (m) return k * 64 + __ffsll((long long)m) - 1;
                }
                return 0;
            };
            auto row_hi = [&](int y) {
                for (int k = wpr - 1; k >= 0; --k) {
                    const uint64_t m = S.rowmask[(size_t)y * wpr + k];
                    if (m) return k * 64 + 63 - __clzll((long long)m);
                }
                return 0;
            };
            int ex = 0, ey = 0;
            switch (e) {
                case 0: ex = row_lo(0); ey = 0; break;
                case 1: ex = row_hi(0); ey = 0; break;
                case 2: ex = w - 1; ey = (int)S.ctop[w - 1]; break;
                case 3: ex = w - 1; ey = (int)S.cbot[w - 1]; break;
                case 4: ex = row_hi(h - 1); ey = h - 1; break;
                case 5: ex = row_lo(h - 1); ey = h - 1; break;
                case 6: ex = 0; ey = (int)S.cbot[0]; break;
                default: ex = 0; ey = (int)S.ctop[0]; break;
            }
            o[22 + 2 * e] = (double)(gx0 + ex);
            o[23 + 2 * e] = (double)(gy0 + ey);
        }
    }
    __syncthreads();
}

__device__ void process_b(uint32_t r, const DevImage& img, const RoiList& rl, Control* ctl,
                          const FeatCfg& cfg, double* __restrict__ out, const DebugOut* dbg,
                          const BSlab& S, const BLayout& B, BShared& sm, uint32_t* dyn) {
    const unsigned tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    const uint32_t label = rl.label[r];
    const int w = (int)rl.w[r], h = (int)rl.h[r];
    const uint32_t x0 = rl.x0[r], y0 = rl.y0[r];
    const long long gx0 = rl.gx[r], gy0 = rl.gy[r];
    const int wpr = (w + 63) >> 6;
    const uint32_t nw = (uint32_t)h * (uint32_t)wpr;
    double* orow = out + (size_t)r * cfg.ncols;
    const bool dbg_on = dbg != nullptr && dbg->label == label;
    const bool want_int = cfg.col_int >= 0, want_mom = cfg.col_mom >= 0, want_glcm = cfg.col_glcm >= 0;
    const bool want_shape = cfg.col_shape >= 0;

    BT_DECL
    // ---- membership words (warp per 64-column word) and popcounts; a warp takes
    // kBU consecutive words per step and issues all their loads before the ballots
    // (one word per step left the loop latency-bound: a slide-tall window's 0.5M
    // words took ~20 ms on one CTA)
    constexpr uint32_t kBU = 8;
    for (uint32_t wb = wid * kBU; wb < nw; wb += kBW * kBU) {
        uint32_t va[kBU], vb[kBU];
#pragma unroll
        for (uint32_t u = 0; u < kBU; ++u) {
            const uint32_t wi = wb + u;
            va[u] = vb[u] = 0u;  // never equal to a label (labels are >= 1)
            if (wi < nw) {
                const int y = (int)(wi / wpr), k = (int)(wi % wpr);
                const uint16_t* row = img.L + (size_t)(y0 + y) * img.pitch + x0;
                const int xa = k * 64 + (int)lane, xb = xa + 32;
                if (xa < w) va[u] = row[xa];
                if (xb < w) vb[u] = row[xb];
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < kBU; ++u) {
            const unsigned lo = __ballot_sync(kFull, va[u] == label);
            const unsigned hi = __ballot_sync(kFull, vb[u] == label);
            if (lane == 0 && wb + u < nw) {
                const uint64_t m = (uint64_t)lo | ((uint64_t)hi << 32);
                S.rowmask[wb + u] = m;
                S.wordoff[wb + u] = __popcll(m);
            }
        }
    }
    for (int i = tid; i < 256; i += kBT) sm.coarse[i] = 0u;
    __syncthreads();
    const uint32_t n = block_exscan(S.wordoff, nw, sm.scan);
    const double dn = (double)n;
    BT(0);

    // ---- pixel list (row-major), intensities, exact integer sums, value histogram
    unsigned long long sS = 0, sQ = 0, sX = 0, sY = 0, sXI = 0, sYI = 0;
    uint32_t vlo = 0xffffu, vhi = 0u;
    // (kBP words per warp step, their intensity loads issued together)
    constexpr uint32_t kBP = 4;
    for (uint32_t wb = wid * kBP; wb < nw; wb += kBW * kBP) {
      uint64_t mw[kBP];
      uint32_t vv[kBP][2];
#pragma unroll
      for (uint32_t u = 0; u < kBP; ++u) {
        const uint32_t wi = wb + u;
        mw[u] = wi < nw ? S.rowmask[wi] : 0ull;
        const uint16_t* Irow = img.I + (size_t)(y0 + wi / wpr) * img.pitch + x0 + (wi % wpr) * 64;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
            vv[u][hf] = ((mw[u] >> ((int)lane + 32 * hf)) & 1ull) ? Irow[(int)lane + 32 * hf] : 0u;
      }
#pragma unroll
      for (uint32_t u = 0; u < kBP; ++u) {
        const uint64_t m = mw[u];
        if (!m) continue;
        const uint32_t wi = wb + u;
        const uint32_t base = S.wordoff[wi];
        const uint32_t y = wi / wpr, k = wi % wpr;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int bit = (int)lane + 32 * hf;
            if (!((m >> bit) & 1ull)) continue;
            const uint32_t pos = base + __popcll(m & ((1ull << bit) - 1ull));
            const uint32_t x = k * 64 + bit;
            const uint32_t v = vv[u][hf];
            S.xy[pos] = x | (y << 16);
            S.vals[pos] = (uint16_t)v;
            sS += v;
            sQ += (unsigned long long)v * v;
            sX += x;
            sY += y;
            sXI += (unsigned long long)x * v;
            sYI += (unsigned long long)y * v;
            vlo = min(vlo, v);
            vhi = max(vhi, v);
            if (want_int) {
                atomicAdd(&S.vhist[v], 1u);
                atomicAdd(&sm.coarse[v >> 8], 1u);
            }
        }
      }
    }
    sS = block_all(sS, sm.u64s, OpAdd());
    sQ = block_all(sQ, sm.u64s, OpAdd());
    sX = block_all(sX, sm.u64s, OpAdd());
    sY = block_all(sY, sm.u64s, OpAdd());
    sXI = block_all(sXI, sm.u64s, OpAdd());
    sYI = block_all(sYI, sm.u64s, OpAdd());
    const uint32_t vmin = block_all(vlo, sm.u32s, OpMin());
    const uint32_t vmax = block_all(vhi, sm.u32s, OpMax());
    BT(1);

    bool have_k = false;
    // ------------------------------------------------------------ intensity
    if (want_int) {
        if (wid == 0) {  // coarse exclusive prefix
            uint32_t c[8], t = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = sm.coarse[lane * 8 + j];
                t += c[j];
            }
            uint32_t run = warp_incl_scan(t) - t;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                sm.cpre[lane * 8 + j] = run;
                run += c[j];
            }
            if (lane == 31) sm.cpre[256] = run;
        }
        __syncthreads();
        const double mean = (double)sS / dn;
        // per-pixel passes: central moments, mad partials, mode, entropy bins
        const uint32_t nb32 = (uint32_t)cfg.bins;
        const uint32_t rng = vmax - vmin;
        double acc[5] = {0, 0, 0, 0, 0};
        unsigned long long slo = 0, best = 0;
        uint32_t clo = 0;
        // mode key and entropy bins: per distinct value from the value histogram
        // (coalesced over [vmin, vmax]) when that range is small next to n, else per
        // pixel (a gather from the histogram and a 64-bit division each)
        const bool by_value = rng < 2u * n;
        auto bin_of = [&](uint32_t v) -> uint32_t {
            if (!rng) return 0u;
            const unsigned long long q = (unsigned long long)nb32 * (v - vmin) / rng;
            return q < nb32 - 1 ? (uint32_t)q : nb32 - 1;
        };
        for (uint32_t i = tid; i < n; i += kBT) {
            const uint32_t v = S.vals[i];
            const double d = (double)v - mean, d2 = d * d;
            acc[0] += d2;
            acc[1] += d2 * d;
            acc[2] += d2 * d2;
            acc[3] += d2 * d2 * d;
            acc[4] += d2 * d2 * d2;
            if ((double)v < mean) {
                slo += v;
                ++clo;
            }
            if (!by_value) {
                const unsigned long long key = ((unsigned long long)S.vhist[v] << 16) | (0xffffu - v);
                best = key > best ? key : best;
                atomicAdd(&S.bins[bin_of(v)], 1u);
            }
        }
        if (by_value) {
            for (uint32_t v = vmin + tid; v <= vmax; v += kBT) {
                const uint32_t c = S.vhist[v];
                if (!c) continue;
                const unsigned long long key = ((unsigned long long)c << 16) | (0xffffu - v);
                best = key > best ? key : best;
                atomicAdd(&S.bins[bin_of(v)], c);
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[k] = block_all(acc[k], sm.f64s, OpAdd());
        slo = block_all(slo, sm.u64s, OpAdd());
        clo = block_all(clo, sm.u32s, OpAdd());
        best = block_all(best, sm.u64s, OpMax());
        // entropy / uniformity over the bins; bins left zero
        const double logn = nlog2(dn);
        double ent = 0;
        unsigned long long usq = 0;
        for (uint32_t b = tid; b < nb32; b += kBT) {
            const uint32_t c = S.bins[b];
            if (c) {
                ent += (double)c * (logn - log2_int(c));
                usq += (unsigned long long)c * c;
                S.bins[b] = 0u;
                if (dbg_on) dbg->hist[b] = c;
            }
        }
        ent = block_all(ent, sm.f64s, OpAdd());
        usq = block_all(usq, sm.u64s, OpAdd());
        // order statistics, one query set per warp, shared through sm.red[0]:
        // warp 0 median + deviation k = n/2, warp 1 deviation k = n/2 - 1 (even n),
        // warps 2..7 the percentiles 1, 10, 25, 75, 90, 99
        if (wid < 8) {
            double r = 0;
            if (wid < 2) {
                const uint32_t shi = kth_value(n / 2, sm.cpre, S.vhist);
                const uint32_t slo = (n & 1) ? shi : kth_value(n / 2 - 1, sm.cpre, S.vhist);
                const uint32_t M2 = (n & 1) ? 2u * shi : slo + shi;
                if (wid == 0) {
                    const uint32_t d_hi = kth_dev_h(n / 2, M2, sm.cpre, S.vhist);
                    if (lane == 0) {
                        sm.red[0][0] = (n & 1) ? (double)shi : 0.5 * ((double)slo + (double)shi);
                        sm.red[0][8] = (double)d_hi;
                    }
                } else {
                    r = (n & 1) ? -1.0 : (double)kth_dev_h(n / 2 - 1, M2, sm.cpre, S.vhist);
                    if (lane == 0) sm.red[0][9] = r;
                }
            } else {
                const double pv = wid == 2 ? 1.0 : wid == 3 ? 10.0 : wid == 4 ? 25.0
                                : wid == 5 ? 75.0 : wid == 6 ? 90.0 : 99.0;
                r = percentile_h(pv, n, sm.cpre, S.vhist);
                if (lane == 0) sm.red[0][wid - 1] = r;
            }
        }
        __syncthreads();
        if (tid == 0) {  // median absolute deviation (intensity_features.cpp), exact
            const double d_hi = sm.red[0][8], d_lo = sm.red[0][9];
            sm.red[0][7] = (n & 1) ? 0.5 * d_hi : 0.5 * (0.5 * d_lo + 0.5 * d_hi);
        }
        __syncthreads();
        const double median = sm.red[0][0], p10 = sm.red[0][2], p25 = sm.red[0][3];
        const double p75 = sm.red[0][4], p90 = sm.red[0][5], median_ad = sm.red[0][7];
        double pct[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) pct[j] = sm.red[0][1 + j];
        __syncthreads();
        // robust mean absolute deviation over [p10, p90]
        unsigned long long rsum = 0;
        uint32_t rn = 0;
        for (uint32_t i = tid; i < n; i += kBT) {
            const double x = (double)S.vals[i];
            if (x >= p10 && x <= p90) {
                rsum += S.vals[i];
                ++rn;
            }
        }
        rsum = block_all(rsum, sm.u64s, OpAdd());
        rn = block_all(rn, sm.u32s, OpAdd());
        double rmad = 0;
        if (rn > 0) {
            const double rmean = (double)rsum / (double)rn;
            unsigned long long rlo = 0;
            uint32_t rcl = 0;
            for (uint32_t i = tid; i < n; i += kBT) {
                const double x = (double)S.vals[i];
                if (x >= p10 && x <= p90 && x < rmean) {
                    rlo += S.vals[i];
                    ++rcl;
                }
            }
            rlo = block_all(rlo, sm.u64s, OpAdd());
            rcl = block_all(rcl, sm.u32s, OpAdd());
            rmad = ((double)(long long)(rsum - 2 * rlo) +
                    (double)((long long)rcl - (long long)(rn - rcl)) * rmean) / (double)rn;
        }
        // value histogram back to zero (the value range, or the pixels' values)
        if (by_value)
            for (uint32_t v = vmin + tid; v <= vmax; v += kBT) S.vhist[v] = 0u;
        else
            for (uint32_t i = tid; i < n; i += kBT) S.vhist[S.vals[i]] = 0u;
        BT(2);

        // ---- edge set: K = largest 8-connected component, E = 4-connected exterior
        double e_mean = 0, e_min = 0, e_max = 0, e_std = 0, e_int = 0;
        {
            if (!block_ke(h, w, wpr, nw, S, B, sm)) {
                if (tid == 0) atomicOr(&ctl->error, kErrRuns);
                return;
            }
            have_k = true;
            // edge = K & (4-neighbour in E, or on the window border); exact integer sums
            unsigned long long es = 0, esq = 0;
            uint32_t en = 0, emn = 0xffffffffu, emx = 0;
            for (uint32_t wi = tid; wi < nw; wi += kBT) {
                const int y = (int)(wi / wpr), k = (int)(wi % wpr);
                const uint64_t kk = S.kmask[wi];
                uint32_t cnt = 0;
                if (kk) {
                    const uint64_t e = S.emask[wi];
                    const uint64_t el = k ? S.emask[wi - 1] : 0ull, er = k + 1 < wpr ? S.emask[wi + 1] : 0ull;
                    uint64_t g = (e << 1) | (el >> 63) | (e >> 1) | (er << 63);
                    if (y > 0) g |= S.emask[wi - wpr];
                    if (y + 1 < h) g |= S.emask[wi + wpr];
                    if (y == 0 || y == h - 1) g = ~0ull;
                    if (k == 0) g |= 1ull;
                    if (k == (w - 1) >> 6) g |= 1ull << ((w - 1) & 63);
                    uint64_t ed = kk & g;
                    cnt = __popcll(ed);
                    const uint64_t m = S.rowmask[wi];
                    const uint32_t base = S.wordoff[wi];
                    while (ed) {
                        const int b = __ffsll((long long)ed) - 1;
                        ed &= ed - 1;
                        const uint32_t v = S.vals[base + __popcll(m & ((1ull << b) - 1ull))];
                        es += v;
                        esq += (unsigned long long)v * v;
                        emn = min(emn, v);
                        emx = max(emx, v);
                    }
                }
                en += cnt;
                if (dbg_on) S.tmpw[wi] = cnt;
            }
            es = block_all(es, sm.u64s, OpAdd());
            esq = block_all(esq, sm.u64s, OpAdd());
            en = block_all(en, sm.u32s, OpAdd());
            emn = block_all(emn, sm.u32s, OpMin());
            emx = block_all(emx, sm.u32s, OpMax());
            if (en) {
                const double den = (double)en;
                e_mean = (double)es / den;
                e_min = (double)emn;
                e_max = (double)emx;
                e_int = (double)es;
                const unsigned __int128 var =
                    (unsigned __int128)en * esq - (unsigned __int128)es * es;  // n^2 var, exact
                e_std = sqrt((double)var / (den * den));
            }
            if (dbg_on) {  // edge pixels in row-major order
                __syncthreads();
                const uint32_t ne = block_exscan(S.tmpw, nw, sm.scan);
                for (uint32_t wi = tid; wi < nw; wi += kBT) {
                    const int y = (int)(wi / wpr), k = (int)(wi % wpr);
                    const uint64_t kk = S.kmask[wi];
                    if (!kk) continue;
                    const uint64_t e = S.emask[wi];
                    const uint64_t el = k ? S.emask[wi - 1] : 0ull, er = k + 1 < wpr ? S.emask[wi + 1] : 0ull;
                    uint64_t g = (e << 1) | (el >> 63) | (e >> 1) | (er << 63);
                    if (y > 0) g |= S.emask[wi - wpr];
                    if (y + 1 < h) g |= S.emask[wi + wpr];
                    if (y == 0 || y == h - 1) g = ~0ull;
                    if (k == 0) g |= 1ull;
                    if (k == (w - 1) >> 6) g |= 1ull << ((w - 1) & 63);
                    uint64_t ed = kk & g;
                    uint32_t j = S.tmpw[wi];
                    while (ed) {
                        const int b = __ffsll((long long)ed) - 1;
                        ed &= ed - 1;
                        if (j < dbg->cap_edge) {
                            dbg->edge_xy[2 * j] = (int32_t)(gx0 + k * 64 + b);
                            dbg->edge_xy[2 * j + 1] = (int32_t)(gy0 + y);
                        }
                        ++j;
                    }
                }
                if (tid == 0) *dbg->n_edge = ne;
            }
        }
        // ---- intensity columns (intensity_features.cpp:42-215), as the S kernel
        if (wid == 0) {
            double wcx = 0, wcy = 0;
            if (sS > 0) {
                wcx = (double)((unsigned long long)gx0 * sS + sXI) / (double)sS;
                wcy = (double)((unsigned long long)gy0 * sS + sYI) / (double)sS;
            }
            const double m2 = acc[0] / dn, m3 = acc[1] / dn, m4 = acc[2] / dn, m5 = acc[3] / dn,
                         m6 = acc[4] / dn;
            const double mad = ((double)(long long)(sS - 2 * slo) +
                                (double)((long long)clo - (long long)(n - clo)) * mean) / dn;
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
            const double energy = (double)sQ, sdev = sqrt(var), iqr = p75 - p25;
            const double mn = (double)vmin, mxv = (double)vmax;
            double o = 0;
            switch (lane) {
                case 0: o = mean; break;
                case 1: o = median; break;
                case 2: o = mode; break;
                case 3: o = mn; break;
                case 4: o = mxv; break;
                case 5: o = mxv - mn; break;
                case 6: o = var; break;
                case 7: o = m2; break;
                case 8: o = sdev; break;
                case 9: o = sqrt(m2); break;
                case 10: o = mad; break;
                case 11: o = median_ad; break;
                case 12: o = rmad; break;
                case 13: o = iqr; break;
                case 14: o = pct[0]; break;
                case 15: o = pct[1]; break;
                case 16: o = pct[2]; break;
                case 17: o = pct[3]; break;
                case 18: o = pct[4]; break;
                case 19: o = pct[5]; break;
                case 20: o = skew; break;
                case 21: o = kurt; break;
                case 22: o = m2 > 0 ? kurt - 3.0 : 0.0; break;
                case 23: o = hsk; break;
                case 24: o = hfl; break;
                case 25: o = energy; break;
                case 26: o = sqrt(energy / dn); break;
                case 27: o = ent / dn; break;
                case 28: o = (double)usq / (dn * dn); break;
                case 29: o = (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0; break;
                case 30: o = mean != 0 ? sdev / mean : 0.0; break;
                default: o = (double)sS; break;
            }
            double* oi = orow + cfg.col_int;
            oi[lane] = o;
            if (lane < 7) {
                const double t[7] = {e_mean, e_min, e_max, e_std, e_int, wcx, wcy};
                double v = t[0];
#pragma unroll
                for (int k = 1; k < 7; ++k)
                    if ((int)lane == k) v = t[k];
                oi[32 + lane] = v;
            }
        }
        __syncthreads();
    }

    // --------------------------------------------------------------- shape
    if (want_shape) {
        if (!have_k && !block_ke(h, w, wpr, nw, S, B, sm)) {
            if (tid == 0) atomicOr(&ctl->error, kErrRuns);
            return;
        }
        shape_b(h, w, wpr, nw, n, gx0, gy0, sX, sY, S, sm, orow + cfg.col_shape);
    }
    BT(3);
    // ------------------------------------------------------------- moments
    if (want_mom) {
        // integer anchors (rounded centroids); binary uses unit mass, weighted I
        const long long nb_ = (long long)n;
        const long long axb = (2 * (long long)sX + nb_) / (2 * nb_);
        const long long ayb = (2 * (long long)sY + nb_) / (2 * nb_);
        const long long W = (long long)sS;
        const long long axw = W > 0 ? (2 * (long long)sXI + W) / (2 * W) : 0;
        const long long ayw = W > 0 ? (2 * (long long)sYI + W) / (2 * W) : 0;
        // warp per row: separable row sums of w dx^p (warp-reduced), then lane i
        // accumulates its own moment N_i += rowsum_p * dy^q (i: grp<<4 | p<<2 | q)
        const int grp = lane >> 4, pp = (lane >> 2) & 3, qq = lane & 3;
        double acc = 0;
        for (int y = wid; y < h; y += kBW) {
            const uint32_t a = S.wordoff[(size_t)y * wpr], e = S.wordoff[(size_t)(y + 1) * wpr];
            double r8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // b^0..3, w b^0..3
            for (uint32_t i = a + lane; i < e; i += 32) {
                const long long x = (long long)(S.xy[i] & 0xffffu);
                const double wv = (double)S.vals[i];
                const double db = (double)(x - axb), dw = (double)(x - axw);
                const double db2 = db * db, dw2 = dw * dw;
                r8[0] += 1.0;
                r8[1] += db;
                r8[2] += db2;
                r8[3] += db2 * db;
                r8[4] += wv;
                r8[5] += wv * dw;
                r8[6] += wv * dw2;
                r8[7] += wv * dw2 * dw;
            }
            warp_sum8(r8);
            const double dy = grp ? (double)((long long)y - ayw) : (double)((long long)y - ayb);
            double rp = r8[0];
#pragma unroll
            for (int k = 1; k < 8; ++k)
                if (k == grp * 4 + pp) rp = r8[k];
            const double qy = qq == 0 ? 1.0 : qq == 1 ? dy : qq == 2 ? dy * dy : dy * dy * dy;
            acc += rp * qy;
        }
        sm.red[wid][lane] = acc;
        __syncthreads();
        if (wid == 0) {
            double N = 0;
            for (int k = 0; k < kBW; ++k) N += sm.red[k][lane];
            moments_epilogue(N, dn, n, sS, sX, sY, sXI, sYI, axb, ayb, axw, ayw, gx0, gy0,
                             orow + cfg.col_mom);
        }
        __syncthreads();
    }

    BT(4);
    // ---------------------------------------------------------------- glcm
    if (want_glcm) {
        const int ng = cfg.ng, A = cfg.n_angles;
        const bool sym = cfg.symmetric != 0;
        const uint32_t span = vmax - vmin + 1u, mdiv = 0xffffffffu / span;
        // dense windows (cells <= raster capacity, ~4 n): a level raster of the window
        // (u16, kNoLevel outside the ROI) lets pair counting walk window cells
        // coalesced with one load per neighbour; sparse windows (multi-component ROIs
        // spread over a large bbox) walk the pixel list instead
        constexpr uint16_t kNoLevel = 0xffffu;
        const uint32_t cells = (uint32_t)w * (uint32_t)h;
        const bool dense = (unsigned long long)w * h <= B.RCAP;
        auto level = [&](uint32_t v) -> uint32_t {  // floor(ng (v - vmin) / span), ng <= 256
            if (vmax <= vmin) return 0u;
            const uint32_t num = (uint32_t)ng * (v - vmin);
            uint32_t q = __umulhi(num, mdiv);
            if (num - q * span >= span) ++q;
            return min((uint32_t)(ng - 1), q);
        };
        // window cells c = tid + k kBT walked as (x, y) with one division per ROI
        const uint32_t uw = (uint32_t)w, step_y = (uint32_t)kBT / uw, step_x = (uint32_t)kBT % uw;
        auto advance = [&](uint32_t& x, uint32_t& y) {
            x += step_x;
            y += step_y;
            if (x >= uw) {
                x -= uw;
                ++y;
            }
        };
        if (dense) {
            uint32_t xc = tid % uw, yc = tid / uw;
            for (uint32_t c = tid; c < cells; c += kBT) {
                const uint32_t y = yc, x = xc;
                advance(xc, yc);
                uint16_t lv = kNoLevel;
                if ((S.rowmask[y * wpr + (x >> 6)] >> (x & 63)) & 1ull)
                    lv = (uint16_t)level(img.I[(size_t)(y0 + y) * img.pitch + x0 + x]);
                S.lraster[c] = lv;
            }
        } else {
            for (uint32_t i = tid; i < n; i += kBT) S.lvl[i] = (uint8_t)level(S.vals[i]);
        }
        __syncthreads();
        BT(5);
        // pair histograms: shared memory when ng*ng fits (kept zero), else the slab's.
        // Dense windows with ng <= 64 and <= 4 angles count every angle in one pass
        // over the cells (4 shared histograms of 64 x 64)
        const bool fused = dense && ng <= 64 && A <= 4;
        uint32_t npa0 = 0, npa1 = 0, npa2 = 0, npa3 = 0;
        if (fused) {
            const uint32_t ngu = (uint32_t)ng;
            uint32_t xc = tid % uw, yc = tid / uw;
            for (uint32_t c = tid; c < cells; c += kBT) {
                const int y = (int)yc, x = (int)xc;
                advance(xc, yc);
                const uint32_t la = S.lraster[c];
                if (la == kNoLevel) continue;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    if (a >= A) break;
                    const int nx = x + cfg.dx[a], ny = y + cfg.dy[a];
                    if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
                    const uint32_t lb = S.lraster[(uint32_t)ny * (uint32_t)w + (uint32_t)nx];
                    if (lb == kNoLevel) continue;
                    const uint32_t key = sym ? min(la, lb) * ngu + max(la, lb) : la * ngu + lb;
                    atomicAdd(&dyn[a * 4096 + key], 1u);
                    if (a == 0) ++npa0;
                    else if (a == 1) ++npa1;
                    else if (a == 2) ++npa2;
                    else ++npa3;
                }
            }
        }
        __syncthreads();
        double sacc = 0;
        for (int a = 0; a < A; ++a) {
            const int ddx = cfg.dx[a], ddy = cfg.dy[a];
            uint32_t* hist = fused ? dyn + a * 4096
                                   : ((uint32_t)ng * (uint32_t)ng <= kSmemCells ? dyn : S.ghist);
            for (int k = tid; k < 256; k += kBT) {
                sm.px[k] = 0u;
                sm.py[k] = 0u;
                sm.pdif[k] = 0u;
            }
            for (int k = tid; k < 512; k += kBT) sm.psum[k] = 0u;
            __syncthreads();
            // pairs (x, y) -> (x + dx, y + dy), both in the ROI
            uint32_t npr = a == 0 ? npa0 : a == 1 ? npa1 : a == 2 ? npa2 : npa3;
            auto count = [&](uint32_t la, uint32_t lb) {
                ++npr;
                const uint32_t key = sym ? min(la, lb) * (uint32_t)ng + max(la, lb)
                                         : la * (uint32_t)ng + lb;
                atomicAdd(&hist[key], 1u);
            };
            if (fused) {
                // counted above
            } else if (dense) {  // window cells whose neighbour is inside the window
                const int xa = ddx < 0 ? -ddx : 0, xb = ddx > 0 ? w - ddx : w;
                const int ya = ddy < 0 ? -ddy : 0, yb = ddy > 0 ? h - ddy : h;
                const uint32_t cw = xb > xa ? (uint32_t)(xb - xa) : 0u;
                const uint32_t ch = yb > ya ? (uint32_t)(yb - ya) : 0u;
                for (uint32_t c = tid; c < cw * ch; c += kBT) {
                    const uint32_t yy = c / cw, xx = c - yy * cw;
                    const int x = (int)xx + xa, y = (int)yy + ya;
                    const uint32_t la = S.lraster[(uint32_t)y * (uint32_t)w + (uint32_t)x];
                    const uint32_t lb =
                        S.lraster[(uint32_t)(y + ddy) * (uint32_t)w + (uint32_t)(x + ddx)];
                    if (la != kNoLevel && lb != kNoLevel) count(la, lb);
                }
            } else {  // member pixels; neighbour by row mask + word offsets
                for (uint32_t i = tid; i < n; i += kBT) {
                    const uint32_t p = S.xy[i];
                    const int x = (int)(p & 0xffffu), y = (int)(p >> 16);
                    const int nx = x + ddx, ny = y + ddy;
                    if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
                    const uint32_t wi = (uint32_t)ny * wpr + (uint32_t)(nx >> 6);
                    const uint64_t m = S.rowmask[wi];
                    if (!((m >> (nx & 63)) & 1ull)) continue;
                    const uint32_t jn = S.wordoff[wi] + __popcll(m & ((1ull << (nx & 63)) - 1ull));
                    count(S.lvl[i], S.lvl[jn]);
                }
            }
            const unsigned long long np = block_all((unsigned long long)npr, sm.u64s, OpAdd());
            const uint32_t ncells = (uint32_t)ng * (uint32_t)ng;
            if (dbg_on && dbg->pairs && tid == 0) dbg->pairs[a] = np;
            double st[29];
#pragma unroll
            for (int k = 0; k < 29; ++k) st[k] = 0;
            if (np > 0) {
                const double T = sym ? 2.0 * (double)np : (double)np;
                const double logT = nlog2(T);
                unsigned long long s2 = 0, sa = 0;
                uint32_t jm = 0;
                double el = 0;
                // dense pass in fixed thread order (deterministic fp64 entropy sum)
                for (uint32_t key = tid; key < ncells; key += kBT) {
                    const uint32_t c = hist[key];
                    if (!c) continue;
                    hist[key] = 0u;  // leave the histogram empty
                    const uint32_t ga = key / (uint32_t)ng, gb = key % (uint32_t)ng;
                    const bool off = sym && ga != gb;
                    const uint32_t cc = (sym && !off) ? 2u * c : c;
                    const uint32_t mcc = off ? 2u * cc : cc;
                    s2 += (unsigned long long)mcc * cc;
                    sa += (unsigned long long)((ga + 1) * (gb + 1)) * mcc;
                    jm = max(jm, cc);
                    el += (double)mcc * (logT - log2_int(cc));
                    atomicAdd(&sm.px[ga], cc);
                    if (off) atomicAdd(&sm.px[gb], cc);
                    if (!sym) atomicAdd(&sm.py[gb], cc);
                    atomicAdd(&sm.psum[ga + gb], mcc);
                    atomicAdd(&sm.pdif[ga > gb ? ga - gb : gb - ga], mcc);
                    if (dbg_on && dbg->glcm) {
                        dbg->glcm[((size_t)a * ng + ga) * ng + gb] = cc;
                        if (off) dbg->glcm[((size_t)a * ng + gb) * ng + ga] = cc;
                    }
                }
                s2 = block_all(s2, sm.u64s, OpAdd());
                sa = block_all(sa, sm.u64s, OpAdd());
                jm = block_all(jm, sm.u32s, OpMax());
                el = block_all(el, sm.f64s, OpAdd());
                if (wid == 0)
                    haralick_finish(sm.px, sym ? sm.px : sm.py, sm.psum, sm.pdif, ng, sym, T, logT, s2,
                                    sa, jm, el, st);
            }
            if (wid == 0) {
                double mine = 0;
#pragma unroll
                for (int k = 0; k < 29; ++k)
                    if ((int)lane == k) mine = st[k];
                if (lane < 29) {
                    orow[cfg.col_glcm + lane * (A + 1) + a] = mine;
                    sacc += mine;
                }
            }
            __syncthreads();
        }
        if (wid == 0 && lane < 29) orow[cfg.col_glcm + lane * (A + 1) + A] = sacc / (double)A;
    }
    __syncthreads();
    BT(6);
}

__global__ void __launch_bounds__(kBT, FXG_B_MINB) k_roi_b(DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                                               double* out, const DebugOut* dbg, uint8_t* scratch,
                                               BLayout B) {
    __shared__ BShared sm;
    extern __shared__ uint32_t dyn[];  // [kSmemCells] GLCM pair histogram, kept zero
    for (uint32_t i = threadIdx.x; i < kSmemCells; i += kBT) dyn[i] = 0u;
    __syncthreads();
    const BSlab S = bslab(scratch + (size_t)blockIdx.x * B.bytes, B);
    const uint32_t nl = ctl->class_count[kClassL];
    const uint32_t total = nl + ctl->overflow_count;  // S kernels have finished
    // sweep 0 claims the L list for windows of > kBigCells cells only; sweep 1 takes
    // every other job (longest jobs first, so none starts at the end of the launch)
    for (int sweep = 0; sweep < 2;) {
        if (threadIdx.x == 0) sm.job = atomicAdd(sweep ? &ctl->class_next[kClassL] : &ctl->b_next_big, 1u);
        __syncthreads();
        const uint32_t idx = sm.job;
        __syncthreads();
        if (idx >= (sweep ? total : nl)) {
            ++sweep;
            continue;
        }
        const uint32_t r = idx < nl ? rl.cls_list[kClassL][idx] : rl.overflow[idx - nl];
        const uint32_t w = rl.w[r], h = rl.h[r];
        const bool big = idx < nl && (unsigned long long)w * h > kBigCells;
        if (big != (sweep == 0)) continue;
        if (h > B.H || (w + 63) / 64 > B.WPR || rl.n[r] > (unsigned long long)B.NMAX) {
            if (threadIdx.x == 0) atomicOr(&ctl->error, kErrCapacity);
            continue;
        }
        process_b(r, img, rl, ctl, cfg, out, dbg, S, B, sm, dyn);
    }
}

}  // namespace

// phase clocks of k_roi_b (tools/phase_clocks.py via fx_debug_phase_clocks)
int roi_b_phase_clocks(unsigned long long* out, int reset) {
#ifdef FXG_PHASE_TIMING
    if (cudaMemcpyFromSymbol(out, g_phase_clk_b, 8 * sizeof(unsigned long long)) != cudaSuccess)
        return 7;
    if (reset) {
        const unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_phase_clk_b, z, sizeof z);
    }
    return 0;
#else
    (void)out;
    (void)reset;
    return 1;
#endif
}

cudaError_t roi_b_setup() {
    k_init_log2_tab<<<4, 256>>>();
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_roi_b, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kSmemCells * sizeof(uint32_t)));
    return e;
}

BLayout make_blayout(uint32_t H, uint32_t WPR, uint32_t NMAX, uint32_t RUNMAX, uint32_t NB,
                     unsigned long long CELLS) {
    BLayout B{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (o + bytes + 255) & ~(size_t)255;
        return at;
    };
    const size_t NW = (size_t)H * WPR;
    B.rowmask = take(NW * 8);
    B.kmask = take(NW * 8);
    B.emask = take(NW * 8);
    B.wordoff = take((NW + 1) * 4);
    B.tmpw = take((NW + 1) * 4);
    B.xy = take((size_t)NMAX * 4);
    B.vals = take((size_t)NMAX * 2);
    B.RCAP = CELLS < 4ull * NMAX ? CELLS : 4ull * NMAX;
    B.lraster = take((size_t)B.RCAP * 2);
    B.lvl = take((size_t)NMAX);
    B.vhist = take(65536 * 4);
    B.runoff = take(((size_t)H + 1) * 4);
    B.rs = take((size_t)RUNMAX * 2);
    B.re = take((size_t)RUNMAX * 2);
    B.parent = take((size_t)RUNMAX * 4);
    B.rsize = take((size_t)RUNMAX * 4);
    B.bins = take((size_t)NB * 4);
    B.ghist = take(65536 * 4);
    B.ctop = take((size_t)WPR * 64 * 4);
    B.cbot = take((size_t)WPR * 64 * 4);
    B.hv = take(((size_t)WPR * 64 * 4 + 8) * 4);
    B.bytes = o;
    B.H = H;
    B.WPR = WPR;
    B.NMAX = NMAX;
    B.RUNMAX = RUNMAX;
    B.NB = NB;
    return B;
}

void launch_roi_b(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                  double* out, const DebugOut* dbg, uint8_t* scratch, const BLayout& B) {
    k_roi_b<<<grid, kBT, kSmemCells * sizeof(uint32_t), s>>>(img, rl, ctl, cfg, out, dbg, scratch, B);
}

}  // namespace fxg
