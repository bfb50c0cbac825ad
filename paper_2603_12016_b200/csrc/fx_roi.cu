// Per-ROI feature kernels (see fx_roi.cuh for the reference mapping).
#include <math.h>

#include "fx_roi.cuh"

namespace fxg {

namespace {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT%=:\n\t"
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

template <typename XY>
struct XYP {
    static constexpr int SH = sizeof(XY) == 2 ? 8 : 16;
    static constexpr uint32_t M = (1u << SH) - 1u;
    __device__ static XY pack(uint32_t x, uint32_t y) { return (XY)(x | (y << SH)); }
    __device__ static uint32_t x(XY v) { return (uint32_t)v & M; }
    __device__ static uint32_t y(XY v) { return (uint32_t)v >> SH; }
};

struct Slab {
    uint64_t* rowmask;
    uint32_t* rowoff;
    uint16_t* vals;
    void* xy;
    uint16_t* stage;
    uint16_t *tmp, *sorted;
    uint32_t* cnt;
    uint64_t *kmask, *emask;
    uint32_t* runoff;
    uint16_t *rs, *re;
    uint32_t *parent, *rsize;
    uint8_t* lvl;
    uint16_t *keys, *keys2;
    uint32_t* gcnt;
    uint32_t* marg;
    double* gstat;
    uint32_t NMAX, RUNMAX;
};

__device__ __forceinline__ Slab slab_at(uint8_t* base, const Layout& L) {
    Slab s;
    s.rowmask = (uint64_t*)(base + L.rowmask);
    s.rowoff = (uint32_t*)(base + L.rowoff);
    s.vals = (uint16_t*)(base + L.vals);
    s.xy = (void*)(base + L.xy);
    s.stage = (uint16_t*)(base + L.stage);
    s.tmp = (uint16_t*)(base + L.tmp);
    s.sorted = (uint16_t*)(base + L.sorted);
    s.cnt = (uint32_t*)(base + L.cnt);
    s.kmask = (uint64_t*)(base + L.kmask);
    s.emask = (uint64_t*)(base + L.emask);
    s.runoff = (uint32_t*)(base + L.runoff);
    s.rs = (uint16_t*)(base + L.rs);
    s.re = (uint16_t*)(base + L.re);
    s.parent = (uint32_t*)(base + L.parent);
    s.rsize = (uint32_t*)(base + L.rsize);
    s.lvl = (uint8_t*)(base + L.lvl);
    s.keys = (uint16_t*)(base + L.keys);
    s.keys2 = (uint16_t*)(base + L.keys2);
    s.gcnt = (uint32_t*)(base + L.gcnt);
    s.marg = (uint32_t*)(base + L.marg);
    s.gstat = (double*)(base + L.gstat);
    s.NMAX = L.NMAX;
    s.RUNMAX = L.RUNMAX;
    return s;
}

struct Job {
    uint32_t label, x0, y0, w, h, row;
    unsigned long long n;
};

__device__ __forceinline__ bool mask_bit(const uint64_t* m, int wpr, int x, int y) {
    return (m[(size_t)y * wpr + (x >> 6)] >> (x & 63)) & 1ull;
}
__device__ __forceinline__ uint32_t mask_rank(const uint64_t* m, const uint32_t* rowoff, int wpr,
                                              int x, int y) {
    const uint64_t* r = m + (size_t)y * wpr;
    uint32_t k = rowoff[y];
    const int wk = x >> 6;
    for (int i = 0; i < wk; ++i) k += __popcll(r[i]);
    return k + __popcll(r[wk] & ((1ull << (x & 63)) - 1ull));
}

// ---- edge phase helpers -------------------------------------------------

// count maximal runs of set bits in a multi-word row
__device__ __forceinline__ uint32_t row_runs(const uint64_t* r, int wpr) {
    uint32_t c = 0;
    uint64_t carry = 0;
    for (int k = 0; k < wpr; ++k) {
        const uint64_t m = r[k];
        c += __popcll(m & ~((m << 1) | carry));
        carry = m >> 63;
    }
    return c;
}
__device__ __forceinline__ void row_emit_runs(const uint64_t* r, int wpr, uint32_t off,
                                              uint16_t* rs, uint16_t* re) {
    uint32_t j = off;
    uint64_t carry = 0;
    for (int k = 0; k < wpr; ++k) {
        const uint64_t m = r[k];
        uint64_t st = m & ~((m << 1) | carry);
        carry = m >> 63;
        while (st) {
            rs[j++] = (uint16_t)(k * 64 + __ffsll((long long)st) - 1);
            st &= st - 1;
        }
    }
    j = off;
    for (int k = 0; k < wpr; ++k) {
        const uint64_t m = r[k];
        const uint64_t nx = (k + 1 < wpr) ? (r[k + 1] & 1ull) : 0ull;
        uint64_t en = m & ~((m >> 1) | (nx << 63));
        while (en) {
            re[j++] = (uint16_t)(k * 64 + __ffsll((long long)en) - 1);
            en &= en - 1;
        }
    }
}
__device__ __forceinline__ void row_or_run(uint64_t* r, int s, int e) {
    for (int k = s >> 6; k <= (e >> 6); ++k) {
        const int a = (k == (s >> 6)) ? (s & 63) : 0;
        const int b = (k == (e >> 6)) ? (e & 63) : 63;
        r[k] |= bits_between(a, b);
    }
}

// Builds run lists of `mask` rows (warp), returns total runs or ~0u on overflow.
__device__ uint32_t build_runs(const uint64_t* mask, int h, int wpr, Slab& S) {
    const unsigned lane = lane_id();
    uint32_t total = 0;
    for (int yb = 0; yb < h; yb += 32) {
        const int y = yb + lane;
        const uint32_t c = (y < h) ? row_runs(mask + (size_t)y * wpr, wpr) : 0u;
        const uint32_t incl = warp_incl_scan(c);
        if (y < h) S.runoff[y] = total + incl - c;
        total += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) S.runoff[h] = total;
    __syncwarp();
    if (total > S.RUNMAX) return ~0u;
    for (int y = lane; y < h; y += 32) row_emit_runs(mask + (size_t)y * wpr, wpr, S.runoff[y], S.rs, S.re);
    for (uint32_t r = lane; r < total; r += 32) S.parent[r] = r;
    __syncwarp();
    return total;
}

// union runs of adjacent rows; ext = 1 for 8-connectivity, 0 for 4-connectivity
__device__ void union_rows(int h, int ext, Slab& S) {
    const unsigned lane = lane_id();
    for (int y = 1 + lane; y < h; y += 32) {
        uint32_t i = S.runoff[y], ie = S.runoff[y + 1];
        uint32_t j = S.runoff[y - 1], je = S.runoff[y];
        while (i < ie && j < je) {
            const int as = S.rs[i], ae = S.re[i], bs = S.rs[j], be = S.re[j];
            if (be + ext < as) {
                ++j;
            } else if (ae + ext < bs) {
                ++i;
            } else {
                uf_union(S.parent, i, j);
                if (ae < be) ++i;
                else ++j;
            }
        }
    }
    __syncwarp();
    for (uint32_t r = lane; r < S.runoff[h]; r += 32) S.parent[r] = uf_find(S.parent, r);
    __syncwarp();
}

// ---- the pipeline ---------------------------------------------------------

template <int WMAX, typename XY, bool TMA>
__device__ __forceinline__ void process_roi(const Job& J, Slab& S, const DevImage& img, const FeatCfg& cfg,
                            double* __restrict__ out, const CUtensorMap* tmapL, uint64_t* mbar,
                            uint32_t& mbar_phase, Control* ctl, RoiList rl, int rank,
                            bool allow_overflow, const DebugOut* dbg) {
    const unsigned lane = lane_id();
    const int w = (int)J.w, h = (int)J.h;
    const int wpr = WMAX > 0 ? WMAX : (w + 63) >> 6;
    const uint32_t label = J.label;
    const bool dbg_on = dbg != nullptr && dbg->label == label;
    double* orow = out + (size_t)J.row * cfg.ncols;
    XY* xy = (XY*)S.xy;

    // ------------------------------------------------------------ load ---
    // pass 1: membership masks, row offsets, compact pixel coordinates
    uint32_t npx = 0;
    const int nchunks = (w + 31) >> 5;
    if (TMA) {
        // the window's label tile was requested by the caller (issue_tma_window)
        mbar_wait(mbar, mbar_phase);
        mbar_phase ^= 1u;
        for (int y = 0; y < h; ++y) {
            if (lane == 0) S.rowoff[y] = npx;
            for (int c = 0; c < nchunks; ++c) {
                const int x = c * 32 + (int)lane;
                const bool in = x < w && S.stage[y * kStageW + (J.x0 & 7u) + x] == label;
                const unsigned b = __ballot_sync(kFull, in);
                if (lane == 0) {
                    uint64_t* mw = &S.rowmask[(size_t)y * wpr + (c >> 1)];
                    if (c & 1) *mw |= (uint64_t)b << 32;
                    else *mw = (uint64_t)b;
                }
                if (in) xy[npx + __popc(b & lanemask_lt())] = XYP<XY>::pack(x, y);
                npx += __popc(b);
            }
        }
    } else {
        const int nq = h * nchunks;
        for (int q0 = 0; q0 < nq; q0 += 8) {
            uint16_t lb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u;
                const int y = q / nchunks, x = (q % nchunks) * 32 + (int)lane;
                lb[u] = (q < nq && x < w) ? img.L[(size_t)(J.y0 + y) * img.pitch + J.x0 + x] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u;
                if (q >= nq) break;
                const int y = q / nchunks, c = q % nchunks, x = c * 32 + (int)lane;
                if (c == 0 && lane == 0) S.rowoff[y] = npx;
                const bool in = x < w && lb[u] == label;
                const unsigned b = __ballot_sync(kFull, in);
                if (lane == 0) {
                    uint64_t* mw = &S.rowmask[(size_t)y * wpr + (c >> 1)];
                    if (c & 1) *mw |= (uint64_t)b << 32;
                    else *mw = (uint64_t)b;
                }
                if (in) xy[npx + __popc(b & lanemask_lt())] = XYP<XY>::pack(x, y);
                npx += __popc(b);
            }
        }
    }
    if (lane == 0) S.rowoff[h] = npx;
    __syncwarp();
    const uint32_t n = npx;

    // pass 2: gather intensities of member pixels; exact integer sums
    unsigned long long sS = 0, sQ = 0, sXI = 0, sYI = 0, sLX = 0, sLY = 0;
    for (uint32_t base = 0; base < n; base += 32 * 8) {
        uint16_t v[8];
        uint32_t px[8], py[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            if (i < n) {
                const XY p = xy[i];
                px[u] = XYP<XY>::x(p);
                py[u] = XYP<XY>::y(p);
                v[u] = __ldg(img.I + (size_t)(J.y0 + py[u]) * img.pitch + J.x0 + px[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            if (i < n) {
                S.vals[i] = v[u];
                const unsigned long long vv = v[u];
                sS += vv;
                sQ += vv * vv;
                sXI += vv * px[u];
                sYI += vv * py[u];
                sLX += px[u];
                sLY += py[u];
            }
        }
    }
    sS = warp_sum(sS);
    sQ = warp_sum(sQ);
    sXI = warp_sum(sXI);
    sYI = warp_sum(sYI);
    sLX = warp_sum(sLX);
    sLY = warp_sum(sLY);
    __syncwarp();

    const double dn = (double)n;
    const long long gx0 = rl.gx[rank], gy0 = rl.gy[rank];
    uint16_t vmin = 0, vmax = 0;
    bool have_minmax = false;

    // ------------------------------------------------------- intensity ---
    if (cfg.col_int >= 0) {
        double* o = orow + cfg.col_int;
        warp_sort16(S.vals, S.tmp, S.sorted, n, S.cnt, false);
        __syncwarp();
        const uint16_t* s = S.sorted;
        vmin = s[0];
        vmax = s[n - 1];
        have_minmax = true;
        const double mean = (double)sS / dn;
        const double mn = (double)vmin, mxv = (double)vmax, range = mxv - mn;
        const double median =
            (n & 1) ? (double)s[n / 2] : 0.5 * ((double)s[n / 2 - 1] + (double)s[n / 2]);

        // central moments m2..m6 and mad (fp64, fixed order)
        double a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, am = 0;
        for (uint32_t i = lane; i < n; i += 32) {
            const double d = (double)s[i] - mean;
            const double d2 = d * d;
            a2 += d2;
            a3 += d2 * d;
            a4 += d2 * d2;
            a5 += d2 * d2 * d;
            a6 += d2 * d2 * d2;
            am += fabs(d);
        }
        const double m2 = warp_sum(a2) / dn, m3 = warp_sum(a3) / dn, m4 = warp_sum(a4) / dn;
        const double m5 = warp_sum(a5) / dn, m6 = warp_sum(a6) / dn, mad = warp_sum(am) / dn;
        const double var_b = m2;
        const double var = n > 1 ? m2 * dn / (dn - 1.0) : 0.0;
        double skew = 0, kurt = 0, exk = 0, hsk = 0, hfl = 0;
        if (m2 > 0) {
            skew = m3 / pow(m2, 1.5);
            kurt = m4 / (m2 * m2);
            exk = kurt - 3.0;
            hsk = m5 / pow(m2, 2.5);
            hfl = m6 / (m2 * m2 * m2);
        }
        // percentiles: lanes 0..5
        const double pvals[6] = {1, 10, 25, 75, 90, 99};
        double myp = 0;
        if (lane < 6) myp = percentile_exact(s, n, pvals[lane]);
        const double p1 = __shfl_sync(kFull, myp, 0), p10 = __shfl_sync(kFull, myp, 1);
        const double p25 = __shfl_sync(kFull, myp, 2), p75 = __shfl_sync(kFull, myp, 3);
        const double p90 = __shfl_sync(kFull, myp, 4), p99 = __shfl_sync(kFull, myp, 5);
        const double iqr = p75 - p25;
        const double qcod = (p75 + p25) != 0 ? iqr / (p75 + p25) : 0.0;
        // median absolute deviation from the median (exact)
        double median_ad;
        {
            const uint32_t M2 = (n & 1) ? 2u * s[n / 2] : (uint32_t)s[n / 2 - 1] + s[n / 2];
            uint32_t d_hi = 0, d_lo = 0;
            if (lane == 0) d_hi = kth_dev2(s, n, M2, n / 2);
            if (lane == 1 && !(n & 1)) d_lo = kth_dev2(s, n, M2, n / 2 - 1);
            d_hi = __shfl_sync(kFull, d_hi, 0);
            d_lo = __shfl_sync(kFull, d_lo, 1);
            median_ad = (n & 1) ? 0.5 * (double)d_hi
                                : 0.5 * (0.5 * (double)d_lo + 0.5 * (double)d_hi);
        }
        // rmad over [p10, p90]
        double rmad = 0;
        {
            unsigned long long rs_ = 0, rn_ = 0;
            for (uint32_t i = lane; i < n; i += 32) {
                const double x = (double)s[i];
                if (x >= p10 && x <= p90) {
                    rs_ += s[i];
                    rn_ += 1;
                }
            }
            rs_ = warp_sum(rs_);
            rn_ = warp_sum(rn_);
            if (rn_ > 0) {
                const double rmean = (double)rs_ / (double)rn_;
                double acc = 0;
                for (uint32_t i = lane; i < n; i += 32) {
                    const double x = (double)s[i];
                    if (x >= p10 && x <= p90) acc += fabs(x - rmean);
                }
                rmad = warp_sum(acc) / (double)rn_;
            }
        }
        // mode (ties -> smallest) and histogram entropy/uniformity via runs
        double mode, entropy, uniformity;
        {
            const unsigned long long nb = (unsigned long long)cfg.bins;
            const unsigned long long rng = (unsigned long long)(vmax - vmin);
            unsigned long long best = 0;  // (len << 16) | (0xffff - value)
            double ent = 0, uni = 0;
            uint32_t carry_v = 0, carry_b = 0;
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                const bool ok = i < n;
                const uint32_t v = ok ? s[i] : 0u;
                const uint32_t bin =
                    ok ? (rng == 0 ? 0u
                                   : (uint32_t)min(nb - 1, nb * (unsigned long long)(v - vmin) / rng))
                       : 0u;
                const uint32_t pv = (ok && i > 0) ? s[i - 1] : 0u;
                const uint32_t pbin =
                    (ok && i > 0)
                        ? (rng == 0 ? 0u
                                    : (uint32_t)min(nb - 1, nb * (unsigned long long)(pv - vmin) / rng))
                        : 0u;
                const bool vstart = ok && (i == 0 || pv != v);
                const bool bstart = ok && (i == 0 || pbin != bin);
                const bool last = ok && (i + 1 == n);
                const uint32_t nv = (ok && !last) ? s[i + 1] : 0u;
                const uint32_t nbin =
                    (ok && !last)
                        ? (rng == 0 ? 0u
                                    : (uint32_t)min(nb - 1, nb * (unsigned long long)(nv - vmin) / rng))
                        : 0u;
                const bool vend = ok && (last || nv != v);
                const bool bend = ok && (last || nbin != bin);
                const unsigned vs = __ballot_sync(kFull, vstart), bs = __ballot_sync(kFull, bstart);
                const unsigned le = lanemask_lt() | (1u << lane);
                const uint32_t vst = (vs & le) ? base + 31 - __clz(vs & le) : carry_v;
                const uint32_t bst = (bs & le) ? base + 31 - __clz(bs & le) : carry_b;
                if (vend) {
                    const unsigned long long len = i - vst + 1;
                    const unsigned long long key = (len << 16) | (0xffffu - v);
                    best = key > best ? key : best;
                }
                if (bend) {
                    const double p = (double)(i - bst + 1) / dn;
                    ent -= p * log2(p);
                    uni += p * p;
                    if (dbg_on && bin < (uint32_t)dbg->nb) dbg->hist[bin] = i - bst + 1;
                }
                if (vs) carry_v = base + 31 - __clz(vs);
                if (bs) carry_b = base + 31 - __clz(bs);
            }
            best = warp_max(best);
            mode = (double)(0xffffu - (uint32_t)(best & 0xffffu));
            entropy = warp_sum(ent);
            uniformity = warp_sum(uni);
        }
        const double energy = (double)sQ;
        const double rms = sqrt(energy / dn);
        const double sdev = sqrt(var);
        const double cov = mean != 0 ? sdev / mean : 0.0;

        // ---------------- edge set (trace_contour visited set, def. B) ---
        double e_mean = 0, e_min = 0, e_max = 0, e_std = 0, e_int = 0;
        {
            bool ok = true;
            uint32_t nr = build_runs(S.rowmask, h, wpr, S);
            if (nr == ~0u) ok = false;
            uint64_t* K = S.kmask;
            if (ok) {
                union_rows(h, 1, S);
                for (uint32_t r = lane; r < nr; r += 32) S.rsize[r] = 0;
                __syncwarp();
                for (uint32_t r = lane; r < nr; r += 32)
                    atomicAdd(&S.rsize[S.parent[r]], (uint32_t)(S.re[r] - S.rs[r] + 1));
                __syncwarp();
                unsigned long long bestk = 0;
                uint32_t nroots = 0;
                for (uint32_t r = lane; r < nr; r += 32)
                    if (S.parent[r] == r) {
                        ++nroots;
                        const unsigned long long k =
                            ((unsigned long long)S.rsize[r] << 32) | (0xffffffffu - r);
                        bestk = k > bestk ? k : bestk;
                    }
                bestk = warp_max(bestk);
                nroots = warp_sum(nroots);
                const uint32_t broot = 0xffffffffu - (uint32_t)(bestk & 0xffffffffu);
                for (int y = lane; y < h; y += 32) {
                    uint64_t* kr = K + (size_t)y * wpr;
                    if (nroots == 1) {
                        for (int k = 0; k < wpr; ++k) kr[k] = S.rowmask[(size_t)y * wpr + k];
                    } else {
                        for (int k = 0; k < wpr; ++k) kr[k] = 0;
                        for (uint32_t r = S.runoff[y]; r < S.runoff[y + 1]; ++r)
                            if (S.parent[r] == broot) row_or_run(kr, S.rs[r], S.re[r]);
                    }
                }
                __syncwarp();
                // free (non-K) cells, as rows in emask (temporarily)
                uint64_t* E = S.emask;
                for (int y = lane; y < h; y += 32)
                    for (int k = 0; k < wpr; ++k) {
                        const int rem = w - k * 64;
                        const uint64_t wm = rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
                        E[(size_t)y * wpr + k] = ~K[(size_t)y * wpr + k] & wm;
                    }
                __syncwarp();
                const uint32_t nf = build_runs(E, h, wpr, S);
                if (nf == ~0u) ok = false;
                if (ok) {
                    union_rows(h, 0, S);
                    for (uint32_t r = lane; r < nf; r += 32) S.rsize[r] = 0;
                    __syncwarp();
                    for (int y = lane; y < h; y += 32)
                        for (uint32_t r = S.runoff[y]; r < S.runoff[y + 1]; ++r)
                            if (y == 0 || y == h - 1 || S.rs[r] == 0 || S.re[r] == w - 1)
                                S.rsize[S.parent[r]] = 1u;
                    __syncwarp();
                    for (int y = lane; y < h; y += 32) {
                        uint64_t* er = E + (size_t)y * wpr;
                        for (int k = 0; k < wpr; ++k) er[k] = 0;
                        for (uint32_t r = S.runoff[y]; r < S.runoff[y + 1]; ++r)
                            if (S.rsize[S.parent[r]]) row_or_run(er, S.rs[r], S.re[r]);
                    }
                    __syncwarp();
                    // edge = K & (4-neighbour in E or outside the window)
                    unsigned long long es = 0, en = 0;
                    uint32_t emn = 0xffffffffu, emx = 0;
                    for (int pass = 0; pass < 2; ++pass) {
                        double ev = 0;
                        for (int y = lane; y < h; y += 32) {
                            uint32_t idx = S.rowoff[y];
                            for (int k = 0; k < wpr; ++k) {
                                const uint64_t kr = K[(size_t)y * wpr + k];
                                const uint64_t e0 = E[(size_t)y * wpr + k];
                                const uint64_t el = (k > 0) ? E[(size_t)y * wpr + k - 1] : 0ull;
                                const uint64_t eh = (k + 1 < wpr) ? E[(size_t)y * wpr + k + 1] : 0ull;
                                uint64_t nb4 = (e0 << 1) | (el >> 63) | (e0 >> 1) | (eh << 63);
                                if (y > 0) nb4 |= E[(size_t)(y - 1) * wpr + k];
                                if (y + 1 < h) nb4 |= E[(size_t)(y + 1) * wpr + k];
                                if (y == 0 || y == h - 1) nb4 = ~0ull;
                                if (k == 0) nb4 |= 1ull;
                                if (k == ((w - 1) >> 6)) nb4 |= 1ull << ((w - 1) & 63);
                                uint64_t edge = kr & nb4;
                                const uint64_t rm = S.rowmask[(size_t)y * wpr + k];
                                while (edge) {
                                    const int b = __ffsll((long long)edge) - 1;
                                    edge &= edge - 1;
                                    const uint32_t v =
                                        S.vals[idx + __popcll(rm & ((1ull << b) - 1ull))];
                                    if (pass == 0) {
                                        es += v;
                                        en += 1;
                                        emn = min(emn, v);
                                        emx = max(emx, v);
                                    } else {
                                        const double d = (double)v - e_mean;
                                        ev += d * d;
                                    }
                                }
                                idx += __popcll(rm);
                            }
                        }
                        if (pass == 0) {
                            es = warp_sum(es);
                            en = warp_sum(en);
                            emn = warp_min(emn);
                            emx = warp_max(emx);
                            if (en == 0) break;
                            e_mean = (double)es / (double)en;
                            e_min = (double)emn;
                            e_max = (double)emx;
                            e_int = (double)es;
                        } else {
                            e_std = sqrt(warp_sum(ev) / (double)en);
                        }
                    }
                    if (dbg_on) {
                        // row-major edge pixel list (single lane, debug only)
                        if (lane == 0) {
                            uint32_t ne = 0;
                            for (int y = 0; y < h; ++y)
                                for (int x = 0; x < w; ++x) {
                                    if (!mask_bit(K, wpr, x, y)) continue;
                                    bool e = (y == 0 || y == h - 1 || x == 0 || x == w - 1);
                                    if (!e) e = mask_bit(E, wpr, x - 1, y) || mask_bit(E, wpr, x + 1, y) ||
                                                mask_bit(E, wpr, x, y - 1) || mask_bit(E, wpr, x, y + 1);
                                    if (!e) continue;
                                    if (ne < dbg->cap_edge) {
                                        dbg->edge_xy[2 * ne] = (int32_t)(gx0 + x);
                                        dbg->edge_xy[2 * ne + 1] = (int32_t)(gy0 + y);
                                    }
                                    ++ne;
                                }
                            *dbg->n_edge = ne;
                        }
                        __syncwarp();  // lane 0 reads K/E, which later phases reuse
                    }
                }
            }
            if (!ok) {
                // run capacity exceeded: re-queue to the L path (slab sized for it)
                if (allow_overflow) {
                    if (lane == 0) {
                        const uint32_t pos = atomicAdd(&ctl->overflow_count, 1u);
                        rl.overflow[pos] = (uint32_t)rank;
                    }
                } else if (lane == 0) {
                    atomicOr(&ctl->error, kErrRuns);
                }
                __syncwarp();
                return;
            }
        }

        // weighted centroid in global coordinates (intensity_features.cpp:31-40)
        double wcx = 0, wcy = 0;
        if (sS > 0) {
            const unsigned long long sx = (unsigned long long)gx0 * sS + sXI;
            const unsigned long long sy = (unsigned long long)gy0 * sS + sYI;
            wcx = (double)sx / (double)sS;
            wcy = (double)sy / (double)sS;
        }
        if (lane < 6) o[14 + lane] = myp;
        if (lane == 0) {
            o[0] = mean;
            o[1] = median;
            o[2] = mode;
            o[3] = mn;
            o[4] = mxv;
            o[5] = range;
            o[6] = var;
            o[7] = var_b;
            o[8] = sdev;
            o[9] = sqrt(var_b);
            o[10] = mad;
            o[11] = median_ad;
            o[12] = rmad;
            o[13] = iqr;
            o[20] = skew;
            o[21] = kurt;
            o[22] = exk;
            o[23] = hsk;
            o[24] = hfl;
            o[25] = energy;
            o[26] = rms;
            o[27] = entropy;
            o[28] = uniformity;
            o[29] = qcod;
            o[30] = cov;
            o[31] = (double)sS;
            o[32] = e_mean;
            o[33] = e_min;
            o[34] = e_max;
            o[35] = e_std;
            o[36] = e_int;
            o[37] = wcx;
            o[38] = wcy;
        }
    }

    // --------------------------------------------------------- moments ---
    if (cfg.col_mom >= 0) {
        // integer anchors (rounded centroids); binary uses unit mass, weighted I
        const long long nb_ = (long long)n;
        const long long axb = (2 * (long long)sLX + nb_) / (2 * nb_);
        const long long ayb = (2 * (long long)sLY + nb_) / (2 * nb_);
        const long long W = (long long)sS;
        const long long axw = W > 0 ? (2 * (long long)sXI + W) / (2 * W) : 0;
        const long long ayw = W > 0 ? (2 * (long long)sYI + W) / (2 * W) : 0;
        double acc[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) acc[k] = 0;
        for (int y = lane; y < h; y += 32) {
            double rb1 = 0, rb2 = 0, rb3 = 0, rw0 = 0, rw1 = 0, rw2 = 0, rw3 = 0;
            uint32_t cntb = 0;
            uint32_t idx = S.rowoff[y];
            for (int k = 0; k < wpr; ++k) {
                uint64_t m = S.rowmask[(size_t)y * wpr + k];
                while (m) {
                    const int b = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    const long long x = (long long)k * 64 + b;
                    const double wv = (double)S.vals[idx++];
                    const double db = (double)(x - axb), dw = (double)(x - axw);
                    const double db2 = db * db, dw2 = dw * dw;
                    ++cntb;
                    rb1 += db;
                    rb2 += db2;
                    rb3 += db2 * db;
                    rw0 += wv;
                    rw1 += wv * dw;
                    rw2 += wv * dw2;
                    rw3 += wv * dw2 * dw;
                }
            }
            const double yb = (double)((long long)y - ayb), yw = (double)((long long)y - ayw);
            const double rb[4] = {(double)cntb, rb1, rb2, rb3};
            const double rw[4] = {rw0, rw1, rw2, rw3};
            const double qb[4] = {1.0, yb, yb * yb, yb * yb * yb};
            const double qw[4] = {1.0, yw, yw * yw, yw * yw * yw};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[p * 4 + q] += rb[p] * qb[q];
                    acc[16 + p * 4 + q] += rw[p] * qw[q];
                }
        }
        const double N = reduce_scatter32(acc);  // lane i: binary (i<16) / weighted N_pq
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
        double* o = orow + cfg.col_mom + grp * 52;
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

    // ------------------------------------------------------------ glcm ---
    if (cfg.col_glcm >= 0) {
        const int ng = cfg.ng, A = cfg.n_angles;
        if (!have_minmax) {
            uint32_t lo = 0xffffu, hi = 0;
            for (uint32_t i = lane; i < n; i += 32) {
                lo = min(lo, (uint32_t)S.vals[i]);
                hi = max(hi, (uint32_t)S.vals[i]);
            }
            vmin = (uint16_t)warp_min(lo);
            vmax = (uint16_t)warp_max(hi);
        }
        // discretize (texture.cpp:45-53): floor(ng*(v-lo)/(hi-lo+1)), exact in integers
        const uint32_t span = (uint32_t)vmax - vmin + 1u;
        for (uint32_t i = lane; i < n; i += 32) {
            uint32_t lv = 0;
            if (vmax > vmin) lv = min((uint32_t)(ng - 1), ((uint32_t)ng * (S.vals[i] - vmin)) / span);
            S.lvl[i] = (uint8_t)lv;
        }
        __syncwarp();
        const bool sym = cfg.symmetric != 0;
        double* og = orow + cfg.col_glcm;
        double sacc = 0;  // lane s < 29: running sum over angles of stat s
        const uint32_t* px = S.marg;
        const uint32_t* py = S.marg + 256;
        const uint32_t* pxy = S.marg + 512;
        const uint32_t* pxmy = S.marg + 1024;
        for (int a = 0; a < A; ++a) {
            const int ddx = cfg.dx[a], ddy = cfg.dy[a];
            // pair keys
            uint32_t np = 0;
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                bool ok = false;
                uint32_t key = 0;
                if (i < n) {
                    const XY pp = xy[i];
                    const int x = (int)XYP<XY>::x(pp), y = (int)XYP<XY>::y(pp);
                    const int nx = x + ddx, ny = y + ddy;
                    if (nx >= 0 && nx < w && ny >= 0 && ny < h && mask_bit(S.rowmask, wpr, nx, ny)) {
                        const uint32_t la = S.lvl[i];
                        const uint32_t lb = S.lvl[mask_rank(S.rowmask, S.rowoff, wpr, nx, ny)];
                        if (sym) key = min(la, lb) * (uint32_t)ng + max(la, lb);
                        else key = la * (uint32_t)ng + lb;
                        ok = true;
                    }
                }
                const unsigned b = __ballot_sync(kFull, ok);
                if (ok) S.keys[np + __popc(b & lanemask_lt())] = (uint16_t)key;
                np += __popc(b);
            }
            __syncwarp();
            for (int k = lane; k < 1280; k += 32) S.marg[k] = 0;
            double st[29];
#pragma unroll
            for (int k = 0; k < 29; ++k) st[k] = 0;
            if (dbg_on && dbg->pairs && lane == 0) dbg->pairs[a] = np;
            if (np > 0) {
                const uint16_t* keys =
                    warp_sort16(S.keys, S.keys2, S.keys, np, S.gcnt, ng * ng <= 256);
                __syncwarp();
                const double T = sym ? 2.0 * (double)np : (double)np;
                double asm_ = 0, ent = 0, acor = 0, jmax = 0;
                uint32_t carry = 0;
                for (uint32_t base = 0; base < np; base += 32) {
                    const uint32_t i = base + lane;
                    const bool ok = i < np;
                    const uint32_t k = ok ? keys[i] : 0u;
                    const bool st_ = ok && (i == 0 || keys[i - 1] != k);
                    const bool en_ = ok && (i + 1 == np || keys[i + 1] != k);
                    const unsigned sb = __ballot_sync(kFull, st_);
                    const unsigned le = lanemask_lt() | (1u << lane);
                    const uint32_t s0 = (sb & le) ? base + 31 - __clz(sb & le) : carry;
                    if (en_) {
                        const uint32_t c = i - s0 + 1;
                        const uint32_t ga = k / (uint32_t)ng, gb = k % (uint32_t)ng;
                        const double gi = ga + 1.0, gj = gb + 1.0;
                        if (sym && ga != gb) {
                            const double p = (double)c / T;
                            asm_ += 2.0 * p * p;
                            ent -= 2.0 * p * log2(p);
                            acor += 2.0 * gi * gj * p;
                            jmax = fmax(jmax, p);
                            atomicAdd(&S.marg[ga], c);
                            atomicAdd(&S.marg[gb], c);
                            atomicAdd(&S.marg[256 + ga], c);
                            atomicAdd(&S.marg[256 + gb], c);
                            atomicAdd(&S.marg[512 + ga + gb], 2u * c);
                            atomicAdd(&S.marg[1024 + gb - ga], 2u * c);
                            if (dbg_on && dbg->glcm) {
                                dbg->glcm[((size_t)a * ng + ga) * ng + gb] = c;
                                dbg->glcm[((size_t)a * ng + gb) * ng + ga] = c;
                            }
                        } else {
                            const uint32_t cc = sym ? 2u * c : c;
                            const double p = (double)cc / T;
                            asm_ += p * p;
                            ent -= p * log2(p);
                            acor += gi * gj * p;
                            jmax = fmax(jmax, p);
                            atomicAdd(&S.marg[ga], cc);
                            atomicAdd(&S.marg[256 + gb], cc);
                            atomicAdd(&S.marg[512 + ga + gb], cc);
                            atomicAdd(&S.marg[1024 + (ga > gb ? ga - gb : gb - ga)], cc);
                            if (dbg_on && dbg->glcm) dbg->glcm[((size_t)a * ng + ga) * ng + gb] = cc;
                        }
                    }
                    if (sb) carry = base + 31 - __clz(sb);
                }
                asm_ = warp_sum(asm_);
                ent = warp_sum(ent);
                acor = warp_sum(acor);
                jmax = warp_max(jmax);
                __syncwarp();
                // marginals px, py (texture.cpp:127-141)
                double mux = 0, muy = 0;
                for (int g = lane; g < ng; g += 32) {
                    mux += (g + 1) * ((double)px[g] / T);
                    muy += (g + 1) * ((double)py[g] / T);
                }
                mux = warp_sum(mux);
                muy = warp_sum(muy);
                double vx = 0, vy = 0, hx = 0, hy = 0;
                for (int g = lane; g < ng; g += 32) {
                    const double a1 = (double)px[g] / T, b1 = (double)py[g] / T;
                    vx += (g + 1 - mux) * (g + 1 - mux) * a1;
                    vy += (g + 1 - muy) * (g + 1 - muy) * b1;
                    if (a1 > 0) hx -= a1 * log2(a1);
                    if (b1 > 0) hy -= b1 * log2(b1);
                }
                vx = warp_sum(vx);
                vy = warp_sum(vy);
                hx = warp_sum(hx);
                hy = warp_sum(hy);
                // p_{x+y} (index k = i+j-2), p_{x-y} (index |i-j|)
                double sumave = 0, sument = 0;
                for (int k = lane; k < 2 * ng - 1; k += 32) {
                    const double p = (double)pxy[k] / T;
                    if (p > 0) {
                        sumave += (k + 2) * p;
                        sument -= p * log2(p);
                    }
                }
                sumave = warp_sum(sumave);
                sument = warp_sum(sument);
                double sumvar = 0, clut = 0, clus = 0, clup = 0;
                for (int k = lane; k < 2 * ng - 1; k += 32) {
                    const double p = (double)pxy[k] / T;
                    if (p > 0) {
                        sumvar += (k + 2 - sumave) * (k + 2 - sumave) * p;
                        const double s = k + 2 - mux - muy;
                        clut += s * s * p;
                        clus += s * s * s * p;
                        clup += s * s * s * s * p;
                    }
                }
                sumvar = warp_sum(sumvar);
                clut = warp_sum(clut);
                clus = warp_sum(clus);
                clup = warp_sum(clup);
                double difave = 0, difent = 0, contrast = 0, idm = 0, id = 0, idn = 0, idmn = 0,
                       iv = 0;
                const double dng = (double)ng;
                for (int d = lane; d < ng; d += 32) {
                    const double p = (double)pxmy[d] / T;
                    if (p > 0) {
                        const double dd = (double)d;
                        difave += dd * p;
                        difent -= p * log2(p);
                        contrast += dd * dd * p;
                        idm += p / (1.0 + dd * dd);
                        id += p / (1.0 + dd);
                        idn += p / (1.0 + dd / dng);
                        idmn += p / (1.0 + dd * dd / (dng * dng));
                        if (d > 0) iv += p / (dd * dd);
                    }
                }
                difave = warp_sum(difave);
                difent = warp_sum(difent);
                contrast = warp_sum(contrast);
                idm = warp_sum(idm);
                id = warp_sum(id);
                idn = warp_sum(idn);
                idmn = warp_sum(idmn);
                iv = warp_sum(iv);
                double difvar = 0;
                for (int d = lane; d < ng; d += 32) {
                    const double p = (double)pxmy[d] / T;
                    if (p > 0) difvar += (d - difave) * (d - difave) * p;
                }
                difvar = warp_sum(difvar);
                double corr = 0;
                if (vx > 0 && vy > 0) corr = (acor - mux * muy) / sqrt(vx * vy);
                const double hxy = hx + hy;  // == hxy1 == hxy2
                const double hmax = fmax(hx, hy);
                const double im1 = hmax > 0 ? (ent - hxy) / hmax : 0.0;
                const double im2 = sqrt(fmax(0.0, 1.0 - exp(-2.0 * (hxy - ent))));
                const double v29[29] = {asm_,   acor,   clup,   clus,     clut, contrast, corr,
                                        difave, difent, difvar, difave,   sqrt(asm_), ent, id,
                                        idm,    id,     idn,    idm,      idmn, im1,      im2,
                                        iv,     mux,    ent,    jmax,     vx,   sumave,   sument,
                                        sumvar};
#pragma unroll
                for (int k = 0; k < 29; ++k) st[k] = v29[k];
            }
            // stat s -> lane s; columns stat-major: glcm_<s>_<angle>, then _ave
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
    }
    __syncwarp();
}

}  // namespace

// ---------------------------------------------------------------- kernels --

constexpr uint32_t kSmemSlack = 128 + 16;  // base alignment + mbarrier

// L path: one warp per CTA, slab in global scratch, plain loads.  Consumes the
// L class list, then the overflow list re-queued by the S kernels.
__global__ void __launch_bounds__(32)
    k_roi_l(DevImage img, RoiList rl, Control* ctl, FeatCfg cfg, double* out, const DebugOut* dbg,
            uint8_t* scratch, Layout L) {
    const unsigned lane = lane_id();
    Slab S = slab_at(scratch + (size_t)blockIdx.x * L.bytes, L);
    uint32_t phase = 0;
    const uint32_t nl = ctl->class_count[kClassL];
    for (;;) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(&ctl->class_next[kClassL], 1u);
        idx = __shfl_sync(kFull, idx, 0);
        const uint32_t total = nl + ctl->overflow_count;
        if (idx >= total) break;
        const uint32_t r = idx < nl ? rl.cls_list[kClassL][idx] : rl.overflow[idx - nl];
        Job J{rl.label[r], rl.x0[r], rl.y0[r], rl.w[r], rl.h[r], r, rl.n[r]};
        const int wpr = ((int)J.w + 63) >> 6;
        if (J.h > L.H || (uint32_t)wpr > L.WPR || J.n > L.NMAX) {
            if (lane == 0) atomicOr(&ctl->error, kErrCapacity);
            continue;
        }
        process_roi<0, uint32_t, false>(J, S, img, cfg, out, nullptr, nullptr, phase, ctl, rl,
                                        (int)r, false, dbg);
    }
}

// ---- host-side launch helpers (keep template instantiation in this TU) ----

void launch_roi_l(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                  double* out, const DebugOut* dbg, uint8_t* scratch, const Layout& L) {
    k_roi_l<<<grid, 32, 0, s>>>(img, rl, ctl, cfg, out, dbg, scratch, L);
}

}  // namespace fxg
