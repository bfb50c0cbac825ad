// Label scan + ROI compaction (replaces RoiRegistry::accumulate / labels(),
// reference roi.cpp:76-117).
//
// k_label_scan: one coalesced HBM sweep over the uint16 label raster (16 B vector
// loads, 8 labels per lane, software-pipelined row batches).  Each lane owns an
// 8-pixel-wide x kStripRows-row strip and folds it into a 2-entry register cache using SIMD-in-word
// tests (one label per chunk is the fast path); the warp then merges equal
// labels with REDUX and issues one set of global atomics per (strip, label) into
// the direct-mapped LabelTable.  Integer min/max/sum are order-free, so the
// table is bit-exact and deterministic.  Intensities are not read here (the
// per-ROI kernels gather them), so the sweep moves 2 B/px.
//
// k_compact_count / k_compact_emit: ascending list of present labels (rank =
// output row), bbox -> window, window-size class lists for the per-ROI kernels.
#include "fx_dev.cuh"
#include "fx_pack.hpp"

namespace fxg {

namespace {

// Warp tile: 32 lanes x 8 px = 256 px wide, kStripRows rows tall.  Each lane
// owns an 8-px-wide column strip and folds what it sees into a 2-entry register
// cache (blob ROIs give 1-2 labels per strip); at the end of the strip the warp
// merges equal labels with REDUX and one lane issues the global atomics.
//
// A lane's column strip is fixed for the whole tile, so a cache entry keeps the
// OR of its per-row pixel masks (one byte per pixel, built by two PRMTs from the
// SIMD compares) instead of a per-row x min/max: the x extent is decoded once,
// at the flush.  Interior tiles (every row and column inside the slot, 16 B
// aligned) run a loop without bounds checks or 64-bit address arithmetic; the
// instruction count per row, not bandwidth, bounded the previous version
// (ncu: 67% issue-active at 2.2 TB/s).
constexpr int kScanThreads = 128;
constexpr int kStripRows = FXG_SCAN_ROWS;
constexpr int kBatch = FXG_SCAN_BATCH;  // rows per load batch (16 B per lane each)

struct CacheEnt {
    uint32_t label, cnt, occ_lo, occ_hi, y0, y1;  // occ_*: pixels 0-3 / 4-7, 0xFF per pixel seen
};

__device__ __forceinline__ void global_fold(const LabelTable& t, uint32_t l, uint32_t cnt,
                                            uint32_t x0, uint32_t x1, uint32_t y0, uint32_t y1) {
    atomicAdd(&t.cnt[l], (unsigned long long)cnt);
    atomicMin(&t.xmin[l], x0);
    atomicMax(&t.xmax[l], x1);
    atomicMin(&t.ymin[l], y0);
    atomicMax(&t.ymax[l], y1);
}

// first / last pixel (0..7) present in an entry's occupancy bytes
__device__ __forceinline__ uint32_t occ_first(const CacheEnt& e) {
    return e.occ_lo ? (uint32_t)(__ffs(e.occ_lo) - 1) >> 3 : 4u + ((uint32_t)(__ffs(e.occ_hi) - 1) >> 3);
}
__device__ __forceinline__ uint32_t occ_last(const CacheEnt& e) {
    return e.occ_hi ? 7u - ((uint32_t)__clz(e.occ_hi) >> 3) : 3u - ((uint32_t)__clz(e.occ_lo) >> 3);
}

// an entry evicted mid-strip is not in the end-of-strip caches the warp reduces
// for maxlab, so its label raises the lane's running maximum lmax (compaction
// skips 1024-label blocks above the slot's maxlab; a global atomic per eviction
// cost the C2 scan 23 us of contention on one address)
__device__ __forceinline__ void evict(const LabelTable& t, const CacheEnt& e, uint32_t x, uint32_t& lmax) {
    if (e.label) {
        global_fold(t, e.label, e.cnt, x + occ_first(e), x + occ_last(e), e.y0, e.y1);
        lmax = max(lmax, e.label & 0xffffu);
    }
}

// fold a row's pixels of label l (pixel bytes olo/ohi, cnt of them) into the cache
__device__ __forceinline__ void cache_put(CacheEnt& c0, CacheEnt& c1, uint32_t& lmax, const LabelTable& t,
                                          uint32_t x, uint32_t l, uint32_t cnt, uint32_t olo,
                                          uint32_t ohi, uint32_t y) {
    if (l == c0.label) {
        c0.cnt += cnt;
        c0.occ_lo |= olo;
        c0.occ_hi |= ohi;
        c0.y1 = y;
    } else if (l == c1.label) {
        c1.cnt += cnt;
        c1.occ_lo |= olo;
        c1.occ_hi |= ohi;
        c1.y1 = y;
    } else {
        evict(t, c1, x, lmax);
        c1 = c0;
        c0 = CacheEnt{l, cnt, olo, ohi, y, y};
    }
}

// several distinct labels inside one 8-px chunk: per pixel, the chunk shifted
// through a register pair (no runtime-indexed array)
__device__ __forceinline__ void chunk_slow(uint4 v, uint32_t x, uint32_t y, uint32_t sb,
                                           CacheEnt& c0, CacheEnt& c1, uint32_t& lmax,
                                           const LabelTable& t) {
    unsigned long long q0 = v.x | ((unsigned long long)v.y << 32);
    unsigned long long q1 = v.z | ((unsigned long long)v.w << 32);
#pragma unroll 1
    for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t l = (uint32_t)q0 & 0xffffu;
        q0 = (q0 >> 16) | (q1 << 48);
        q1 >>= 16;
        const uint32_t byte = 0xffu << (8 * (k & 3));
        if (l) cache_put(c0, c1, lmax, t, x, sb | l, 1u, k < 4 ? byte : 0u, k < 4 ? 0u : byte, y);
    }
}

// sb = slot << 16: cache keys and table indices are slot * 65536 + label
__device__ __forceinline__ void chunk(uint4 v, uint32_t x, uint32_t y, uint32_t sb, CacheEnt& c0,
                                      CacheEnt& c1, uint32_t& lmax, const LabelTable& t) {
    if ((v.x | v.y | v.z | v.w) == 0u) return;
    // the largest label of the chunk (paired-halfword max, VIMNMX.U16x2)
    const uint32_t mx2 = __vmaxu2(__vmaxu2(v.x, v.y), __vmaxu2(v.z, v.w));
    const uint32_t L = max(mx2 & 0xffffu, mx2 >> 16);
    const uint32_t LL = L | (L << 16);
    // a halfword h is 0 or L  <=>  min(h, h ^ L) == 0: one XOR and one paired min
    // per word instead of the emulated SIMD compares
    const uint32_t bad = __vminu2(v.x, v.x ^ LL) | __vminu2(v.y, v.y ^ LL) |
                         __vminu2(v.z, v.z ^ LL) | __vminu2(v.w, v.w ^ LL);
    if (bad) {
        chunk_slow(v, x, y, sb, c0, c1, lmax, t);
        return;
    }
    // nonzero halfwords (SWAR: bit 15 of each half set iff the half is nonzero), then
    // one byte per pixel carrying that bit (PRMT of the high bytes)
    auto nz = [](uint32_t q) { return ((q & 0x7fff7fffu) + 0x7fff7fffu) | q; };
    const uint32_t olo = __byte_perm(nz(v.x), nz(v.y), 0x7531) & 0x80808080u;
    const uint32_t ohi = __byte_perm(nz(v.z), nz(v.w), 0x7531) & 0x80808080u;
    cache_put(c0, c1, lmax, t, x, sb | L, (uint32_t)(__popc(olo) + __popc(ohi)), olo, ohi, y);
}

__device__ __forceinline__ uint4 load_chunk(const uint16_t* __restrict__ L, size_t pitch, int W,
                                            int H, int x, int y, bool vec) {
    if (y >= H || x >= W) return make_uint4(0, 0, 0, 0);  // H: end row of the slot
    const uint16_t* p = L + (size_t)y * pitch + x;
    if (vec && x + 8 <= W) return __ldg(reinterpret_cast<const uint4*>(p));
    uint32_t wv[4] = {0, 0, 0, 0};
    for (int k = 0; k < 8; ++k)
        if (x + k < W) wv[k >> 1] |= (uint32_t)p[k] << (16 * (k & 1));
    return make_uint4(wv[0], wv[1], wv[2], wv[3]);
}

// warp-aggregated flush of one cache entry per lane (REDUX per distinct label)
__device__ __forceinline__ void warp_flush(const CacheEnt& e, uint32_t x, const LabelTable& t) {
    const unsigned lane = lane_id();
    unsigned todo = __ballot_sync(kFull, e.label != 0);
    const uint32_t ex0 = e.label ? x + occ_first(e) : 0xffffffffu;
    const uint32_t ex1 = e.label ? x + occ_last(e) : 0u;
    while (todo) {
        const int leader = __ffs(todo) - 1;
        const uint32_t L = __shfl_sync(kFull, e.label, leader);
        const bool mine = e.label == L;
        const unsigned peers = __ballot_sync(kFull, mine);
        todo &= ~peers;
        const uint32_t cnt = __reduce_add_sync(kFull, mine ? e.cnt : 0u);
        const uint32_t x0 = __reduce_min_sync(kFull, mine ? ex0 : 0xffffffffu);
        const uint32_t x1 = __reduce_max_sync(kFull, mine ? ex1 : 0u);
        const uint32_t y0 = __reduce_min_sync(kFull, mine ? e.y0 : 0xffffffffu);
        const uint32_t y1 = __reduce_max_sync(kFull, mine ? e.y1 : 0u);
        if ((int)lane == leader) global_fold(t, L, cnt, x0, x1, y0, y1);
    }
}

}  // namespace

__global__ void __launch_bounds__(kScanThreads, FXG_SCAN_MINB)
    k_label_scan(const uint16_t* __restrict__ L, int W, int H, size_t pitch, int vec_ok, SlotMap m,
                 LabelTable t) {
    const unsigned lane = lane_id();
    const int warps_total = gridDim.x * (kScanThreads / 32);
    const int gw = blockIdx.x * (kScanThreads / 32) + (threadIdx.x >> 5);
    const int tiles_x = (W + 255) / 256;
    const int n_tiles = tiles_x * ((H + kStripRows - 1) / kStripRows);
    for (int tile = gw; tile < n_tiles; tile += warps_total) {
        const int strip = tile / tiles_x;
        const uint32_t slot = m.strip_slot ? m.strip_slot[(strip * kStripRows) >> 6] : 0u;
        const SlotInfo si = m.info ? m.info[slot] : m.s0;
        const int sw = si.w, send = si.row0 + si.h;  // slot bounds in the stack
        const uint32_t sb = slot << 16;
        const uint32_t gxo = (uint32_t)si.ox, gyo = (uint32_t)(si.oy - si.row0);
        const int tx0 = (tile % tiles_x) * 256;
        const int x = tx0 + (int)lane * 8;
        const int y0 = strip * kStripRows;
        const uint32_t gx = (uint32_t)x + gxo;
        CacheEnt c0{0, 0, 0, 0, 0, 0}, c1{0, 0, 0, 0, 0, 0};
        uint32_t lmax = 0;  // largest label this lane evicted in the tile
        if (vec_ok && tx0 + 256 <= sw && y0 + kStripRows <= send) {
            // interior tile: plain pointer walk, kBatch rows of 16 B in flight per lane
            const uint4* p = reinterpret_cast<const uint4*>(L + (size_t)y0 * pitch + x);
            const uint32_t step = (uint32_t)(pitch >> 3);  // uint4 per row
            uint32_t gy = (uint32_t)y0 + gyo;
#pragma unroll 1
            for (int r0 = 0; r0 < kStripRows; r0 += kBatch) {
                uint4 v[kBatch];
#pragma unroll
                for (int r = 0; r < kBatch; ++r) v[r] = __ldg(p + (size_t)r * step);
                p += (size_t)kBatch * step;
#pragma unroll
                for (int r = 0; r < kBatch; ++r) chunk(v[r], gx, gy + r, sb, c0, c1, lmax, t);
                gy += kBatch;
            }
        } else {
            // edge tile (image borders, batch slots): bounds-checked loads, one row at
            // a time (rare; kept simple so the interior loop keeps its registers)
#pragma unroll 1
            for (int r = 0; r < kStripRows; ++r)
                chunk(load_chunk(L, pitch, sw, send, x, y0 + r, vec_ok), gx, (uint32_t)(y0 + r) + gyo, sb,
                      c0, c1, lmax, t);
        }
        warp_flush(c0, gx, t);
        warp_flush(c1, gx, t);
        const uint32_t mx = warp_max(max(lmax, max(c0.label & 0xffffu, c1.label & 0xffffu)));
        if (lane == 0 && mx) atomicMax(&t.maxlab[slot], mx);
    }
}

// --- compaction -------------------------------------------------------------
//
// Work unit: a "pair" = (slot, 1024-label block); pairs above the slot's max
// label are dead (no table reads).  k_compact_count (persistent, grid-stride over
// pairs) counts present + owned labels per live pair; the last block to finish
// turns the counts into output rows (slot-major, labels ascending = the order of
// running the images one by one), lists the live pairs and clears maxlab.
// k_compact_emit walks the live pairs only, writes the ROI list and resets every
// table entry it consumed, so the next scan starts from a clean table without a
// memset.

// a label is emitted when present and owned (its first row in [own_y0, own_y1))
__device__ __forceinline__ bool owned(const LabelTable& t, uint32_t key, const CompactArgs& a) {
    if ((key & 0xffffu) == 0 || t.cnt[key] == 0ull) return false;
    const uint32_t y = t.ymin[key];
    return y >= a.own_y0 && y < a.own_y1;
}

__global__ void __launch_bounds__(1024) k_compact_count(LabelTable t, Control* ctl, CompactArgs a,
                                                        int nslots) {
    extern __shared__ uint32_t s_max[];  // [nslots]
    __shared__ uint32_t wt_n[32], wt_l[32];
    __shared__ uint32_t carry_n, carry_l;
    __shared__ int is_last;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = (int)tid; i < nslots; i += 1024) s_max[i] = t.maxlab[i];
    __syncthreads();
    const int nb = nslots * kBlocksPerSlot;
    for (int pair = blockIdx.x; pair < nb; pair += gridDim.x) {
        const uint32_t slot = pair / kBlocksPerSlot, blk = pair % kBlocksPerSlot;
        if (blk * 1024u > s_max[slot]) {  // uniform per block
            if (tid == 0) a.block_sum[pair] = 0u;
            continue;
        }
        const uint32_t key = slot * (uint32_t)kMaxLabels + blk * 1024u + tid;
        const int c = __syncthreads_count(owned(t, key, a));
        if (tid == 0) a.block_sum[pair] = (uint32_t)c | kBlockLive;
    }
    // last block: exclusive scans of the counts and of the live flags
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    if (tid == 0) carry_n = carry_l = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int b = b0 + (int)tid;
        const uint32_t raw = b < nb ? __ldcg(&a.block_sum[b]) : 0u;
        const uint32_t v = raw & ~kBlockLive, f = raw >> 31;
        const uint32_t in_n = warp_incl_scan(v), in_l = warp_incl_scan(f);
        if (lane == 31) {
            wt_n[warp] = in_n;
            wt_l[warp] = in_l;
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t x = wt_n[lane], y = wt_l[lane];
            wt_n[lane] = warp_incl_scan(x) - x;
            wt_l[lane] = warp_incl_scan(y) - y;
        }
        __syncthreads();
        const uint32_t ex_n = carry_n + wt_n[warp] + in_n - v;
        const uint32_t ex_l = carry_l + wt_l[warp] + in_l - f;
        if (b < nb) {
            a.block_base[b] = ex_n;
            if (f) a.live[ex_l] = (uint32_t)b;
            if (b % kBlocksPerSlot == 0) a.slot_base[b / kBlocksPerSlot] = ex_n;
        }
        __syncthreads();
        if (tid == 1023) {
            carry_n = ex_n + v;
            carry_l = ex_l + f;
        }
        __syncthreads();
    }
    if (tid == 0) {
        ctl->n_rois = carry_n;
        a.slot_base[nslots] = carry_n;
        a.done[1] = carry_l;  // live pair count
        a.done[0] = 0u;       // ready for the next compaction
    }
    for (int i = (int)tid; i < nslots; i += 1024) t.maxlab[i] = 0u;
}

// class of a window (w x h) with n pixels
__device__ __forceinline__ int roi_class(uint32_t w, uint32_t h, unsigned long long n) {
    if (w <= (uint32_t)kS0W && h <= (uint32_t)kS0H && n <= (unsigned long long)kS0N) return kClassS0;
    if (w <= (uint32_t)kSW && h <= (uint32_t)kSH) return n <= (unsigned long long)kS1N ? kClassS1 : kClassS2;
    return kClassL;
}

__global__ void __launch_bounds__(1024) k_compact_emit(LabelTable t, Control* ctl, RoiList r,
                                                       CompactArgs a, SlotMap m) {
    __shared__ uint32_t warp_cnt[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n_live = a.done[1];
    // more ROIs than output rows: the table is still consumed and the ROI list
    // written, but no ROI is queued, so no per-ROI kernel writes a row
    const bool fits = ctl->n_rois <= a.cap_rows;
    if (!fits && blockIdx.x == 0 && tid == 0) atomicOr(&ctl->error, kErrOutCap);
    for (uint32_t i = blockIdx.x; i < n_live; i += gridDim.x) {
        const uint32_t pair = a.live[i];
        const uint32_t slot = pair / kBlocksPerSlot, blk = pair % kBlocksPerSlot;
        const uint32_t l = blk * 1024u + tid;
        const uint32_t key = slot * (uint32_t)kMaxLabels + l;
        const unsigned long long n = t.cnt[key];
        const bool present = owned(t, key, a);
        const unsigned msk = __ballot_sync(kFull, present);
        if (lane == 0) warp_cnt[warp] = __popc(msk);
        __syncthreads();
        if (warp == 0) {
            const uint32_t c = warp_cnt[lane];
            warp_cnt[lane] = warp_incl_scan(c) - c;
        }
        __syncthreads();
        const uint32_t wbase = warp_cnt[warp];
        __syncthreads();  // warp_cnt is rewritten by the next pair
        if (n == 0ull) continue;
        const uint32_t gx0 = t.xmin[key], gy0 = t.ymin[key], gx1 = t.xmax[key], gy1 = t.ymax[key];
        // consume: reset the entry for the next scan
        t.cnt[key] = 0ull;
        t.xmin[key] = 0xffffffffu;
        t.ymin[key] = 0xffffffffu;
        t.xmax[key] = 0u;
        t.ymax[key] = 0u;
        if (!present) continue;
        const uint32_t rank = a.block_base[pair] + wbase + __popc(msk & lanemask_lt());
        // table holds global coordinates; windows are local to the (stacked) raster read
        const SlotInfo si = m.info ? m.info[slot] : m.s0;
        const uint32_t x0 = gx0 - (uint32_t)si.ox, ly0 = gy0 - (uint32_t)si.oy;
        const uint32_t w = gx1 - gx0 + 1, h = gy1 - gy0 + 1;
        if (gx0 < (uint32_t)si.ox || gy0 < (uint32_t)si.oy || x0 + w > (uint32_t)si.w ||
            ly0 + h > (uint32_t)si.h)
            atomicOr(&ctl->error, kErrWindow);  // window not inside the image (halo too small)
        r.label[rank] = l;
        r.gx[rank] = (int32_t)gx0;
        r.gy[rank] = (int32_t)gy0;
        r.x0[rank] = x0;
        r.y0[rank] = ly0 + (uint32_t)si.row0;
        r.w[rank] = w;
        r.h[rank] = h;
        r.n[rank] = n;
        if (!fits) continue;
        const int c = roi_class(w, h, n);
        // one atomic per (warp, class): the class lists are consumed in any order
        const unsigned peers = __match_any_sync(__activemask(), c);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if ((int)lane == leader) base = atomicAdd(&ctl->class_count[c], (uint32_t)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        const uint32_t pos = base + __popc(peers & lanemask_lt());
        // select, not a runtime index into the kernel-parameter array (a local copy)
        uint32_t* lst = c == kClassS0 ? r.cls_list[kClassS0]
                        : c == kClassS1 ? r.cls_list[kClassS1]
                        : c == kClassS2 ? r.cls_list[kClassS2] : r.cls_list[kClassL];
        lst[pos] = rank;
        if (c == kClassL) {
            atomicMax(&ctl->l_max_h, h);
            atomicMax(&ctl->l_max_wpr, (w + 63) / 64);
            atomicMax(&ctl->l_max_n, n);
            atomicMax(&ctl->l_max_cells, (unsigned long long)w * h);
        }
    }
}


// --- banded host path (fx_capi.cu featurize_banded) --------------------------
//
// After the one compaction of a banded call, every queued ROI is bucketed by the
// band holding its window's last row (its pixels are all on the device once that
// band's intensities have arrived): per (band, class) counts and the smallest
// rank per band, then the band-major lists and one control block per band, so the
// host issues the per-band kernels without copying anything to the device.

__device__ __forceinline__ bool band_item(const RoiList& rl, const Control* ctl, uint32_t i,
                                          const BandPlan& bp, uint32_t& r, uint32_t& b,
                                          uint32_t& k) {
    uint32_t base = 0;
    for (k = 0; k < (uint32_t)kNumClasses; ++k) {
        const uint32_t n = ctl->class_count[k];
        if (i < base + n) break;
        base += n;
    }
    if (k == (uint32_t)kNumClasses) return false;
    const uint32_t* lst = k == kClassS0 ? rl.cls_list[kClassS0]
                          : k == kClassS1 ? rl.cls_list[kClassS1]
                          : k == kClassS2 ? rl.cls_list[kClassS2] : rl.cls_list[kClassL];
    r = lst[i - base];
    b = bp.band_of(rl.y0[r] + rl.h[r] - 1);
    return true;
}

__global__ void k_band_count(RoiList rl, const Control* ctl, BandPlan bp, uint32_t* cnt,
                             uint32_t* first) {
    const uint32_t total = ctl->class_count[0] + ctl->class_count[1] + ctl->class_count[2] +
                           ctl->class_count[3];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        uint32_t r, b, k;
        if (!band_item(rl, ctl, i, bp, r, b, k)) continue;
        atomicAdd(&cnt[b * kNumClasses + k], 1u);
        atomicMin(&first[b], r);
    }
}

__global__ void k_band_scatter(RoiList rl, const Control* ctl, BandPlan bp, const uint32_t* cnt,
                               uint32_t* cursor, uint32_t* seg, Control* band_ctl) {
    const uint32_t nb = bp.nb;
    __shared__ uint32_t off[kMaxBands * kNumClasses];
    if (threadIdx.x == 0) {  // class-major exclusive offsets: off[k nb + b] (<= 256 entries),
        uint32_t acc = 0;      // so a run of consecutive bands is one range per class
        for (uint32_t k = 0; k < (uint32_t)kNumClasses; ++k)
            for (uint32_t b = 0; b < nb; ++b) {
                off[k * nb + b] = acc;
                acc += cnt[b * kNumClasses + k];
            }
    }
    __syncthreads();
    const uint32_t total = ctl->class_count[0] + ctl->class_count[1] + ctl->class_count[2] +
                           ctl->class_count[3];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        uint32_t r, b, k;
        if (!band_item(rl, ctl, i, bp, r, b, k)) continue;
        seg[off[k * nb + b] + atomicAdd(&cursor[b * kNumClasses + k], 1u)] = r;
    }
    if (blockIdx.x == 0 && threadIdx.x < nb) {  // control block of each band
        Control c = *ctl;
        const uint32_t b = threadIdx.x;
        for (int k = 0; k < kNumClasses; ++k) {
            c.class_count[k] = cnt[b * kNumClasses + k];
            c.class_next[k] = 0;
        }
        c.overflow_count = c.overflow_next = 0;
        c.t_next[0] = c.t_next[1] = 0;
        c.mom_alloc = c.int_alloc = 0;
        c.w_next = c.b_next_big = 0;
        c.error = 0;
        band_ctl[b] = c;
    }
}


// --- whole slide over several devices (fx_multi_featurize_slide) ---------------
//
// Each device scans its own row band into its own label table.  The tables are
// merged by peer reads over NVLink (a device listed twice reads its own memory):
// every device sums the counts and takes the min / max of the boxes of all bands
// for labels [0, lmax] into a scratch table (the peers' tables are only read, so
// no device sees a half-merged table), then commits it.  Integer sums and min /
// max are order-free, so every device ends with the table a whole-slide scan
// would give, bit for bit.

__global__ void k_table_merge(TablePeers tp, uint32_t lmax, unsigned long long* out_cnt,
                              uint32_t* out_bb, size_t out_pitch) {
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l <= lmax; l += gridDim.x * blockDim.x) {
        unsigned long long c = 0;
        uint32_t x0 = 0xffffffffu, y0 = 0xffffffffu, x1 = 0u, y1 = 0u;
        for (int e = 0; e < tp.n; ++e) {
            const unsigned long long ce = tp.cnt[e][l];
            if (!ce) continue;
            c += ce;
            const uint32_t* b = tp.bb[e];
            const size_t pp = tp.pitch[e];
            x0 = min(x0, b[l]);
            y0 = min(y0, b[pp + l]);
            x1 = max(x1, b[2 * pp + l]);
            y1 = max(y1, b[3 * pp + l]);
        }
        out_cnt[l] = c;
        out_bb[l] = x0;
        out_bb[out_pitch + l] = y0;
        out_bb[2 * out_pitch + l] = x1;
        out_bb[3 * out_pitch + l] = y1;
    }
}

// Straddling windows: rectangle k covers slide rows [y_lo, y_hi) and columns
// [x_lo, x_hi) of the owner's window below its band; the rows come from the band
// of device src (peer pointers), into the owner's raster at row (y - y_own).
// One block per (rectangle, row chunk), 16 B copies where the columns allow.
__global__ void k_halo_gather(const HaloRect* rects, int n_rects, const uint16_t* const* srcL,
                              const uint16_t* const* srcI, const size_t* src_pitch,
                              const int* src_y0, uint16_t* dstL, uint16_t* dstI, size_t dst_pitch,
                              int dst_y0) {
    for (int k = blockIdx.y; k < n_rects; k += gridDim.y) {
        const HaloRect r = rects[k];
        const uint16_t* sL = srcL[r.src];
        const uint16_t* sI = srcI[r.src];
        const size_t sp = src_pitch[r.src];
        const int sy0 = src_y0[r.src];
        const int w = r.x_hi - r.x_lo;
        for (int y = r.y_lo + blockIdx.x; y < r.y_hi; y += gridDim.x) {
            const size_t so = (size_t)(y - sy0) * sp + r.x_lo;
            const size_t dof = (size_t)(y - dst_y0) * dst_pitch + r.x_lo;
            for (int x = threadIdx.x; x < w; x += blockDim.x) {
                dstL[dof + x] = sL[so + x];
                dstI[dof + x] = sI[so + x];
            }
        }
    }
}


// --- pixel clouds (RoiRegistry::cloud, roi.cpp:76-148) --------------------------
//
// One warp per ROI walks its window row by row, 32 columns at a time; member
// pixels are ballot-compacted, so each cloud comes out in mask scan order (the
// reference's order) at its offset in label order: (x, y) global, intensity.
__global__ void k_cloud_gather(DevImage img, RoiList rl, const Control* ctl,
                               const unsigned long long* offsets, uint32_t* xs, uint32_t* ys,
                               uint16_t* vs) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    const uint32_t n = ctl->n_rois;
    for (uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const uint32_t L = rl.label[r], x0 = rl.x0[r], y0 = rl.y0[r], w = rl.w[r], h = rl.h[r];
        unsigned long long at = offsets[r];
        for (uint32_t y = 0; y < h; ++y) {
            const size_t row = (size_t)(y0 + y) * img.pitch + x0;
            for (uint32_t x = 0; x < w; x += 32) {
                const bool in = x + lane < w && img.L[row + x + lane] == L;
                const unsigned m = __ballot_sync(kFull, in);
                if (in) {
                    const unsigned long long k = at + __popc(m & lanemask_lt());
                    xs[k] = (uint32_t)rl.gx[r] + x + lane;
                    ys[k] = (uint32_t)rl.gy[r] + y;
                    vs[k] = img.I[row + x + lane];
                }
                at += __popc(m);
            }
        }
    }
}


// --- packed host rows (fx_pack.hpp) -------------------------------------------
//
// One 256-thread CTA per (row, 2048-pixel tile) of a packed block, 8 pixels per
// thread (16 B stores).  Labels: a binary search from the tile's first segment
// for the one covering the thread's first pixel, then a walk over the (rarely
// more than one or two) change points inside its 8 pixels.  Intensities: the
// labelled pixels' values follow in row order, so a thread's first value sits at
// the tile's count plus the labelled pixels before it in the tile (block scan).
__global__ void __launch_bounds__(256) k_unpack_labels(const uint8_t* __restrict__ region, int rows,
                                                       int W, uint16_t* __restrict__ L, size_t P) {
    const int tiles = pk_tiles(W), t = (int)blockIdx.x, row = (int)blockIdx.y;
    const uint32_t* tile_seg = reinterpret_cast<const uint32_t*>(region);
    const uint32_t* seg = reinterpret_cast<const uint32_t*>(region + pk_index_bytes(rows, W));
    const size_t ti = (size_t)row * tiles + t;
    const uint32_t rs = tile_seg[(size_t)row * tiles], re = tile_seg[(size_t)(row + 1) * tiles];
    const int x0 = t * kPackTile + (int)threadIdx.x * 8;
    if (x0 >= W) return;
    auto x_of = [&](uint32_t k) -> uint32_t { return k < re ? (seg[k] & 0xffffu) : 0x10000u; };
    // the segment covering the tile's first pixel is the tile's first or the one before
    uint32_t lo = max(rs, tile_seg[ti] ? tile_seg[ti] - 1u : 0u), hi = re - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (x_of(mid) <= (uint32_t)x0) lo = mid;
        else hi = mid - 1;
    }
    uint32_t k = lo, nx = x_of(k + 1), lab = seg[k] >> 16;
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        while ((uint32_t)(x0 + j) >= nx) {
            ++k;
            lab = seg[k] >> 16;
            nx = x_of(k + 1);
        }
        v[j] = lab;
    }
    uint16_t* out = L + (size_t)row * P;
    if (x0 + 8 <= W) {
        *reinterpret_cast<uint4*>(out + x0) =
            make_uint4(v[0] | v[1] << 16, v[2] | v[3] << 16, v[4] | v[5] << 16, v[6] | v[7] << 16);
    } else {
        for (int j = 0; j < 8 && x0 + j < W; ++j) out[x0 + j] = (uint16_t)v[j];
    }
}

__global__ void __launch_bounds__(256) k_unpack_intensity(const uint8_t* __restrict__ region, int rows,
                                                          int W, const uint16_t* __restrict__ L,
                                                          uint16_t* __restrict__ I, size_t P) {
    __shared__ uint32_t warp_tot[8];
    const int tiles = pk_tiles(W), t = (int)blockIdx.x, row = (int)blockIdx.y;
    const uint32_t* tile_pix = reinterpret_cast<const uint32_t*>(region);
    const uint16_t* pix = reinterpret_cast<const uint16_t*>(region + pk_index_bytes(rows, W));
    const int x0 = t * kPackTile + (int)threadIdx.x * 8;
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint16_t* lrow = L + (size_t)row * P;
    uint32_t lab[8];
    if (x0 + 8 <= W) {
        const uint4 q = *reinterpret_cast<const uint4*>(lrow + x0);
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) lab[j] = (w4[j >> 1] >> (16 * (j & 1))) & 0xffffu;
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) lab[j] = x0 + j < W ? lrow[x0 + j] : 0u;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) cnt += lab[j] != 0u;
    const uint32_t incl = warp_incl_scan(cnt);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (unsigned q = 0; q < wid; ++q) before += warp_tot[q];
    if (x0 >= W) return;
    uint32_t at = tile_pix[(size_t)row * tiles + t] + before + incl - cnt;
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = lab[j] ? pix[at++] : 0u;
    uint16_t* out = I + (size_t)row * P;
    if (x0 + 8 <= W) {
        *reinterpret_cast<uint4*>(out + x0) =
            make_uint4(v[0] | v[1] << 16, v[2] | v[3] << 16, v[4] | v[5] << 16, v[6] | v[7] << 16);
    } else {
        for (int j = 0; j < 8 && x0 + j < W; ++j) out[x0 + j] = (uint16_t)v[j];
    }
}

}  // namespace fxg
