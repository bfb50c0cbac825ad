// Label scan + ROI compaction (replaces RoiRegistry::accumulate / labels(),
// reference roi.cpp:76-117).
//
// k_label_scan: one coalesced HBM sweep over the uint16 label raster (16 B vector
// loads, 8 labels per thread).  Each thread owns an 8-pixel-wide x 8-row strip
// and folds the pixels it sees into a 2-entry register cache; evictions go to a
// per-CTA shared-memory hash table (smem atomics), which is flushed to the
// direct-mapped global LabelTable with one set of global atomics per (tile,
// label).  Integer min/max/sum are order-free, so the table is bit-exact and
// deterministic.  Intensities are not read here (the per-ROI kernels gather
// them), so the sweep moves 2 B/px.
//
// k_compact_count / k_compact_emit: ascending list of present labels (rank =
// output row), bbox -> window, window-size class lists for the per-ROI kernels.
#include "fx_dev.cuh"

namespace fxg {

namespace {

constexpr int kScanThreads = 256;  // 8 warps
constexpr int kTileW = 256;        // 32 lanes x 8 px
constexpr int kRowsPerWarp = 8;
constexpr int kTileH = 8 * kRowsPerWarp;  // 64
constexpr int kHashBits = 9;
constexpr int kHash = 1 << kHashBits;

struct CacheEnt {
    uint32_t label, cnt, x0, x1, y0, y1;
};

struct ScanSmem {
    uint32_t key[kHash];
    uint32_t cnt[kHash];
    uint32_t x0[kHash], x1[kHash], y0[kHash], y1[kHash];
};

__device__ __forceinline__ void global_fold(const LabelTable& t, uint32_t l, uint32_t cnt,
                                            uint32_t x0, uint32_t x1, uint32_t y0,
                                            uint32_t y1) {
    atomicAdd(&t.cnt[l], (unsigned long long)cnt);
    atomicMin(&t.xmin[l], x0);
    atomicMax(&t.xmax[l], x1);
    atomicMin(&t.ymin[l], y0);
    atomicMax(&t.ymax[l], y1);
}

__device__ __forceinline__ void hash_fold(ScanSmem& s, const LabelTable& t, const CacheEnt& e) {
    if (e.label == 0) return;
    uint32_t slot = (e.label * 2654435761u) >> (32 - kHashBits);
    for (int probe = 0; probe < kHash; ++probe) {
        uint32_t k = s.key[slot];
        if (k == 0) {
            k = atomicCAS(&s.key[slot], 0u, e.label);
            if (k == 0) k = e.label;
        }
        if (k == e.label) {
            atomicAdd(&s.cnt[slot], e.cnt);
            atomicMin(&s.x0[slot], e.x0);
            atomicMax(&s.x1[slot], e.x1);
            atomicMin(&s.y0[slot], e.y0);
            atomicMax(&s.y1[slot], e.y1);
            return;
        }
        slot = (slot + 1) & (kHash - 1);
    }
    global_fold(t, e.label, e.cnt, e.x0, e.x1, e.y0, e.y1);  // table full: direct
}

__device__ __forceinline__ void cache_add(CacheEnt& c0, CacheEnt& c1, ScanSmem& s,
                                          const LabelTable& t, uint32_t l, uint32_t x,
                                          uint32_t y) {
    if (l == c0.label) {
        c0.cnt++;
        c0.x0 = min(c0.x0, x);
        c0.x1 = max(c0.x1, x);
        c0.y1 = y;  // rows are visited in increasing order
    } else if (l == c1.label) {
        c1.cnt++;
        c1.x0 = min(c1.x0, x);
        c1.x1 = max(c1.x1, x);
        c1.y1 = y;
    } else {
        hash_fold(s, t, c1);
        c1 = c0;
        c0 = CacheEnt{l, 1u, x, x, y, y};
    }
}

}  // namespace

__global__ void __launch_bounds__(kScanThreads)
    k_label_scan(const uint16_t* __restrict__ L, int W, int H, size_t pitch, int vec_ok,
                 LabelTable t) {
    __shared__ ScanSmem s;
    for (int i = threadIdx.x; i < kHash; i += kScanThreads) {
        s.key[i] = 0;
        s.cnt[i] = 0;
        s.x0[i] = 0xffffffffu;
        s.x1[i] = 0;
        s.y0[i] = 0xffffffffu;
        s.y1[i] = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tiles_x = (W + kTileW - 1) / kTileW;
    const int tiles_y = (H + kTileH - 1) / kTileH;
    const int n_tiles = tiles_x * tiles_y;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int x = tx * kTileW + lane * 8;
        const int ybase = ty * kTileH + warp * kRowsPerWarp;
        CacheEnt c0{0, 0, 0, 0, 0, 0}, c1{0, 0, 0, 0, 0, 0};
        uint4 v[kRowsPerWarp];
        if (vec_ok && x + 8 <= W) {
#pragma unroll
            for (int r = 0; r < kRowsPerWarp; ++r) {
                const int y = ybase + r;
                v[r] = (y < H) ? __ldcs(reinterpret_cast<const uint4*>(L + (size_t)y * pitch + x))
                               : make_uint4(0, 0, 0, 0);
            }
        } else {
#pragma unroll
            for (int r = 0; r < kRowsPerWarp; ++r) {
                const int y = ybase + r;
                uint32_t wv[4] = {0, 0, 0, 0};
                if (y < H) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (x + k < W)
                            wv[k >> 1] |= (uint32_t)L[(size_t)y * pitch + x + k] << (16 * (k & 1));
                }
                v[r] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
        }
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r) {
            const uint32_t wv[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
            if ((wv[0] | wv[1] | wv[2] | wv[3]) == 0) continue;
            const uint32_t y = (uint32_t)(ybase + r);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t l = (wv[k >> 1] >> (16 * (k & 1))) & 0xffffu;
                if (l) cache_add(c0, c1, s, t, l, (uint32_t)(x + k), y);
            }
        }
        hash_fold(s, t, c0);
        hash_fold(s, t, c1);
        __syncthreads();
        for (int i = threadIdx.x; i < kHash; i += kScanThreads) {
            const uint32_t k = s.key[i];
            if (k) {
                global_fold(t, k, s.cnt[i], s.x0[i], s.x1[i], s.y0[i], s.y1[i]);
                s.key[i] = 0;
                s.cnt[i] = 0;
                s.x0[i] = 0xffffffffu;
                s.x1[i] = 0;
                s.y0[i] = 0xffffffffu;
                s.y1[i] = 0;
            }
        }
        __syncthreads();
    }
}

// --- compaction -------------------------------------------------------------

__global__ void __launch_bounds__(1024) k_compact_count(LabelTable t, Control* ctl) {
    const uint32_t l = blockIdx.x * 1024 + threadIdx.x;
    const int present = (l != 0 && t.cnt[l] != 0ull);
    const int c = __syncthreads_count(present);
    if (threadIdx.x == 0) ctl->block_sum[blockIdx.x] = (uint32_t)c;
}

// class of a window (w x h) with n pixels
__device__ __forceinline__ int roi_class(uint32_t w, uint32_t h, unsigned long long n) {
    if (w <= (uint32_t)kSW && h <= (uint32_t)kSH) return n <= (unsigned long long)kS1N ? kClassS1 : kClassS2;
    return kClassL;
}

__global__ void __launch_bounds__(1024) k_compact_emit(LabelTable t, Control* ctl, RoiList r) {
    __shared__ uint32_t warp_cnt[32];
    __shared__ uint32_t block_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) {
        uint32_t a = (lane < blockIdx.x) ? ctl->block_sum[lane] : 0;
        uint32_t b = (lane + 32 < blockIdx.x) ? ctl->block_sum[lane + 32] : 0;
        uint32_t s = warp_sum(a + b);
        if (lane == 0) block_base = s;
        if (blockIdx.x == gridDim.x - 1) {
            uint32_t tot = warp_sum((lane < gridDim.x ? ctl->block_sum[lane] : 0u) +
                                    (lane + 32 < gridDim.x ? ctl->block_sum[lane + 32] : 0u));
            if (lane == 0) ctl->n_rois = tot;
        }
    }
    const uint32_t l = blockIdx.x * 1024 + tid;
    const unsigned long long n = (l != 0) ? t.cnt[l] : 0ull;
    const bool present = n != 0ull;
    const unsigned m = __ballot_sync(kFull, present);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
        uint32_t c = warp_cnt[lane];
        uint32_t incl = warp_incl_scan(c);
        warp_cnt[lane] = incl - c;
    }
    __syncthreads();
    if (!present) return;
    const uint32_t rank = block_base + warp_cnt[warp] + __popc(m & lanemask_lt());
    const uint32_t x0 = t.xmin[l], y0 = t.ymin[l];
    const uint32_t w = t.xmax[l] - x0 + 1, h = t.ymax[l] - y0 + 1;
    r.label[rank] = l;
    r.x0[rank] = x0;
    r.y0[rank] = y0;
    r.w[rank] = w;
    r.h[rank] = h;
    r.n[rank] = n;
    const int c = roi_class(w, h, n);
    const uint32_t pos = atomicAdd(&ctl->class_count[c], 1u);
    r.cls_list[c][pos] = rank;
    if (c == kClassL) {
        atomicMax(&ctl->l_max_h, h);
        atomicMax(&ctl->l_max_wpr, (w + 63) / 64);
        atomicMax(&ctl->l_max_n, n);
        atomicMax(&ctl->l_max_cells, (unsigned long long)w * h);
    }
}

}  // namespace fxg
