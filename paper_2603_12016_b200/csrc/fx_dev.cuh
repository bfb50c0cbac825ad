// Shared device-side definitions for libfxg (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fxg {

// label-scan tuning (rows per load batch, min blocks/SM, grid waves, strip rows;
// the strip height divides the 64-row slot-map granularity).  Measured on C2
// (tools/kbench.py): 8 rows x 1 block/SM 130 us, 2 rows x 8 blocks/SM 86 us --
// the sweep is latency-bound, occupancy (bytes in flight) is the lever.
#ifndef FXG_SCAN_BATCH
#define FXG_SCAN_BATCH 4
#endif
#ifndef FXG_SCAN_MINB
#define FXG_SCAN_MINB 8
#endif
#ifndef FXG_SCAN_WAVES
#define FXG_SCAN_WAVES 16
#endif
#ifndef FXG_B_MINB
#define FXG_B_MINB 2  // large-ROI kernel: min CTAs per SM (register cap; 2: 7.1 -> 5.2 ms on C5-regime)
#endif
#ifndef FXG_SCAN_ROWS
#define FXG_SCAN_ROWS 64
#endif

constexpr int kMaxLabels = 65536;  // uint16 labels (reference image.hpp:24)
constexpr unsigned kFull = 0xffffffffu;

// Per-label accumulators of the label scan, direct-mapped by (slot, label value)
// (replaces RoiRegistry's std::map<label, Entry>, roi.cpp:76-110).  A slot is one
// image of a batch; slot s owns entries [s*65536, (s+1)*65536).  Entries are left
// in the reset state (cnt 0, min ~0, max 0) by the compaction that consumes them.
struct LabelTable {
    unsigned long long* cnt;  // [slots*65536] pixel count
    uint32_t* xmin;           // inclusive bbox, global coordinates (origin added)
    uint32_t* ymin;
    uint32_t* xmax;
    uint32_t* ymax;
    uint32_t* maxlab;         // [slots] largest label seen (bounds the compaction)
};

// One image of a batch, stacked row-wise in one pitched raster: image rows
// [row0, row0+h) of the stack, columns [0, w); origin (ox, oy) is added to the
// table coordinates.  row0 is a multiple of the scan strip height (64).
struct SlotInfo {
    int32_t row0, w, h, ox, oy;
};
struct SlotMap {
    const SlotInfo* info;        // [nslots] device; null -> single image s0
    const uint16_t* strip_slot;  // [stack rows / 64] slot of each 64-row strip
    SlotInfo s0;
    int nslots;
};

// ROI classes by window (bbox) size; each is consumed by its own persistent kernel.
enum RoiClass { kClassS0 = 0, kClassS1 = 1, kClassS2 = 2, kClassL = 3, kNumClasses = 4 };

// S-class limits: window fits a 64x64 TMA staging tile, one u64 mask word per row.
constexpr int kSW = 64, kSH = 64;
// TMA staging tile: box x origin must be 16 B aligned (multiple of 8 u16) on
// sm_100a (an unaligned innermost coordinate raises "illegal instruction"),
// so the box starts at x0 & ~7 and is 72 wide to cover any 64-wide window.
constexpr int kStageW = 72;
// S0: small windows (w <= 33, h <= 40) staged in a 40-wide tile -> half the slab
// S0 staging tile width (TMA boxes start at x0 & ~7, so windows up to kStageW0 - 7 wide)
#ifndef FXG_STAGEW0
#define FXG_STAGEW0 40
#endif
constexpr int kStageW0 = FXG_STAGEW0, kS0W = kStageW0 - 7, kS0H = 40;
constexpr int kS1N = 1024;  // max ROI pixels for S1
// max ROI pixels for S0: sizes the per-warp buffers (vals, xy, sort), so it sets how
// many S0 warps fit an SM; S0-shaped windows with more pixels go to S1
#ifndef FXG_S0N
#define FXG_S0N 768
#endif
constexpr int kS0N = FXG_S0N;
constexpr int kS2N = 4096;  // = kSW*kSH
constexpr int kS1Runs = 512;
constexpr int kS2Runs = 2176;  // >= worst case (33 free runs x 64 rows + 64)

// k_roi_b takes the windows above this many cells first (one sweep of the L list),
// then the rest: a few slide-tall windows picked up last would otherwise run alone
// at the end of the launch
constexpr unsigned long long kBigCells = 1ull << 20;

// Device-side control block, zeroed per featurize call.
struct Control {
    uint32_t n_rois;
    uint32_t class_count[kNumClasses];
    uint32_t class_next[kNumClasses];
    uint32_t overflow_count;  // S ROIs re-queued to the L path (run capacity)
    uint32_t overflow_next;
    uint32_t l_max_h;         // max window height among L ROIs
    uint32_t l_max_wpr;       // max 64-bit words per row among L ROIs
    unsigned long long l_max_n;      // max pixel count among L ROIs
    unsigned long long l_max_cells;  // max window cells among L ROIs
    uint32_t t_next[2];              // GLRLM/GLSZM/NGTDM work counters (S lists, L list)
    unsigned long long mom_alloc;    // moments: pixels staged so far (bump allocator)
    unsigned long long int_alloc;    // intensity: sorted values staged so far
    uint32_t w_next;                 // wide texture kernel (ng > 256) work counter
    uint32_t b_next_big;             // k_roi_b: first sweep, windows of > kBigCells cells
    // sticky across the sub-batches of one API call: compact_stage clears only the
    // fields above (offsetof(Control, error) bytes); the call's first stage clears all
    uint32_t error;                  // bit flags, see kErr*
    uint32_t pad_;
};

// whole slide over several devices: the label tables of the bands (peer pointers)
constexpr int kMaxPeers = 16;
struct TablePeers {
    const unsigned long long* cnt[kMaxPeers];
    const uint32_t* bb[kMaxPeers];  // xmin | ymin | xmax | ymax rows, pitch[e] apart
    size_t pitch[kMaxPeers];
    int n;
};
// one rectangle of a straddling window to fetch from band src
struct HaloRect {
    int src, y_lo, y_hi, x_lo, x_hi;
};

// banded host path: at most this many row bands per call
constexpr int kMaxBands = 64;
// Row bands of a banded call: nb1 bands of `rows` rows from row 0, then the rest
// (from split_y) in bands of `rows2` (the last band is cut finer, so the work left
// after the last copy is small).
struct BandPlan {
    uint32_t rows, rows2, split_y, nb1, nb;
    __host__ __device__ uint32_t band_of(uint32_t y) const {
        const uint32_t b = y < split_y ? y / rows : nb1 + (y - split_y) / rows2;
        return b < nb ? b : nb - 1;
    }
    __host__ __device__ uint32_t y0_of(uint32_t b) const {
        return b < nb1 ? b * rows : split_y + (b - nb1) * rows2;
    }
};

// compaction scratch: per (slot, 1024-label block) counts and exclusive bases
constexpr int kBlocksPerSlot = kMaxLabels / 1024;
constexpr uint32_t kBlockLive = 0x80000000u;  // block_sum flag: block <= maxlab

constexpr uint32_t kErrCapacity = 1u;  // L slab too small for a ROI
constexpr uint32_t kErrRuns = 2u;      // L run capacity exceeded
constexpr uint32_t kErrWindow = 4u;    // an owned ROI window is not inside the image
constexpr uint32_t kErrOutCap = 8u;    // more ROIs than output rows: no per-ROI kernel ran

// compaction parameters: owned row range (band sharding; [0, ~0) = all), in
// global coordinates, and the scratch arrays
struct CompactArgs {
    uint32_t own_y0, own_y1;
    uint32_t cap_rows;     // output rows available; above it no ROI is queued (kErrOutCap)
    uint32_t* block_sum;   // [nslots*64]
    uint32_t* block_base;  // [nslots*64]
    uint32_t* slot_base;   // [nslots+1] first output row of each slot, + total
    uint32_t* live;        // [nslots*64] live pairs, ascending
    uint32_t* done;        // [2]: blocks finished (last-block scan), live pair count
};

// Compacted ROI list: rank r == output row r (labels ascending).
struct RoiList {
    uint32_t* label;
    int32_t* gx;  // global coordinates of the window origin (table xmin, ymin)
    int32_t* gy;
    uint32_t* x0;  // window origin in the (stacked) raster being read
    uint32_t* y0;
    uint32_t* w;
    uint32_t* h;
    unsigned long long* n;
    uint32_t* cls_list[kNumClasses];  // ranks per class, [65536] each
    uint32_t* overflow;               // ranks re-queued from S to L
};

struct DevImage {
    const uint16_t* I;
    const uint16_t* L;
    int w, h;
    size_t pitch;  // elements
    int ox, oy;    // global origin
};

// Feature configuration for the per-ROI kernels (resolved on the host).
struct FeatCfg {
    uint32_t groups;
    int ncols;
    int col_int, col_shape, col_mom, col_glcm;  // column offsets, -1 if absent
    int col_glrlm, col_glszm, col_ngtdm;
    int bins;                        // max(2, histogram_bins)
    int ng, symmetric, n_angles;
    int angle[8];                    // sorted (engine.cpp:36-40)
    int dx[8], dy[8];                // angle_offset (texture.cpp:15-23)
    uint64_t* shape_rows;            // shape: per ROI rank, 64 rows of all pixels + 64 of K
    uint32_t* shape_hdr;             // shape: per ROI rank, h | w << 8 | staged << 16
    uint32_t* mom_px;                // moments: staged pixels (x | y << 8 | v << 16), or null
    unsigned long long* mom_off;     // moments: per ROI rank, offset into mom_px (~0: not staged)
    unsigned long long* mom_sums;    // moments: per ROI rank, sS, sXI, sYI, sLX, sLY (exact)
    unsigned long long mom_cap;      // moments: capacity of mom_px (pixels)
    uint16_t* int_vals;              // intensity: staged sorted values, or null
    unsigned long long* int_off;     // intensity: per ROI rank, offset (~0: not staged)
    unsigned long long* int_sums;    // intensity: per ROI rank, sum v, sum v^2 (exact)
    unsigned long long int_cap;      // intensity: capacity of int_vals (values)
};

// GLCM variants of the S kernels: none, key sort (ng > 64), shared histogram
// (ng <= 64: keys la*64+lb < 4096, packed u16 counts)
enum GlcmMode { kGlNone = 0, kGlSort = 1, kGlHist = 2 };
constexpr int kGlHistMaxNg = 64;
__host__ __device__ inline int s_glcm_mode(const FeatCfg& c) {
    return c.col_glcm < 0 ? kGlNone : (c.ng <= kGlHistMaxNg ? kGlHist : kGlSort);
}

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T u = __shfl_xor_sync(kFull, v, o);
        v = u < v ? u : v;
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T u = __shfl_xor_sync(kFull, v, o);
        v = u > v ? u : v;
    }
    return v;
}
// inclusive prefix sum across the warp
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(kFull, v, o);
        if (lane >= (unsigned)o) v += u;
    }
    return v;
}

}  // namespace fxg
