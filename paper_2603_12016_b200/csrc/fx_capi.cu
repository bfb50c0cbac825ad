// Device context + orchestration of the featurize pipeline (C ABI, fxg.h).
//
//   H2D (host inputs only) -> k_label_scan -> k_compact_count -> k_compact_emit
//   -> k_roi_s<S1> / k_roi_s<S2> (TMA-staged windows, warp per ROI)
//   -> k_roi_b (large windows + S overflow: one CTA per ROI, global slabs) -> D2H table
//
// The only host synchronisation before the table readback is a small
// side-stream copy of the compaction counters (L-path slab sizing), which
// overlaps the S kernels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstddef>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fx_dev.cuh"
#include "fx_host.hpp"
#include "fx_pack.hpp"
#include "fx_roi.cuh"
#include "fxg.h"

namespace fxg {
__global__ void k_label_scan(const uint16_t* L, int W, int H, size_t pitch, int vec_ok, SlotMap m,
                             LabelTable t);
__global__ void k_compact_count(LabelTable t, Control* ctl, CompactArgs a, int nslots);
__global__ void k_compact_emit(LabelTable t, Control* ctl, RoiList r, CompactArgs a, SlotMap m);
__global__ void k_table_merge(TablePeers tp, uint32_t lmax, unsigned long long* out_cnt,
                              uint32_t* out_bb, size_t out_pitch);
__global__ void k_halo_gather(const HaloRect* rects, int n_rects, const uint16_t* const* srcL,
                              const uint16_t* const* srcI, const size_t* src_pitch,
                              const int* src_y0, uint16_t* dstL, uint16_t* dstI, size_t dst_pitch,
                              int dst_y0);
__global__ void k_cloud_gather(DevImage img, RoiList rl, const Control* ctl,
                               const unsigned long long* offsets, uint32_t* xs, uint32_t* ys,
                               uint16_t* vs);
__global__ void k_band_count(RoiList rl, const Control* ctl, BandPlan bp, uint32_t* cnt,
                             uint32_t* first);
__global__ void k_unpack_labels(const uint8_t* region, int rows, int W, uint16_t* L, size_t P);
__global__ void k_unpack_intensity(const uint8_t* region, int rows, int W, const uint16_t* L,
                                   uint16_t* I, size_t P);
__global__ void k_band_scatter(RoiList rl, const Control* ctl, BandPlan bp, const uint32_t* cnt,
                               uint32_t* cursor, uint32_t* seg, Control* band_ctl);
cudaError_t roi_s_setup(int* occ /* [3][3]: class x GlcmMode */);
void launch_roi_s(int cls, int grid, cudaStream_t s, const CUtensorMap* tmaps, int tma40, int tma72,
                  DevImage img, RoiList rl, Control* ctl, FeatCfg cfg, double* out,
                  const DebugOut* dbg);
cudaError_t roi_b_setup();
void launch_shape_serial(int n_s, cudaStream_t s, RoiList rl, Control* ctl, FeatCfg cfg,
                         double* out);
cudaError_t roi_t_setup();
void launch_serial_stats(int n_s, bool intensity, bool moments, cudaStream_t s, RoiList rl,
                         Control* ctl, FeatCfg cfg, double* out, cudaStream_t s2, cudaEvent_t fork,
                         cudaEvent_t join);
TLayout make_tlayout(unsigned long long CELLS, uint32_t NMAX);
void launch_roi_t(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                  double* out, uint8_t* scratch, const TLayout& T, int which, bool init);
BLayout make_blayout(uint32_t H, uint32_t WPR, uint32_t NMAX, uint32_t RUNMAX, uint32_t NB,
                     unsigned long long CELLS);
void launch_roi_b(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                  double* out, const DebugOut* dbg, uint8_t* scratch, const BLayout& B);
WLayout make_wlayout(unsigned long long cells, unsigned long long nmax, int ng);
cudaError_t wide_setup();
void launch_texture_wide(int grid, cudaStream_t s, DevImage img, RoiList rl, Control* ctl, FeatCfg cfg,
                         double* out, uint8_t* scratch, const WLayout& L);
}  // namespace fxg

using namespace fxg;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess)                                                       \
            return set_error(e_ == cudaErrorMemoryAllocation ? FX_E_OOM : FX_E_CUDA, \
                             std::string(#x) + ": " + cudaGetErrorString(e_));      \
    } while (0)


struct KTime {
    double ms = 0;
    uint64_t count = 0;
};

struct fx_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own_stream = nullptr, stream = nullptr, side = nullptr;
    cudaStream_t copy = nullptr;  // batch staging (H2D of the next sub-batch)
    cudaStream_t d2h = nullptr;   // banded host path: feature rows back while bands compute
    cudaStream_t copy2 = nullptr; // packed host path: packed blocks next to the raw ones
    // banded host path (featurize_banded): per-band events and pinned host staging
    std::vector<cudaEvent_t> ev_band;  // 3 per band: labels in, intensities in, rows done
    uint32_t* d_band = nullptr;        // [cnt kMaxBands*4][cursor kMaxBands*4][first kMaxBands]
    uint32_t* h_band = nullptr;        // pinned mirror of d_band
    Control* d_band_ctl = nullptr;     // one control block per band
    Control* h_band_ctl = nullptr;     // pinned mirror (error flags)
    uint32_t* d_band_seg = nullptr;    // class-major band lists [roi_cap] (band_range_lists)
    size_t band_seg_cap = 0;
    // whole slide over several devices (fx_multi_featurize_slide)
    unsigned long long* d_mcnt = nullptr;  // merged table scratch (slot-0 layout)
    uint32_t* d_mbb = nullptr;
    uint8_t* d_slide = nullptr;            // halo rects + peer pointer arrays
    size_t slide_bytes = 0;
    uint16_t* d_work = nullptr;            // band + halo raster when the reserve is too small
    size_t work_elems = 0;
    uint8_t* d_wscratch = nullptr;         // wide texture kernel slabs (ng > 256)
    size_t wscratch_bytes = 0;
    cudaEvent_t ev_compact = nullptr, ev_stats = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // the serial passes on two streams
    cudaEvent_t ev_staged[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    // label table: tab_slots slices of 65536 entries, left reset by each compaction
    int tab_slots = 0;
    bool table_clean = false;  // every entry in the reset state
    unsigned long long* d_cnt = nullptr;
    uint32_t* d_bb = nullptr;  // xmin | ymin | xmax | ymax, tab_slots*65536 each
    uint32_t* d_maxlab = nullptr;
    uint32_t* d_csum = nullptr;       // block_sum | block_base | live | slot_base | done
    uint32_t* h_slot_base = nullptr;  // pinned [tab_slots+1]
    Control* d_ctl = nullptr;
    Control* h_ctl = nullptr;  // pinned
    // ROI list: roi_cap entries (tab_slots * 65536)
    size_t roi_cap = 0;
    uint32_t* d_roi32 = nullptr;  // label,gx,gy,x0,y0,w,h + 4 class lists + overflow
    unsigned long long* d_roin = nullptr;
    // batch slot maps (double-buffered with pinned host mirrors)
    SlotInfo* d_slots[2] = {nullptr, nullptr};
    uint16_t* d_strips[2] = {nullptr, nullptr};
    SlotInfo* h_slots[2] = {nullptr, nullptr};
    uint16_t* h_strips[2] = {nullptr, nullptr};
    size_t map_slots_cap = 0, map_strips_cap = 0;
    // batch staging rasters (intensity then labels), double-buffered
    uint16_t* d_stage[2] = {nullptr, nullptr};
    size_t stage_elems = 0;  // per raster
    uint32_t* d_blab = nullptr;  // batch output labels (host outputs)
    size_t blab_cap = 0;
    // GLRLM/GLSZM/NGTDM slabs: [0] S-class windows, [1] large windows
    uint8_t* d_tscratch[2] = {nullptr, nullptr};
    size_t tscratch_bytes[2] = {0, 0};
    TLayout tlay_prev[2] = {};
    int tlay_grid[2] = {0, 0};
    // moments: staged pixels of the S ROIs for k_moments_serial
    uint32_t* d_mom_px = nullptr;
    unsigned long long* d_mom_off = nullptr;
    unsigned long long* d_mom_sums = nullptr;
    uint16_t* d_int_vals = nullptr;  // intensity: staged sorted values of the S ROIs
    unsigned long long* d_int_off = nullptr;
    unsigned long long* d_int_sums = nullptr;
    size_t int_cap = 0, int_off_cap = 0;
    size_t mom_cap = 0, mom_off_cap = 0;
    // shape group: per-ROI staged row masks (S ROIs) for k_shape_serial
    uint64_t* d_shape_rows = nullptr;
    uint32_t* d_shape_hdr = nullptr;
    size_t shape_cap = 0;
    // staging for host inputs / outputs
    uint16_t* d_img = nullptr;  // intensity then labels, pitched
    size_t img_pitch = 0, img_rows_cap = 0;
    double* d_out = nullptr;
    size_t out_cap = 0;  // doubles
    // L-path slabs
    uint8_t* d_lscratch = nullptr;
    size_t lscratch_bytes = 0;
    BLayout lay_prev{};  // layout of the last large-ROI launch (zeroed regions valid)
    int lay_grid = 0;
    // debug capture
    DebugOut* d_dbg = nullptr;
    // accounting
    uint64_t launches = 0;
    bool timing = false;
    std::string timing_only;  // non-empty: time only the kernel of this name
    std::map<std::string, KTime> ktimes;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> ev_pool;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    int occ_s[3][3] = {{1, 1, 1}, {1, 1, 1}, {1, 1, 1}};
    bool sync_debug = false;
    bool no_tma = false;
    bool no_stage = false;  // FXG_NO_STAGE=1: in-warp intensity / moments (tests)
    int band_rows = 0;      // FXG_BAND_ROWS: banded host path band height (0 auto, <0 off)
    // packed host rows (fx_pack.hpp): worker pool, pinned + device block staging,
    // the host's nonzero masks; FXG_PACK=0 / fx_ctx_set_packing(0) sends raw rows
    bool packing = true;
    int pack_raw_pct = 25;  // FXG_PACK_RAW: % of row blocks sent raw (DMA next to the packers)
    uint8_t* h_pack = nullptr;
    // batch path: packed staging in two halves (by staging buffer); events: a half's
    // host-to-device copies done, its unpack kernels done; one per shipped block
    size_t pack_half = 0;
    cudaEvent_t ev_pack_free[2] = {nullptr, nullptr}, ev_unpacked[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_blocks;
    std::vector<uint32_t> pack_mask_b[2];
    uint8_t* d_pack = nullptr;
    size_t pack_bytes = 0;
    std::vector<uint32_t> pack_mask;
    // bytes moved by the last call (host paths)
    uint64_t h2d_bytes = 0, d2h_bytes = 0;
};

namespace {

constexpr int kRoiArrays = 8 + kNumClasses;  // u32 arrays of the ROI list

RoiList roi_list(fx_ctx* c) {
    RoiList r;
    uint32_t* b = c->d_roi32;
    const size_t N = c->roi_cap;
    r.label = b;
    r.gx = reinterpret_cast<int32_t*>(b + 1 * N);
    r.gy = reinterpret_cast<int32_t*>(b + 2 * N);
    r.x0 = b + 3 * N;
    r.y0 = b + 4 * N;
    r.w = b + 5 * N;
    r.h = b + 6 * N;
    for (int k = 0; k < kNumClasses; ++k) r.cls_list[k] = b + (7 + k) * N;
    r.overflow = b + (7 + kNumClasses) * N;
    r.n = c->d_roin;
    return r;
}

LabelTable label_table(fx_ctx* c) {
    LabelTable t;
    const size_t N = (size_t)c->tab_slots * kMaxLabels;
    t.cnt = c->d_cnt;
    t.xmin = c->d_bb;
    t.ymin = c->d_bb + N;
    t.xmax = c->d_bb + 2 * N;
    t.ymax = c->d_bb + 3 * N;
    t.maxlab = c->d_maxlab;
    return t;
}

CompactArgs compact_args(fx_ctx* c, uint32_t own_y0, uint32_t own_y1, size_t cap_rows = ~size_t(0)) {
    const size_t nb = (size_t)c->tab_slots * kBlocksPerSlot;
    uint32_t* b = c->d_csum;
    const uint32_t cap = (uint32_t)std::min<size_t>(cap_rows, 0xffffffffu);
    return CompactArgs{own_y0,     own_y1,     cap, b, b + nb, b + 3 * nb, b + 2 * nb,
                       b + 3 * nb + c->tab_slots + 1};
}

// memset the whole table to the reset state (cnt 0, min ~0, max 0, maxlab 0)
int reset_table(fx_ctx* c) {
    const size_t N = (size_t)c->tab_slots * kMaxLabels;
    cudaStream_t s = c->stream;
    CK(cudaMemsetAsync(c->d_cnt, 0, N * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(c->d_bb, 0xff, 2 * N * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(c->d_bb + 2 * N, 0, 2 * N * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(c->d_maxlab, 0, (size_t)c->tab_slots * sizeof(uint32_t), s));
    c->table_clean = true;
    return FX_OK;
}

// table, compaction scratch and ROI list for `slots` images per launch
int ensure_slots(fx_ctx* c, int slots) {
    if (slots <= c->tab_slots) return FX_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->d_cnt);
    cudaFree(c->d_bb);
    cudaFree(c->d_maxlab);
    cudaFree(c->d_csum);
    if (c->h_slot_base) cudaFreeHost(c->h_slot_base);
    cudaFree(c->d_roi32);
    cudaFree(c->d_roin);
    c->d_cnt = nullptr;
    c->d_bb = c->d_maxlab = c->d_csum = c->h_slot_base = c->d_roi32 = nullptr;
    c->d_roin = nullptr;
    c->tab_slots = 0;
    c->roi_cap = 0;
    const size_t N = (size_t)slots * kMaxLabels;
    CK(cudaMalloc(&c->d_cnt, N * sizeof(unsigned long long)));
    CK(cudaMalloc(&c->d_bb, 4 * N * sizeof(uint32_t)));
    CK(cudaMalloc(&c->d_maxlab, (size_t)slots * sizeof(uint32_t)));
    const size_t csum = 3 * (size_t)slots * kBlocksPerSlot + slots + 1 + 2;
    CK(cudaMalloc(&c->d_csum, csum * sizeof(uint32_t)));
    CK(cudaMemset(c->d_csum, 0, csum * sizeof(uint32_t)));
    CK(cudaMallocHost(&c->h_slot_base, ((size_t)slots + 1) * sizeof(uint32_t)));
    CK(cudaMalloc(&c->d_roi32, (size_t)kRoiArrays * N * sizeof(uint32_t)));
    CK(cudaMalloc(&c->d_roin, N * sizeof(unsigned long long)));
    c->tab_slots = slots;
    c->roi_cap = N;
    return reset_table(c);
}

SlotMap single_map(const DevImage& img) {
    SlotMap m;
    m.info = nullptr;
    m.strip_slot = nullptr;
    m.s0 = SlotInfo{0, img.w, img.h, img.ox, img.oy};
    m.nslots = 1;
    return m;
}

cudaEvent_t get_event(fx_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Launch bracket: counts launches; with timing on, records events on the stream.
struct Launch {
    fx_ctx* c;
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    bool timed = false;
    Launch(fx_ctx* c_, const char* n, cudaStream_t on = nullptr)
        : c(c_), name(n), st(on ? on : c_->stream) {
        c->launches++;
        // each timing event between launches costs ~3 us of device time (it breaks
        // launch pipelining), so a filter can restrict timing to one kernel
        timed = c->timing && (c->timing_only.empty() || c->timing_only == n);
        if (timed) {
            a = get_event(c);
            b = get_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~Launch() {
        if (timed) {
            cudaEventRecord(b, st);
            c->pending.push_back({name, {a, b}});
        }
        if (c->sync_debug) {  // FXG_SYNC_DEBUG=1: attribute device faults to a kernel
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) fprintf(stderr, "[fxg] %s: %s\n", name, cudaGetErrorString(e));
        }
    }
};

void collect_times(fx_ctx* c) {
    for (auto& p : c->pending) {
        float ms = 0;
        cudaEventSynchronize(p.second.second);
        cudaEventElapsedTime(&ms, p.second.first, p.second.second);
        auto& k = c->ktimes[p.first];
        k.ms += ms;
        k.count++;
        c->ev_pool.push_back(p.second.first);
        c->ev_pool.push_back(p.second.second);
    }
    c->pending.clear();
}

// texture groups with more than 256 grey levels run on the wide kernel (fx_wide.cu)
constexpr int kWideNg = 256, kWideMaxNg = 32768;
bool wide_texture(const FeatCfg& f) {
    return f.ng > kWideNg && (f.col_glcm >= 0 || f.col_glrlm >= 0 || f.col_glszm >= 0 || f.col_ngtdm >= 0);
}
// the same configuration without the texture groups (their columns stay reserved)
FeatCfg core_cfg(FeatCfg f) {
    f.col_glcm = f.col_glrlm = f.col_glszm = f.col_ngtdm = -1;
    return f;
}

int validate_texture(unsigned groups, const fx_texture_params& p) {
    if (!(groups & (FX_GROUP_GLCM | FX_GROUP_GLRLM | FX_GROUP_GLSZM | FX_GROUP_NGTDM)))
        return FX_OK;
    if (p.ng < 2) return set_error(FX_E_CONFIG, "grey level count must be >= 2");
    if (p.ng > kWideMaxNg)  // the reference's level grid is int16 (texture.hpp:15-28)
        return set_error(FX_E_CONFIG, "grey level count above 32768");
    if (p.n_angles < 1 || p.n_angles > 8) return set_error(FX_E_CONFIG, "1..8 angles supported");
    for (int i = 0; i < p.n_angles; ++i) {
        const int a = p.angles[i];
        if (a != 0 && a != 45 && a != 90 && a != 135)
            return set_error(FX_E_CONFIG, "unsupported angle " + std::to_string(a));
    }
    return FX_OK;
}

FeatCfg make_cfg(unsigned groups, const fx_texture_params& p) {
    FeatCfg f{};
    f.groups = groups;
    int col = 0;
    f.col_int = f.col_shape = f.col_mom = f.col_glcm = -1;
    if (groups & FX_GROUP_INTENSITY) {
        f.col_int = col;
        col += 39;
    }
    if (groups & FX_GROUP_SHAPE) {  // engine.cpp:22-23 canonical order
        f.col_shape = col;
        col += 38;
    }
    if (groups & FX_GROUP_MOMENTS) {
        f.col_mom = col;
        col += 104;
    }
    if (groups & FX_GROUP_GLCM) {
        f.col_glcm = col;
        col += 29 * (p.n_angles + 1);
    }
    f.col_glrlm = f.col_glszm = f.col_ngtdm = -1;
    if (groups & FX_GROUP_GLRLM) {
        f.col_glrlm = col;
        col += 16 * (p.n_angles + 1);
    }
    if (groups & FX_GROUP_GLSZM) {
        f.col_glszm = col;
        col += 16;
    }
    if (groups & FX_GROUP_NGTDM) {
        f.col_ngtdm = col;
        col += 5;
    }
    f.ncols = col;
    f.bins = std::max(2, p.histogram_bins);
    f.ng = p.ng;
    f.symmetric = p.symmetric;
    const std::vector<int> a = sorted_angles(p);
    f.n_angles = (int)a.size();
    for (int i = 0; i < f.n_angles; ++i) {
        f.angle[i] = a[i];
        const int d = p.offset;
        switch (a[i]) {  // angle_offset, texture.cpp:15-23 (y points down)
            case 0: f.dx[i] = d; f.dy[i] = 0; break;
            case 45: f.dx[i] = d; f.dy[i] = -d; break;
            case 90: f.dx[i] = 0; f.dy[i] = -d; break;
            default: f.dx[i] = -d; f.dy[i] = -d; break;
        }
    }
    return f;
}

int ensure_out(fx_ctx* c, size_t doubles) {
    if (doubles <= c->out_cap) return FX_OK;
    if (c->d_out) cudaFree(c->d_out);
    c->d_out = nullptr;
    c->out_cap = 0;
    CK(cudaMalloc(&c->d_out, doubles * sizeof(double)));
    c->out_cap = doubles;
    return FX_OK;
}

int ensure_lscratch(fx_ctx* c, size_t bytes) {
    if (bytes <= c->lscratch_bytes) return FX_OK;
    if (c->d_lscratch) {
        cudaStreamSynchronize(c->stream);
        cudaFree(c->d_lscratch);
    }
    c->d_lscratch = nullptr;
    c->lscratch_bytes = 0;
    c->lay_grid = 0;
    CK(cudaMalloc(&c->d_lscratch, bytes));
    c->lscratch_bytes = bytes;
    return FX_OK;
}

int ensure_img(fx_ctx* c, int w, int h) {
    const size_t pitch = ((size_t)w + 63) / 64 * 64;  // elements; 128 B rows for TMA
    if (pitch <= c->img_pitch && (size_t)h <= c->img_rows_cap) return FX_OK;
    if (c->d_img) cudaFree(c->d_img);
    c->d_img = nullptr;
    c->img_pitch = c->img_rows_cap = 0;
    CK(cudaMalloc(&c->d_img, pitch * (size_t)h * 2 * sizeof(uint16_t)));
    c->img_pitch = pitch;
    c->img_rows_cap = (size_t)h;
    return FX_OK;
}

bool make_tmap(fx_ctx* c, const DevImage& img, const uint16_t* raster, CUtensorMap* m, int box_w) {
    if (!c->encode) return false;
    if ((reinterpret_cast<uintptr_t>(raster) & 15u) || ((img.pitch * 2) & 15u)) return false;
    if (img.w < box_w || img.h < 8) return false;
    cuuint64_t dims[2] = {(cuuint64_t)img.w, (cuuint64_t)img.h};
    cuuint64_t strides[1] = {(cuuint64_t)img.pitch * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_w, 8};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = c->encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)raster, dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// large-ROI slab layout from the compaction maxima (>= an S2 window, for overflow)
BLayout b_layout(const Control& h, int bins) {
    const uint32_t H = std::max<uint32_t>(h.l_max_h, kSH);
    const uint32_t WPR = std::max<uint32_t>(h.l_max_wpr, 1);
    const uint32_t NMAX = (uint32_t)std::max<unsigned long long>(h.l_max_n, kS2N);
    const unsigned long long cells = std::max<unsigned long long>(h.l_max_cells, (unsigned long long)kSW * kSH);
    // runs of the member mask: <= n and <= cells / 2 + H; runs of the window cells
    // outside K: <= (runs of K) + 1 per row <= n + H.  Bounding by n as well keeps a
    // tall, sparse window (a two-component ROI spanning a slide) from sizing every
    // CTA's slab by its cell count (C5: 13M -> 0.2M runs, 26 -> 296 CTAs)
    const uint32_t RUNMAX = (uint32_t)std::min<unsigned long long>(
        std::min<unsigned long long>(cells / 2 + H + 64, (unsigned long long)NMAX + H + 64), 64ull << 20);
    return make_blayout(H, WPR, NMAX, RUNMAX, (uint32_t)std::max(bins, 2), cells);
}

struct DebugHost {
    uint32_t label = 0;
    int nb = 0;
    unsigned long long* hist = nullptr;  // device
    int32_t* edge = nullptr;
    uint32_t cap_edge = 0;
    uint32_t* n_edge = nullptr;
    uint32_t* glcm = nullptr;
    unsigned long long* pairs = nullptr;
};

// Label scan of one image (or band) into the ctx's label table, in global
// coordinates (image origin added).  reset clears the table first.
// moments staging: pixels of the S ROIs (bounded; ROIs past the capacity keep the
// in-warp path) and per-ROI offsets
constexpr size_t kMomStagePixels = 64ull << 20;
int ensure_moments(fx_ctx* c, size_t img_pixels) {
    const size_t want = std::min(kMomStagePixels, std::max<size_t>(img_pixels, 1 << 20));
    if (want > c->mom_cap || c->roi_cap > c->mom_off_cap) {
        if (c->stream) cudaStreamSynchronize(c->stream);
        cudaFree(c->d_mom_px);
        cudaFree(c->d_mom_off);
        cudaFree(c->d_mom_sums);
        c->d_mom_px = nullptr;
        c->d_mom_off = nullptr;
        c->d_mom_sums = nullptr;
        c->mom_cap = c->mom_off_cap = 0;
        // +4 elements: the serial pass reads staged pixels in 16 B vectors
        CK(cudaMalloc(&c->d_mom_px, (want + 4) * sizeof(uint32_t)));
        CK(cudaMalloc(&c->d_mom_off, c->roi_cap * sizeof(unsigned long long)));
        CK(cudaMalloc(&c->d_mom_sums, c->roi_cap * 5 * sizeof(unsigned long long)));
        c->mom_cap = want;
        c->mom_off_cap = c->roi_cap;
    }
    return FX_OK;
}

int ensure_intensity(fx_ctx* c, size_t img_pixels) {
    const size_t want = std::min(kMomStagePixels, std::max<size_t>(img_pixels, 1 << 20));
    if (want > c->int_cap || c->roi_cap > c->int_off_cap) {
        if (c->stream) cudaStreamSynchronize(c->stream);
        cudaFree(c->d_int_vals);
        cudaFree(c->d_int_off);
        cudaFree(c->d_int_sums);
        c->d_int_vals = nullptr;
        c->d_int_off = nullptr;
        c->d_int_sums = nullptr;
        c->int_cap = c->int_off_cap = 0;
        // +8 elements: the serial pass reads staged values in 16 B vectors
        CK(cudaMalloc(&c->d_int_vals, (want + 8) * sizeof(uint16_t)));
        CK(cudaMalloc(&c->d_int_off, c->roi_cap * sizeof(unsigned long long)));
        CK(cudaMalloc(&c->d_int_sums, c->roi_cap * 2 * sizeof(unsigned long long)));
        c->int_cap = want;
        c->int_off_cap = c->roi_cap;
    }
    return FX_OK;
}

// shape staging for roi_cap ROIs: 128 row masks each, headers zeroed (consumed
// and reset by k_shape_serial)
int ensure_shape(fx_ctx* c) {
    if (c->roi_cap <= c->shape_cap) return FX_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->d_shape_rows);
    cudaFree(c->d_shape_hdr);
    c->d_shape_rows = nullptr;
    c->d_shape_hdr = nullptr;
    c->shape_cap = 0;
    CK(cudaMalloc(&c->d_shape_rows, c->roi_cap * 128 * sizeof(uint64_t)));
    CK(cudaMalloc(&c->d_shape_hdr, c->roi_cap * sizeof(uint32_t)));
    CK(cudaMemset(c->d_shape_hdr, 0, c->roi_cap * sizeof(uint32_t)));
    c->shape_cap = c->roi_cap;
    return FX_OK;
}

// reset: start from an empty table (a memset only when the last use left it dirty).
int scan_stage(fx_ctx* c, const DevImage& img, const SlotMap& m, bool reset) {
    if (reset && !c->table_clean) {
        int rc = reset_table(c);
        if (rc) return rc;
    }
    LabelTable t = label_table(c);
    cudaStream_t s = c->stream;
    const int vec_ok = ((reinterpret_cast<uintptr_t>(img.L) & 15u) == 0) && (img.pitch % 8 == 0);
    const int tiles = ((img.w + 255) / 256) * ((img.h + FXG_SCAN_ROWS - 1) / FXG_SCAN_ROWS);
    const int grid = std::max(1, std::min((tiles + 3) / 4, c->sm_count * FXG_SCAN_WAVES));
    Launch l(c, "k_label_scan");
    k_label_scan<<<grid, 128, 0, s>>>(img.L, img.w, img.h, img.pitch, vec_ok, m, t);
    CK(cudaGetLastError());
    return FX_OK;
}

// compaction of the table (slots of m) into the ROI list; consumes the table.
// More ROIs than cap_rows: none is queued for the per-ROI kernels (kErrOutCap).
// first: the first stage of an API call also clears the sticky error word.
int compact_stage(fx_ctx* c, const SlotMap& m, uint32_t own_y0, uint32_t own_y1, size_t cap_rows,
                  bool first) {
    LabelTable t = label_table(c);
    RoiList rl = roi_list(c);
    const CompactArgs ca = compact_args(c, own_y0, own_y1, cap_rows);
    cudaStream_t s = c->stream;
    const int nb = m.nslots * kBlocksPerSlot;
    const int grid = std::min(nb, 2 * c->sm_count);
    CK(cudaMemsetAsync(c->d_ctl, 0, first ? sizeof(Control) : offsetof(Control, error), s));
    {
        Launch l(c, "k_compact_count");
        k_compact_count<<<grid, 1024, m.nslots * sizeof(uint32_t), s>>>(t, c->d_ctl, ca, m.nslots);
    }
    {
        Launch l(c, "k_compact_emit");
        k_compact_emit<<<grid, 1024, 0, s>>>(t, c->d_ctl, rl, ca, m);
    }
    CK(cudaGetLastError());
    return FX_OK;
}

// Staging buffers of the serial passes for one call (intensity / moments / shape),
// unless debugging or FXG_NO_STAGE=1 (the in-warp paths, otherwise taken only when
// the staging buffers overflow, e.g. huge images).
int prepare_cfg(fx_ctx* c, const DevImage& img, unsigned groups, const fx_texture_params& p,
                const DebugOut* dbg_dev, FeatCfg* out) {
    FeatCfg cfg = make_cfg(groups, p);
    if (cfg.col_shape >= 0) {
        const int rs = ensure_shape(c);
        if (rs) return rs;
        cfg.shape_rows = c->d_shape_rows;
        cfg.shape_hdr = c->d_shape_hdr;
    }
    if (cfg.col_int >= 0 && !dbg_dev && !c->no_stage) {
        const int ri = ensure_intensity(c, (size_t)img.w * (size_t)img.h);
        if (ri) return ri;
        cfg.int_vals = c->d_int_vals;
        cfg.int_off = c->d_int_off;
        cfg.int_sums = c->d_int_sums;
        cfg.int_cap = c->int_cap;
    }
    if (cfg.col_mom >= 0 && !dbg_dev && !c->no_stage) {
        const int rm = ensure_moments(c, (size_t)img.w * (size_t)img.h);
        if (rm) return rm;
        cfg.mom_px = c->d_mom_px;
        cfg.mom_off = c->d_mom_off;
        cfg.mom_sums = c->d_mom_sums;
        cfg.mom_cap = c->mom_cap;
    }
    *out = cfg;
    return FX_OK;
}

// TMA descriptors of img's label / intensity rasters (40- and 72-wide boxes)
struct TmaSet {
    CUtensorMap m[4];
    int tma40 = 0, tma72 = 0;
};
void make_tmaps(fx_ctx* c, const DevImage& img, TmaSet* t) {
    std::memset(t->m, 0, sizeof t->m);
    t->tma40 = (!c->no_tma && make_tmap(c, img, img.L, &t->m[0], kStageW0) &&
                make_tmap(c, img, img.I, &t->m[1], kStageW0)) ? 1 : 0;
    t->tma72 = (!c->no_tma && make_tmap(c, img, img.L, &t->m[2], kStageW) &&
                make_tmap(c, img, img.I, &t->m[3], kStageW)) ? 1 : 0;
}

const char* const kSName[3] = {"k_roi_s0", "k_roi_s1", "k_roi_s2"};

// Per-ROI kernels over the ROIs queued in the device control block, whose class
// counts the host knows (hc): S classes from cls_first on, GLRLM/GLSZM/NGTDM, the
// serial passes over the staged S ROIs, then the large-ROI kernel (L ROIs + S
// overflow).
int roi_work(fx_ctx* c, const DevImage& img, const FeatCfg& cfg, const Control& hc,
             const TmaSet& tm, double* out_dev, const DebugOut* dbg_dev, int cls_first,
             Control* ctl, const RoiList& rl, const FeatCfg* wide = nullptr, bool split_serial = true) {
    cudaStream_t s = c->stream;
    const int glcm = s_glcm_mode(cfg);
    for (int cls = cls_first; cls <= kClassS2; ++cls) {
        if (hc.class_count[cls] == 0) continue;
        Launch l(c, kSName[cls]);
        launch_roi_s(cls, c->sm_count * c->occ_s[cls][glcm], s, tm.m, tm.tma40, tm.tma72, img,
                     rl, ctl, cfg, out_dev, dbg_dev);
    }
    CK(cudaGetLastError());
    const bool texture = cfg.col_glrlm >= 0 || cfg.col_glszm >= 0 || cfg.col_ngtdm >= 0;
    const uint64_t n_s_rois = (uint64_t)hc.class_count[kClassS0] + hc.class_count[kClassS1] +
                              hc.class_count[kClassS2];
    const uint64_t n_l = hc.class_count[kClassL];
    // (running the serial passes on a second stream next to k_roi_t measured slower:
    // its persistent CTAs leave no room, and 512-image batches fill the GPU anyway)
    if (texture) {
        // GLRLM/GLSZM/NGTDM: S-class windows, then large windows (own slabs)
        for (int which = 0; which < 2; ++which) {
            const uint64_t nw = which ? n_l : n_s_rois;
            if (!nw) continue;
            const TLayout T = which ? make_tlayout(std::max<unsigned long long>(hc.l_max_cells, 4096ull),
                                                   (uint32_t)std::max<unsigned long long>(hc.l_max_n, 4096ull))
                                    : make_tlayout(4096ull, 4096u);
            uint64_t grid = std::min<uint64_t>((uint64_t)c->sm_count * 4, nw);
            grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, (4ull << 30) / std::max<size_t>(T.bytes, 1)));
            const size_t need = (size_t)T.bytes * grid;
            if (need > c->tscratch_bytes[which]) {
                cudaStreamSynchronize(s);
                cudaFree(c->d_tscratch[which]);
                c->d_tscratch[which] = nullptr;
                c->tscratch_bytes[which] = 0;
                c->tlay_grid[which] = 0;
                CK(cudaMalloc(&c->d_tscratch[which], need));
                c->tscratch_bytes[which] = need;
            }
            const bool same = c->tlay_grid[which] >= (int)grid && T.bytes == c->tlay_prev[which].bytes &&
                              T.HC == c->tlay_prev[which].HC && T.hjk == c->tlay_prev[which].hjk;
            Launch l(c, which ? "k_roi_t_large" : "k_roi_t");
            launch_roi_t((int)grid, s, img, rl, ctl, cfg, out_dev, c->d_tscratch[which], T,
                         which, !same);
            if (!same) {
                c->tlay_prev[which] = T;
                c->tlay_grid[which] = (int)grid;
            }
        }
    }
    // intensity statistics, moments and serial shape columns of the staged S ROIs,
    // before k_roi_b (which rewrites the rows of overflowed S ROIs).  (Fusing these
    // into the S kernels, one lane per finished ROI, measured 30% slower: the S slabs
    // leave the serial loads almost no L1.)
    if (n_s_rois > 0) {
        if (cfg.int_vals || cfg.mom_px) {
            Launch l(c, "k_serial_stats");
            launch_serial_stats((int)n_s_rois, cfg.int_vals != nullptr, cfg.mom_px != nullptr, s, rl,
                                ctl, cfg, out_dev, split_serial ? c->side : nullptr, c->ev_fork, c->ev_join);
        }
        if (cfg.col_shape >= 0) {
            Launch l(c, "k_shape_serial");
            launch_shape_serial((int)n_s_rois, s, rl, ctl, cfg, out_dev);
        }
    }
    if (n_l == 0 && n_s_rois == 0) return FX_OK;
    {
        // large ROIs + S overflow: one CTA per ROI; the slabs' histograms are kept
        // zero by the kernel, so they are cleared only when the layout changes
        const BLayout B = b_layout(hc, cfg.bins);
        uint64_t grid = std::min<uint64_t>((uint64_t)c->sm_count * 2,
                                           std::max<uint64_t>(std::max<uint64_t>(n_l, 1),
                                                              n_s_rois > 0 ? 16 : 1));
        const uint64_t budget = 8ull << 30;  // scratch cap: fewer CTAs for huge windows
        grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, budget / std::max<size_t>(B.bytes, 1)));
        int rc = ensure_lscratch(c, (size_t)B.bytes * grid);
        if (rc) return rc;
        const bool same = c->lay_grid >= (int)grid && B.bytes == c->lay_prev.bytes &&
                          B.vhist == c->lay_prev.vhist && B.ghist == c->lay_prev.ghist &&
                          B.bins == c->lay_prev.bins && B.NB == c->lay_prev.NB;
        if (!same) {
            CK(cudaMemsetAsync(c->d_lscratch, 0, (size_t)B.bytes * grid, s));
            c->lay_prev = B;
            c->lay_grid = (int)grid;
        }
        Launch l(c, "k_roi_b");
        launch_roi_b((int)grid, s, img, rl, ctl, cfg, out_dev, dbg_dev, c->d_lscratch, B);
    }
    CK(cudaGetLastError());
    if (wide) {
        // texture groups above 256 grey levels: every queued ROI's texture columns
        const uint64_t total = n_s_rois + n_l;
        const WLayout W = make_wlayout(std::max<unsigned long long>(hc.l_max_cells, (unsigned long long)kSW * kSH),
                                       std::max<unsigned long long>(hc.l_max_n, (unsigned long long)kS2N), wide->ng);
        uint64_t grid = std::min<uint64_t>((uint64_t)c->sm_count * 2, total);
        grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, (4ull << 30) / std::max<size_t>(W.bytes, 1)));
        const size_t need = W.bytes * grid;
        if (need > c->wscratch_bytes) {
            cudaStreamSynchronize(s);
            cudaFree(c->d_wscratch);
            c->d_wscratch = nullptr;
            c->wscratch_bytes = 0;
            CK(cudaMalloc(&c->d_wscratch, need));
            c->wscratch_bytes = need;
        }
        Launch l(c, "k_texture_wide");
        launch_texture_wide((int)grid, s, img, rl, ctl, *wide, out_dev, c->d_wscratch, W);
        CK(cudaGetLastError());
    }
    return FX_OK;
}

// Compaction (owned rows [own_y0, own_y1)) + per-ROI kernels over the ctx's label
// table, reading pixels of img.  out_dev: [cap_rois x ncols] device.
// With slot_base (host, [m.nslots+1]) the first output row of every slot is returned.
int featurize_stage(fx_ctx* c, const DevImage& img, const SlotMap& m, uint32_t own_y0,
                    uint32_t own_y1, unsigned groups, const fx_texture_params& p, double* out_dev,
                    size_t cap_rois, size_t* n_rois, const DebugOut* dbg_dev,
                    uint32_t* slot_base = nullptr, bool first = true) {
    FeatCfg cfg;
    int rc = prepare_cfg(c, img, groups, p, dbg_dev, &cfg);
    if (rc) return rc;
    const int vrc = validate_texture(groups, p);
    const FeatCfg wcfg = cfg;
    const bool wide = vrc == FX_OK && wide_texture(cfg);
    if (wide) cfg = core_cfg(cfg);
    cudaStream_t s = c->stream;
    rc = compact_stage(c, m, own_y0, own_y1, cap_rois, first);
    if (rc) return rc;
    CK(cudaEventRecord(c->ev_compact, s));
    CK(cudaStreamWaitEvent(c->side, c->ev_compact, 0));
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, c->side));
    if (slot_base)
        CK(cudaMemcpyAsync(c->h_slot_base, compact_args(c, 0, 0).slot_base,
                           ((size_t)m.nslots + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           c->side));
    CK(cudaEventRecord(c->ev_stats, c->side));

    if (vrc != FX_OK) {  // texture parameters are only an error when a ROI exists
        CK(cudaEventSynchronize(c->ev_stats));
        *n_rois = c->h_ctl->n_rois;
        return c->h_ctl->n_rois ? vrc : FX_OK;
    }
    TmaSet tm;
    make_tmaps(c, img, &tm);
    const int glcm = s_glcm_mode(cfg);
    {
        // S0 before the class counts are known (its persistent grid finds its list
        // empty when there is none), overlapping the counters' readback
        Launch l(c, kSName[kClassS0]);
        launch_roi_s(kClassS0, c->sm_count * c->occ_s[kClassS0][glcm], s, tm.m, tm.tma40, tm.tma72,
                     img, roi_list(c), c->d_ctl, cfg, out_dev, dbg_dev);
    }
    CK(cudaGetLastError());
    // the class counts arrive while S0 runs; S1 / S2 launch only when they have ROIs
    // (an empty persistent grid still costs ~7 us).  With more ROIs than cap_rois the
    // compaction queued none, so S0 found no work and wrote no row.
    CK(cudaEventSynchronize(c->ev_stats));
    const Control hc = *c->h_ctl;
    *n_rois = hc.n_rois;
    if (slot_base) std::memcpy(slot_base, c->h_slot_base, ((size_t)m.nslots + 1) * sizeof(uint32_t));
    if (hc.error & kErrWindow) {
        cudaStreamSynchronize(s);
        return set_error(FX_E_ARG, "an owned ROI window extends beyond the image (halo too small)");
    }
    if (hc.n_rois > cap_rois) {
        cudaStreamSynchronize(s);
        return set_error(FX_E_CAPACITY, "output capacity " + std::to_string(cap_rois) +
                                            " < " + std::to_string(hc.n_rois) + " ROIs");
    }
    rc = roi_work(c, img, cfg, hc, tm, out_dev, dbg_dev, kClassS1, c->d_ctl, roi_list(c),
                  wide ? &wcfg : nullptr);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    return FX_OK;
}

int run_pipeline(fx_ctx* c, const DevImage& img, unsigned groups, const fx_texture_params& p,
                 double* out_dev, size_t cap_rois, size_t* n_rois, const DebugOut* dbg_dev) {
    const SlotMap m = single_map(img);
    int rc = scan_stage(c, img, m, true);
    if (rc) return rc;
    return featurize_stage(c, img, m, 0u, 0xffffffffu, groups, p, out_dev, cap_rois, n_rois, dbg_dev);
}

int finish(fx_ctx* c) {
    CK(cudaStreamSynchronize(c->stream));
    // per-kernel event pairs are resolved when the times are queried, so timed
    // steps carry no event synchronisation on the host (bounded backlog)
    if (c->timing && c->pending.size() > 8192) collect_times(c);
    if (c->h_ctl->error & kErrCapacity)
        return set_error(FX_E_CAPACITY, "a large ROI exceeded the L-path slab");
    if (c->h_ctl->error & kErrRuns)
        return set_error(FX_E_CAPACITY, "a large ROI exceeded the run-list capacity");
    if (c->h_ctl->error & kErrOutCap)
        return set_error(FX_E_CAPACITY, "more ROIs than output rows");
    return FX_OK;
}

DevImage to_dev(const fx_image& im) {
    DevImage d;
    d.I = im.intensity;
    d.L = im.labels;
    d.w = im.width;
    d.h = im.height;
    d.pitch = im.pitch ? im.pitch : (size_t)im.width;
    d.ox = im.origin_x;
    d.oy = im.origin_y;
    return d;
}

int check_groups(unsigned groups) {
    if (groups == 0) return set_error(FX_E_CONFIG, "feature list is empty");
    if (groups & ~FX_GROUP_ALL) return set_error(FX_E_CONFIG, "unknown feature group bit");
    const unsigned missing = groups & ~FX_GROUP_DEVICE;
    if (missing) {
        std::string names;
        for (int i = 0; i < 7; ++i)
            if (missing & (1u << i)) names += (names.empty() ? "" : ",") + all_group_names()[i];
        return set_error(FX_E_CONFIG, "feature group(s) '" + names +
                                          "' have no device kernel in this build (no CPU fallback)");
    }
    return FX_OK;
}

// Device image from the caller's image; host rasters are staged into pitched buffers.
int stage_image(fx_ctx* c, const fx_image* im, DevImage* d) {
    *d = to_dev(*im);
    if (im->mem_kind == FX_MEM_DEVICE) return FX_OK;
    int rc = ensure_img(c, im->width, im->height);
    if (rc) return rc;
    uint16_t* dI = c->d_img;
    uint16_t* dL = c->d_img + c->img_pitch * c->img_rows_cap;
    const size_t sp = (im->pitch ? im->pitch : (size_t)im->width) * 2;
    if (sp == c->img_pitch * 2 && (size_t)im->width == c->img_pitch) {  // linear copies
        CK(cudaMemcpyAsync(dI, im->intensity, sp * (size_t)im->height, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dL, im->labels, sp * (size_t)im->height, cudaMemcpyHostToDevice, c->stream));
    } else {
        CK(cudaMemcpy2DAsync(dI, c->img_pitch * 2, im->intensity, sp, (size_t)im->width * 2,
                             (size_t)im->height, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpy2DAsync(dL, c->img_pitch * 2, im->labels, sp, (size_t)im->width * 2,
                             (size_t)im->height, cudaMemcpyHostToDevice, c->stream));
    }
    d->I = dI;
    d->L = dL;
    d->pitch = c->img_pitch;
    return FX_OK;
}

// images per launch set: each is one label-table slot (65536 labels x 24 B); the
// thread-per-ROI passes want many ROIs per launch (C4: 100 per tile)
#ifndef FXG_BATCH_SLOTS
#define FXG_BATCH_SLOTS 512
#endif
constexpr int kBatchSlots = FXG_BATCH_SLOTS;
constexpr size_t kStageBudget = (size_t)kBatchSlots << 19;  // staged elements per raster per sub-batch

int ensure_maps(fx_ctx* c, size_t slots, size_t strips) {
    if (slots <= c->map_slots_cap && strips <= c->map_strips_cap) return FX_OK;
    cudaStreamSynchronize(c->copy);
    cudaStreamSynchronize(c->stream);
    slots = std::max(slots, c->map_slots_cap);
    strips = std::max(strips, c->map_strips_cap);
    for (int b = 0; b < 2; ++b) {
        cudaFree(c->d_slots[b]);
        cudaFree(c->d_strips[b]);
        if (c->h_slots[b]) cudaFreeHost(c->h_slots[b]);
        if (c->h_strips[b]) cudaFreeHost(c->h_strips[b]);
        c->d_slots[b] = nullptr;
        c->d_strips[b] = nullptr;
        c->h_slots[b] = nullptr;
        c->h_strips[b] = nullptr;
    }
    c->map_slots_cap = c->map_strips_cap = 0;
    for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&c->d_slots[b], slots * sizeof(SlotInfo)));
        CK(cudaMalloc(&c->d_strips[b], strips * sizeof(uint16_t)));
        CK(cudaMallocHost(&c->h_slots[b], slots * sizeof(SlotInfo)));
        CK(cudaMallocHost(&c->h_strips[b], strips * sizeof(uint16_t)));
    }
    c->map_slots_cap = slots;
    c->map_strips_cap = strips;
    return FX_OK;
}

int ensure_stage(fx_ctx* c, size_t elems) {
    if (elems <= c->stage_elems) return FX_OK;
    cudaStreamSynchronize(c->copy);
    cudaStreamSynchronize(c->stream);
    for (int b = 0; b < 2; ++b) {
        cudaFree(c->d_stage[b]);
        c->d_stage[b] = nullptr;
    }
    c->stage_elems = 0;
    elems = (elems + 63) / 64 * 64;
    for (int b = 0; b < 2; ++b) CK(cudaMalloc(&c->d_stage[b], 2 * elems * sizeof(uint16_t)));
    c->stage_elems = elems;
    return FX_OK;
}

int ensure_blab(fx_ctx* c, size_t n) {
    if (n <= c->blab_cap) return FX_OK;
    cudaStreamSynchronize(c->stream);
    cudaFree(c->d_blab);
    c->d_blab = nullptr;
    c->blab_cap = 0;
    CK(cudaMalloc(&c->d_blab, n * sizeof(uint32_t)));
    c->blab_cap = n;
    return FX_OK;
}

// ---- host rasters in row bands (the end-to-end path of fx_featurize) ----------
//
// PCIe moves ~55 GB/s: a C2 image (268 MB of rasters) takes ~4.9 ms to arrive and
// its 57 MB table ~1 ms to leave, against ~0.6 ms of kernels.  Instead of copy ->
// compute -> copy back, the rasters move in row bands on the copy stream (all
// labels first, then the intensities):
//   - the label scan runs band by band as the labels arrive;
//   - the compaction runs once over the whole table (a ROI's bbox is only final when
//     every row has been scanned); the host reads the ROI windows back and sorts
//     each class list by the band holding the window's last row;
//   - band b's ROIs are featurized as soon as band b's intensities are in (the
//     unchanged per-ROI kernels over a control block holding that band's lists);
//   - output rows [r_(b-1), r_b) leave on the d2h stream as soon as every ROI of
//     rank < r_b is final (blob grids: about one band's rows per band), so the D2H
//     overlaps the remaining H2D (PCIe is full duplex).
// Results are identical to the unbanded path: the same kernels on the same ROIs.

int ensure_band(fx_ctx* c, int bands) {
    if (!c->d_band) {
        CK(cudaMalloc(&c->d_band, (size_t)kMaxBands * (2 * kNumClasses + 1) * sizeof(uint32_t)));
        CK(cudaMallocHost(&c->h_band, (size_t)kMaxBands * (2 * kNumClasses + 1) * sizeof(uint32_t)));
        CK(cudaMalloc(&c->d_band_ctl, (size_t)kMaxBands * sizeof(Control)));
        CK(cudaMallocHost(&c->h_band_ctl, (size_t)kMaxBands * sizeof(Control)));
    }
    if (c->roi_cap > c->band_seg_cap) {
        cudaFree(c->d_band_seg);
        c->d_band_seg = nullptr;
        c->band_seg_cap = 0;
        CK(cudaMalloc(&c->d_band_seg, c->roi_cap * sizeof(uint32_t)));
        c->band_seg_cap = c->roi_cap;
    }
    while ((int)c->ev_band.size() < 3 * bands) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_band.push_back(e);
    }
    return FX_OK;
}

// band height for a host image (0: unbanded); FXG_BAND_ROWS overrides (<0: off)
int band_rows_for(const fx_ctx* c, int w, int h) {
    if (c->band_rows < 0) return 0;
    if (c->band_rows > 0) return (c->band_rows + 63) / 64 * 64;
    if (h < 2048 || (size_t)w * (size_t)h < (8u << 20)) return 0;  // not worth it
    return std::max(256, (h / 8 + 63) / 64 * 64);                   // ~8 bands
}

// band plan of an image of h rows: bands of band_rows (at least h / kMaxBands), the
// last one cut into quarters (>= 64 rows each) so little work follows the last copy
BandPlan band_plan(int band_rows, int h) {
    const int min_rows = ((h + kMaxBands - 4 - 1) / (kMaxBands - 4) + 63) / 64 * 64;
    const uint32_t R = (uint32_t)std::max(band_rows, min_rows);
    BandPlan bp{};
    bp.rows = R;
    const uint32_t nb0 = ((uint32_t)h + R - 1) / R;
    bp.nb1 = nb0 - 1;
    bp.split_y = bp.nb1 * R;
    bp.rows2 = std::max<uint32_t>(64, (R / 4 + 63) / 64 * 64);
    bp.nb = bp.nb1 + ((uint32_t)h - bp.split_y + bp.rows2 - 1) / bp.rows2;
    return bp;
}

// The ROI lists of bands [b0, b1] after k_band_scatter (class-major segments of
// d_band_seg: class k's lists of bands 0..nb-1 are consecutive, so a run of bands
// is one range per class); bc: the host copy of the counts for launch decisions.
uint64_t band_range_lists(const fx_ctx* c, const uint32_t* h_cnt, int nb, int b0, int b1,
                          const Control& hc, const RoiList& rl, Control& bc, RoiList& rb) {
    bc = hc;
    rb = rl;
    size_t base = 0;
    uint64_t total = 0;
    for (int k = 0; k < kNumClasses; ++k) {
        size_t before = 0, in = 0, all = 0;
        for (int b = 0; b < nb; ++b) {
            const uint32_t v = h_cnt[b * kNumClasses + k];
            all += v;
            if (b < b0) before += v;
            else if (b <= b1) in += v;
        }
        rb.cls_list[k] = c->d_band_seg + base + before;
        bc.class_count[k] = (uint32_t)in;
        base += all;
        total += in;
    }
    return total;
}

// Row blocks of the packed host path: each band cut into pieces of at most
// kPackRows rows (a block never straddles a band, so a band's intensities are
// complete once its last block has been unpacked).
#ifndef FXG_PACK_ROWS
#define FXG_PACK_ROWS 256
#endif
constexpr int kPackRows = FXG_PACK_ROWS;
struct PackBlock {
    int y0, rows, band;
    bool raw;  // sent raw by DMA (both rasters) while the workers pack the others
    size_t lab_off, int_off;  // region offsets in the staging buffers
    size_t lab_cap_seg, int_cap_pix;
};

// One packer pool per process (the packers are bound by the host's memory
// bandwidth, which every context shares); one packing call at a time holds it.
std::mutex& packer_mutex() {
    static std::mutex m;
    return m;
}
// Threads: FXG_PACK_THREADS, else the host's cores shared among the processes of
// a torchrun job on this node (LOCAL_WORLD_SIZE), less one for the caller, <= 15.
PackPool* packer_pool() {
    static PackPool* const pool = [] {
        int n = 0;
        if (const char* e = getenv("FXG_PACK_THREADS")) n = atoi(e);
        if (n <= 0) {
            const int hw = std::max(1, (int)std::thread::hardware_concurrency());
            const char* lw = getenv("LOCAL_WORLD_SIZE");
            const int procs = lw ? std::max(1, atoi(lw)) : 1;
            n = std::min(hw / procs - 1, 15);
        }
        return new PackPool(std::max(1, n));  // lives for the process
    }();
    return pool;
}

// pinned + device staging for packed blocks (both paths)
int ensure_pack(fx_ctx* c, size_t bytes) {
    if (bytes <= c->pack_bytes) return FX_OK;
    cudaStreamSynchronize(c->copy);
    cudaStreamSynchronize(c->copy2);
    cudaStreamSynchronize(c->stream);
    cudaFreeHost(c->h_pack);
    cudaFree(c->d_pack);
    c->h_pack = nullptr;
    c->d_pack = nullptr;
    c->pack_bytes = 0;
    CK(cudaMallocHost(&c->h_pack, bytes));
    CK(cudaMalloc(&c->d_pack, bytes));
    c->pack_bytes = bytes;
    c->pack_half = 0;  // the caller re-lays its halves
    return FX_OK;
}

bool packing_usable(const fx_ctx* c, const fx_image* im) {
    return c->packing && pack_isa() == 2 && im->width <= 65536;
}

// Host rasters as packed row blocks (fx_pack.hpp): the pool's workers pack every
// block's labels (change points + nonzero masks), then every block's labelled
// intensities; this thread ships each block as soon as it is packed, unpacks it
// on the device, scans the whole label raster after the last label block,
// compacts, and runs each band's ROIs once that band's intensities are unpacked
// (the per-band ROI work and row readback of featurize_banded).  A block whose
// labels do not pack into half their raw size goes raw (both rasters).
int featurize_packed(fx_ctx* c, const fx_image* im, int band_rows, unsigned groups,
                     const fx_texture_params& p, uint32_t* out_labels, double* out_values,
                     size_t cap_rois, size_t* n_rois) {
    const int W = im->width, H = im->height;
    const BandPlan bp = band_plan(band_rows, H);
    const int nb = (int)bp.nb;
    int rc = ensure_img(c, W, H);
    if (!rc) rc = ensure_band(c, nb);
    if (rc) return rc;
    cudaStream_t s = c->stream;
    const size_t P = c->img_pitch, spe = im->pitch ? im->pitch : (size_t)W, sp = spe * 2;
    DevImage d;
    d.I = c->d_img;
    d.L = c->d_img + P * c->img_rows_cap;
    d.w = W;
    d.h = H;
    d.pitch = P;
    d.ox = im->origin_x;
    d.oy = im->origin_y;
    // blocks and their staging regions
    std::vector<PackBlock> blk;
    size_t bytes = 0;
    for (int b = 0; b < nb; ++b) {
        const int ya = (int)bp.y0_of((uint32_t)b), yb = b + 1 < nb ? (int)bp.y0_of((uint32_t)b + 1) : H;
        for (int y = ya; y < yb; y += kPackRows) {
            PackBlock k;
            k.y0 = y;
            k.rows = std::min(kPackRows, yb - y);
            k.band = b;
            k.raw = false;
            k.lab_cap_seg = (size_t)k.rows * (size_t)W / 4;  // half the raw label bytes
            k.lab_off = bytes;
            bytes += pk_align16(pk_lab_bytes(k.rows, W, k.lab_cap_seg));
            k.int_off = bytes;
            k.int_cap_pix = (size_t)k.rows * (size_t)W / 2;  // half the raw intensity bytes
            bytes += pk_align16(pk_int_bytes(k.rows, W, k.int_cap_pix));
            blk.push_back(k);
        }
    }
    const int NB = (int)blk.size();
    // The host's memory bandwidth bounds the packers (~2.6 B read per pixel) and
    // PCIe the raw DMA (4 B per pixel): a share of the blocks goes raw so both run
    // from the start (spread evenly: block j raw when floor((j+1) r) > floor(j r)).
    for (int q = 0; q < NB; ++q)
        blk[q].raw = (q + 1) * c->pack_raw_pct / 100 > q * c->pack_raw_pct / 100;
    rc = ensure_pack(c, bytes);
    if (rc) return rc;
    const size_t mp = ((size_t)W + 31) / 32;  // mask words per row
    if (c->pack_mask.size() < mp * (size_t)H) c->pack_mask.resize(mp * (size_t)H);
    std::unique_lock<std::mutex> pool_lock(packer_mutex());
    PackPool* const shared_pool = packer_pool();
    std::vector<size_t> lab_bytes(NB, 0), int_bytes(NB, 0);
    // FXG_PACK_TRACE=1: host timeline of the call on stderr (tools)
    static const bool trace = getenv("FXG_PACK_TRACE") && atoi(getenv("FXG_PACK_TRACE"));
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, int k) {
        if (trace)
            fprintf(stderr, "pack-trace %8.3f ms %s %d\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(),
                    what, k);
    };
    uint8_t* hp = c->h_pack;
    uint32_t* mask = c->pack_mask.data();
    PackPool* pool = shared_pool;
    // the previous call's copies out of the staging buffers are complete (its
    // finish() synchronised every stream)
    pool->start(2 * NB, [&, pool](int t) {
        const PackBlock& k = blk[t < NB ? t : t - NB];
        uint32_t* m = mask + (size_t)k.y0 * mp;
        if (k.raw) return;
        if (t < NB) {
            lab_bytes[t] = pack_labels(im->labels, spe, W, k.y0, k.y0 + k.rows, hp + k.lab_off,
                                       k.lab_cap_seg, m, mp);
        } else {
            const int j = t - NB;
            while (!pool->done(j)) std::this_thread::yield();  // claimed earlier, running
            if (lab_bytes[j])
                int_bytes[j] = pack_intensity(im->intensity, spe, W, k.y0, k.y0 + k.rows, m, mp,
                                              hp + k.int_off, k.int_cap_pix);
        }
    });
    // the workers read the caller's rasters and write the staging buffers: every
    // return waits for them
    struct Join {
        PackPool* p;
        std::unique_lock<std::mutex>* lk;
        void release() {
            if (!lk) return;
            p->wait();
            lk->unlock();
            lk = nullptr;
        }
        ~Join() { release(); }
    } join{pool, &pool_lock};
    auto spin = [&](int t) {
        while (!pool->done(t)) std::this_thread::yield();
    };
    // events: [nb+b] band b's rows final (as featurize_banded), [2nb+j] label block
    // j shipped, [2nb+NB+j] intensity block j shipped
    while (c->ev_band.size() < (size_t)(2 * nb + 2 * NB)) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_band.push_back(e);
    }
    cudaEvent_t* ev = c->ev_band.data();
    CK(cudaEventRecord(c->ev_compact, s));
    CK(cudaStreamWaitEvent(c->copy, c->ev_compact, 0));
    c->h2d_bytes = c->d2h_bytes = 0;
    // trace: device timeline (timing events on s / d2h, read at the end)
    std::vector<std::pair<std::string, cudaEvent_t>> tev;
    auto dmark = [&](const std::string& what, cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.emplace_back(what, e);
    };
    dmark("start", s);
    auto raw_rows = [&](const uint16_t* src, uint16_t* dst, const PackBlock& k) -> int {
        CK(cudaMemcpy2DAsync(dst + (size_t)k.y0 * P, P * 2, src + (size_t)k.y0 * spe, sp, (size_t)W * 2,
                             (size_t)k.rows, cudaMemcpyHostToDevice, c->copy));
        c->h2d_bytes += (size_t)W * 2 * (size_t)k.rows;
        return FX_OK;
    };
    // 0. the raw blocks' labels, then their intensities, on the copy stream at once
    CK(cudaStreamWaitEvent(c->copy2, c->ev_compact, 0));
    for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < NB; ++j) {
            if (!blk[j].raw) continue;
            if ((rc = raw_rows(pass ? im->intensity : im->labels, const_cast<uint16_t*>(pass ? d.I : d.L),
                               blk[j])))
                return rc;
            CK(cudaEventRecord(ev[2 * nb + pass * NB + j], c->copy));
        }
    // 1. label blocks: ship the packed ones as they are done (copy2), unpack
    for (int j = 0; j < NB; ++j) {
        const PackBlock& k = blk[j];
        cudaEvent_t e = ev[2 * nb + j];
        if (!k.raw) {
            spin(j);
            mark("labels packed", j);
            if (lab_bytes[j]) {
                CK(cudaMemcpyAsync(c->d_pack + k.lab_off, hp + k.lab_off, lab_bytes[j],
                                   cudaMemcpyHostToDevice, c->copy2));
                c->h2d_bytes += lab_bytes[j];
                CK(cudaEventRecord(e, c->copy2));
            } else {  // did not pack: raw after all (copy stream, behind the raw blocks)
                if ((rc = raw_rows(im->labels, const_cast<uint16_t*>(d.L), k))) return rc;
                CK(cudaEventRecord(e, c->copy));
            }
        }
        CK(cudaStreamWaitEvent(s, e, 0));
        if (lab_bytes[j]) {
            Launch l(c, "k_unpack_labels");
            k_unpack_labels<<<dim3(pk_tiles(W), k.rows), 256, 0, s>>>(c->d_pack + k.lab_off, k.rows, W,
                                                           const_cast<uint16_t*>(d.L) + (size_t)k.y0 * P, P);
        }
    }
    CK(cudaGetLastError());
    dmark("labels unpacked", s);
    rc = scan_stage(c, d, single_map(d), true);
    if (rc) return rc;
    FeatCfg cfg;
    rc = prepare_cfg(c, d, groups, p, nullptr, &cfg);
    if (rc) return rc;
    const int vrc = validate_texture(groups, p);
    const FeatCfg wcfg = cfg;
    const bool wide = vrc == FX_OK && wide_texture(cfg);
    if (wide) cfg = core_cfg(cfg);
    rc = compact_stage(c, single_map(d), 0u, 0xffffffffu, cap_rois, true);
    if (rc) return rc;
    RoiList rl = roi_list(c);
    uint32_t* cnt = c->d_band;
    uint32_t* cursor = cnt + kMaxBands * kNumClasses;
    uint32_t* first = cursor + kMaxBands * kNumClasses;
    CK(cudaMemsetAsync(cnt, 0, 2 * kMaxBands * kNumClasses * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(first, 0xff, kMaxBands * sizeof(uint32_t), s));
    {
        const int grid = 2 * c->sm_count;
        Launch l(c, "k_band_count");
        k_band_count<<<grid, 256, 0, s>>>(rl, c->d_ctl, bp, cnt, first);
        Launch l2(c, "k_band_scatter");
        k_band_scatter<<<grid, 256, 0, s>>>(rl, c->d_ctl, bp, cnt, cursor, c->d_band_seg, c->d_band_ctl);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->h_band, c->d_band, (size_t)kMaxBands * (2 * kNumClasses + 1) * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(c->ev_stats, s));
    mark("compaction queued", 0);
    CK(cudaStreamSynchronize(s));
    mark("compaction done", 0);
    const Control hc = *c->h_ctl;
    const size_t n = hc.n_rois;
    *n_rois = n;
    if (vrc != FX_OK) return n ? vrc : FX_OK;
    if (hc.error & kErrWindow)
        return set_error(FX_E_ARG, "an owned ROI window extends beyond the image (halo too small)");
    if (n > cap_rois)
        return set_error(FX_E_CAPACITY, "output capacity " + std::to_string(cap_rois) + " < " +
                                            std::to_string(n) + " ROIs");
    if (n == 0) return FX_OK;
    if (out_labels) {
        CK(cudaStreamWaitEvent(c->d2h, c->ev_stats, 0));
        CK(cudaMemcpyAsync(out_labels, rl.label, n * 4, cudaMemcpyDeviceToHost, c->d2h));
        c->d2h_bytes += n * 4;
    }
    const uint32_t* h_cnt = c->h_band;
    const uint32_t* h_first = c->h_band + 2 * kMaxBands * kNumClasses;
    std::vector<uint32_t> final_after(nb);
    uint32_t later = (uint32_t)n;
    for (int b = nb - 1; b >= 0; --b) {
        final_after[b] = later;
        later = std::min(later, h_first[b]);
    }
    const size_t ncols = (size_t)cfg.ncols;
    TmaSet tm;
    make_tmaps(c, d, &tm);
    size_t rows_out = 0;
    int j = 0;
    // 2. ship and unpack one intensity block (waiting for its packing if needed)
    auto ship_int = [&](int q) -> int {
        const PackBlock& k = blk[q];
        cudaEvent_t e = ev[2 * nb + NB + q];
        if (!k.raw) {
            spin(NB + q);
            mark("intensity packed", q);
            if (int_bytes[q]) {
                CK(cudaMemcpyAsync(c->d_pack + k.int_off, hp + k.int_off, int_bytes[q],
                                   cudaMemcpyHostToDevice, c->copy2));
                c->h2d_bytes += int_bytes[q];
                CK(cudaEventRecord(e, c->copy2));
            } else {
                int r2 = raw_rows(im->intensity, const_cast<uint16_t*>(d.I), k);
                if (r2) return r2;
                CK(cudaEventRecord(e, c->copy));
            }
        }
        CK(cudaStreamWaitEvent(s, e, 0));
        if (int_bytes[q]) {
            Launch l(c, "k_unpack_intensity");
            k_unpack_intensity<<<dim3(pk_tiles(W), k.rows), 256, 0, s>>>(
                c->d_pack + k.int_off, k.rows, W, d.L + (size_t)k.y0 * P,
                const_cast<uint16_t*>(d.I) + (size_t)k.y0 * P, P);
        }
        return FX_OK;
    };
    // a band is ready when every one of its intensity blocks is packed (raw ones are
    // queued from the start)
    auto band_ready = [&](int bb, int from) -> bool {
        for (int q = from; q < NB && blk[q].band == bb; ++q)
            if (!blk[q].raw && !pool->done(NB + q)) return false;
        return true;
    };
    for (int b = 0; b < nb;) {
        // this band's blocks (waiting for them), then every following band whose blocks
        // are already packed: one set of ROI launches for the run of bands (each band's
        // launches have a fixed latency, and the packers often finish several at once)
        for (; j < NB && blk[j].band == b; ++j)
            if ((rc = ship_int(j))) return rc;
        int b2 = b;
        static const bool merge = !getenv("FXG_PACK_MERGE") || atoi(getenv("FXG_PACK_MERGE"));
        while (merge && b2 + 1 < nb && band_ready(b2 + 1, j)) {
            ++b2;
            for (; j < NB && blk[j].band == b2; ++j)
                if ((rc = ship_int(j))) return rc;
        }
        CK(cudaGetLastError());
        dmark("bands " + std::to_string(b) + "-" + std::to_string(b2) + " intensities unpacked", s);
        Control bc;
        RoiList rb;
        const uint64_t band_rois = band_range_lists(c, h_cnt, nb, b, b2, hc, rl, bc, rb);
        if (band_rois) {
            Control* dctl = c->d_band_ctl + b;
            if (b2 > b) {  // the run's own control block (as k_band_scatter builds a band's)
                Control cb = hc;
                for (int q = 0; q < kNumClasses; ++q) {
                    cb.class_count[q] = bc.class_count[q];
                    cb.class_next[q] = 0;
                }
                cb.overflow_count = cb.overflow_next = 0;
                cb.t_next[0] = cb.t_next[1] = 0;
                cb.mom_alloc = cb.int_alloc = 0;
                cb.w_next = cb.b_next_big = 0;
                cb.error = 0;
                c->h_band_ctl[b] = cb;
                CK(cudaMemcpyAsync(dctl, c->h_band_ctl + b, sizeof(Control), cudaMemcpyHostToDevice, s));
            }
            rc = roi_work(c, d, cfg, bc, tm, c->d_out, nullptr, kClassS0, dctl, rb,
                          wide ? &wcfg : nullptr, false);
            if (rc) return rc;
        }
        const size_t upto = std::max<size_t>(rows_out, b2 == nb - 1 ? n : final_after[b2]);
        if (upto > rows_out) {
            CK(cudaEventRecord(ev[nb + b], s));
            CK(cudaStreamWaitEvent(c->d2h, ev[nb + b], 0));
            CK(cudaMemcpyAsync(out_values + rows_out * ncols, c->d_out + rows_out * ncols,
                               (upto - rows_out) * ncols * sizeof(double), cudaMemcpyDeviceToHost,
                               c->d2h));
            c->d2h_bytes += (upto - rows_out) * ncols * sizeof(double);
            rows_out = upto;
            dmark("bands " + std::to_string(b) + "-" + std::to_string(b2) + " rows back", c->d2h);
        }
        b = b2 + 1;
    }
    join.release();  // every block packed and shipped: the pool is free for other contexts
    CK(cudaMemcpyAsync(c->h_band_ctl, c->d_band_ctl, (size_t)nb * sizeof(Control),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    mark("compute done", 0);
    for (int b = 0; b < nb; ++b) c->h_ctl->error |= c->h_band_ctl[b].error;
    CK(cudaStreamSynchronize(c->d2h));
    mark("d2h done", 0);
    if (trace) {
        for (auto& te : tev) {
            float ms = 0;
            cudaEventElapsedTime(&ms, tev[0].second, te.second);
            fprintf(stderr, "pack-trace device %8.3f ms %s\n", ms, te.first.c_str());
        }
        for (auto& te : tev) cudaEventDestroy(te.second);
    }
    return FX_OK;
}

int featurize_banded(fx_ctx* c, const fx_image* im, int band_rows, unsigned groups,
                     const fx_texture_params& p, uint32_t* out_labels, double* out_values,
                     size_t cap_rois, size_t* n_rois) {
    const int W = im->width, H = im->height;
    const BandPlan bp = band_plan(band_rows, H);
    const int nb = (int)bp.nb;
    int rc = ensure_img(c, W, H);
    if (!rc) rc = ensure_band(c, nb);
    if (rc) return rc;
    cudaStream_t s = c->stream;
    const size_t P = c->img_pitch, sp = (im->pitch ? im->pitch : (size_t)W) * 2;
    DevImage d;
    d.I = c->d_img;
    d.L = c->d_img + P * c->img_rows_cap;
    d.w = W;
    d.h = H;
    d.pitch = P;
    d.ox = im->origin_x;
    d.oy = im->origin_y;
    cudaEvent_t* ev = c->ev_band.data();  // [b]: labels in, [nb+b]: intensities in, [2nb+b]: rows
    // the copy stream starts after this stream's earlier work (staging buffer reuse)
    CK(cudaEventRecord(c->ev_compact, s));
    CK(cudaStreamWaitEvent(c->copy, c->ev_compact, 0));
    c->h2d_bytes = c->d2h_bytes = 0;
    auto rows_of = [&](int b) {
        const int y0 = (int)bp.y0_of((uint32_t)b);
        return (b + 1 < nb ? (int)bp.y0_of((uint32_t)b + 1) : H) - y0;
    };
    for (int pass = 0; pass < 2; ++pass)  // all labels, then all intensities
        for (int b = 0; b < nb; ++b) {
            const size_t y0 = bp.y0_of((uint32_t)b);
            const uint16_t* src = (pass ? im->intensity : im->labels) + y0 * (sp / 2);
            uint16_t* dst = const_cast<uint16_t*>(pass ? d.I : d.L) + y0 * P;
            if (sp == P * 2 && (size_t)W == P)  // rows contiguous on both sides: one linear copy
                CK(cudaMemcpyAsync(dst, src, sp * (size_t)rows_of(b), cudaMemcpyHostToDevice, c->copy));
            else
                CK(cudaMemcpy2DAsync(dst, P * 2, src, sp, (size_t)W * 2, (size_t)rows_of(b),
                                     cudaMemcpyHostToDevice, c->copy));
            c->h2d_bytes += (size_t)W * 2 * (size_t)rows_of(b);
            CK(cudaEventRecord(ev[pass * nb + b], c->copy));
        }
    // label scan band by band, in global coordinates
    for (int b = 0; b < nb; ++b) {
        CK(cudaStreamWaitEvent(s, ev[b], 0));
        DevImage band = d;
        band.L = d.L + (size_t)bp.y0_of((uint32_t)b) * P;
        band.I = band.L;
        band.h = rows_of(b);
        band.oy = d.oy + (int)bp.y0_of((uint32_t)b);
        rc = scan_stage(c, band, single_map(band), b == 0);
        if (rc) return rc;
    }
    FeatCfg cfg;
    rc = prepare_cfg(c, d, groups, p, nullptr, &cfg);
    if (rc) return rc;
    const int vrc = validate_texture(groups, p);
    const FeatCfg wcfg = cfg;
    const bool wide = vrc == FX_OK && wide_texture(cfg);
    if (wide) cfg = core_cfg(cfg);
    rc = compact_stage(c, single_map(d), 0u, 0xffffffffu, cap_rois, true);
    if (rc) return rc;
    // bucket the queued ROIs by band on the device (nothing queued when the ROIs
    // exceed cap_rois); the host reads back the control block, the per-(band,
    // class) counts and first ranks in one round trip, while the intensities keep
    // arriving; no host-to-device copy competes with them
    RoiList rl = roi_list(c);
    uint32_t* cnt = c->d_band;
    uint32_t* cursor = cnt + kMaxBands * kNumClasses;
    uint32_t* first = cursor + kMaxBands * kNumClasses;
    CK(cudaMemsetAsync(cnt, 0, 2 * kMaxBands * kNumClasses * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(first, 0xff, kMaxBands * sizeof(uint32_t), s));
    {
        const int grid = 2 * c->sm_count;
        Launch l(c, "k_band_count");
        k_band_count<<<grid, 256, 0, s>>>(rl, c->d_ctl, bp, cnt, first);
        Launch l2(c, "k_band_scatter");
        k_band_scatter<<<grid, 256, 0, s>>>(rl, c->d_ctl, bp, cnt, cursor, c->d_band_seg, c->d_band_ctl);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->h_band, c->d_band, (size_t)kMaxBands * (2 * kNumClasses + 1) * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(c->ev_stats, s));
    CK(cudaStreamSynchronize(s));
    const Control hc = *c->h_ctl;
    const size_t n = hc.n_rois;
    *n_rois = n;
    if (vrc != FX_OK) return n ? vrc : FX_OK;
    if (hc.error & kErrWindow)
        return set_error(FX_E_ARG, "an owned ROI window extends beyond the image (halo too small)");
    if (n > cap_rois)
        return set_error(FX_E_CAPACITY, "output capacity " + std::to_string(cap_rois) + " < " +
                                            std::to_string(n) + " ROIs");
    if (n == 0) {
        CK(cudaStreamSynchronize(c->copy));
        return FX_OK;
    }
    if (out_labels) {
        CK(cudaStreamWaitEvent(c->d2h, c->ev_stats, 0));
        CK(cudaMemcpyAsync(out_labels, rl.label, n * 4, cudaMemcpyDeviceToHost, c->d2h));
        c->d2h_bytes += n * 4;
    }
    const uint32_t* h_cnt = c->h_band;
    const uint32_t* h_first = c->h_band + 2 * kMaxBands * kNumClasses;
    // rows final after band b: every rank below the first rank of any later band
    std::vector<uint32_t> final_after(nb);
    uint32_t later = (uint32_t)n;
    for (int b = nb - 1; b >= 0; --b) {
        final_after[b] = later;
        later = std::min(later, h_first[b]);
    }
    const size_t ncols = (size_t)cfg.ncols;
    TmaSet tm;
    make_tmaps(c, d, &tm);
    size_t rows_out = 0;
    for (int b = 0; b < nb; ++b) {
        Control bc;  // host copy of the band's counts (launch decisions)
        RoiList rb;  // the band's lists: segments of d_band_seg
        const uint64_t band_rois = band_range_lists(c, h_cnt, nb, b, b, hc, rl, bc, rb);
        CK(cudaStreamWaitEvent(s, ev[nb + b], 0));
        if (band_rois) {
            // (one stream per band: the serial passes' second stream only added
            // per-band event latency to this pipeline, 5.23 -> 5.29 ms on C2)
            rc = roi_work(c, d, cfg, bc, tm, c->d_out, nullptr, kClassS0, c->d_band_ctl + b, rb,
                          wide ? &wcfg : nullptr, false);
            if (rc) return rc;
        }
        const size_t upto = std::max<size_t>(rows_out, b == nb - 1 ? n : final_after[b]);
        if (upto > rows_out) {
            CK(cudaEventRecord(ev[2 * nb + b], s));
            CK(cudaStreamWaitEvent(c->d2h, ev[2 * nb + b], 0));
            CK(cudaMemcpyAsync(out_values + rows_out * ncols, c->d_out + rows_out * ncols,
                               (upto - rows_out) * ncols * sizeof(double), cudaMemcpyDeviceToHost,
                               c->d2h));
            c->d2h_bytes += (upto - rows_out) * ncols * sizeof(double);
            rows_out = upto;
        }
    }
    // the bands' error flags into the call's control block
    CK(cudaMemcpyAsync(c->h_band_ctl, c->d_band_ctl, (size_t)nb * sizeof(Control),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int b = 0; b < nb; ++b) c->h_ctl->error |= c->h_band_ctl[b].error;
    CK(cudaStreamSynchronize(c->d2h));
    return FX_OK;
}

// per-image checks of a batch; row_offsets[1..n] zeroed
int validate_batch(const fx_image* ims, int n, size_t* row_offsets) {
    const int kind = ims[0].mem_kind;
    for (int i = 0; i < n; ++i) {
        const fx_image& im = ims[i];
        if (!im.intensity || !im.labels) return set_error(FX_E_ARG, "null raster in batch");
        if (im.width < 1 || im.height < 1) return set_error(FX_E_PAIRING, "empty raster in batch");
        if (im.pitch && im.pitch < (size_t)im.width) return set_error(FX_E_ARG, "pitch < width");
        if (im.mem_kind != kind) return set_error(FX_E_ARG, "mixed host/device images in one batch");
        row_offsets[i + 1] = 0;
    }
    return FX_OK;
}

// Host image runs of a batch sub-batch (images back to back with the staging
// pitch, whole 64-row strips) staged packed: blocks of up to kBatchPackRows rows
// packed by the shared pool into half `buf` of the packed staging while this
// thread ships finished blocks (copy2: never waits for compute) and unpacks them
// on the copy stream (which waits until compute has released staging buffer buf);
// a share of the blocks goes raw by DMA meanwhile (as featurize_packed).  Packing
// into a half waits only for that half's previous copies (ev_pack_free), and its
// device half is rewritten only after its previous unpacks (ev_unpacked).
struct PackRun {
    const uint16_t *I, *L;
    size_t row0, rows;
};
constexpr int kBatchPackRows = 4096;
int stage_packed_runs(fx_ctx* c, const std::vector<PackRun>& runs, int P, int buf) {
    struct Blk {
        const uint16_t *I, *L;
        size_t row0;
        int rows;
        bool raw;
        size_t lab_off, int_off, cap_seg, cap_pix, mask_row;
    };
    std::vector<Blk> blk;
    size_t bytes = 0, mask_rows = 0;
    for (const PackRun& r : runs)
        for (size_t y = 0; y < r.rows; y += kBatchPackRows) {
            Blk b;
            b.rows = (int)std::min<size_t>(kBatchPackRows, r.rows - y);
            b.I = r.I + y * (size_t)P;
            b.L = r.L + y * (size_t)P;
            b.row0 = r.row0 + y;
            b.cap_seg = (size_t)b.rows * (size_t)P / 4;  // half the raw label bytes
            b.cap_pix = (size_t)b.rows * (size_t)P / 2;  // half the raw intensity bytes
            b.lab_off = bytes;
            bytes += pk_align16(pk_lab_bytes(b.rows, P, b.cap_seg));
            b.int_off = bytes;
            bytes += pk_align16(pk_int_bytes(b.rows, P, b.cap_pix));
            b.mask_row = mask_rows;
            mask_rows += (size_t)b.rows;
            b.raw = false;
            blk.push_back(b);
        }
    const int NB = (int)blk.size();
    for (int q = 0; q < NB; ++q) blk[q].raw = (q + 1) * c->pack_raw_pct / 100 > q * c->pack_raw_pct / 100;
    // staging halves sized for the largest sub-batch seen
    const size_t half = std::max(c->pack_half, pk_align16(bytes));
    int rc = FX_OK;
    if (half > c->pack_half) {  // re-lay the halves: nothing may still use the old ones
        CK(cudaStreamSynchronize(c->copy));
        CK(cudaStreamSynchronize(c->copy2));
        rc = ensure_pack(c, 2 * half);
        if (rc) return rc;
        c->pack_half = half;
    }
    for (int h = 0; h < 2; ++h) {
        if (!c->ev_pack_free[h]) CK(cudaEventCreateWithFlags(&c->ev_pack_free[h], cudaEventDisableTiming));
        if (!c->ev_unpacked[h]) CK(cudaEventCreateWithFlags(&c->ev_unpacked[h], cudaEventDisableTiming));
    }
    while ((int)c->ev_blocks.size() < NB) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_blocks.push_back(e);
    }
    CK(cudaEventSynchronize(c->ev_pack_free[buf]));  // this half's previous copies are done
    uint8_t* hp = c->h_pack + (size_t)buf * c->pack_half;
    uint8_t* dp = c->d_pack + (size_t)buf * c->pack_half;
    const size_t mp = (size_t)P / 32;
    std::vector<uint32_t>& maskv = c->pack_mask_b[buf];
    if (maskv.size() < mp * mask_rows) maskv.resize(mp * mask_rows);
    uint32_t* mask = maskv.data();
    std::vector<size_t> lab_bytes(NB, 0), int_bytes(NB, 0);
    std::unique_lock<std::mutex> lock(packer_mutex());
    PackPool* pool = packer_pool();
    pool->start(NB, [&](int t) {
        const Blk& b = blk[t];
        if (b.raw) return;
        uint32_t* m = mask + b.mask_row * mp;
        lab_bytes[t] = pack_labels(b.L, (size_t)P, P, 0, b.rows, hp + b.lab_off, b.cap_seg, m, mp);
        if (lab_bytes[t])
            int_bytes[t] = pack_intensity(b.I, (size_t)P, P, 0, b.rows, m, mp, hp + b.int_off, b.cap_pix);
    });
    struct Join {
        PackPool* p;
        ~Join() { p->wait(); }
    } join{pool};
    uint16_t* sI = c->d_stage[buf];
    uint16_t* sL = c->d_stage[buf] + c->stage_elems;
    auto raw = [&](const uint16_t* src, uint16_t* dst, const Blk& b) -> int {
        const size_t n = (size_t)b.rows * (size_t)P * 2;
        CK(cudaMemcpyAsync(dst + b.row0 * P, src, n, cudaMemcpyHostToDevice, c->copy));
        c->h2d_bytes += n;
        return FX_OK;
    };
    for (const Blk& b : blk)
        if (b.raw && ((rc = raw(b.L, sL, b)) || (rc = raw(b.I, sI, b)))) return rc;
    CK(cudaStreamWaitEvent(c->copy2, c->ev_unpacked[buf], 0));  // device half free
    for (int t = 0; t < NB; ++t) {
        const Blk& b = blk[t];
        if (b.raw) continue;
        while (!pool->done(t)) std::this_thread::yield();
        if (!lab_bytes[t]) {
            if ((rc = raw(b.L, sL, b)) || (rc = raw(b.I, sI, b))) return rc;
            continue;
        }
        CK(cudaMemcpyAsync(dp + b.lab_off, hp + b.lab_off, lab_bytes[t], cudaMemcpyHostToDevice, c->copy2));
        if (int_bytes[t])
            CK(cudaMemcpyAsync(dp + b.int_off, hp + b.int_off, int_bytes[t], cudaMemcpyHostToDevice,
                               c->copy2));
        c->h2d_bytes += lab_bytes[t] + int_bytes[t];
        CK(cudaEventRecord(c->ev_blocks[t], c->copy2));
        CK(cudaStreamWaitEvent(c->copy, c->ev_blocks[t], 0));
        const dim3 grid(pk_tiles(P), b.rows);
        Launch l(c, "k_unpack_labels", c->copy);
        k_unpack_labels<<<grid, 256, 0, c->copy>>>(dp + b.lab_off, b.rows, P, sL + b.row0 * P, P);
        if (int_bytes[t]) {
            Launch l2(c, "k_unpack_intensity", c->copy);
            k_unpack_intensity<<<grid, 256, 0, c->copy>>>(dp + b.int_off, b.rows, P, sL + b.row0 * P,
                                                          sI + b.row0 * P, P);
        } else if ((rc = raw(b.I, sI, b))) {
            return rc;
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_pack_free[buf], c->copy2));
    CK(cudaEventRecord(c->ev_unpacked[buf], c->copy));
    return FX_OK;
}

// The sub-batch pipeline of fx_featurize_batch with device outputs (out_dev,
// lab_dev: [cap_rois] rows): images stacked per sub-batch (one label-table slot
// each, staging double-buffered on the copy stream).  After each sub-batch's
// work is enqueued, on_sub(first_row, rows) may enqueue its readback (rows are
// final once the stream reaches that point).  Inputs validated by the caller.
int batch_core(fx_ctx* c, const fx_image* ims, int n, unsigned groups, const fx_texture_params* p,
               double* out_dev, uint32_t* lab_dev, size_t cap_rois, size_t* row_offsets,
               const std::function<int(size_t, size_t)>& on_sub) {
    const int kind = ims[0].mem_kind;
    int maxw = 0;
    for (int i = 0; i < n; ++i) maxw = std::max(maxw, ims[i].width);
    int rc = FX_OK;
    const FeatCfg cfg = make_cfg(groups, *p);
    const size_t P = ((size_t)maxw + 63) / 64 * 64;  // staging pitch (elements)
    auto pitch_of = [](const fx_image& im) { return im.pitch ? im.pitch : (size_t)im.width; };
    // plan: sub-batches of <= kBatchSlots images within the staging budget
    struct Sub {
        int first, count;
        size_t rows;  // stacked rows (each image padded to a multiple of 64)
        bool zero_copy;
    };
    std::vector<Sub> plan;
    for (int i = 0; i < n; ++i) {
        const size_t r = ((size_t)ims[i].height + 63) / 64 * 64;
        if (plan.empty() || plan.back().count == kBatchSlots ||
            (plan.back().rows + r) * P > kStageBudget)
            plan.push_back(Sub{i, 0, 0, false});
        plan.back().count++;
        plan.back().rows += r;
    }
    size_t max_rows = 0, max_strips = 0;
    int max_count = 0;
    bool need_stage = false;
    for (Sub& b : plan) {
        // device images already stacked in one pitched allocation are read in place
        bool zc = kind == FX_MEM_DEVICE;
        const size_t pt = pitch_of(ims[b.first]);
        for (int j = b.first; zc && j < b.first + b.count; ++j) {
            const fx_image& im = ims[j];
            zc = pitch_of(im) == pt;
            if (zc && j + 1 < b.first + b.count) {
                const size_t step = pt * (size_t)im.height;
                zc = im.height % 64 == 0 && ims[j + 1].labels == im.labels + step &&
                     ims[j + 1].intensity == im.intensity + step;
            }
        }
        b.zero_copy = zc;
        if (zc) {
            b.rows = 0;
            for (int j = b.first; j < b.first + b.count; ++j) b.rows += (size_t)ims[j].height;
        } else {
            need_stage = true;
            max_rows = std::max(max_rows, b.rows);
        }
        max_strips = std::max(max_strips, (b.rows + 63) / 64);
        max_count = std::max(max_count, b.count);
    }
    rc = ensure_slots(c, max_count);
    if (!rc) rc = ensure_maps(c, (size_t)max_count, max_strips);
    if (!rc && need_stage) rc = ensure_stage(c, P * max_rows);
    if (rc) return rc;
    // stage sub-batch k into buffer k%2 on the copy stream (slot map included)
    auto stage = [&](int k) -> int {
        const Sub& b = plan[k];
        const int buf = k % 2;
        CK(cudaStreamWaitEvent(c->copy, c->ev_free[buf], 0));
        SlotInfo* hs = c->h_slots[buf];
        uint16_t* hst = c->h_strips[buf];
        size_t row0 = 0;
        const cudaMemcpyKind mk = kind == FX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        // images that sit back to back in the caller's memory with the staging pitch
        // and whole 64-row strips (e.g. a [T, H, W] stack) go in one linear copy per
        // raster: one call per run instead of two per image (host enqueue time
        // bounded the C4 end-to-end path)
        const uint16_t *runI = nullptr, *runL = nullptr;
        size_t run_row0 = 0, run_rows = 0;
        // host runs are packed (label change points + labelled intensities) where the
        // host can (fx_pack.hpp), else copied raw
        const bool pack = kind == FX_MEM_HOST && c->packing && pack_isa() == 2 && P <= 65536;
        std::vector<PackRun> runs;
        auto flush = [&]() -> int {
            if (run_rows) {
                if (pack) {
                    runs.push_back(PackRun{runI, runL, run_row0, run_rows});
                } else {
                    CK(cudaMemcpyAsync(c->d_stage[buf] + run_row0 * P, runI, run_rows * P * 2, mk, c->copy));
                    CK(cudaMemcpyAsync(c->d_stage[buf] + c->stage_elems + run_row0 * P, runL,
                                       run_rows * P * 2, mk, c->copy));
                    c->h2d_bytes += run_rows * P * 4;
                }
            }
            run_rows = 0;
            return FX_OK;
        };
        for (int j = 0; j < b.count; ++j) {
            const fx_image& im = ims[b.first + j];
            hs[j] = SlotInfo{(int32_t)row0, im.width, im.height, im.origin_x, im.origin_y};
            const size_t r = b.zero_copy ? (size_t)im.height : ((size_t)im.height + 63) / 64 * 64;
            for (size_t st = row0 / 64; st < (row0 + r + 63) / 64; ++st) hst[st] = (uint16_t)j;
            if (!b.zero_copy) {
                const bool linear = pitch_of(im) == P && (size_t)im.height == r;
                if (linear && run_rows && im.intensity == runI + run_rows * P && im.labels == runL + run_rows * P) {
                    run_rows += r;  // extends the current run
                } else {
                    if (flush()) return FX_E_CUDA;
                    if (linear) {
                        runI = im.intensity;
                        runL = im.labels;
                        run_row0 = row0;
                        run_rows = r;
                    } else {
                        const size_t sp = pitch_of(im) * 2;
                        uint16_t* dI = c->d_stage[buf] + row0 * P;
                        uint16_t* dL = c->d_stage[buf] + c->stage_elems + row0 * P;
                        CK(cudaMemcpy2DAsync(dI, P * 2, im.intensity, sp, (size_t)im.width * 2,
                                             (size_t)im.height, mk, c->copy));
                        CK(cudaMemcpy2DAsync(dL, P * 2, im.labels, sp, (size_t)im.width * 2,
                                             (size_t)im.height, mk, c->copy));
                        if (kind == FX_MEM_HOST) c->h2d_bytes += (size_t)im.width * im.height * 4;
                    }
                }
            }
            row0 += r;
        }
        if (flush()) return FX_E_CUDA;
        if (!runs.empty()) {
            const int prc = stage_packed_runs(c, runs, (int)P, buf);
            if (prc) return prc;
        }
        CK(cudaMemcpyAsync(c->d_slots[buf], hs, (size_t)b.count * sizeof(SlotInfo),
                           cudaMemcpyHostToDevice, c->copy));
        CK(cudaMemcpyAsync(c->d_strips[buf], hst, ((b.rows + 63) / 64) * sizeof(uint16_t),
                           cudaMemcpyHostToDevice, c->copy));
        CK(cudaEventRecord(c->ev_staged[buf], c->copy));
        return FX_OK;
    };
    size_t base = 0;
    std::vector<uint32_t> sb((size_t)max_count + 1);
    rc = stage(0);
    for (size_t k = 0; !rc && k < plan.size(); ++k) {
        if (k + 1 < plan.size()) rc = stage((int)k + 1);
        if (rc) break;
        const Sub& b = plan[k];
        const int buf = (int)(k % 2);
        CK(cudaStreamWaitEvent(c->stream, c->ev_staged[buf], 0));
        DevImage d;
        int wmax = 0;
        for (int j = b.first; j < b.first + b.count; ++j) wmax = std::max(wmax, ims[j].width);
        if (b.zero_copy) {
            d.I = ims[b.first].intensity;
            d.L = ims[b.first].labels;
            d.pitch = pitch_of(ims[b.first]);
        } else {
            d.I = c->d_stage[buf];
            d.L = c->d_stage[buf] + c->stage_elems;
            d.pitch = P;
        }
        d.w = wmax;
        d.h = (int)b.rows;
        d.ox = d.oy = 0;
        SlotMap m;
        m.info = c->d_slots[buf];
        m.strip_slot = c->d_strips[buf];
        m.s0 = SlotInfo{0, 0, 0, 0, 0};
        m.nslots = b.count;
        size_t nr = 0;
        rc = scan_stage(c, d, m, true);
        if (!rc)
            rc = featurize_stage(c, d, m, 0u, 0xffffffffu, groups, *p, out_dev + base * cfg.ncols,
                                 cap_rois >= base ? cap_rois - base : 0, &nr, nullptr, sb.data(),
                                 k == 0);
        if (rc) {
            if (rc == FX_E_CAPACITY) row_offsets[n] = base + nr;  // rows needed so far
            break;
        }
        for (int j = 0; j < b.count; ++j) row_offsets[b.first + j] = base + sb[j];
        if (nr)
            CK(cudaMemcpyAsync(lab_dev + base, roi_list(c).label, nr * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaEventRecord(c->ev_free[buf], c->stream));
        if (on_sub) {
            rc = on_sub(base, nr);
            if (rc) break;
        }
        base += nr;
    }
    if (rc) {
        cudaStreamSynchronize(c->copy);
        cudaStreamSynchronize(c->stream);
        return rc;
    }
    row_offsets[n] = base;
    return FX_OK;
}


}  // namespace

// ---- internal entry points for fx_multi.cu (not part of the C ABI) ------------
namespace fxg {
int ictx_validate_batch(const fx_image* ims, int n, size_t* row_offsets) {
    return validate_batch(ims, n, row_offsets);
}
int ictx_check_groups(unsigned groups) { return check_groups(groups); }
int ictx_ncols(unsigned groups, const fx_texture_params& p) { return make_cfg(groups, p).ncols; }
int ictx_batch_device(fx_ctx* c, const fx_image* ims, int n, unsigned groups,
                      const fx_texture_params* p, double* out_dev, uint32_t* lab_dev,
                      size_t cap_rows, size_t* row_offsets) {
    return batch_core(c, ims, n, groups, p, out_dev, lab_dev, cap_rows, row_offsets, nullptr);
}
// ---- whole slide over several devices: one row band per context ---------------
// (driven by fx_multi_featurize_slide, fx_multi.cu; every step is enqueued on the
// context's stream, the order across devices is kept by events)

// H2D of rows [y0, y1) of the host slide into this context's raster (with
// `reserve` spare rows below for the halo), then the label scan of the band into
// a fresh table (global rows).  *lmax: the band's largest label.
int islide_load_scan(fx_ctx* c, const fx_image* im, int y0, int y1, int reserve,
                     cudaEvent_t loaded, cudaEvent_t scanned, uint32_t* lmax) {
    CK(cudaSetDevice(c->device));
    const int rows = y1 - y0, W = im->width;
    int rc = ensure_img(c, W, rows + reserve);
    if (rc) return rc;
    cudaStream_t s = c->stream;
    const size_t P = c->img_pitch, sp = (im->pitch ? im->pitch : (size_t)W) * 2;
    uint16_t* dI = c->d_img;
    uint16_t* dL = c->d_img + P * c->img_rows_cap;
    CK(cudaMemcpy2DAsync(dL, P * 2, im->labels + (size_t)y0 * (sp / 2), sp, (size_t)W * 2, rows,
                         cudaMemcpyHostToDevice, s));
    CK(cudaMemcpy2DAsync(dI, P * 2, im->intensity + (size_t)y0 * (sp / 2), sp, (size_t)W * 2, rows,
                         cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(loaded, s));
    DevImage band{dI, dL, W, rows, P, im->origin_x, im->origin_y + y0};
    rc = scan_stage(c, band, single_map(band), true);
    if (rc) return rc;
    CK(cudaEventRecord(scanned, s));
    CK(cudaMemcpyAsync(c->h_slot_base, c->d_maxlab, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *lmax = c->h_slot_base[0];
    return FX_OK;
}

// this context's band raster and label table, for its peers
void islide_band(fx_ctx* c, const uint16_t** L, const uint16_t** I, size_t* pitch,
                 const unsigned long long** cnt, const uint32_t** bb, size_t* bb_pitch) {
    *I = c->d_img;
    *L = c->d_img + c->img_pitch * c->img_rows_cap;
    *pitch = c->img_pitch;
    *cnt = c->d_cnt;
    *bb = c->d_bb;
    *bb_pitch = (size_t)c->tab_slots * kMaxLabels;
}

// the table of labels [0, lmax] merged from every band's table (peer reads, after
// every band's scan) into this context's scratch
int islide_merge(fx_ctx* c, const TablePeers& tp, uint32_t lmax, const cudaEvent_t* scanned,
                 cudaEvent_t merged) {
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    if (!c->d_mcnt) {
        CK(cudaMalloc(&c->d_mcnt, (size_t)kMaxLabels * sizeof(unsigned long long)));
        CK(cudaMalloc(&c->d_mbb, 4 * (size_t)kMaxLabels * sizeof(uint32_t)));
    }
    for (int e = 0; e < tp.n; ++e) CK(cudaStreamWaitEvent(s, scanned[e], 0));
    {
        Launch l(c, "k_table_merge");
        const int grid = std::max(1, std::min<int>((int)(lmax / 256) + 1, 4 * c->sm_count));
        k_table_merge<<<grid, 256, 0, s>>>(tp, lmax, c->d_mcnt, c->d_mbb, kMaxLabels);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(merged, s));
    return FX_OK;
}

// after every context merged (its peers stop reading this table): the merged
// table becomes this context's table, and is read back (host cnt [lmax+1],
// bbox [4][lmax+1]) for the ownership and halo plan
int islide_commit(fx_ctx* c, uint32_t lmax, const cudaEvent_t* merged, int n_peers,
                  uint64_t* h_cnt, uint32_t* h_bb) {
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    for (int e = 0; e < n_peers; ++e) CK(cudaStreamWaitEvent(s, merged[e], 0));
    const size_t n = (size_t)lmax + 1, bp = (size_t)c->tab_slots * kMaxLabels;
    CK(cudaMemcpyAsync(c->d_cnt, c->d_mcnt, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpy2DAsync(c->d_bb, bp * 4, c->d_mbb, (size_t)kMaxLabels * 4, n * 4, 4,
                         cudaMemcpyDeviceToDevice, s));
    c->h_slot_base[0] = lmax;  // the compaction walks labels up to the table's max label
    CK(cudaMemcpyAsync(c->d_maxlab, c->h_slot_base, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(h_cnt, c->d_mcnt, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(h_bb, n * 4, c->d_mbb, (size_t)kMaxLabels * 4, n * 4, 4,
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->table_clean = false;
    return FX_OK;
}

// Halo of the owned straddling windows: `need` rows below the band with zeroed
// labels, the windows' rectangles gathered from the peers' band rasters (peer
// reads after their loads), then the owned ROIs featurized on band + halo.  Rows
// (labels ascending) and labels are read back into host buffers.
int islide_featurize(fx_ctx* c, const fx_image* im, int y0, int y1, int need,
                     const std::vector<HaloRect>& rects, const std::vector<const uint16_t*>& pL,
                     const std::vector<const uint16_t*>& pI, const std::vector<size_t>& pp,
                     const std::vector<int>& py0, const cudaEvent_t* loaded, unsigned groups,
                     const fx_texture_params& p, size_t cap, uint32_t* h_labels, double* h_values,
                     size_t* n_rois) {
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int W = im->width, rows = y1 - y0, total = rows + need;
    const size_t P = c->img_pitch;
    uint16_t* bandI = c->d_img;
    uint16_t* bandL = c->d_img + P * c->img_rows_cap;
    uint16_t *wI = bandI, *wL = bandL;
    if ((size_t)total > c->img_rows_cap) {
        // too few reserve rows: a separate band + halo raster (the band buffer stays
        // in place: the peers may be reading it)
        const size_t elems = P * (size_t)total * 2;
        if (elems > c->work_elems) {
            cudaStreamSynchronize(s);
            cudaFree(c->d_work);
            c->d_work = nullptr;
            c->work_elems = 0;
            CK(cudaMalloc(&c->d_work, elems * sizeof(uint16_t)));
            c->work_elems = elems;
        }
        wI = c->d_work;
        wL = c->d_work + P * (size_t)total;
        CK(cudaMemcpy2DAsync(wI, P * 2, bandI, P * 2, (size_t)W * 2, rows, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpy2DAsync(wL, P * 2, bandL, P * 2, (size_t)W * 2, rows, cudaMemcpyDeviceToDevice, s));
    }
    if (need > 0) {
        CK(cudaMemset2DAsync(wL + (size_t)rows * P, P * 2, 0, (size_t)W * 2, need, s));
        const int nr = (int)rects.size(), np = (int)pL.size();
        std::vector<uint8_t> h;
        auto put = [&](const void* src, size_t n) {
            const size_t at = (h.size() + 15) / 16 * 16;
            h.resize(at + n);
            std::memcpy(h.data() + at, src, n);
            return at;
        };
        const size_t oR = put(rects.data(), nr * sizeof(HaloRect));
        const size_t oL = put(pL.data(), np * sizeof(void*)), oI = put(pI.data(), np * sizeof(void*));
        const size_t oP = put(pp.data(), np * sizeof(size_t)), oY = put(py0.data(), np * sizeof(int));
        if (h.size() > c->slide_bytes) {
            cudaStreamSynchronize(s);
            cudaFree(c->d_slide);
            c->d_slide = nullptr;
            c->slide_bytes = 0;
            CK(cudaMalloc(&c->d_slide, h.size()));
            c->slide_bytes = h.size();
        }
        CK(cudaMemcpyAsync(c->d_slide, h.data(), h.size(), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // h is a pageable local
        for (int e = 0; e < np; ++e) CK(cudaStreamWaitEvent(s, loaded[e], 0));
        if (nr) {
            const uint8_t* b = c->d_slide;
            Launch l(c, "k_halo_gather");
            k_halo_gather<<<dim3(64, std::min(nr, 1024)), 256, 0, s>>>(
                (const HaloRect*)(b + oR), nr, (const uint16_t* const*)(b + oL),
                (const uint16_t* const*)(b + oI), (const size_t*)(b + oP), (const int*)(b + oY), wL, wI,
                P, y0);
        }
        CK(cudaGetLastError());
    }
    const FeatCfg cfg = make_cfg(groups, p);
    int rc = ensure_out(c, std::max<size_t>(1, cap) * (size_t)cfg.ncols);
    if (rc) return rc;
    DevImage d{wI, wL, W, total, P, im->origin_x, im->origin_y + y0};
    rc = featurize_stage(c, d, single_map(d), (uint32_t)(im->origin_y + y0),
                         (uint32_t)(im->origin_y + y1), groups, p, c->d_out, cap, n_rois, nullptr);
    if (rc) {
        cudaStreamSynchronize(s);
        return rc;
    }
    if (*n_rois) {
        CK(cudaMemcpyAsync(h_values, c->d_out, *n_rois * cfg.ncols * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h_labels, roi_list(c).label, *n_rois * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    }
    return finish(c);
}

cudaStream_t ictx_stream(fx_ctx* c) { return c->stream; }
cudaStream_t ictx_d2h(fx_ctx* c) { return c->d2h; }
int ictx_device(const fx_ctx* c) { return c->device; }
int ictx_finish(fx_ctx* c) { return finish(c); }
}  // namespace fxg

extern "C" {

int fx_ctx_create(int device, fx_ctx** out) {
    if (!out) return set_error(FX_E_ARG, "null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_error(FX_E_CUDA, "no CUDA device visible (the device path has no CPU fallback)");
    if (device < 0 || device >= ndev) return set_error(FX_E_ARG, "bad device index");
    fx_ctx* c = new fx_ctx();
    c->device = device;
    auto fail = [&](int rc) {
        fx_ctx_destroy(c);
        return rc;
    };
#define CKC(x)                                                                     \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            return fail(set_error(e_ == cudaErrorMemoryAllocation ? FX_E_OOM : FX_E_CUDA, \
                                  std::string(#x) + ": " + cudaGetErrorString(e_))); \
    } while (0)
    CKC(cudaSetDevice(device));
    cudaDeviceProp prop;
    CKC(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(set_error(FX_E_CUDA, "libfxg is built for sm_100a (B200); device is sm_" +
                                             std::to_string(prop.major * 10 + prop.minor)));
    c->sm_count = prop.multiProcessorCount;
    if (const char* e = getenv("FXG_SYNC_DEBUG")) c->sync_debug = atoi(e) != 0;
    if (const char* e = getenv("FXG_NO_TMA")) c->no_tma = atoi(e) != 0;
    if (const char* e = getenv("FXG_NO_STAGE")) c->no_stage = atoi(e) != 0;
    CKC(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    CKC(cudaEventCreateWithFlags(&c->ev_compact, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_stats, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CKC(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->copy2, cudaStreamNonBlocking));
    if (const char* e = getenv("FXG_BAND_ROWS")) c->band_rows = atoi(e);
    if (const char* e = getenv("FXG_PACK")) c->packing = atoi(e) != 0;
    if (const char* e = getenv("FXG_PACK_RAW")) c->pack_raw_pct = std::max(0, std::min(100, atoi(e)));
    for (int b = 0; b < 2; ++b) {
        CKC(cudaEventCreateWithFlags(&c->ev_staged[b], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&c->ev_free[b], cudaEventDisableTiming));
    }
    CKC(cudaMalloc(&c->d_ctl, sizeof(Control)));
    CKC(cudaMallocHost(&c->h_ctl, sizeof(Control)));
    CKC(cudaMalloc(&c->d_dbg, sizeof(DebugOut)));
    {
        int rc = ensure_slots(c, 1);
        if (rc) return fail(rc);
        CKC(cudaStreamSynchronize(c->stream));
    }
    CKC(roi_s_setup(&c->occ_s[0][0]));
    CKC(roi_b_setup());
    CKC(roi_t_setup());
    CKC(wide_setup());
    for (auto& row : c->occ_s)
        for (int& o : row) o = std::max(1, o);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        c->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
#undef CKC
    *out = c;
    return FX_OK;
}

int fx_ctx_destroy(fx_ctx* c) {
    if (!c) return FX_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy) cudaStreamSynchronize(c->copy);
    if (c->d2h) cudaStreamSynchronize(c->d2h);
    collect_times(c);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    c->ev_pool.clear();
    cudaFreeHost(c->h_pack);
    cudaFree(c->d_pack);
    for (int h = 0; h < 2; ++h) {
        if (c->ev_pack_free[h]) cudaEventDestroy(c->ev_pack_free[h]);
        if (c->ev_unpacked[h]) cudaEventDestroy(c->ev_unpacked[h]);
    }
    for (cudaEvent_t e : c->ev_blocks) cudaEventDestroy(e);
    cudaFree(c->d_cnt);
    cudaFree(c->d_bb);
    cudaFree(c->d_maxlab);
    cudaFree(c->d_csum);
    if (c->h_slot_base) cudaFreeHost(c->h_slot_base);
    cudaFree(c->d_ctl);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    cudaFree(c->d_roi32);
    cudaFree(c->d_roin);
    for (int b = 0; b < 2; ++b) {
        cudaFree(c->d_slots[b]);
        cudaFree(c->d_strips[b]);
        if (c->h_slots[b]) cudaFreeHost(c->h_slots[b]);
        if (c->h_strips[b]) cudaFreeHost(c->h_strips[b]);
        cudaFree(c->d_stage[b]);
        if (c->ev_staged[b]) cudaEventDestroy(c->ev_staged[b]);
        if (c->ev_free[b]) cudaEventDestroy(c->ev_free[b]);
    }
    cudaFree(c->d_blab);
    cudaFree(c->d_shape_rows);
    cudaFree(c->d_shape_hdr);
    cudaFree(c->d_tscratch[0]);
    cudaFree(c->d_tscratch[1]);
    cudaFree(c->d_mom_px);
    cudaFree(c->d_mom_off);
    cudaFree(c->d_mom_sums);
    cudaFree(c->d_int_vals);
    cudaFree(c->d_int_off);
    cudaFree(c->d_int_sums);
    cudaFree(c->d_img);
    cudaFree(c->d_out);
    cudaFree(c->d_lscratch);
    cudaFree(c->d_dbg);
    for (auto& p : c->pending) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->ev_compact) cudaEventDestroy(c->ev_compact);
    if (c->ev_stats) cudaEventDestroy(c->ev_stats);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->d2h) cudaStreamDestroy(c->d2h);
    if (c->copy2) cudaStreamDestroy(c->copy2);
    for (cudaEvent_t e : c->ev_band) cudaEventDestroy(e);
    cudaFree(c->d_band);
    cudaFree(c->d_band_ctl);
    cudaFree(c->d_band_seg);
    cudaFree(c->d_mcnt);
    cudaFree(c->d_mbb);
    cudaFree(c->d_slide);
    cudaFree(c->d_work);
    cudaFree(c->d_wscratch);
    if (c->h_band) cudaFreeHost(c->h_band);
    if (c->h_band_ctl) cudaFreeHost(c->h_band_ctl);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return FX_OK;
}

int fx_host_alloc(size_t bytes, void** out) {
    if (!out) return set_error(FX_E_ARG, "null argument");
    *out = nullptr;
    if (bytes == 0) return FX_OK;
    if (cudaMallocHost(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return set_error(FX_E_OOM, "pinned host allocation failed");
    }
    return FX_OK;
}

int fx_host_free(void* p) {
    if (p && cudaFreeHost(p) != cudaSuccess) {
        cudaGetLastError();
        return set_error(FX_E_CUDA, "cudaFreeHost failed");
    }
    return FX_OK;
}

int fx_ctx_set_stream(fx_ctx* c, void* stream) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    return FX_OK;
}

int fx_ctx_set_band_rows(fx_ctx* c, int rows) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    c->band_rows = rows;
    return FX_OK;
}

int fx_debug_pack_rows(const uint16_t* labels, const uint16_t* intensity, size_t pitch, int width,
                       int rows, uint8_t* lab_region, size_t lab_cap, uint8_t* int_region,
                       size_t int_cap, size_t* lab_bytes, size_t* int_bytes) {
    if (!labels || !intensity || !lab_region || !int_region || !lab_bytes || !int_bytes || width < 1 ||
        rows < 1 || pitch < (size_t)width)
        return set_error(FX_E_ARG, "bad argument");
    if (pack_isa() != 2) return set_error(FX_E_CONFIG, "this host has no AVX-512 VBMI2 packer");
    const size_t idx = pk_index_bytes(rows, width);
    if (lab_cap < idx + 128 || int_cap < idx + 64) return set_error(FX_E_ARG, "region too small");
    const size_t cap_seg = (lab_cap - idx - 128) / 4, cap_pix = (int_cap - idx - 64) / 2;
    const size_t mp = ((size_t)width + 31) / 32;
    std::vector<uint32_t> mask(mp * (size_t)rows);
    *lab_bytes = pack_labels(labels, pitch, width, 0, rows, lab_region, cap_seg, mask.data(), mp);
    *int_bytes = *lab_bytes ? pack_intensity(intensity, pitch, width, 0, rows, mask.data(), mp, int_region,
                                             cap_pix)
                            : 0;
    return FX_OK;
}

int fx_ctx_set_packing(fx_ctx* c, int on) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    c->packing = on != 0;
    return FX_OK;
}

int fx_ctx_last_transfer(const fx_ctx* c, uint64_t* h2d, uint64_t* d2h) {
    if (!c || !h2d || !d2h) return set_error(FX_E_ARG, "null argument");
    *h2d = c->h2d_bytes;
    *d2h = c->d2h_bytes;
    return FX_OK;
}

uint64_t fx_ctx_launch_count(const fx_ctx* c) { return c ? c->launches : 0; }

int fx_ctx_enable_timing(fx_ctx* c, int enable) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    c->timing = enable != 0;
    return FX_OK;
}

int fx_ctx_timing_filter(fx_ctx* c, const char* kernel) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    c->timing_only = kernel ? kernel : "";
    return FX_OK;
}

int fx_ctx_kernel_times(fx_ctx* c, char* names, size_t names_cap, double* ms, uint64_t* counts,
                        int cap, int* n) {
    if (!c || !n) return set_error(FX_E_ARG, "null argument");
    collect_times(c);
    std::string joined;
    int i = 0;
    for (auto& kv : c->ktimes) {
        if (i < cap) {
            if (ms) ms[i] = kv.second.ms;
            if (counts) counts[i] = kv.second.count;
        }
        if (i) joined += '\n';
        joined += kv.first;
        ++i;
    }
    *n = i;
    if (names) {
        if (names_cap < joined.size() + 1) return set_error(FX_E_CAPACITY, "names buffer too small");
        std::memcpy(names, joined.c_str(), joined.size() + 1);
    }
    return FX_OK;
}

int fx_ctx_reset_kernel_times(fx_ctx* c) {
    if (!c) return set_error(FX_E_ARG, "null ctx");
    collect_times(c);
    c->ktimes.clear();
    return FX_OK;
}

int fx_featurize(fx_ctx* c, const fx_image* im, unsigned groups, const fx_texture_params* p,
                 uint32_t* out_labels, double* out_values, size_t cap_rois, size_t* n_rois) {
    if (!c || !im || !p || !n_rois) return set_error(FX_E_ARG, "null argument");
    if (!im->intensity || !im->labels) return set_error(FX_E_ARG, "null raster");
    if (im->width < 1 || im->height < 1) return set_error(FX_E_PAIRING, "empty raster");
    if (im->pitch && im->pitch < (size_t)im->width) return set_error(FX_E_ARG, "pitch < width");
    *n_rois = 0;
    int rc = check_groups(groups);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    const FeatCfg cfg = make_cfg(groups, *p);
    if (im->mem_kind == FX_MEM_HOST) {
        const int br = band_rows_for(c, im->width, im->height);
        if (br > 0) {
            rc = ensure_out(c, std::max<size_t>(1, cap_rois) * (size_t)cfg.ncols);
            if (!rc)
                rc = packing_usable(c, im)
                         ? featurize_packed(c, im, br, groups, *p, out_labels, out_values, cap_rois, n_rois)
                         : featurize_banded(c, im, br, groups, *p, out_labels, out_values, cap_rois, n_rois);
            // no copy may still read the caller's rasters once the call returns
            cudaStreamSynchronize(c->copy);
            cudaStreamSynchronize(c->copy2);
            if (rc) {
                cudaStreamSynchronize(c->copy);
                cudaStreamSynchronize(c->d2h);
                cudaStreamSynchronize(c->stream);
                return rc;
            }
            return finish(c);
        }
    }
    DevImage d;
    rc = stage_image(c, im, &d);
    if (rc) return rc;
    double* out_dev = out_values;
    if (im->mem_kind == FX_MEM_HOST) {
        rc = ensure_out(c, std::max<size_t>(1, cap_rois) * (size_t)cfg.ncols);
        if (rc) return rc;
        out_dev = c->d_out;
    }
    rc = run_pipeline(c, d, groups, *p, out_dev, cap_rois, n_rois, nullptr);
    if (rc) {
        cudaStreamSynchronize(c->stream);
        return rc;
    }
    const size_t nr = *n_rois;
    if (im->mem_kind == FX_MEM_HOST) {
        if (nr) {
            CK(cudaMemcpyAsync(out_values, out_dev, nr * cfg.ncols * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(out_labels, roi_list(c).label, nr * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, c->stream));
        }
    } else if (nr) {
        CK(cudaMemcpyAsync(out_labels, roi_list(c).label, nr * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, c->stream));
    }
    return finish(c);
}

int fx_scan_accumulate(fx_ctx* c, const fx_image* im, int reset) {
    if (!c || !im || !im->labels) return set_error(FX_E_ARG, "null argument");
    if (im->width < 1 || im->height < 1) return set_error(FX_E_PAIRING, "empty raster");
    CK(cudaSetDevice(c->device));
    fx_image lab_only = *im;
    if (!lab_only.intensity) lab_only.intensity = lab_only.labels;  // scan reads labels only
    DevImage d;
    int rc = stage_image(c, &lab_only, &d);
    if (!rc) rc = scan_stage(c, d, single_map(d), reset != 0);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));
    return FX_OK;
}

int fx_label_table_copy(fx_ctx* c, uint64_t* cnt, uint32_t* bbox, int to_ctx, int mem_kind) {
    if (!c || !cnt || !bbox) return set_error(FX_E_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    const cudaMemcpyKind k = to_ctx ? (mem_kind == FX_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                 : cudaMemcpyHostToDevice)
                                    : (mem_kind == FX_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                 : cudaMemcpyDeviceToHost);
    // slot 0 of the ctx table; its bbox rows are tab_slots*65536 apart
    const size_t bc = kMaxLabels * sizeof(unsigned long long), row = kMaxLabels * sizeof(uint32_t);
    const size_t tab_pitch = (size_t)c->tab_slots * row;
    if (to_ctx) {
        CK(cudaMemcpyAsync(c->d_cnt, cnt, bc, k, c->stream));
        CK(cudaMemcpy2DAsync(c->d_bb, tab_pitch, bbox, row, row, 4, k, c->stream));
        // the loaded table is consumed by the next compaction over all labels
        const uint32_t full = kMaxLabels - 1;
        CK(cudaMemcpyAsync(c->d_maxlab, &full, sizeof full, cudaMemcpyHostToDevice, c->stream));
        c->table_clean = false;
    } else {
        CK(cudaMemcpyAsync(cnt, c->d_cnt, bc, k, c->stream));
        CK(cudaMemcpy2DAsync(bbox, row, c->d_bb, tab_pitch, row, 4, k, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return FX_OK;
}

int fx_featurize_owned(fx_ctx* c, const fx_image* im, int own_y0, int own_y1, unsigned groups,
                       const fx_texture_params* p, uint32_t* out_labels, double* out_values,
                       size_t cap_rois, size_t* n_rois) {
    if (!c || !im || !p || !n_rois) return set_error(FX_E_ARG, "null argument");
    if (!im->intensity || !im->labels) return set_error(FX_E_ARG, "null raster");
    if (own_y0 < 0 || own_y1 < own_y0) return set_error(FX_E_ARG, "bad owned row range");
    *n_rois = 0;
    int rc = check_groups(groups);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    DevImage d;
    rc = stage_image(c, im, &d);
    if (rc) return rc;
    const FeatCfg cfg = make_cfg(groups, *p);
    double* out_dev = out_values;
    if (im->mem_kind == FX_MEM_HOST) {
        rc = ensure_out(c, std::max<size_t>(1, cap_rois) * (size_t)cfg.ncols);
        if (rc) return rc;
        out_dev = c->d_out;
    }
    rc = featurize_stage(c, d, single_map(d), (uint32_t)own_y0, (uint32_t)own_y1, groups, *p,
                         out_dev, cap_rois, n_rois, nullptr);
    if (rc) {
        cudaStreamSynchronize(c->stream);
        return rc;
    }
    const size_t nr = *n_rois;
    if (nr) {
        const cudaMemcpyKind k = im->mem_kind == FX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (im->mem_kind == FX_MEM_HOST)
            CK(cudaMemcpyAsync(out_values, out_dev, nr * cfg.ncols * sizeof(double), k, c->stream));
        CK(cudaMemcpyAsync(out_labels, roi_list(c).label, nr * sizeof(uint32_t), k, c->stream));
    }
    return finish(c);
}

// ---- batch of images (C4): stacked in HBM, one table slot per image -------------

int fx_featurize_batch(fx_ctx* c, const fx_image* ims, int n, unsigned groups,
                       const fx_texture_params* p, uint32_t* out_labels, double* out_values,
                       size_t cap_rois, size_t* row_offsets) {
    if (!c || (n && !ims) || !p || !row_offsets || n < 0) return set_error(FX_E_ARG, "null argument");
    row_offsets[0] = 0;
    if (n == 0) return FX_OK;
    int rc = validate_batch(ims, n, row_offsets);
    if (!rc) rc = check_groups(groups);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    const FeatCfg cfg = make_cfg(groups, *p);
    if (ims[0].mem_kind == FX_MEM_DEVICE) {
        rc = batch_core(c, ims, n, groups, p, out_values, out_labels, cap_rois, row_offsets, nullptr);
        return rc ? rc : finish(c);
    }
    // host images: each sub-batch's rows leave on the d2h stream while the next
    // sub-batch computes
    c->h2d_bytes = c->d2h_bytes = 0;
    rc = ensure_out(c, std::max<size_t>(1, cap_rois) * (size_t)cfg.ncols);
    if (!rc) rc = ensure_blab(c, std::max<size_t>(1, cap_rois));
    if (rc) return rc;
    const size_t nc = (size_t)cfg.ncols;
    auto readback = [&](size_t first, size_t rows) -> int {
        if (!rows) return FX_OK;
        cudaEvent_t e = get_event(c);
        CK(cudaEventRecord(e, c->stream));
        CK(cudaStreamWaitEvent(c->d2h, e, 0));
        c->ev_pool.push_back(e);  // reusable once recorded work is queued behind it
        CK(cudaMemcpyAsync(out_values + first * nc, c->d_out + first * nc, rows * nc * sizeof(double),
                           cudaMemcpyDeviceToHost, c->d2h));
        CK(cudaMemcpyAsync(out_labels + first, c->d_blab + first, rows * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, c->d2h));
        c->d2h_bytes += rows * (nc * sizeof(double) + sizeof(uint32_t));
        return FX_OK;
    };
    rc = batch_core(c, ims, n, groups, p, c->d_out, c->d_blab, cap_rois, row_offsets, readback);
    cudaStreamSynchronize(c->d2h);
    cudaStreamSynchronize(c->copy);  // no copy may still read the caller's rasters
    return rc ? rc : finish(c);
}

int fx_featurize_u16(fx_ctx* c, const uint16_t* intensity, const uint16_t* labels, int width,
                     int height, size_t pitch, int mem_kind, unsigned groups,
                     const fx_texture_params* p, uint32_t* out_labels, double* out_values,
                     size_t cap_rois, size_t* n_rois) {
    fx_image im{intensity, labels, width, height, pitch, 0, 0, mem_kind};
    return fx_featurize(c, &im, groups, p, out_labels, out_values, cap_rois, n_rois);
}

int fx_roi_features(fx_ctx* c, const uint32_t* xs, const uint32_t* ys, const uint16_t* is,
                    size_t n, unsigned groups, const fx_texture_params* p, double* out,
                    size_t cap) {
    if (!c || !p || !out || (n && (!xs || !ys || !is))) return set_error(FX_E_ARG, "null argument");
    int rc = check_groups(groups);
    if (rc) return rc;
    const FeatCfg cfg = make_cfg(groups, *p);
    if (cap < (size_t)cfg.ncols) return set_error(FX_E_CAPACITY, "output buffer too small");
    if (n == 0) {  // empty cloud: every group reports zeros (engine.cpp:138-209)
        std::fill(out, out + cfg.ncols, 0.0);
        return FX_OK;
    }
    uint32_t x0 = xs[0], x1 = xs[0], y0 = ys[0], y1 = ys[0];
    for (size_t i = 0; i < n; ++i) {
        x0 = std::min(x0, xs[i]);
        x1 = std::max(x1, xs[i]);
        y0 = std::min(y0, ys[i]);
        y1 = std::max(y1, ys[i]);
    }
    if ((uint64_t)(x1 - x0 + 1) * (uint64_t)(y1 - y0 + 1) > (1ull << 31))
        return set_error(FX_E_ARG, "cloud bounding box above 2^31 cells");
    const int w = (int)(x1 - x0 + 1), h = (int)(y1 - y0 + 1);
    std::vector<uint16_t> I((size_t)w * h, 0), L((size_t)w * h, 0);
    for (size_t i = 0; i < n; ++i) {
        const size_t k = (size_t)(ys[i] - y0) * w + (xs[i] - x0);
        if (L[k])  // each pixel once (fx_roi_features_batch)
            return set_error(FX_E_ARG, "duplicate pixel (" + std::to_string(xs[i]) + ", " +
                                           std::to_string(ys[i]) + ") in cloud");
        I[k] = is[i];
        L[k] = 1;
    }
    fx_image im{I.data(), L.data(), w, h, (size_t)w, (int)x0, (int)y0, FX_MEM_HOST};
    uint32_t lab = 0;
    size_t nr = 0;
    rc = fx_featurize(c, &im, groups, p, &lab, out, 1, &nr);
    if (rc) return rc;
    if (nr != 1) return set_error(FX_E_INTERNAL, "rasterized cloud did not yield one ROI");
    return FX_OK;
}

int fx_roi_features_batch(fx_ctx* c, const uint32_t* xs, const uint32_t* ys, const uint16_t* is,
                          const size_t* offsets, size_t n_clouds, unsigned groups,
                          const fx_texture_params* p, double* out, size_t cap_rows) {
    if (!c || !p || !offsets || (n_clouds && !out)) return set_error(FX_E_ARG, "null argument");
    int rc = check_groups(groups);
    if (rc) return rc;
    const FeatCfg cfg = make_cfg(groups, *p);
    if (cap_rows < n_clouds) return set_error(FX_E_CAPACITY, "output rows < clouds");
    const size_t nc = (size_t)cfg.ncols;
    // each non-empty cloud becomes its own bbox image (label 1, origin at the bbox
    // corner), all of them in one fx_featurize_batch call
    std::vector<size_t> which;  // cloud of each image
    std::vector<std::vector<uint16_t>> rI, rL;
    std::vector<fx_image> ims;
    for (size_t k = 0; k < n_clouds; ++k) {
        const size_t a = offsets[k], b = offsets[k + 1];
        if (b < a) return set_error(FX_E_ARG, "offsets not ascending");
        if (a == b) {  // empty cloud: zeros (engine.cpp:138-209)
            std::fill(out + k * nc, out + (k + 1) * nc, 0.0);
            continue;
        }
        if (!xs || !ys || !is) return set_error(FX_E_ARG, "null argument");
        uint32_t x0 = xs[a], x1 = xs[a], y0 = ys[a], y1 = ys[a];
        for (size_t i = a; i < b; ++i) {
            x0 = std::min(x0, xs[i]);
            x1 = std::max(x1, xs[i]);
            y0 = std::min(y0, ys[i]);
            y1 = std::max(y1, ys[i]);
        }
        if ((uint64_t)(x1 - x0 + 1) * (uint64_t)(y1 - y0 + 1) > (1ull << 31))
            return set_error(FX_E_ARG, "cloud " + std::to_string(k) + ": bounding box above 2^31 cells");
        const int w = (int)(x1 - x0 + 1), h = (int)(y1 - y0 + 1);
        rI.emplace_back((size_t)w * h, (uint16_t)0);
        rL.emplace_back((size_t)w * h, (uint16_t)0);
        for (size_t i = a; i < b; ++i) {
            const size_t q = (size_t)(ys[i] - y0) * w + (xs[i] - x0);
            // a PixelCloud holds each pixel once (roi.cpp:76-117 builds it from a mask);
            // a repeated pixel would be counted once here and twice by the reference
            if (rL.back()[q])
                return set_error(FX_E_ARG, "cloud " + std::to_string(k) + ": duplicate pixel (" +
                                               std::to_string(xs[i]) + ", " + std::to_string(ys[i]) + ")");
            rI.back()[q] = is[i];
            rL.back()[q] = 1;
        }
        which.push_back(k);
        ims.push_back(fx_image{nullptr, nullptr, w, h, (size_t)w, (int)x0, (int)y0, FX_MEM_HOST});
    }
    if (which.empty()) return FX_OK;
    for (size_t j = 0; j < ims.size(); ++j) {  // raster storage is stable now
        ims[j].intensity = rI[j].data();
        ims[j].labels = rL[j].data();
    }
    std::vector<uint32_t> labs(which.size());
    std::vector<double> vals(which.size() * nc);
    std::vector<size_t> offs(which.size() + 1);
    rc = fx_featurize_batch(c, ims.data(), (int)ims.size(), groups, p, labs.data(), vals.data(),
                            which.size(), offs.data());
    if (rc) return rc;
    for (size_t j = 0; j < which.size(); ++j) {
        if (offs[j + 1] - offs[j] != 1)
            return set_error(FX_E_INTERNAL, "a rasterized cloud did not yield one ROI");
        std::copy(vals.begin() + offs[j] * nc, vals.begin() + (offs[j] + 1) * nc, out + which[j] * nc);
    }
    return FX_OK;
}

int fx_roi_table(fx_ctx* c, const fx_image* im, uint32_t* out_labels, uint64_t* out_count,
                 uint32_t* out_bbox, size_t cap, size_t* n_rois) {
    if (!c || !im || !n_rois) return set_error(FX_E_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    DevImage d;
    int rc = stage_image(c, im, &d);
    if (rc) return rc;
    RoiList rl = roi_list(c);
    cudaStream_t s = c->stream;
    const SlotMap m = single_map(d);
    rc = scan_stage(c, d, m, true);
    if (!rc) rc = compact_stage(c, m, 0u, 0xffffffffu, ~size_t(0), true);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const size_t nr = c->h_ctl->n_rois;
    *n_rois = nr;
    if (nr > cap) return set_error(FX_E_CAPACITY, "output capacity too small");
    if (!nr) return finish(c);
    std::vector<int32_t> x0(nr), y0(nr);
    std::vector<uint32_t> w(nr), h(nr);
    std::vector<unsigned long long> cnt(nr);
    CK(cudaMemcpy(out_labels, rl.label, nr * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(x0.data(), rl.gx, nr * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y0.data(), rl.gy, nr * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(w.data(), rl.w, nr * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.data(), rl.h, nr * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cnt.data(), rl.n, nr * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nr; ++i) {
        out_count[i] = cnt[i];
        out_bbox[4 * i + 0] = (uint32_t)x0[i];
        out_bbox[4 * i + 1] = (uint32_t)y0[i];
        out_bbox[4 * i + 2] = (uint32_t)x0[i] + w[i] - 1;
        out_bbox[4 * i + 3] = (uint32_t)y0[i] + h[i] - 1;
    }
    return finish(c);
}

int fx_roi_clouds(fx_ctx* c, const fx_image* im, uint32_t* out_labels, uint64_t* out_offsets,
                  uint32_t* out_bbox, size_t cap_rois, uint32_t* xs, uint32_t* ys, uint16_t* vs,
                  size_t cap_px, size_t* n_rois, size_t* n_px) {
    if (!c || !im || !n_rois || !n_px) return set_error(FX_E_ARG, "null argument");
    if (!im->intensity || !im->labels) return set_error(FX_E_ARG, "null raster");
    if (im->width < 1 || im->height < 1) return set_error(FX_E_PAIRING, "empty raster");
    *n_rois = *n_px = 0;
    CK(cudaSetDevice(c->device));
    DevImage d;
    int rc = stage_image(c, im, &d);
    if (rc) return rc;
    const SlotMap m = single_map(d);
    rc = scan_stage(c, d, m, true);
    if (!rc) rc = compact_stage(c, m, 0u, 0xffffffffu, ~size_t(0), true);
    if (rc) return rc;
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(Control), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const size_t nr = c->h_ctl->n_rois;
    RoiList rl = roi_list(c);
    std::vector<unsigned long long> cnt(nr), off(nr + 1, 0);
    if (nr) CK(cudaMemcpy(cnt.data(), rl.n, nr * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nr; ++i) off[i + 1] = off[i] + cnt[i];
    *n_rois = nr;
    *n_px = off[nr];
    if (!xs || !ys || !vs || !out_labels || !out_offsets || !out_bbox) return finish(c);  // size query
    if (nr > cap_rois || off[nr] > cap_px) return set_error(FX_E_CAPACITY, "cloud buffers too small");
    if (nr) {
        std::vector<int32_t> gx(nr), gy(nr);
        std::vector<uint32_t> w(nr), h(nr);
        CK(cudaMemcpy(out_labels, rl.label, nr * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(gx.data(), rl.gx, nr * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(gy.data(), rl.gy, nr * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(w.data(), rl.w, nr * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(h.data(), rl.h, nr * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < nr; ++i) {
            out_offsets[i] = off[i];
            out_bbox[4 * i + 0] = (uint32_t)gx[i];
            out_bbox[4 * i + 1] = (uint32_t)gy[i];
            out_bbox[4 * i + 2] = (uint32_t)gx[i] + w[i] - 1;
            out_bbox[4 * i + 3] = (uint32_t)gy[i] + h[i] - 1;
        }
        out_offsets[nr] = off[nr];
        const size_t np = off[nr];
        void* buf = nullptr;  // offsets | xs | ys | vs, device
        const size_t bytes = (nr + 1) * 8 + np * 10 + 64;
        CK(cudaMalloc(&buf, bytes));
        uint8_t* b = (uint8_t*)buf;
        unsigned long long* d_off = (unsigned long long*)b;
        uint32_t* d_x = (uint32_t*)(b + (nr + 1) * 8);
        uint32_t* d_y = d_x + np;
        uint16_t* d_v = (uint16_t*)(d_y + np);
        cudaError_t e = cudaMemcpyAsync(d_off, off.data(), (nr + 1) * 8, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
            Launch l(c, "k_cloud_gather");
            k_cloud_gather<<<std::max<int>(1, std::min<int>((int)((nr + 7) / 8), 8 * c->sm_count)), 256, 0, s>>>(
                d, rl, c->d_ctl, d_off, d_x, d_y, d_v);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(xs, d_x, np * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(ys, d_y, np * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(vs, d_v, np * 2, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(buf);
        if (e != cudaSuccess) return set_error(FX_E_CUDA, std::string("fx_roi_clouds: ") + cudaGetErrorString(e));
    }
    return finish(c);
}

int fx_debug_roi(fx_ctx* c, const fx_image* im, uint32_t label, const fx_texture_params* p,
                 uint64_t* hist, int32_t* edge_xy, size_t cap_edge, size_t* n_edge,
                 uint32_t* glcm_counts, uint64_t* glcm_pairs) {
    if (!c || !im || !p) return set_error(FX_E_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    unsigned groups = FX_GROUP_INTENSITY | FX_GROUP_GLCM;
    const FeatCfg cfg = make_cfg(groups, *p);
    int rc = validate_texture(groups, *p);
    if (rc) return rc;
    if (p->ng > kWideNg) return set_error(FX_E_CONFIG, "fx_debug_roi captures GLCM counts for ng <= 256");
    DevImage d;
    rc = stage_image(c, im, &d);
    if (rc) return rc;
    const int nb = cfg.bins, A = cfg.n_angles, ng = cfg.ng;
    DebugOut h{};
    h.label = label;
    h.nb = nb;
    h.cap_edge = (uint32_t)std::min<size_t>(cap_edge, 1u << 26);
    void* buf = nullptr;
    const size_t bytes = (size_t)nb * 8 + (size_t)h.cap_edge * 8 + 8 + (size_t)A * ng * ng * 4 + A * 8 + 64;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemsetAsync(buf, 0, bytes, c->stream));
    uint8_t* b = (uint8_t*)buf;
    h.hist = (unsigned long long*)b;
    b += (size_t)nb * 8;
    h.pairs = (unsigned long long*)b;
    b += (size_t)A * 8;
    h.n_edge = (uint32_t*)b;
    b += 8;
    h.edge_xy = (int32_t*)b;
    b += (size_t)h.cap_edge * 8;
    h.glcm = (uint32_t*)b;
    CK(cudaMemcpyAsync(c->d_dbg, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
    rc = ensure_out(c, (size_t)kMaxLabels * cfg.ncols);
    size_t nr = 0;
    if (!rc) rc = run_pipeline(c, d, groups, *p, c->d_out, kMaxLabels, &nr, c->d_dbg);
    if (!rc) rc = finish(c);
    if (!rc) {
        uint32_t ne = 0;
        cudaMemcpy(&ne, h.n_edge, 4, cudaMemcpyDeviceToHost);
        if (n_edge) *n_edge = ne;
        if (hist) cudaMemcpy(hist, h.hist, (size_t)nb * 8, cudaMemcpyDeviceToHost);
        if (edge_xy) cudaMemcpy(edge_xy, h.edge_xy, (size_t)std::min<uint32_t>(ne, h.cap_edge) * 8,
                                cudaMemcpyDeviceToHost);
        if (glcm_counts) cudaMemcpy(glcm_counts, h.glcm, (size_t)A * ng * ng * 4, cudaMemcpyDeviceToHost);
        if (glcm_pairs) cudaMemcpy(glcm_pairs, h.pairs, (size_t)A * 8, cudaMemcpyDeviceToHost);
    }
    cudaFree(buf);
    return rc;
}

}  // extern "C"
