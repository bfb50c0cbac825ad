/*
 * fxg.h -- C ABI of the B200-native featurex hot path (libfxg.so).
 *
 * Drop-in boundary for the reference's featurize path (featurex, /root/reference/proj):
 * plain pointers and sizes only, no C++ or torch types.  Each entry point names
 * the reference interface it replaces (paths relative to /root/reference/proj).
 * The C++ host layer (include/featurex_gpu/engine.hpp) re-exposes the
 * reference's engine.hpp signatures on top of these calls.
 *
 * Conventions
 *  - Return value: FX_OK (0) or an fx_status code; fx_last_error() returns a
 *    thread-local message for the last failure on the calling thread.
 *  - Error codes map 1:1 onto the reference exception types
 *    (include/featurex/errors.hpp:8-58) plus device-side failures.
 *  - The caller owns every buffer.  The library never returns memory to free;
 *    device scratch belongs to the fx_ctx.
 *  - A fx_ctx is not thread-safe; distinct contexts on distinct host threads are.
 *  - There is no CPU fallback: every fx_featurize* call runs sm_100a kernels and
 *    fails with FX_E_CUDA when no usable device/kernel image is present.
 */
#ifndef FXG_H
#define FXG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FXG_ABI_VERSION 1

typedef enum fx_status {
    FX_OK = 0,
    FX_E_CONFIG = 1,          /* featurex::ConfigError    (errors.hpp:56-58) */
    FX_E_UNKNOWN_PROFILE = 2, /* featurex::UnknownProfile (errors.hpp:48-50) */
    FX_E_PAIRING = 3,         /* featurex::PairingError   (errors.hpp:16-18) */
    FX_E_IO = 4,              /* featurex::IoError        (errors.hpp:8-10)  */
    FX_E_FORMAT = 5,          /* featurex::FormatError    (errors.hpp:12-14) */
    FX_E_ZERO_MASS = 6,       /* featurex::ZeroMassError  (errors.hpp:24-26) */
    FX_E_CUDA = 7,            /* CUDA runtime / launch failure, no device     */
    FX_E_OOM = 8,             /* device or pinned allocation failed           */
    FX_E_NCCL = 9,            /* collective failure (sharded entry points)    */
    FX_E_CAPACITY = 10,       /* caller's output buffer too small             */
    FX_E_ARG = 11,            /* invalid argument (null pointer, bad size)    */
    FX_E_INTERNAL = 12
} fx_status;

typedef enum fx_mem_kind { FX_MEM_HOST = 0, FX_MEM_DEVICE = 1 } fx_mem_kind;

/* Feature group bits, canonical order of engine.cpp:22-23. */
#define FX_GROUP_INTENSITY 0x01u
#define FX_GROUP_SHAPE 0x02u
#define FX_GROUP_MOMENTS 0x04u
#define FX_GROUP_GLCM 0x08u
#define FX_GROUP_GLRLM 0x10u
#define FX_GROUP_GLSZM 0x20u
#define FX_GROUP_NGTDM 0x40u
#define FX_GROUP_ALL 0x7Fu
/* Groups with device kernels in this build (all seven). */
#define FX_GROUP_DEVICE FX_GROUP_ALL

/* TextureParams (engine.hpp:14-17) + GlcmParams (texture.hpp:30-35). */
typedef struct fx_texture_params {
    int ng;             /* grey levels; >= 2 (discretize, texture.cpp:30)       */
    int offset;         /* pixel distance d                                     */
    int n_angles;       /* number of entries used in angles[] (1..8)            */
    int angles[8];      /* each in {0,45,90,135}; columns use sorted order      */
    int symmetric;      /* count (b,a) with (a,b)                               */
    int histogram_bins; /* intensity entropy/uniformity bins, max(2, bins)      */
} fx_texture_params;

/* One image pair: row-major uint16 rasters.  pitch is in elements (>= width).
 * origin_x/origin_y are the global coordinates of pixel (0,0); raw moments and
 * weighted centroids are reported in global coordinates (a band shard or a
 * rasterized PixelCloud passes its offset here).  mem_kind says where the two
 * rasters live; outputs of fx_featurize live in the same kind of memory. */
typedef struct fx_image {
    const uint16_t* intensity;
    const uint16_t* labels;
    int width;
    int height;
    size_t pitch;
    int origin_x;
    int origin_y;
    int mem_kind;
} fx_image;

int fx_abi_version(void);
const char* fx_last_error(void);

/* ---- pure host helpers (no device) ------------------------------------- */

/* resolve_profile (engine.hpp:22, engine.cpp:71-86): "default",
 * "performance", "ibsi-like"; FX_E_UNKNOWN_PROFILE otherwise. */
int fx_resolve_profile(const char* name, fx_texture_params* out);

/* resolve_feature_groups (engine.hpp:60, engine.cpp:88-105): names
 * (incl. "*ALL*") -> canonical group bit mask; FX_E_CONFIG on empty/unknown. */
int fx_resolve_groups(const char* const* names, int n_names, unsigned* out_mask);

/* feature_columns (engine.hpp:64-65, engine.cpp:107-136): '\n'-joined names
 * into buf (may be NULL for a size query); *need = bytes incl. NUL. */
int fx_columns(unsigned groups, const fx_texture_params* params, char* buf, size_t cap,
               size_t* need, int* n_cols);

/* ---- device context ------------------------------------------------------ */

typedef struct fx_ctx fx_ctx;

int fx_ctx_create(int device, fx_ctx** out);
int fx_ctx_destroy(fx_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (NULL restores the ctx's own stream). */
int fx_ctx_set_stream(fx_ctx* ctx, void* cuda_stream);
/* Host rasters of fx_featurize move in row bands of this many rows (multiple of
 * 64), overlapping H2D, kernels and D2H; 0 = automatic (~8 bands for images of
 * >= 2048 rows and >= 8 Mpx, else unbanded), < 0 = never banded.  Results are
 * identical either way. */
int fx_ctx_set_band_rows(fx_ctx* ctx, int rows);
/* Banded host rasters cross PCIe packed (default on when the host has AVX-512
 * VBMI2 and width <= 65536): per row the label change points and only the
 * intensities of labelled pixels, packed by a pool of host threads and unpacked
 * on the device (the features never read an unlabelled pixel's intensity).
 * 0 sends raw rows.  Results are identical either way. */
int fx_ctx_set_packing(fx_ctx* ctx, int on);
/* Bytes the last fx_featurize call on host rasters moved host-to-device and
 * device-to-host (0 for device-resident calls). */
int fx_ctx_last_transfer(const fx_ctx* ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* Kernel launches issued by this ctx since creation (evidence counter). */
uint64_t fx_ctx_launch_count(const fx_ctx* ctx);
/* Optional per-kernel CUDA-event timing on the launching stream. */
int fx_ctx_enable_timing(fx_ctx* ctx, int enable);
/* Restrict timing to the kernel of this name (NULL or "" = every kernel): each
 * timing event between launches costs device time, so a timed region that must
 * not be perturbed times only the kernel it reports. */
int fx_ctx_timing_filter(fx_ctx* ctx, const char* kernel);
/* names: '\n'-joined kernel names; ms[i]: accumulated device ms; count[i]:
 * launches.  Returns the number of kernels in *n. */
int fx_ctx_kernel_times(fx_ctx* ctx, char* names, size_t names_cap, double* ms,
                        uint64_t* counts, int cap, int* n);
int fx_ctx_reset_kernel_times(fx_ctx* ctx);

/* Page-locked host memory for the input pipeline (decode straight into the
 * buffers the H2D copies read, so the copy engine runs at full rate and
 * overlaps the kernels).  No reference counterpart: the reference has no
 * device.  FX_E_OOM when the allocation fails. */
int fx_host_alloc(size_t bytes, void** out);
int fx_host_free(void* p);

/* ---- the hot path ---------------------------------------------------------- */

/* Replaces the per-pair body of featurex::run (engine.cpp:300-336):
 * RoiRegistry::accumulate (roi.cpp:76-110) + compute_roi_features
 * (engine.cpp:138-209) for every label.  Writes labels ascending into
 * out_labels[0..*n_rois) and the feature table row-major
 * [*n_rois x n_cols] in feature_columns order into out_values.  When the
 * table does not fit (cap_rois), *n_rois is set and FX_E_CAPACITY returned. */
int fx_featurize(fx_ctx* ctx, const fx_image* image, unsigned groups,
                 const fx_texture_params* params, uint32_t* out_labels, double* out_values,
                 size_t cap_rois, size_t* n_rois);

/* A batch of image pairs (the per-file loop of featurex::run, engine.cpp:300-336,
 * and the C4 tile stacks): every image is featurized exactly as by fx_featurize,
 * rows of image i are out_labels/out_values[row_offsets[i] .. row_offsets[i+1]).
 * All images share one mem_kind; outputs live in that kind of memory.  Images
 * are stacked in HBM and processed up to 128 per launch set (one label-table slot
 * each); device images that are already stacked in one pitched allocation
 * (heights multiple of 64, common pitch, contiguous) are read in place.  On
 * FX_E_CAPACITY, row_offsets[n] holds a lower bound of the rows needed. */
int fx_featurize_batch(fx_ctx* ctx, const fx_image* images, int n_images, unsigned groups,
                       const fx_texture_params* params, uint32_t* out_labels, double* out_values,
                       size_t cap_rois, size_t* row_offsets);

/* Convenience form of fx_featurize with origin (0,0). */
int fx_featurize_u16(fx_ctx* ctx, const uint16_t* intensity, const uint16_t* labels, int width,
                     int height, size_t pitch, int mem_kind, unsigned groups,
                     const fx_texture_params* params, uint32_t* out_labels,
                     double* out_values, size_t cap_rois, size_t* n_rois);

/* The per-ROI operator compute_roi_features(PixelCloud, groups, params)
 * (engine.hpp:68-70): host arrays of pixel x, y, intensity, each pixel once
 * (FX_E_ARG on a repeated pixel or a bounding box above 2^31 cells).  The cloud
 * is rasterized into its bbox window and run through the same device kernels (a
 * batch of one).  out receives n_cols values. */
int fx_roi_features(fx_ctx* ctx, const uint32_t* xs, const uint32_t* ys,
                    const uint16_t* intensities, size_t n, unsigned groups,
                    const fx_texture_params* params, double* out, size_t cap);

/* featurex::run (engine.hpp:77, engine.cpp:283-350) on PGM directories: pairs
 * by basename under `pattern`, featurizes every pair on `device` through the
 * batched pipeline of the C++ engine (include/featurex_gpu/engine.hpp) and
 * writes the sorted "%.10g" CSV.  groups_csv: comma-separated group names.
 * Per-pair failures are counted in failed_pairs, not returned. */
typedef struct fx_run_summary {
    int images;
    uint64_t rois;
    uint64_t rows;
    double elapsed_seconds;
    int failed_pairs;
} fx_run_summary;
int fx_run(const char* intensity_dir, const char* mask_dir, const char* pattern,
           const char* groups_csv, const char* profile, int threads, int parallel, int device,
           const char* output_path, fx_run_summary* out);

/* Many clouds at once (extension; the reference operator takes one cloud per
 * call): cloud k is pixels [offsets[k], offsets[k+1]) of xs / ys / intensities;
 * row k of out ([n_clouds x n_cols]) equals fx_roi_features on cloud k.  The
 * clouds run as one fx_featurize_batch (one bbox image each), so the per-call
 * launch and synchronisation cost is paid once. */
int fx_roi_features_batch(fx_ctx* ctx, const uint32_t* xs, const uint32_t* ys,
                          const uint16_t* intensities, const size_t* offsets, size_t n_clouds,
                          unsigned groups, const fx_texture_params* params, double* out,
                          size_t cap_rows);

/* ---- band sharding (C5: a whole slide split into row bands across GPUs) -----
 * 1. every rank: fx_scan_accumulate(own band, reset=1)  -> partial label table in
 *    GLOBAL coordinates (origin_x/origin_y of the band image);
 * 2. merge the partial tables across ranks (count: sum; xmin,ymin: min; xmax,ymax:
 *    max) -- fx_label_table_copy out, NCCL all-reduce, copy back in;
 * 3. every rank: fx_featurize_owned(band + halo rows, own rows [y0, y1)) -> rows of
 *    the ROIs whose first row lies in its band (the owner holds the whole window,
 *    so order statistics and the contour edge set need no merging).
 * Results are identical to fx_featurize on the whole image, for any band count. */
int fx_scan_accumulate(fx_ctx* ctx, const fx_image* band, int reset);
/* cnt: u64[65536]; bbox: u32[4][65536] = xmin | ymin | xmax | ymax (global coords).
 * to_ctx = 0 copies the ctx's table out, 1 loads it in.  mem_kind: the buffers. */
int fx_label_table_copy(fx_ctx* ctx, uint64_t* cnt, uint32_t* bbox, int to_ctx, int mem_kind);
int fx_featurize_owned(fx_ctx* ctx, const fx_image* image, int own_y0, int own_y1,
                       unsigned groups, const fx_texture_params* params, uint32_t* out_labels,
                       double* out_values, size_t cap_rois, size_t* n_rois);

/* Label scan only (RoiRegistry::accumulate + labels(), roi.cpp:76-117):
 * ascending labels, pixel counts and inclusive bboxes [xmin,ymin,xmax,ymax]
 * in image coordinates (origin added).  Host output buffers. */
int fx_roi_table(fx_ctx* ctx, const fx_image* image, uint32_t* out_labels, uint64_t* out_count,
                 uint32_t* out_bbox, size_t cap, size_t* n_rois);

/* RoiRegistry::accumulate + cloud (roi.cpp:76-148) on the device: every ROI's
 * pixel cloud, clouds in label order (ascending), each in mask scan order, (x, y)
 * with the image origin added.  offsets[n_rois + 1] index xs / ys / vs; bbox
 * [n_rois][4] = x_min, y_min, x_max, y_max.  With any output pointer NULL only
 * *n_rois / *n_px are returned (size query); FX_E_CAPACITY if a buffer is short. */
int fx_roi_clouds(fx_ctx* ctx, const fx_image* image, uint32_t* out_labels, uint64_t* offsets,
                  uint32_t* bbox, size_t cap_rois, uint32_t* xs, uint32_t* ys, uint16_t* vs,
                  size_t cap_px, size_t* n_rois, size_t* n_px);

/* Introspection of one ROI's integer intermediates, for the bit-exact tests:
 *  hist      : intensity histogram counts over max(2,bins) bins
 *              (intensity_features.cpp:156-167)                 [nb]
 *  edge_xy   : edge pixel set used by the edge_* columns, interleaved x,y in
 *              row-major order (== trace_contour's visited set)  [2*cap_edge]
 *  glcm      : raw co-occurrence counts per sorted angle, dense [A][ng][ng]
 *              (texture.cpp:58-80) and pair counts [A]
 * Any output pointer may be NULL.  All host buffers. */
int fx_debug_roi(fx_ctx* ctx, const fx_image* image, uint32_t label,
                 const fx_texture_params* params, uint64_t* hist, int32_t* edge_xy,
                 size_t cap_edge, size_t* n_edge, uint32_t* glcm_counts, uint64_t* glcm_pairs);

/* ---- several devices of this process ----------------------- */

typedef struct fx_multi fx_multi;
/* One fx_ctx and one host thread per listed device (a device may be listed more
 * than once: several contexts share it). */
int fx_multi_create(const int* devices, int n_devices, fx_multi** out);
int fx_multi_destroy(fx_multi* m);
int fx_multi_device_count(const fx_multi* m);
/* The i-th device's context (owned by m), e.g. for fx_ctx_set_band_rows. */
fx_ctx* fx_multi_ctx(fx_multi* m, int i);
/* C4 across devices: the batch is cut into chunks (up to 512 images, at least
 * one chunk per device when the batch allows), chunk j
 * runs on device j mod N through the fx_featurize_batch pipeline, and rows come
 * back straight into their place: output identical to fx_featurize_batch (rows in
 * input order, row_offsets[n+1]).  Host images only when N > 1. */
int fx_multi_featurize_batch(fx_multi* m, const fx_image* images, int n, unsigned groups,
                             const fx_texture_params* params, uint32_t* out_labels,
                             double* out_values, size_t cap_rois, size_t* row_offsets);
/* C5 across devices: one host image in row bands, one band per device.  Each
 * device scans its band; the label tables are merged by peer reads (NVLink);
 * a ROI belongs to the band of its first row, and an owner gathers only its
 * straddling windows' rectangles from the other bands (peer reads) before
 * featurizing its ROIs.  Output identical to fx_featurize on the whole image
 * (labels ascending).  Bands are whole 64-row strips: an image of fewer strips
 * than devices uses its first max(1, height / 64) devices.  Replaces the
 * per-pair body of run() (engine.cpp:300-336) for one image too large for one
 * device's pass. */
int fx_multi_featurize_slide(fx_multi* m, const fx_image* image, unsigned groups,
                             const fx_texture_params* params, uint32_t* out_labels,
                             double* out_values, size_t cap_rois, size_t* n_rois);

/* Per-phase clock totals of the S-class ROI kernels (summed over ROIs, lane 0's
 * clock64 deltas): 0 load+gather, 1 intensity sort, 2 intensity statistics,
 * 3 edge set + edge statistics, 4 moments, 5 GLCM levels+pair keys, 6 GLCM key
 * sort, 7 GLCM run-length counts, 8 Haralick.  Only in builds with
 * -DFXG_PHASE_TIMING (tools/); others return FX_E_CONFIG. */
int fx_debug_phase_clocks(unsigned long long* out, int n, int reset);
/* Host packer of the packed host rows (fx_ctx_set_packing), for tests: packs
 * `rows` rows of width `width` (pitch in elements) into a label region of
 * lab_cap bytes and an intensity region of int_cap bytes, in the layout the
 * device unpacks (csrc/fx_pack.hpp).  *lab_bytes / *int_bytes receive the bytes
 * used (0: does not fit, the block goes raw).  FX_E_CONFIG when this host has no
 * AVX-512 VBMI2 (packing is then off). */
int fx_debug_pack_rows(const uint16_t* labels, const uint16_t* intensity, size_t pitch, int width,
                       int rows, uint8_t* lab_region, size_t lab_cap, uint8_t* int_region,
                       size_t int_cap, size_t* lab_bytes, size_t* int_bytes);
/* Same for the GLRLM/GLSZM/NGTDM kernel (thread 0 per ROI): 0 discretize,
 * 1 GLRLM (other), 2 GLSZM, 3 NGTDM, 4 GLRLM run counting, 5 GLRLM features. */
int fx_debug_texture_clocks(unsigned long long* out, int n, int reset);


#ifdef __cplusplus
}
#endif
#endif /* FXG_H */
