/* TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
 *
 * fx_oracle: a plain-C CPU restatement of the reference featurex hot path
 * (label scan, intensity group incl. the Moore contour, moments, discretize +
 * GLCM + Haralick, column naming).  Used only by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the parity checker.  Every function cites
 * the reference file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity of this restatement is PINNED against the compiled reference
 * (oracle/_ref/libfxref.so, tests/test_oracle_pin.py) and against the golden
 * vectors of the reference's own unit tests (tests/golden/, tests/test_golden.py).
 */
#ifndef FX_ORACLE_H
#define FX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* group bits, canonical order (engine.cpp:22-23) */
#define FXO_INTENSITY 1u
#define FXO_SHAPE 2u
#define FXO_MOMENTS 4u
#define FXO_GLCM 8u
#define FXO_GLRLM 16u
#define FXO_GLSZM 32u
#define FXO_NGTDM 64u

typedef struct {
    int ng;
    int offset;
    int n_angles;
    int angles[8];
    int symmetric;
    int histogram_bins;
} fxo_params;

/* number of feature columns (feature_columns, engine.cpp:107-136) */
int fxo_n_cols(unsigned groups, const fxo_params* p);

/* RoiRegistry::accumulate + labels (roi.cpp:76-117): ascending labels, count, bbox. */
int fxo_roi_table(const uint16_t* labels, int w, int h, uint32_t* out_labels,
                  uint64_t* out_count, uint32_t* out_bbox, size_t cap, size_t* n);

/* in-memory engine path: accumulate + compute_roi_features per label
 * (engine.cpp:300-333, 138-209) for groups in {intensity, moments, glcm}. */
int fxo_featurize(const uint16_t* intensity, const uint16_t* labels, int w, int h,
                  unsigned groups, const fxo_params* p, uint32_t* out_labels,
                  double* out_values, size_t cap_rois, size_t* n_rois, int* n_cols);

/* compute_roi_features on one cloud (engine.cpp:138-209). */
int fxo_roi_features(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                     unsigned groups, const fxo_params* p, double* out, size_t cap,
                     int* n_cols);

/* trace_contour (contour.cpp:70-144): visit order, interleaved x,y. */
int fxo_trace_contour(const uint32_t* xs, const uint32_t* ys, size_t n, int32_t* out_xy,
                      size_t cap, size_t* n_points);

/* discretize + glcm raw counts (texture.cpp:29-85): counts[ng*ng], pair_count. */
int fxo_glcm_counts(const uint32_t* xs, const uint32_t* ys, const uint16_t* is, size_t n,
                    int ng, int offset, int angle, int symmetric, uint64_t* counts,
                    uint64_t* pair_count);

/* 256-bin (nb-bin) intensity histogram of intensity_features.cpp:156-167. */
int fxo_intensity_hist(const uint16_t* is, size_t n, int bins, uint64_t* hist);

const char* fxo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
