// Host-side packing of a (labels, intensities) row block for the H2D link.
//
// The per-ROI features read an intensity only where a label is set (the
// reference computes every feature from its PixelCloud, roi.cpp:76-117), and a
// label raster is runs of equal values.  A block of rows therefore crosses PCIe
// as two regions:
//   labels:      row_seg[rows + 1], then per row its label change points
//                seg = x | label << 16 (a segment runs to the next change point
//                or the row end; x = 0 always starts one);
//   intensities: row_pix[rows + 1], then the intensities of the labelled pixels
//                only, row-major.
// k_unpack_labels / k_unpack_intensity (fx_scan.cu) rebuild the rasters in HBM
// (intensity 0 where the label is 0).  The C2 image packs to ~35 MB instead of
// 268 MB.  The host passes are branch-free: 32 labels per step, change and
// nonzero masks by AVX-512 compares, VPCOMPRESSW appends (fx_pack.cpp).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#ifdef __CUDACC__
#define FXP_HD __host__ __device__
#else
#define FXP_HD
#endif

namespace fxg {

// Rows are indexed in tiles of kPackTile pixels (one 256-thread CTA of the
// unpack kernels, 8 pixels per thread): per (row, tile) the label region records
// the segment count before the tile and the intensity region the labelled-pixel
// count before it, so every tile unpacks on its own.
constexpr int kPackTile = 2048;
FXP_HD inline int pk_tiles(int width) { return (width + kPackTile - 1) / kPackTile; }
// region layouts (byte offsets); every array starts 16-byte aligned:
//   labels:      tile_seg[rows * tiles + 1] u32 | seg[nseg] u32 (x | label << 16)
//   intensities: tile_pix[rows * tiles + 1] u32 | pix[npix] u16
FXP_HD inline size_t pk_align16(size_t b) { return (b + 15) & ~(size_t)15; }
FXP_HD inline size_t pk_index_bytes(int rows, int width) {
    return pk_align16(4 * ((size_t)rows * (size_t)pk_tiles(width) + 1));
}
// capacity of a label region of `cap_seg` segments / an intensity region of
// `cap_pix` pixels, including the vector stores' slack
inline size_t pk_lab_bytes(int rows, int width, size_t cap_seg) {
    return pk_index_bytes(rows, width) + 4 * cap_seg + 128;
}
inline size_t pk_int_bytes(int rows, int width, size_t cap_pix) {
    return pk_index_bytes(rows, width) + 2 * cap_pix + 64;
}

// Labels of rows [y0, y1) (pitch in elements, width <= 65536) into a label region
// of capacity cap_seg segments, and the rows' nonzero masks (one bit per pixel,
// mask_pitch u32 words per row, rows from 0) for pack_intensity.  Returns the
// region bytes to send, or 0 when a row might not fit (send the block raw).
size_t pack_labels(const uint16_t* labels, size_t pitch, int width, int y0, int y1, uint8_t* region,
                   size_t cap_seg, uint32_t* mask, size_t mask_pitch);
// Intensities of the labelled pixels of rows [y0, y1) (mask from pack_labels)
// into an intensity region of capacity cap_pix pixels.  Returns the region bytes,
// or 0 when a row might not fit (send the block's intensities raw).
size_t pack_intensity(const uint16_t* intensity, size_t pitch, int width, int y0, int y1,
                      const uint32_t* mask, size_t mask_pitch, uint8_t* region, size_t cap_pix);

// 2: AVX-512 VBMI2 packers; 0: none on this host (the banded path sends raw rows)
int pack_isa();

// Persistent host workers for the packing tasks of one call: start() hands out
// task indices in order and returns at once; done(i) turns true when task i has
// finished (its writes visible); wait() returns when every task has.
class PackPool {
public:
    explicit PackPool(int nthreads);
    ~PackPool();
    int threads() const { return (int)workers_.size(); }
    void start(int ntasks, std::function<void(int)> fn);
    bool done(int i) const { return flags_[i].load(std::memory_order_acquire) != 0; }
    void wait();

private:
    void loop();
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, cv_done_;
    std::function<void(int)> fn_;
    std::vector<std::atomic<int>> flags_;
    std::atomic<int> next_{0};
    int ntasks_ = 0, remaining_ = 0, busy_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace fxg
