// Host packing of row blocks (fx_pack.hpp) and the worker pool that runs it.
#include "fx_pack.hpp"

#include <immintrin.h>

#include <cstring>

namespace fxg {

namespace {

bool have_vbmi2() {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
           __builtin_cpu_supports("avx512vbmi2");
}

#define FXP_TARGET __attribute__((target("avx512f,avx512bw,avx512vbmi2,avx512vl,popcnt")))

// 32 labels per step: change mask (label != left neighbour; x = 0 always a
// change) and nonzero mask; the change positions and labels are compressed in
// registers, interleaved into u32 segments and stored whole (the region has
// 128 B of slack past its capacity).
FXP_TARGET size_t pack_labels_vbmi2(const uint16_t* labels, size_t pitch, uint32_t w, int y0, int y1,
                                    uint8_t* region, size_t cap_seg, uint32_t* mask, size_t mp) {
    const int rows = y1 - y0, tiles = pk_tiles((int)w);
    uint32_t* tile_seg = reinterpret_cast<uint32_t*>(region);
    uint32_t* seg = reinterpret_cast<uint32_t*>(region + pk_index_bytes(rows, (int)w));
    const __m512i iota = _mm512_set_epi16(31, 30, 29, 28, 27, 26, 25, 24, 23, 22, 21, 20, 19, 18, 17,
                                          16, 15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0);
    // (x_i, label_i) pairs: output lane 2i <- x_i, 2i+1 <- label_i (index 32 + i)
    const __m512i ilo = _mm512_set_epi16(47, 15, 46, 14, 45, 13, 44, 12, 43, 11, 42, 10, 41, 9, 40, 8,
                                         39, 7, 38, 6, 37, 5, 36, 4, 35, 3, 34, 2, 33, 1, 32, 0);
    const __m512i ihi = _mm512_set_epi16(63, 31, 62, 30, 61, 29, 60, 28, 59, 27, 58, 26, 57, 25, 56, 24,
                                         55, 23, 54, 22, 53, 21, 52, 20, 51, 19, 50, 18, 49, 17, 48, 16);
    const __m512i zero = _mm512_setzero_si512();
    size_t ns = 0;
    for (int y = y0; y < y1; ++y) {
        if (ns + w > cap_seg) return 0;
        const uint16_t* l = labels + (size_t)y * pitch;
        uint32_t* mrow = mask + (size_t)(y - y0) * mp;
        uint32_t* ts = tile_seg + (size_t)(y - y0) * tiles;
        for (uint32_t x = 0; x < w; x += 32) {
            if (!(x & (kPackTile - 1))) ts[x / kPackTile] = (uint32_t)ns;
            const uint32_t left = w - x;
            const __mmask32 k = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
            const __m512i a = _mm512_maskz_loadu_epi16(k, l + x);
            // left neighbours (masked: lane 0 of the row reads nothing)
            const __m512i b = _mm512_maskz_loadu_epi16(x ? k : (k & ~1u), l + x - 1);
            const __mmask32 chg = _mm512_mask_cmpneq_epi16_mask(k, a, b) | (x ? 0u : 1u);
            mrow[x >> 5] = (uint32_t)_mm512_mask_cmpneq_epi16_mask(k, a, zero);
            const __m512i pos = _mm512_add_epi16(iota, _mm512_set1_epi16((short)x));
            const __m512i cp = _mm512_maskz_compress_epi16(chg, pos);
            const __m512i cl = _mm512_maskz_compress_epi16(chg, a);
            _mm512_storeu_si512(seg + ns, _mm512_permutex2var_epi16(cp, ilo, cl));
            _mm512_storeu_si512(seg + ns + 16, _mm512_permutex2var_epi16(cp, ihi, cl));
            ns += (size_t)_mm_popcnt_u32(chg);
        }
    }
    tile_seg[(size_t)rows * tiles] = (uint32_t)ns;
    return pk_index_bytes(rows, (int)w) + 4 * ns;
}

FXP_TARGET size_t pack_intensity_vbmi2(const uint16_t* intensity, size_t pitch, uint32_t w, int y0,
                                       int y1, const uint32_t* mask, size_t mp, uint8_t* region,
                                       size_t cap_pix) {
    const int rows = y1 - y0, tiles = pk_tiles((int)w);
    uint32_t* tile_pix = reinterpret_cast<uint32_t*>(region);
    uint16_t* pix = reinterpret_cast<uint16_t*>(region + pk_index_bytes(rows, (int)w));
    size_t np = 0;
    for (int y = y0; y < y1; ++y) {
        if (np + w > cap_pix) return 0;
        const uint16_t* iv = intensity + (size_t)y * pitch;
        const uint32_t* mrow = mask + (size_t)(y - y0) * mp;
        uint32_t* tp = tile_pix + (size_t)(y - y0) * tiles;
        for (uint32_t x = 0; x < w; x += 32) {
            if (!(x & (kPackTile - 1))) tp[x / kPackTile] = (uint32_t)np;
            const __mmask32 m = mrow[x >> 5];
            if (!m) continue;  // no intensity of this word is read
            const __m512i v = _mm512_maskz_loadu_epi16(m, iv + x);
            _mm512_storeu_si512(pix + np, _mm512_maskz_compress_epi16(m, v));
            np += (size_t)_mm_popcnt_u32(m);
        }
    }
    tile_pix[(size_t)rows * tiles] = (uint32_t)np;
    return pk_index_bytes(rows, (int)w) + 2 * np;
}

}  // namespace

int pack_isa() {
    static const int isa = have_vbmi2() ? 2 : 0;
    return isa;
}

size_t pack_labels(const uint16_t* labels, size_t pitch, int width, int y0, int y1, uint8_t* region,
                   size_t cap_seg, uint32_t* mask, size_t mask_pitch) {
    if (pack_isa() != 2 || width > 65536) return 0;
    return pack_labels_vbmi2(labels, pitch, (uint32_t)width, y0, y1, region, cap_seg, mask, mask_pitch);
}

size_t pack_intensity(const uint16_t* intensity, size_t pitch, int width, int y0, int y1,
                      const uint32_t* mask, size_t mask_pitch, uint8_t* region, size_t cap_pix) {
    if (pack_isa() != 2 || width > 65536) return 0;
    return pack_intensity_vbmi2(intensity, pitch, (uint32_t)width, y0, y1, mask, mask_pitch, region,
                                cap_pix);
}

// ---------------------------------------------------------------- pool ----

PackPool::PackPool(int nthreads) {
    for (int t = 0; t < nthreads; ++t) workers_.emplace_back([this] { loop(); });
}

PackPool::~PackPool() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void PackPool::start(int ntasks, std::function<void(int)> fn) {
    wait();
    std::lock_guard<std::mutex> g(mu_);
    if ((int)flags_.size() < ntasks) flags_ = std::vector<std::atomic<int>>(ntasks);
    for (int i = 0; i < ntasks; ++i) flags_[i].store(0, std::memory_order_relaxed);
    fn_ = std::move(fn);
    ntasks_ = remaining_ = ntasks;
    next_.store(0, std::memory_order_relaxed);
    ++gen_;
    cv_.notify_all();
}

void PackPool::wait() {
    std::unique_lock<std::mutex> g(mu_);
    // every task done and every worker back from the claim loop (a worker still
    // claiming with the old task count must not see the next generation)
    cv_done_.wait(g, [this] { return remaining_ == 0 && busy_ == 0; });
}

void PackPool::loop() {
    uint64_t seen = 0;
    for (;;) {
        int n;
        {
            std::unique_lock<std::mutex> g(mu_);
            cv_.wait(g, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            n = ntasks_;
            ++busy_;
        }
        int finished = 0;
        for (int i; (i = next_.fetch_add(1, std::memory_order_relaxed)) < n;) {
            fn_(i);
            flags_[i].store(1, std::memory_order_release);
            ++finished;
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            remaining_ -= finished;
            --busy_;
            if (remaining_ == 0 && busy_ == 0) cv_done_.notify_all();
        }
    }
}

}  // namespace fxg
