// Several devices of one process: one fx_ctx and one host
// thread per device.
//
// fx_multi_featurize_batch (C4: independent images).  The reference runs its
// pairs one after another (engine.cpp:298-333); here the batch is cut into
// chunks of up to 512 images (one launch set of label-table slots), chunk j goes
// to device j mod N, and every device runs its chunks through the same sub-batch
// pipeline as fx_featurize_batch into device-resident rows.  Rows must come out
// in input order, so a chunk's first output row is the sum of the row counts of
// the chunks before it: each device publishes its chunk's count as soon as the
// compaction has produced it (well before the kernels finish), waits for the
// counts of the earlier chunks, then reads its rows back straight into their
// final place on its own copy stream.  Devices never wait on each other's
// kernels, only on earlier chunks' ROI counts; no collective is needed.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fx_dev.cuh"
#include "fx_host.hpp"
#include "fxg.h"

namespace fxg {
int ictx_validate_batch(const fx_image* ims, int n, size_t* row_offsets);
int ictx_check_groups(unsigned groups);
int ictx_ncols(unsigned groups, const fx_texture_params& p);
int ictx_batch_device(fx_ctx* c, const fx_image* ims, int n, unsigned groups,
                      const fx_texture_params* p, double* out_dev, uint32_t* lab_dev,
                      size_t cap_rows, size_t* row_offsets);
cudaStream_t ictx_stream(fx_ctx* c);
cudaStream_t ictx_d2h(fx_ctx* c);
int ictx_device(const fx_ctx* c);
int ictx_finish(fx_ctx* c);
int islide_load_scan(fx_ctx* c, const fx_image* im, int y0, int y1, int reserve,
                     cudaEvent_t loaded, cudaEvent_t scanned, uint32_t* lmax);
void islide_band(fx_ctx* c, const uint16_t** L, const uint16_t** I, size_t* pitch,
                 const unsigned long long** cnt, const uint32_t** bb, size_t* bb_pitch);
int islide_merge(fx_ctx* c, const TablePeers& tp, uint32_t lmax, const cudaEvent_t* scanned,
                 cudaEvent_t merged);
int islide_commit(fx_ctx* c, uint32_t lmax, const cudaEvent_t* merged, int n_peers,
                  uint64_t* h_cnt, uint32_t* h_bb);
int islide_featurize(fx_ctx* c, const fx_image* im, int y0, int y1, int need,
                     const std::vector<HaloRect>& rects, const std::vector<const uint16_t*>& pL,
                     const std::vector<const uint16_t*>& pI, const std::vector<size_t>& pp,
                     const std::vector<int>& py0, const cudaEvent_t* loaded, unsigned groups,
                     const fx_texture_params& p, size_t cap, uint32_t* h_labels, double* h_values,
                     size_t* n_rois);
}  // namespace fxg

using namespace fxg;

namespace {

constexpr int kChunkImages = 512;  // = one launch set of table slots (fx_capi.cu)

// per-device output rows of one chunk, double-buffered across a device's chunks
struct DevBufs {
    double* vals[2] = {nullptr, nullptr};
    uint32_t* labs[2] = {nullptr, nullptr};
    size_t cap[2] = {0, 0};  // rows
    cudaEvent_t drained[2] = {nullptr, nullptr};  // readback of the buffer's last chunk done
};

}  // namespace

struct fx_multi {
    std::vector<int> devices;
    std::vector<fx_ctx*> ctx;
    std::vector<DevBufs> bufs;
    // slide: per device, events on its own device: band loaded, scanned, table merged
    std::vector<cudaEvent_t> ev_loaded, ev_scanned, ev_merged;
};

namespace {

#define MCK(x)                                                                      \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess)                                                      \
            return set_error(e_ == cudaErrorMemoryAllocation ? FX_E_OOM : FX_E_CUDA, \
                             std::string(#x) + ": " + cudaGetErrorString(e_));     \
    } while (0)

int ensure_buf(DevBufs& b, int k, size_t rows, int ncols) {
    if (rows <= b.cap[k]) return FX_OK;
    cudaFree(b.vals[k]);
    cudaFree(b.labs[k]);
    b.vals[k] = nullptr;
    b.labs[k] = nullptr;
    b.cap[k] = 0;
    rows = std::max<size_t>(rows, 1024);
    MCK(cudaMalloc(&b.vals[k], rows * (size_t)std::max(ncols, 1) * sizeof(double)));
    MCK(cudaMalloc(&b.labs[k], rows * sizeof(uint32_t)));
    b.cap[k] = rows;
    return FX_OK;
}

// counts of the chunks' rows, published as they become known
struct Ledger {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<long long> rows;  // -1 unknown, -2 failed
    explicit Ledger(size_t n) : rows(n, -1) {}
    void publish(size_t j, long long v) {
        {
            std::lock_guard<std::mutex> g(mu);
            rows[j] = v;
        }
        cv.notify_all();
    }
    // sum of rows[0..j); -1 if an earlier chunk failed
    long long base(size_t j) {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] {
            for (size_t i = 0; i < j; ++i)
                if (rows[i] == -1) return false;
            return true;
        });
        long long s = 0;
        for (size_t i = 0; i < j; ++i) {
            if (rows[i] < 0) return -1;
            s += rows[i];
        }
        return s;
    }
};

}  // namespace

extern "C" {

int fx_multi_create(const int* devices, int n_devices, fx_multi** out) {
    if (!out || !devices || n_devices < 1) return set_error(FX_E_ARG, "null argument");
    *out = nullptr;
    fx_multi* m = new fx_multi();
    for (int i = 0; i < n_devices; ++i) {
        fx_ctx* c = nullptr;
        const int rc = fx_ctx_create(devices[i], &c);
        if (rc) {
            fx_multi_destroy(m);
            return rc;
        }
        m->devices.push_back(devices[i]);
        m->ctx.push_back(c);
        m->bufs.emplace_back();
        DevBufs& b = m->bufs.back();
        cudaSetDevice(devices[i]);
        for (int k = 0; k < 2; ++k)
            if (cudaEventCreateWithFlags(&b.drained[k], cudaEventDisableTiming) != cudaSuccess) {
                fx_multi_destroy(m);
                return set_error(FX_E_CUDA, "cudaEventCreate failed");
            }
        cudaEvent_t e[3];
        for (cudaEvent_t& x : e)
            if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) {
                fx_multi_destroy(m);
                return set_error(FX_E_CUDA, "cudaEventCreate failed");
            }
        m->ev_loaded.push_back(e[0]);
        m->ev_scanned.push_back(e[1]);
        m->ev_merged.push_back(e[2]);
    }
    // peer access between distinct devices (the slide's table merge and halo
    // gather read the other bands' memory over NVLink)
    for (int i = 0; i < n_devices; ++i)
        for (int j = 0; j < n_devices; ++j) {
            if (devices[i] == devices[j]) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]);
            if (!ok) {
                fx_multi_destroy(m);
                return set_error(FX_E_CUDA, "no peer access between devices " +
                                                std::to_string(devices[i]) + " and " + std::to_string(devices[j]));
            }
            cudaSetDevice(devices[i]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                fx_multi_destroy(m);
                return set_error(FX_E_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
            }
            cudaGetLastError();
        }
    *out = m;
    return FX_OK;
}

int fx_multi_destroy(fx_multi* m) {
    if (!m) return FX_OK;
    for (size_t d = 0; d < m->ctx.size(); ++d) {
        cudaSetDevice(m->devices[d]);
        fx_ctx_destroy(m->ctx[d]);
        DevBufs& b = m->bufs[d];
        for (int k = 0; k < 2; ++k) {
            cudaFree(b.vals[k]);
            cudaFree(b.labs[k]);
            if (b.drained[k]) cudaEventDestroy(b.drained[k]);
        }
    }
    for (auto* v : {&m->ev_loaded, &m->ev_scanned, &m->ev_merged})
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
    delete m;
    return FX_OK;
}

int fx_multi_device_count(const fx_multi* m) { return m ? (int)m->ctx.size() : 0; }

fx_ctx* fx_multi_ctx(fx_multi* m, int i) {
    return (m && i >= 0 && i < (int)m->ctx.size()) ? m->ctx[i] : nullptr;
}

int fx_multi_featurize_batch(fx_multi* m, const fx_image* ims, int n, unsigned groups,
                             const fx_texture_params* p, uint32_t* out_labels, double* out_values,
                             size_t cap_rois, size_t* row_offsets) {
    if (!m || (n && !ims) || !p || !row_offsets || n < 0) return set_error(FX_E_ARG, "null argument");
    row_offsets[0] = 0;
    if (n == 0) return FX_OK;
    int rc = ictx_validate_batch(ims, n, row_offsets);
    if (!rc) rc = ictx_check_groups(groups);
    if (rc) return rc;
    if (n > 0 && (!out_values || !out_labels)) return set_error(FX_E_ARG, "null output");
    const int kind = ims[0].mem_kind;
    const cudaMemcpyKind back = kind == FX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (kind == FX_MEM_DEVICE && m->ctx.size() > 1)
        return set_error(FX_E_ARG, "device-resident batches live on one device: use fx_featurize_batch");
    const int nc = ictx_ncols(groups, *p);
    const int N = (int)m->ctx.size();
    // chunks of up to one launch set, at least one per device when the batch allows
    const int chunk = std::max(1, std::min(kChunkImages, (n + N - 1) / N));
    const size_t n_chunks = ((size_t)n + chunk - 1) / chunk;
    Ledger ledger(n_chunks);
    double total_px = 0;
    for (int i = 0; i < n; ++i) total_px += (double)ims[i].width * ims[i].height;
    std::vector<int> status(N, FX_OK);
    std::vector<std::string> errs(N);
    auto worker = [&](int d) {
        fx_ctx* c = m->ctx[d];
        DevBufs& B = m->bufs[d];
        cudaSetDevice(m->devices[d]);
        // whatever path leaves the worker, no copy into the caller's buffers is
        // still in flight when the call returns
        struct Drain {
            fx_ctx* c;
            ~Drain() {
                cudaStreamSynchronize(ictx_d2h(c));
                cudaStreamSynchronize(ictx_stream(c));
            }
        } drain{c};
        int use = 0;
        bool ran = false;  // finish() reads this call's control block: only after work
        for (size_t j = (size_t)d; j < n_chunks; j += N, use ^= 1) {
            ran = true;
            const int first = (int)(j * chunk), cnt = std::min(chunk, n - first);
            // rows of this chunk: guess from its pixel share of cap_rois, grow on overflow
            double px = 0;
            for (int i = first; i < first + cnt; ++i) px += (double)ims[i].width * ims[i].height;
            size_t cap = (size_t)(1.25 * (double)cap_rois * px / std::max(total_px, 1.0)) + 4096;
            cap = std::min(cap, std::max<size_t>(cap_rois, 1));
            std::vector<size_t> offs((size_t)cnt + 1, 0);
            int r = FX_OK;
            for (int attempt = 0; attempt < 8; ++attempt) {
                r = ensure_buf(B, use, cap, nc);
                // the buffer's previous chunk must have left the device
                if (!r && cudaStreamWaitEvent(ictx_stream(c), B.drained[use], 0) != cudaSuccess)
                    r = set_error(FX_E_CUDA, "cudaStreamWaitEvent failed");
                if (!r)
                    r = ictx_batch_device(c, ims + first, cnt, groups, p, B.vals[use], B.labs[use], cap,
                                          offs.data());
                if (r != FX_E_CAPACITY || cap >= cap_rois) break;
                // rows needed so far (the failing sub-batch included): grow, rerun the chunk
                cap = std::min<size_t>(std::max<size_t>(cap_rois, 1), std::max(offs[cnt], 2 * cap));
            }
            if (r) {
                status[d] = r;
                errs[d] = fx_last_error();
                ledger.publish(j, -2);
                // later chunks of this device never run: publish them as failed
                for (size_t k = j + N; k < n_chunks; k += N) ledger.publish(k, -2);
                return;
            }
            const size_t rows = offs[cnt];
            ledger.publish(j, (long long)rows);
            const long long base = ledger.base(j);
            if (base < 0) {  // an earlier chunk failed
                for (size_t k = j + N; k < n_chunks; k += N) ledger.publish(k, -2);
                return;
            }
            if ((size_t)base + rows > cap_rois) {
                status[d] = set_error(FX_E_CAPACITY, "output capacity " + std::to_string(cap_rois) +
                                                         " < " + std::to_string(base + rows) + " ROIs");
                errs[d] = fx_last_error();
                for (size_t k = j + N; k < n_chunks; k += N) ledger.publish(k, -2);
                return;
            }
            for (int t = 0; t < cnt; ++t) row_offsets[first + t] = (size_t)base + offs[t];
            cudaEvent_t done = B.drained[use];
            cudaStream_t s = ictx_stream(c), cp = ictx_d2h(c);
            if (rows) {
                cudaEventRecord(done, s);
                cudaStreamWaitEvent(cp, done, 0);
                cudaMemcpyAsync(out_values + (size_t)base * nc, B.vals[use], rows * nc * sizeof(double), back, cp);
                cudaMemcpyAsync(out_labels + base, B.labs[use], rows * sizeof(uint32_t), back, cp);
            }
            cudaEventRecord(done, cp);
        }
        if (!ran) return;
        if (cudaStreamSynchronize(ictx_d2h(c)) != cudaSuccess)
            status[d] = set_error(FX_E_CUDA, "readback failed");
        const int f = ictx_finish(c);
        if (f && !status[d]) {
            status[d] = f;
            errs[d] = fx_last_error();
        }
    };
    std::vector<std::thread> th;
    for (int d = 1; d < N; ++d) th.emplace_back(worker, d);
    worker(0);
    for (auto& t : th) t.join();
    for (int d = 0; d < N; ++d)
        if (status[d]) return set_error(status[d], errs[d].empty() ? "device " + std::to_string(d) + " failed" : errs[d]);
    size_t total = 0;
    for (size_t j = 0; j < n_chunks; ++j) total += (size_t)ledger.rows[j];
    row_offsets[n] = total;
    return FX_OK;
}


// C5 across devices: one host slide in row bands, one band per device.
//   1. every device loads its band (H2D) and scans it into its own label table;
//   2. every device merges the tables of all bands by peer reads (k_table_merge:
//      counts summed, boxes min / max, labels [0, lmax]) and commits the result:
//      each ends with the table of the whole slide, bit for bit;
//   3. a ROI belongs to the band holding its first row; an owner whose ROIs run
//      below its band gathers just those windows' rectangles from the bands that
//      hold them (k_halo_gather, peer reads) -- only straddling ROIs move, not
//      whole rows -- and featurizes its ROIs on band + halo;
//   4. the bands' rows (labels ascending each) are merged by label.
// Every statistic is computed by one device over the ROI's complete window, so
// the table equals fx_featurize on the whole slide for any number of devices.
int fx_multi_featurize_slide(fx_multi* m, const fx_image* im, unsigned groups,
                             const fx_texture_params* p, uint32_t* out_labels, double* out_values,
                             size_t cap_rois, size_t* n_rois) {
    if (!m || !im || !p || !n_rois) return set_error(FX_E_ARG, "null argument");
    *n_rois = 0;
    if (!im->intensity || !im->labels) return set_error(FX_E_ARG, "null raster");
    if (im->width < 1 || im->height < 1) return set_error(FX_E_PAIRING, "empty raster");
    if (im->pitch && im->pitch < (size_t)im->width) return set_error(FX_E_ARG, "pitch < width");
    if (im->mem_kind != FX_MEM_HOST) return set_error(FX_E_ARG, "the slide is read from host memory");
    int rc = ictx_check_groups(groups);
    if (rc) return rc;
    if ((int)m->ctx.size() > kMaxPeers) return set_error(FX_E_ARG, "at most 16 devices per slide");
    const int H = im->height;
    // bands of whole 64-row strips (the last one takes the remainder); a slide of
    // fewer strips than devices runs on its first H / 64 devices (at least one)
    const int N = std::min((int)m->ctx.size(), std::max(1, H / 64));
    const int nc = ictx_ncols(groups, *p);
    std::vector<int> y0(N), y1(N);
    for (int d = 0; d < N; ++d) {
        y0[d] = (int)((long long)H * d / N) / 64 * 64;
        y1[d] = d == N - 1 ? H : (int)((long long)H * (d + 1) / N) / 64 * 64;
    }
    for (int d = 0; d < N; ++d)
        if (y1[d] <= y0[d]) return set_error(FX_E_INTERNAL, "empty slide band");
    std::vector<int> status(N, FX_OK);
    std::vector<std::string> errs(N);
    auto parallel = [&](auto&& fn) {  // fn(d) on one host thread per device
        std::vector<std::thread> th;
        for (int d = 0; d < N; ++d)
            th.emplace_back([&, d] {
                cudaSetDevice(m->devices[d]);
                const int r = fn(d);
                if (r && !status[d]) {
                    status[d] = r;
                    errs[d] = fx_last_error();
                }
            });
        for (auto& t : th) t.join();
        for (int d = 0; d < N; ++d)
            if (status[d]) {
                // the other devices may still read the caller's slide (H2D): drain them
                for (int e = 0; e < N; ++e) {
                    cudaSetDevice(m->devices[e]);
                    cudaStreamSynchronize(ictx_stream(m->ctx[e]));
                }
                return set_error(status[d], errs[d]);
            }
        return (int)FX_OK;
    };
    // 1. load + scan
    std::vector<uint32_t> lmax(N, 0);
    rc = parallel([&](int d) {
        const int reserve = std::min(H - y1[d], std::max(256, (y1[d] - y0[d]) / 4));
        return islide_load_scan(m->ctx[d], im, y0[d], y1[d], reserve, m->ev_loaded[d], m->ev_scanned[d],
                                &lmax[d]);
    });
    if (rc) return rc;
    const uint32_t L = *std::max_element(lmax.begin(), lmax.end());
    if (L == 0) return FX_OK;  // no labelled pixel
    // 2. merge by peer reads, commit
    TablePeers tp{};
    tp.n = N;
    std::vector<const uint16_t*> pL(N), pI(N);
    std::vector<size_t> pp(N);
    for (int d = 0; d < N; ++d)
        islide_band(m->ctx[d], &pL[d], &pI[d], &pp[d], &tp.cnt[d], &tp.bb[d], &tp.pitch[d]);
    std::vector<uint64_t> cnt((size_t)L + 1);
    std::vector<uint32_t> bb(4 * ((size_t)L + 1));
    rc = parallel([&](int d) {
        int r = islide_merge(m->ctx[d], tp, L, m->ev_scanned.data(), m->ev_merged[d]);
        return r;
    });
    if (rc) return rc;
    rc = parallel([&](int d) {
        std::vector<uint64_t> c2;
        std::vector<uint32_t> b2;
        if (d) {  // every device commits; device 0's copy feeds the plan
            c2.resize(cnt.size());
            b2.resize(bb.size());
        }
        return islide_commit(m->ctx[d], L, m->ev_merged.data(), N, d ? c2.data() : cnt.data(),
                             d ? b2.data() : bb.data());
    });
    if (rc) return rc;
    // 3. ownership (first row) and the straddling rectangles per owner
    const size_t nl = (size_t)L + 1;
    const long long oy = im->origin_y, ox = im->origin_x;
    std::vector<int> need(N, 0);
    std::vector<size_t> owned(N, 0);
    std::vector<std::vector<HaloRect>> rects(N);
    size_t total = 0;
    for (size_t l = 1; l < nl; ++l) {
        if (!cnt[l]) continue;
        ++total;
        const long long ymin = (long long)bb[nl + l] - oy, ymax = (long long)bb[3 * nl + l] - oy;
        const int xlo = (int)((long long)bb[l] - ox), xhi = (int)((long long)bb[2 * nl + l] - ox) + 1;
        int d = 0;
        while (d + 1 < N && ymin >= y0[d + 1]) ++d;
        ++owned[d];
        if (ymax < y1[d]) continue;
        need[d] = std::max(need[d], (int)(ymax + 1 - y1[d]));
        for (int e = d + 1; e < N && y0[e] <= ymax; ++e) {
            const int a = std::max(y1[d], y0[e]), b = (int)std::min<long long>(y1[e], ymax + 1);
            if (a < b) rects[d].push_back(HaloRect{e, a, b, xlo, xhi});
        }
    }
    if (total > cap_rois)
        return set_error(FX_E_CAPACITY, "output capacity " + std::to_string(cap_rois) + " < " +
                                            std::to_string(total) + " ROIs");
    std::vector<int> py0(y0.begin(), y0.end());
    std::vector<std::vector<uint32_t>> labs(N);
    std::vector<std::vector<double>> vals(N);
    std::vector<size_t> got(N, 0);
    rc = parallel([&](int d) {
        labs[d].resize(std::max<size_t>(owned[d], 1));
        vals[d].resize(std::max<size_t>(owned[d], 1) * (size_t)std::max(nc, 1));
        return islide_featurize(m->ctx[d], im, y0[d], y1[d], need[d], rects[d], pL, pI, pp, py0,
                                m->ev_loaded.data(), groups, *p, owned[d], labs[d].data(),
                                vals[d].data(), &got[d]);
    });
    if (rc) return rc;
    // 4. merge the bands' rows by label
    std::vector<size_t> at(N, 0);
    size_t k = 0;
    while (k < total) {
        int best = -1;
        for (int d = 0; d < N; ++d)
            if (at[d] < got[d] && (best < 0 || labs[d][at[d]] < labs[best][at[best]])) best = d;
        if (best < 0) break;
        out_labels[k] = labs[best][at[best]];
        std::memcpy(out_values + k * nc, vals[best].data() + at[best] * nc, (size_t)nc * sizeof(double));
        ++at[best];
        ++k;
    }
    if (k != total) return set_error(FX_E_INTERNAL, "bands returned " + std::to_string(k) + " of " +
                                                      std::to_string(total) + " ROIs");
    *n_rois = total;
    return FX_OK;
}

}  // extern "C"
