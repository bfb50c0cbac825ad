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
#include <mutex>
#include <string>
#include <thread>
#include <vector>

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
    const size_t n_chunks = ((size_t)n + kChunkImages - 1) / kChunkImages;
    const int N = (int)m->ctx.size();
    Ledger ledger(n_chunks);
    double total_px = 0;
    for (int i = 0; i < n; ++i) total_px += (double)ims[i].width * ims[i].height;
    std::vector<int> status(N, FX_OK);
    std::vector<std::string> errs(N);
    auto worker = [&](int d) {
        fx_ctx* c = m->ctx[d];
        DevBufs& B = m->bufs[d];
        cudaSetDevice(m->devices[d]);
        int use = 0;
        bool ran = false;  // finish() reads this call's control block: only after work
        for (size_t j = (size_t)d; j < n_chunks; j += N, use ^= 1) {
            ran = true;
            const int first = (int)(j * kChunkImages), cnt = std::min(kChunkImages, n - first);
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

}  // extern "C"
