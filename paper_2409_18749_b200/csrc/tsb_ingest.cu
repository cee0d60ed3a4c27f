// Staged PCIe ingest for pinned-host sample stores.
//
// The reference reads each batch's samples from its DirectorySource into a
// host buffer (pipeline.py:190-210) before the segment memcpy
// (payload.py:234-235).  Here the batch's samples -- scattered rows of a
// pinned host store, in epoch order -- cross PCIe once: one gather kernel per
// batch on a dedicated ingest stream reads the mapped pinned rows with
// 16-byte loads (thousands in flight cover the PCIe latency) and writes them
// into a double-buffered HBM staging area, overlapped with the collate kernel
// of the previous batch on the producer stream.  It co-resides with the
// collate (no shared memory, few registers).  One copy-engine operation per
// sample would cost ~2 us of host API time each (0.5 ms per 256-sample
// batch); SM loads of pinned memory reach ~48 GB/s on B200's PCIe Gen5 x16
// link (profiles/r1/h2d_probe.json).  The collate kernel then reads HBM
// through its TMA path.  Passthrough batches are gathered straight into the
// ring slot.
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "tsb_common.cuh"

using namespace tsb;

struct tsb_ingest {
    int dev;
    int depth;
    int64_t max_batch;
    int64_t sample_bytes;
    uint8_t *staging;     // [depth][max_batch * sample_bytes] HBM
    int64_t *d_idx;       // [depth][max_batch] the batch's real sample indices
    int32_t *d_params;    // [depth][max_batch][3] crop/flip table
    int64_t *d_identity;  // [max_batch] 0..max_batch-1 (rows of a staged batch)
    int64_t *h_idx;       // [depth][max_batch] pinned upload buffer
    int32_t *h_params;    // [depth][max_batch][3] pinned upload buffer (crop-aware batches)
    uint64_t bytes;       // H2D bytes enqueued (tsb_ingest_bytes)
    cudaStream_t stream;  // ingest stream (beside the producer stream)
    cudaStream_t ce_stream;  // copy-engine share of a batch (TSB_INGEST_CE samples)
    cudaEvent_t ce_done;
    std::vector<cudaEvent_t> done, freed;
    std::vector<int> used;
    int next;
    // TSB_INGEST=hostpack: host threads gather the batch's sample rows into a
    // pinned buffer, then ONE contiguous copy-engine transfer per batch
    uint8_t *h_pack = nullptr;  // [depth][max_batch * sample_bytes] pinned
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    uint64_t gen = 0;      // job generation (workers wake on a change)
    int busy = 0;          // workers still on the current job
    bool stop = false;
    struct Job {
        const uint8_t *src;
        const int64_t *idx;
        const int32_t *params;  // crop params (null: whole samples)
        int64_t b, sb;
        int row_bytes, h, pad;
        uint8_t *dst;
    } job{};
    std::atomic<int64_t> next_sample{0};
};

namespace {
__global__ void iota_kernel(int64_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = i;
}

// Sample s of the batch: bytes [lo*row_bytes, hi*row_bytes) of store row
// idx[s] -> out + s*sb (+ the same offset).  With crop params only the rows
// the crop reads (rows [max(0, oy-pad), min(h, h+oy-pad))); else the sample.
// 16-byte vectors when every offset is 16-byte aligned, else bytes.  `line`
// (vector path): the crop's row span widened to whole lines of that many bytes
// (the extra bytes belong to rows the collate does not read).
constexpr int IG_THREADS = 256;
constexpr int IG_U = 4;            // 16-byte loads in flight per thread
constexpr int IG_LINE = 128;       // default line the crop's row span is widened to
__global__ void __launch_bounds__(IG_THREADS)
    ingest_gather_kernel(const uint8_t *__restrict__ host, const int64_t *__restrict__ idx,
                         const int32_t *__restrict__ params, int64_t sb, int row_bytes, int h,
                         int pad, int vec, int line, int64_t chunk, uint8_t *__restrict__ out) {
    const int s = blockIdx.y;
    int64_t begin = 0, end = sb;
    if (params) {
        const int oy = params[3 * s];
        const int lo = max(oy - pad, 0), hi = min(h + oy - pad, h);
        begin = (int64_t)lo * row_bytes;
        end = hi > lo ? (int64_t)hi * row_bytes : begin;
        if (line && end > begin) {  // whole lines: no split PCIe read requests
            begin &= ~(int64_t)(line - 1);
            end = min((end + line - 1) & ~(int64_t)(line - 1), sb);
        }
    }
    const int64_t c0 = begin + (int64_t)blockIdx.x * chunk;
    const int64_t c1 = min(c0 + chunk, end);
    if (c0 >= c1) return;
    const uint8_t *src = host + idx[s] * sb;
    uint8_t *dst = out + (int64_t)s * sb;
    if (vec) {
        for (int64_t o0 = c0 + 16 * (int64_t)threadIdx.x; o0 < c1; o0 += 16 * IG_THREADS * IG_U) {
            uint4 v[IG_U];
#pragma unroll
            for (int u = 0; u < IG_U; ++u) {
                const int64_t o = o0 + 16 * (int64_t)(u * IG_THREADS);
                if (o < c1) v[u] = ld_nc_v4(src + o);
            }
#pragma unroll
            for (int u = 0; u < IG_U; ++u) {
                const int64_t o = o0 + 16 * (int64_t)(u * IG_THREADS);
                if (o < c1) *reinterpret_cast<uint4 *>(dst + o) = v[u];
            }
        }
    } else {
        for (int64_t o = c0 + threadIdx.x; o < c1; o += IG_THREADS) dst[o] = src[o];
    }
}
}  // namespace

namespace tsb {
void preload_ingest() { touch_kernel(iota_kernel); }

// Enqueue the H2D copy of batch rows h_idx[0..b) of `host_store` on the
// ingest stream, into staging buffer k (or `dst` when non-null), plus the
// index upload; `stream` waits for it.  Returns k.
//
// With `crop` (augment batches): the crop/flip params of every sample are
// derived here on the host -- the same pure function of (aug seed, epoch,
// sample index) the device uses (SURVEY.md §8a A6') -- and uploaded with the
// indices, and only the source rows the crop reads cross PCIe: output row y
// reads source row y + oy - pad, so rows [max(0, oy-pad), min(h, h+oy-pad))
// of each sample (on average 8.2 of 224 rows fewer at pad 16).  The collate
// kernel loads exactly those rows of a staged sample, never the others.
// (Columns too would save another 3.7%, but 2D copies -- one op per sample --
// ran ~10x slower: e2e 154 k vs 1.49 M samples/s; profiles/r1/ingest_2d_ab.txt.)
// one sample's rows (all, or the crop's) into the pinned pack buffer
static void pack_sample(const tsb_ingest::Job &j, int64_t i) {
    size_t off = 0, len = (size_t)j.sb;
    if (j.params) {
        const int oy = j.params[3 * i];
        const int lo = oy - j.pad > 0 ? oy - j.pad : 0;
        const int hi = j.h + oy - j.pad < j.h ? j.h + oy - j.pad : j.h;
        off = (size_t)lo * (size_t)j.row_bytes;
        len = hi > lo ? (size_t)(hi - lo) * (size_t)j.row_bytes : 0;
    }
    if (len) memcpy(j.dst + (size_t)i * (size_t)j.sb + off, j.src + (size_t)j.idx[i] * (size_t)j.sb + off, len);
}
static void pack_work(tsb_ingest *g) {
    const tsb_ingest::Job j = g->job;
    for (;;) {
        const int64_t i = g->next_sample.fetch_add(1, std::memory_order_relaxed);
        if (i >= j.b) break;
        pack_sample(j, i);
    }
}
static void pack_worker(tsb_ingest *g) {
    uint64_t seen = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->cv.wait(lk, [&] { return g->stop || g->gen != seen; });
            if (g->stop) return;
            seen = g->gen;
        }
        pack_work(g);
        std::lock_guard<std::mutex> lk(g->mu);
        if (--g->busy == 0) g->cv_done.notify_all();
    }
}
// the calling thread and the workers pack the batch; returns when done
static void pack_batch(tsb_ingest *g, const tsb_ingest::Job &j) {
    if (g->workers.empty()) {
        static const int want = getenv("TSB_INGEST_THREADS")
                                    ? atoi(getenv("TSB_INGEST_THREADS"))
                                    : (int)std::min(7u, std::max(1u, std::thread::hardware_concurrency() / 2));
        for (int t = 0; t < want; ++t) g->workers.emplace_back(pack_worker, g);
    }
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->job = j;
        g->next_sample.store(0, std::memory_order_relaxed);
        g->busy = (int)g->workers.size();
        ++g->gen;
    }
    g->cv.notify_all();
    pack_work(g);
    std::unique_lock<std::mutex> lk(g->mu);
    g->cv_done.wait(lk, [&] { return g->busy == 0; });
}

int ingest_batch(tsb_ingest *g, const void *host_store, const int64_t *h_idx, int64_t b,
                 void *dst, void *stream, int *k_out, bool after_stream, const IngestCrop *crop) {
    TSB_CHECK(g && host_store && h_idx && k_out, "null argument");
    TSB_CHECK(b >= 1 && b <= g->max_batch, "batch %lld exceeds the ingest capacity %lld",
              (long long)b, (long long)g->max_batch);
    const int k = g->next;
    g->next = (g->next + 1) % g->depth;
    // the pinned index buffer k is reused: its previous upload must be done
    if (g->used[k]) TSB_CUDA(cudaEventSynchronize(g->done[k]));
    g->used[k] = 1;
    int64_t *hk = g->h_idx + (size_t)k * g->max_batch;
    memcpy(hk, h_idx, sizeof(int64_t) * (size_t)b);
    // staging buffer k is free once the previous batch staged in it was collated
    TSB_CUDA(cudaStreamWaitEvent(g->stream, g->freed[k], 0));
    if (after_stream) {  // a copy straight into a ring slot must follow the stream's gate
        TSB_CUDA(cudaEventRecord(g->freed[k], as_stream(stream)));
        TSB_CUDA(cudaStreamWaitEvent(g->stream, g->freed[k], 0));
    }
    uint8_t *out = dst ? static_cast<uint8_t *>(dst)
                       : g->staging + (size_t)k * (size_t)(g->max_batch * g->sample_bytes);
    const size_t sb = (size_t)g->sample_bytes;
    int32_t *hp = g->h_params + (size_t)k * g->max_batch * 3;
    size_t nbytes = 0;
    static const bool host_pack = getenv("TSB_INGEST") && !strcmp(getenv("TSB_INGEST"), "hostpack");
    static const bool per_sample = getenv("TSB_INGEST") && !strcmp(getenv("TSB_INGEST"), "memcpy");
    // TSB_IG_ALIGN=bytes (A/B; a power of two, 0 = the crop's exact row span)
    static const int line = getenv("TSB_IG_ALIGN") ? atoi(getenv("TSB_IG_ALIGN")) : IG_LINE;
    static const bool align = line >= 16 && (line & (line - 1)) == 0;
    const bool vec = ((uintptr_t)host_store & 15) == 0 && sb % 16 == 0 &&
                     (!crop || crop->row_bytes % 16 == 0);
    for (int64_t i = 0; i < b; ++i) {
        size_t len = sb;
        if (crop) {
            int oy = 0, ox = 0, fl = 0;
            derive_aug_host(crop->aug_mixed, crop->epoch, h_idx[i], crop->pad, crop->flip, oy, ox,
                            fl);
            hp[3 * i] = oy;
            hp[3 * i + 1] = ox;
            hp[3 * i + 2] = fl;
            const int lo = oy - crop->pad > 0 ? oy - crop->pad : 0;
            const int hi = crop->h + oy - crop->pad < crop->h ? crop->h + oy - crop->pad : crop->h;
            len = hi > lo ? (size_t)(hi - lo) * (size_t)crop->row_bytes : 0;
            if (vec && align && len && !host_pack && !per_sample) {  // the gather kernel reads whole lines
                const size_t b0 = ((size_t)lo * (size_t)crop->row_bytes) & ~(size_t)(line - 1);
                size_t b1 = ((size_t)hi * (size_t)crop->row_bytes + line - 1) & ~(size_t)(line - 1);
                if (b1 > sb) b1 = sb;
                len = b1 - b0;
            }
        }
        nbytes += len;
    }
    int64_t *dk = g->d_idx + (size_t)k * g->max_batch;
    int32_t *pk = g->d_params + (size_t)k * g->max_batch * 3;
    TSB_CUDA(cudaMemcpyAsync(dk, hk, sizeof(int64_t) * (size_t)b, cudaMemcpyHostToDevice,
                             g->stream));
    nbytes += sizeof(int64_t) * (size_t)b;
    if (crop) {
        TSB_CUDA(cudaMemcpyAsync(pk, hp, sizeof(int32_t) * 3 * (size_t)b, cudaMemcpyHostToDevice,
                                 g->stream));
        nbytes += sizeof(int32_t) * 3 * (size_t)b;
    }
    const int row_bytes = crop ? crop->row_bytes : 0;
    if (host_pack) {
        if (!g->h_pack)
            TSB_CUDA(cudaHostAlloc(&g->h_pack, (size_t)g->depth * (size_t)g->max_batch * sb, 0));
        uint8_t *hb = g->h_pack + (size_t)k * (size_t)g->max_batch * sb;  // free: done[k] synced
        tsb_ingest::Job j{static_cast<const uint8_t *>(host_store), h_idx, crop ? hp : nullptr, b,
                          (int64_t)sb, row_bytes, crop ? crop->h : 0, crop ? crop->pad : 0, hb};
        pack_batch(g, j);
        TSB_CUDA(cudaMemcpyAsync(out, hb, (size_t)b * sb, cudaMemcpyHostToDevice, g->stream));
        g->bytes += (size_t)b * sb + sizeof(int64_t) * (size_t)b +
                    (crop ? sizeof(int32_t) * 3 * (size_t)b : 0);
        TSB_CUDA(cudaEventRecord(g->done[k], g->stream));
        TSB_CUDA(cudaStreamWaitEvent(as_stream(stream), g->done[k], 0));
        *k_out = k;
        return TSB_OK;
    }
    // A/B (TSB_INGEST=memcpy): one copy-engine operation per sample instead
    if (per_sample) {
        for (int64_t i = 0; i < b; ++i) {
            size_t off = 0, len = sb;
            if (crop) {
                const int oy = hp[3 * i];
                const int lo = oy - crop->pad > 0 ? oy - crop->pad : 0;
                const int hi = crop->h + oy - crop->pad < crop->h ? crop->h + oy - crop->pad : crop->h;
                off = (size_t)lo * (size_t)row_bytes;
                len = hi > lo ? (size_t)(hi - lo) * (size_t)row_bytes : 0;
            }
            if (len)
                TSB_CUDA(cudaMemcpyAsync(out + (size_t)i * sb + off,
                                         static_cast<const uint8_t *>(host_store) +
                                             (size_t)h_idx[i] * sb + off,
                                         len, cudaMemcpyHostToDevice, g->stream));
        }
        g->bytes += nbytes;
        TSB_CUDA(cudaEventRecord(g->done[k], g->stream));
        TSB_CUDA(cudaStreamWaitEvent(as_stream(stream), g->done[k], 0));
        *k_out = k;
        return TSB_OK;
    }
    // TSB_INGEST_CE=n: the batch's last n samples go by the copy engine (one
    // copy per sample on a second stream, issued from this thread) beside the
    // gather kernel's SM loads of the others -- both share the PCIe link
    static const int64_t n_ce_knob =
        getenv("TSB_INGEST_CE") ? (int64_t)atoll(getenv("TSB_INGEST_CE")) : 0;
    const int64_t n_ce = n_ce_knob < b ? n_ce_knob : b - 1;
    if (n_ce > 0) {
        TSB_CUDA(cudaStreamWaitEvent(g->ce_stream, g->freed[k], 0));
        for (int64_t i = b - n_ce; i < b; ++i) {
            size_t off = 0, len = sb;
            if (crop) {
                const int oy = hp[3 * i];
                const int lo = oy - crop->pad > 0 ? oy - crop->pad : 0;
                const int hi = crop->h + oy - crop->pad < crop->h ? crop->h + oy - crop->pad : crop->h;
                off = (size_t)lo * (size_t)row_bytes;
                len = hi > lo ? (size_t)(hi - lo) * (size_t)row_bytes : 0;
            }
            if (len)
                TSB_CUDA(cudaMemcpyAsync(out + (size_t)i * sb + off,
                                         static_cast<const uint8_t *>(host_store) +
                                             (size_t)h_idx[i] * sb + off,
                                         len, cudaMemcpyHostToDevice, g->ce_stream));
        }
        TSB_CUDA(cudaEventRecord(g->ce_done, g->ce_stream));
    }
    const int64_t b_sm = b - (n_ce > 0 ? n_ce : 0);
    const bool vec_k = vec && ((uintptr_t)out & 15) == 0;
    // bytes per CTA and sample (TSB_IG_CHUNK A/B; 16 KB default)
    static const int64_t chunk =
        getenv("TSB_IG_CHUNK") ? (int64_t)atoll(getenv("TSB_IG_CHUNK")) : 16384;
    dim3 grid((unsigned)((sb + chunk - 1) / chunk), (unsigned)b_sm);
    TSB_CHECK(b <= 65535, "batch %lld exceeds the gather grid", (long long)b);
    ingest_gather_kernel<<<grid, IG_THREADS, 0, g->stream>>>(
        static_cast<const uint8_t *>(host_store), dk, crop ? pk : nullptr, (int64_t)sb, row_bytes,
        crop ? crop->h : 0, crop ? crop->pad : 0, vec_k ? 1 : 0, vec_k && align ? line : 0, chunk, out);
    TSB_LAUNCH_CHECK();
    if (n_ce > 0) TSB_CUDA(cudaStreamWaitEvent(g->stream, g->ce_done, 0));
    g->bytes += nbytes;
    TSB_CUDA(cudaEventRecord(g->done[k], g->stream));
    TSB_CUDA(cudaStreamWaitEvent(as_stream(stream), g->done[k], 0));
    *k_out = k;
    return TSB_OK;
}

// The producer stream is done with staging buffer k.
int ingest_release(tsb_ingest *g, int k, void *stream) {
    TSB_CUDA(cudaEventRecord(g->freed[k], as_stream(stream)));
    return TSB_OK;
}

uint8_t *ingest_staging(tsb_ingest *g, int k) {
    return g->staging + (size_t)k * (size_t)(g->max_batch * g->sample_bytes);
}
int64_t *ingest_indices(tsb_ingest *g, int k) { return g->d_idx + (size_t)k * g->max_batch; }
int32_t *ingest_params(tsb_ingest *g, int k) { return g->d_params + (size_t)k * g->max_batch * 3; }
int64_t *ingest_identity(tsb_ingest *g) { return g->d_identity; }
int64_t ingest_sample_bytes(tsb_ingest *g) { return g->sample_bytes; }
}  // namespace tsb

extern "C" {

int tsb_ingest_create(int dev, int64_t max_batch, int64_t sample_bytes, int depth,
                      tsb_ingest **out) {
    TSB_CHECK(out && max_batch >= 1 && sample_bytes >= 1 && depth >= 1 && depth <= 8,
              "bad ingest geometry");
    CurrentDeviceGuard device_guard;
    TSB_CUDA(cudaSetDevice(dev));
    tsb_ingest *g = new tsb_ingest{};
    g->dev = dev;
    g->depth = depth;
    g->max_batch = max_batch;
    g->sample_bytes = sample_bytes;
    const size_t stage = (size_t)max_batch * (size_t)sample_bytes;
    cudaError_t e = cudaMalloc(&g->staging, stage * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_idx, sizeof(int64_t) * max_batch * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_params, sizeof(int32_t) * 3 * max_batch * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_identity, sizeof(int64_t) * max_batch);
    if (e == cudaSuccess) e = cudaHostAlloc(&g->h_idx, sizeof(int64_t) * max_batch * depth, 0);
    if (e == cudaSuccess)
        e = cudaHostAlloc(&g->h_params, sizeof(int32_t) * 3 * max_batch * depth, 0);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->ce_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ce_done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_error("ingest allocation: %s", cudaGetErrorString(e));
        tsb_ingest_destroy(g);
        return TSB_ERR_CUDA;
    }
    g->done.resize(depth);
    g->freed.resize(depth);
    g->used.assign(depth, 0);
    for (int k = 0; k < depth; ++k) {
        TSB_CUDA(cudaEventCreateWithFlags(&g->done[k], cudaEventDisableTiming));
        TSB_CUDA(cudaEventCreateWithFlags(&g->freed[k], cudaEventDisableTiming));
    }
    iota_kernel<<<(unsigned)((max_batch + 255) / 256), 256, 0, g->stream>>>(g->d_identity,
                                                                          max_batch);
    TSB_LAUNCH_CHECK();
    TSB_CUDA(cudaStreamSynchronize(g->stream));
    *out = g;
    return TSB_OK;
}

int tsb_ingest_destroy(tsb_ingest *g) {
    if (!g) return TSB_OK;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->stop = true;
    }
    g->cv.notify_all();
    for (auto &t : g->workers) t.join();
    if (g->h_pack) {
        if (g->stream) cudaStreamSynchronize(g->stream);
        cudaFreeHost(g->h_pack);
    }
    if (g->stream) cudaStreamSynchronize(g->stream);
    for (auto ev : g->done) cudaEventDestroy(ev);
    for (auto ev : g->freed) cudaEventDestroy(ev);
    if (g->stream) cudaStreamDestroy(g->stream);
    if (g->ce_stream) cudaStreamSynchronize(g->ce_stream);
    if (g->ce_stream) cudaStreamDestroy(g->ce_stream);
    if (g->ce_done) cudaEventDestroy(g->ce_done);
    cudaFree(g->staging);
    cudaFree(g->d_idx);
    cudaFree(g->d_params);
    cudaFree(g->d_identity);
    if (g->h_idx) cudaFreeHost(g->h_idx);
    if (g->h_params) cudaFreeHost(g->h_params);
    delete g;
    return TSB_OK;
}

int tsb_ingest_batch_api(tsb_ingest *g, int *used) {
    TSB_CHECK(g && used, "null argument");
    *used = 1;  // one gather launch per batch
    return TSB_OK;
}

int tsb_ingest_bytes(tsb_ingest *g, uint64_t *bytes) {
    TSB_CHECK(g && bytes, "null argument");
    *bytes = g->bytes;
    return TSB_OK;
}

}  // extern "C"
