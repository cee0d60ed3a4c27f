// Staged PCIe ingest for pinned-host sample stores.
//
// The reference reads each batch's samples from its DirectorySource into a
// host buffer (pipeline.py:190-210) before the segment memcpy
// (payload.py:234-235).  Here the batch's samples -- scattered rows of a
// pinned host store, in epoch order -- cross PCIe once, by the copy engine:
// one cudaMemcpyBatchAsync of B sample rows per batch on a dedicated ingest
// stream into a double-buffered HBM staging area, overlapped with the
// collate kernel of the previous batch on the producer stream.  The copy
// engine sustains ~55 GB/s H2D on B200's PCIe Gen5 x16 link against ~48 GB/s
// for SM loads of pinned memory (profiles/r1), and the collate kernel then
// reads HBM through its TMA path.  Passthrough batches are copied straight
// into the ring slot (no kernel at all).
#include <cstring>
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
    cudaStream_t stream;  // copy-engine stream
    std::vector<cudaEvent_t> done, freed;
    std::vector<int> used;
    int next;
    std::vector<void *> dsts, srcs;
    std::vector<size_t> sizes;
    int batch_api;        // cudaMemcpyBatchAsync usable (else one copy per sample)
};

namespace {
__global__ void iota_kernel(int64_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = i;
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
// (Columns too would save another 3.7%, but 2D copies -- cudaMemcpy3DBatchAsync,
// one op per sample -- run ~10x slower on the copy engine: e2e 154 k vs 1.49 M
// samples/s; profiles/r1/ingest_2d_ab.txt.)
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
    const uint8_t *src = static_cast<const uint8_t *>(host_store);
    const size_t sb = (size_t)g->sample_bytes;
    int32_t *hp = g->h_params + (size_t)k * g->max_batch * 3;
    size_t nbytes = 0;
    bool done = false;
    for (int64_t i = 0; i < b; ++i) {
        size_t off = 0, len = sb;
        if (crop) {
            int oy = 0, ox = 0, fl = 0;
            derive_aug_host(crop->aug_mixed, crop->epoch, h_idx[i], crop->pad, crop->flip, oy, ox,
                            fl);
            hp[3 * i] = oy;
            hp[3 * i + 1] = ox;
            hp[3 * i + 2] = fl;
            const int lo = oy - crop->pad > 0 ? oy - crop->pad : 0;
            const int hi = crop->h + oy - crop->pad < crop->h ? crop->h + oy - crop->pad : crop->h;
            // a sample cropped out entirely (pad >= h) still gets a 1-byte copy
            // (the batch API takes no empty entries); the kernel reads none of it
            off = hi > lo ? (size_t)lo * (size_t)crop->row_bytes : 0;
            len = hi > lo ? (size_t)(hi - lo) * (size_t)crop->row_bytes : 1;
        }
        g->dsts[i] = out + (size_t)i * sb + off;
        g->srcs[i] = const_cast<uint8_t *>(src + (size_t)h_idx[i] * sb + off);
        g->sizes[i] = len;
        nbytes += g->sizes[i];
    }
    if (!done && g->batch_api) {
        cudaMemcpyAttributes attr{};
        attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
        size_t attr_idx = 0, fail = 0;
        cudaError_t e = cudaMemcpyBatchAsync(g->dsts.data(), g->srcs.data(), g->sizes.data(),
                                             (size_t)b, &attr, &attr_idx, 1, &fail, g->stream);
        if (e == cudaSuccess) {
            done = true;
        } else {
            cudaGetLastError();
            g->batch_api = 0;  // driver without the batch API: per-sample copies from now on
        }
    }
    if (!done)
        for (int64_t i = 0; i < b; ++i)
            TSB_CUDA(cudaMemcpyAsync(g->dsts[i], g->srcs[i], g->sizes[i], cudaMemcpyHostToDevice,
                                     g->stream));
    TSB_CUDA(cudaMemcpyAsync(g->d_idx + (size_t)k * g->max_batch, hk, sizeof(int64_t) * (size_t)b,
                             cudaMemcpyHostToDevice, g->stream));
    nbytes += sizeof(int64_t) * (size_t)b;
    if (crop) {
        TSB_CUDA(cudaMemcpyAsync(g->d_params + (size_t)k * g->max_batch * 3, hp,
                                 sizeof(int32_t) * 3 * (size_t)b, cudaMemcpyHostToDevice,
                                 g->stream));
        nbytes += sizeof(int32_t) * 3 * (size_t)b;
    }
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
    g->batch_api = 1;
    const size_t stage = (size_t)max_batch * (size_t)sample_bytes;
    cudaError_t e = cudaMalloc(&g->staging, stage * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_idx, sizeof(int64_t) * max_batch * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_params, sizeof(int32_t) * 3 * max_batch * depth);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_identity, sizeof(int64_t) * max_batch);
    if (e == cudaSuccess) e = cudaHostAlloc(&g->h_idx, sizeof(int64_t) * max_batch * depth, 0);
    if (e == cudaSuccess)
        e = cudaHostAlloc(&g->h_params, sizeof(int32_t) * 3 * max_batch * depth, 0);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
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
    g->dsts.resize(max_batch);
    g->srcs.resize(max_batch);
    g->sizes.resize(max_batch);
    iota_kernel<<<(unsigned)((max_batch + 255) / 256), 256, 0, g->stream>>>(g->d_identity,
                                                                          max_batch);
    TSB_LAUNCH_CHECK();
    TSB_CUDA(cudaStreamSynchronize(g->stream));
    *out = g;
    return TSB_OK;
}

int tsb_ingest_destroy(tsb_ingest *g) {
    if (!g) return TSB_OK;
    if (g->stream) cudaStreamSynchronize(g->stream);
    for (auto ev : g->done) cudaEventDestroy(ev);
    for (auto ev : g->freed) cudaEventDestroy(ev);
    if (g->stream) cudaStreamDestroy(g->stream);
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
    *used = g->batch_api;
    return TSB_OK;
}

int tsb_ingest_bytes(tsb_ingest *g, uint64_t *bytes) {
    TSB_CHECK(g && bytes, "null argument");
    *bytes = g->bytes;
    return TSB_OK;
}

}  // extern "C"
