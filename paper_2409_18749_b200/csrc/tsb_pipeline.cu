// Native producer/consumer loops over the device ring: one host call enqueues
// a whole range of batches (memops + kernels), so the per-batch host cost is
// a few driver calls instead of a Python round trip.
#include <stdlib.h>

#include "tsb_common.cuh"

using namespace tsb;

namespace tsb {
int ring_publish_ptrs(tsb_ring *r, int slot, int writer, uint64_t **ready, unsigned int **counter);
int ring_writers(const tsb_ring *r);
int ring_phys_device(const tsb_ring *r);
void ring_internals(tsb_ring *r, uint8_t **base, int64_t *stride, uint64_t **ready,
                    uint64_t **cursors, unsigned int **counters);
int produce_persistent_crc(const void *src, const int64_t *order, int64_t b, int h, int w, int c,
                           int pad, int flip, uint64_t aug_seed, uint64_t epoch,
                           const float *scale, const float *bias, int out_kind,
                           uint8_t *ring_base, int64_t slot_stride, int slots, uint64_t *ready,
                           const uint64_t *cursors, unsigned int *counters, const int *live,
                           int n_live, int64_t input_bytes, int with_target, uint64_t seq0,
                           int64_t batch0, int n, uint32_t *d_crc, uint32_t *h_crc,
                           void *stream);
int produce_persistent(int mode, const void *src, const int64_t *order, int64_t b,
                       int64_t sample_bytes, uint64_t seed, uint64_t epoch, uint8_t *ring_base,
                       int64_t slot_stride, int slots, uint64_t *ready, const uint64_t *cursors,
                       unsigned int *counters, const int *live, int n_live, int64_t input_bytes,
                       int with_target, uint64_t seq0, int64_t batch0, int n, void *stream,
                       int64_t ep_len, int64_t ep_stride);
int produce_multi(int mode, const void *src, const int64_t *idx, int64_t b, int h, int w, int c,
                  int pad, int flip, uint64_t seed, uint64_t epoch, const float *scale,
                  const float *bias, int out_kind, int64_t sample_bytes, void *const *outs,
                  int64_t *const *tgts, uint64_t *const *readys, int n, unsigned int *counter,
                  uint64_t seq, int pdl, int sys_fence, void *stream);
bool ring_has_host_control(const tsb_ring *r);
int ring_host_gate(tsb_ring *r, const int *live, int n_live, uint64_t need);
int collate_augment_publish(const void *src, const int64_t *d_indices, int64_t b, int h, int w,
                            int c, int pad, int flip, uint64_t aug_seed, uint64_t epoch,
                            const float *scale, const float *bias, int out_kind, void *out,
                            int64_t *tgt, uint64_t *ready, uint64_t seq, unsigned int *counter,
                            int pdl, void *stream, const int32_t *d_params,
                            const int64_t *tgt_idx, uint64_t *release = nullptr,
                            uint32_t *crc_out = nullptr, int *crc_done = nullptr,
                            uint32_t *crc_host = nullptr);
int ingest_batch(tsb_ingest *g, const void *host_store, const int64_t *h_idx, int64_t b,
                 void *dst, void *stream, int *k_out, bool after_stream,
                 const IngestCrop *crop = nullptr);
int ingest_release(tsb_ingest *g, int k, void *stream);
uint8_t *ingest_staging(tsb_ingest *g, int k);
int64_t *ingest_indices(tsb_ingest *g, int k);
int32_t *ingest_params(tsb_ingest *g, int k);
int64_t *ingest_identity(tsb_ingest *g);
int64_t ingest_sample_bytes(tsb_ingest *g);
int jpeg_decode(tsb_jpeg *j, const int64_t *h_idx, int64_t b, void *out, void *stream);
int jpeg_upload_indices(tsb_jpeg *j, const int64_t *h_idx, int64_t b, void *stream);
uint8_t *jpeg_staging(tsb_jpeg *j);
int64_t *jpeg_indices(tsb_jpeg *j);
int32_t *jpeg_params(tsb_jpeg *j);
int64_t *jpeg_identity(tsb_jpeg *j);
int64_t jpeg_sample_bytes(tsb_jpeg *j);
}  // namespace tsb

extern "C" {

int tsb_produce_range(tsb_ring *r, const tsb_produce_args *a, uint64_t seq0, int64_t batch0,
                      int n, const int *live, int n_live, void **ev, void *stream) {
    TSB_CHECK(r && a && a->d_order, "null argument");
    TSB_CHECK(seq0 >= 1 && n >= 0 && batch0 >= 0, "bad range");
    int slots = 0;
    size_t stride = 0;
    if (int rc = tsb_ring_geometry(r, &slots, &stride, nullptr)) return rc;
    const int64_t b = a->batch_size;
    const size_t nbytes = (size_t)a->input_bytes + (a->with_target ? 8 * (size_t)b : 0);
    TSB_CHECK(nbytes <= stride, "batch (%zu B) exceeds the ring slot (%zu B)", nbytes, stride);
    TSB_CHECK(a->wait_stride <= slots, "wait_stride %d exceeds the ring depth %d", a->wait_stride,
              slots);
    auto s = as_stream(stream);
    // Host-shared control words: gate on the host (no device wait in the
    // stream), and chain consecutive fused batches with programmatic dependent
    // launch.  The first batch of a range keeps full stream ordering (the
    // previous op on the stream may be anything).
    TSB_CHECK(a->gate == TSB_GATE_DEVICE || ring_has_host_control(r),
              "TSB_GATE_HOST needs a ring with a host control block");
    const bool host_gate = a->gate == TSB_GATE_HOST;
    TSB_CHECK(a->order_epochs <= 1 || (a->persistent && a->mode != TSB_SRC_AUGMENT),
              "a multi-epoch order (order_epochs > 1) is for the persistent passthrough producer");
    static const bool no_pdl = getenv("TSB_NO_PDL") && atoi(getenv("TSB_NO_PDL"));      // A/B knobs
    static const bool no_fused = getenv("TSB_NO_FUSED") && atoi(getenv("TSB_NO_FUSED"));
    bool prev_fused = a->chain != 0;
    const bool jpeg = a->jpeg && a->h_order;
    if (jpeg) {
        TSB_CHECK(a->mode == TSB_SRC_AUGMENT || a->mode == TSB_SRC_GATHER,
                  "a JPEG source feeds the augment or gather modes");
        TSB_CHECK(jpeg_sample_bytes(a->jpeg) == a->sample_bytes,
                  "decoder geometry (%lld B) does not match the samples (%lld B)",
                  (long long)jpeg_sample_bytes(a->jpeg), (long long)a->sample_bytes);
        TSB_CHECK(!no_fused && ring_writers(r) == 1,
                  "the JPEG source needs the fused single-writer path");
    }
    // TSB_INGEST=direct (A/B): the collate's TMA reads the pinned store's rows
    // itself, no staging copy
    static const bool direct_ingest =
        getenv("TSB_INGEST") && !strcmp(getenv("TSB_INGEST"), "direct");
    const bool staged = !jpeg && a->ingest && a->h_order && !ev && !direct_ingest;
    if (a->persistent && a->d_crc && a->mode == TSB_SRC_AUGMENT && !staged && !jpeg && !ev &&
        !no_fused && ring_has_host_control(r) && ring_writers(r) == 1) {
        // fused collate + CRC, one cooperative launch for the whole range
        uint8_t *base = nullptr;
        int64_t sstride = 0;
        uint64_t *ready = nullptr, *cursors = nullptr;
        unsigned int *counters = nullptr;
        ring_internals(r, &base, &sstride, &ready, &cursors, &counters);
        const int rc = produce_persistent_crc(
            a->src, a->d_order, b, a->h, a->w, a->c, a->pad, a->flip, a->seed, a->epoch, a->scale,
            a->bias, a->out_kind, base, sstride, slots, ready, cursors, counters, live, n_live,
            a->input_bytes, a->with_target, seq0, batch0, n, a->d_crc, a->h_crc, stream);
        if (rc != TSB_ERR_STALE) {
            if (a->crc_fused) *a->crc_fused = rc == TSB_OK && n > 0 ? 1 : 0;
            return rc;
        }
    }
    if (a->persistent && !(a->d_crc && a->mode == TSB_SRC_AUGMENT)) {
        // one cooperative launch for the whole range, gated on the device
        TSB_CHECK(ring_has_host_control(r) && ring_writers(r) == 1 && !staged && !jpeg &&
                      !a->d_crc && !ev,
                  "the persistent producer needs a host-control single-writer ring, a "
                  "device-resident passthrough source and no CRC / events");
        uint8_t *base = nullptr;
        int64_t sstride = 0;
        uint64_t *ready = nullptr, *cursors = nullptr;
        unsigned int *counters = nullptr;
        ring_internals(r, &base, &sstride, &ready, &cursors, &counters);
        int64_t ep_len = 0, ep_stride = 0;
        if (a->order_epochs > 1) {  // one launch across epoch boundaries
            TSB_CHECK(a->epoch_len >= 1 && a->order_stride >= a->epoch_len * b &&
                          batch0 + n <= a->order_epochs * a->epoch_len,
                      "multi-epoch range: batches %lld..%lld exceed %lld epochs of %lld",
                      (long long)batch0, (long long)(batch0 + n), (long long)a->order_epochs,
                      (long long)a->epoch_len);
            ep_len = a->epoch_len;
            ep_stride = a->order_stride;
        }
        return produce_persistent(a->mode, a->src, a->d_order, a->batch_size, a->sample_bytes,
                                  a->seed, a->epoch, base, sstride, slots, ready, cursors,
                                  counters, live, n_live, a->input_bytes, a->with_target, seq0,
                                  batch0, n, stream, ep_len, ep_stride);
    }

    if (staged)
        TSB_CHECK(ingest_sample_bytes(a->ingest) == a->sample_bytes,
                  "ingest staging is for %lld-byte samples, not %lld",
                  (long long)ingest_sample_bytes(a->ingest), (long long)a->sample_bytes);
    bool all_fused = a->d_crc != nullptr;  // every batch's CRC came from the collate kernel
    if (a->crc_fused) *a->crc_fused = 0;
    for (int i = 0; i < n; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        const int slot = (int)((q - 1) % (uint64_t)slots);
        const int64_t bi = batch0 + i;
        const int64_t *idx = a->d_order + bi * b;
        void *out = nullptr;
        if (int rc = tsb_ring_slot_ptr(r, slot, &out)) return rc;
        // reuse gate, amortised over blocks of `stride` batches: one wait on every
        // live cursor covers the slots of the whole block (each device wait on a
        // host-shared word costs a PCIe round trip)
        const uint64_t stride = a->wait_stride > 1 ? (uint64_t)a->wait_stride : 1;
        if (host_gate) {
            if (q > (uint64_t)slots)
                if (int rc = ring_host_gate(r, live, n_live, q - (uint64_t)slots)) return rc;
        } else if (i == 0 || (q - 1) % stride == 0) {
            uint64_t block_end = q + (stride - 1 - (q - 1) % stride);
            const uint64_t last = seq0 + (uint64_t)n - 1;
            if (block_end > last) block_end = last;
            if (block_end > (uint64_t)slots)
                if (int rc = tsb_ring_wait_free(r, live, n_live, block_end - (uint64_t)slots, stream))
                    return rc;
        }
        if (ev) TSB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[2 * i]), s));
        int rc = TSB_OK;
        bool published = false, staged_target = false;
        // per-batch CRC fused into the collate when the geometry allows (the
        // kernel's completing CTA writes d_crc[slot] before the ready word)
        uint32_t *crc_out = a->d_crc ? a->d_crc + slot : nullptr;
        uint32_t *crc_host = a->d_crc && a->h_crc ? a->h_crc + slot : nullptr;
        int crc_done = 0;
        switch (a->mode) {
            case TSB_SRC_AUGMENT:
                if (!no_fused && ring_writers(r) == 1) {  // fused epilogue: target copy + publish from the kernel
                    uint64_t *ready = nullptr;
                    unsigned int *counter = nullptr;
                    if ((rc = ring_publish_ptrs(r, slot, 0, &ready, &counter))) return rc;
                    int64_t *tgt = a->with_target
                                       ? reinterpret_cast<int64_t *>(static_cast<uint8_t *>(out) +
                                                                     a->input_bytes)
                                       : nullptr;
                    const int pdl = prev_fused && host_gate && !ev && !no_pdl;
                    if (jpeg) {  // nvJPEG decode into HBM staging, then collate it
                        const int64_t *hb = a->h_order + bi * b;
                        if ((rc = jpeg_upload_indices(a->jpeg, hb, b, stream))) return rc;
                        if ((rc = jpeg_decode(a->jpeg, hb, b, jpeg_staging(a->jpeg), stream)))
                            return rc;
                        int32_t *params = jpeg_params(a->jpeg);
                        if ((rc = tsb_aug_params(a->seed, a->epoch, jpeg_indices(a->jpeg), b,
                                                 a->pad, a->flip, params, stream)))
                            return rc;
                        rc = collate_augment_publish(jpeg_staging(a->jpeg), jpeg_identity(a->jpeg),
                                                     b, a->h, a->w, a->c, a->pad, a->flip, a->seed,
                                                     a->epoch, a->scale, a->bias, a->out_kind, out,
                                                     tgt, ready, q, counter, 0, stream, params,
                                                     jpeg_indices(a->jpeg), nullptr, crc_out,
                                                     &crc_done, crc_host);
                        published = true;
                        break;
                    }
                    if (staged) {  // PCIe ingest into HBM staging, then collate it
                        // crop-aware: only the rows the crop reads cross PCIe, and the
                        // param table is derived on the host and uploaded with the indices
                        const IngestCrop crop{mix64(a->seed ^ AUG_DOMAIN), a->epoch, a->h, a->w,
                                              a->w * a->c, a->pad, a->flip};
                        int k = 0;
                        if ((rc = ingest_batch(a->ingest, a->src, a->h_order + bi * b, b, nullptr,
                                               stream, &k, false, &crop)))
                            return rc;
                        int32_t *params = ingest_params(a->ingest, k);
                        rc = collate_augment_publish(ingest_staging(a->ingest, k),
                                                     ingest_identity(a->ingest), b, a->h, a->w,
                                                     a->c, a->pad, a->flip, a->seed, a->epoch,
                                                     a->scale, a->bias, a->out_kind, out, tgt,
                                                     ready, q, counter, 0, stream, params,
                                                     ingest_indices(a->ingest, k), nullptr,
                                                     crc_out, &crc_done, crc_host);
                        if (!rc) rc = ingest_release(a->ingest, k, stream);
                        published = true;
                        break;
                    }
                    rc = collate_augment_publish(a->src, idx, b, a->h, a->w, a->c, a->pad,
                                                 a->flip, a->seed, a->epoch, a->scale, a->bias,
                                                 a->out_kind, out, tgt, ready, q, counter, pdl,
                                                 stream, nullptr, nullptr, nullptr, crc_out,
                                                 &crc_done, crc_host);
                    published = true;
                    break;
                }
                rc = tsb_collate_augment(a->src, idx, b, a->h, a->w, a->c, a->pad, a->flip,
                                         a->seed, a->epoch, a->scale, a->bias, a->out_kind,
                                         nullptr, out, stream);
                break;
            case TSB_SRC_GATHER:
                if (jpeg) {  // decode straight into the slot (u8 HWC), then target + publish
                    const int64_t *hb = a->h_order + bi * b;
                    if ((rc = jpeg_upload_indices(a->jpeg, hb, b, stream))) return rc;
                    if ((rc = jpeg_decode(a->jpeg, hb, b, out, stream))) return rc;
                    if (a->with_target) {
                        TSB_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(out) + a->input_bytes,
                                                 jpeg_indices(a->jpeg), 8 * b,
                                                 cudaMemcpyDeviceToDevice, s));
                        staged_target = true;
                    }
                    break;
                }
                if (staged) {  // the ingest gather straight into the slot
                    int k = 0;
                    if ((rc = ingest_batch(a->ingest, a->src, a->h_order + bi * b, b, out, stream,
                                           &k, !host_gate)))
                        return rc;
                    if (a->with_target) {
                        TSB_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(out) + a->input_bytes,
                                                 ingest_indices(a->ingest, k), 8 * b,
                                                 cudaMemcpyDeviceToDevice, s));
                        staged_target = true;
                    }
                    rc = ingest_release(a->ingest, k, stream);
                    break;
                }
                [[fallthrough]];
            case TSB_SRC_SYNTHETIC:
                if (!no_fused && ring_writers(r) == 1 && a->sample_bytes % 16 == 0 &&
                    ((uintptr_t)out & 15) == 0) {
                    // one persistent passthrough launch: samples + target + slot publish
                    uint64_t *ready = nullptr;
                    unsigned int *counter = nullptr;
                    if ((rc = ring_publish_ptrs(r, slot, 0, &ready, &counter))) return rc;
                    int64_t *tgt = a->with_target
                                       ? reinterpret_cast<int64_t *>(static_cast<uint8_t *>(out) +
                                                                     a->input_bytes)
                                       : nullptr;
                    void *outs[1] = {out};
                    int64_t *tgts[1] = {tgt};
                    uint64_t *readys[1] = {ready};
                    const int pdl = prev_fused && host_gate && !ev && !no_pdl;
                    rc = produce_multi(a->mode, a->src, idx, b, a->h, a->w, a->c, a->pad, a->flip,
                                       a->seed, a->epoch, a->scale, a->bias, a->out_kind,
                                       a->sample_bytes, outs, tgts, readys, 1, counter, q, pdl, 0,
                                       stream);
                    published = true;
                    break;
                }
                rc = a->mode == TSB_SRC_GATHER
                         ? tsb_gather(a->src, idx, b, a->sample_bytes, out, stream)
                         : tsb_fill_synthetic(out, idx, b, a->seed, a->epoch, a->sample_bytes,
                                              stream);
                break;
            default:
                TSB_CHECK(false, "bad produce mode %d", a->mode);
        }
        if (rc) return rc;
        // With a separate per-batch CRC the fused kernel still publishes the slot: the
        // checksum only rides in the Announce, which the host sends after
        // reading it, so no consumer fetches the slot before its CRC is known
        // (and nothing rewrites it before every consumer released it).  The
        // CRC launches sit between two collates, so that pair is not PDL-chained.
        prev_fused = published && (!a->d_crc || crc_done);
        all_fused = all_fused && crc_done;
        if (ev) TSB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[2 * i + 1]), s));
        if (published) {
            if (a->d_crc && !crc_done)
                if (int rc2 = tsb_crc32(out, nbytes, a->d_crc + slot, nullptr, stream)) return rc2;
            continue;
        }
        if (a->with_target && !staged_target)
            TSB_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(out) + a->input_bytes, idx, 8 * b,
                                     cudaMemcpyDeviceToDevice, s));
        if (a->d_crc)
            if (int rc2 = tsb_crc32(out, nbytes, a->d_crc + slot, nullptr, stream)) return rc2;
        if (int rc3 = tsb_ring_publish(r, slot, q, stream)) return rc3;
    }
    if (a->crc_fused) *a->crc_fused = all_fused && n > 0 ? 1 : 0;
    return TSB_OK;
}

int tsb_consume_range(tsb_ring *r, int consumer, uint64_t seq0, int n, void **ev, void *stream) {
    TSB_CHECK(r && seq0 >= 1 && n >= 0, "bad argument");
    int slots = 0;
    if (int rc = tsb_ring_geometry(r, &slots, nullptr, nullptr)) return rc;
    auto s = as_stream(stream);
    for (int i = 0; i < n; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        const int slot = (int)((q - 1) % (uint64_t)slots);
        if (int rc = tsb_ring_wait_ready(r, slot, q, stream)) return rc;
        if (ev && i == 0) TSB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[0]), s));
        if (ev && i == n - 1) TSB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[1]), s));
        if (int rc = tsb_ring_ack(r, consumer, q, stream)) return rc;
    }
    return TSB_OK;
}

int tsb_produce_group(tsb_ring *const *rings, int n_rings, int local, const tsb_produce_args *a,
                      int shard, int n_shards, uint64_t seq0, int64_t batch0, int n,
                      const int *live, const int *n_live, void *stream) {
    TSB_CHECK(rings && a && a->d_order && n_live, "null argument");
    TSB_CHECK(n_rings >= 1 && n_rings <= TSB_MAX_DST, "rings must be 1..%d", TSB_MAX_DST);
    TSB_CHECK(local >= 0 && local < n_rings, "bad local ring %d", local);
    TSB_CHECK(n_shards >= 1 && shard >= 0 && shard < n_shards, "bad shard %d/%d", shard, n_shards);
    TSB_CHECK(seq0 >= 1 && n >= 0 && batch0 >= 0, "bad range");
    TSB_CHECK(!a->d_crc, "per-batch CRC is not fused into the fan-out path");
    const int64_t b = a->batch_size;
    TSB_CHECK(b >= n_shards, "batch %lld smaller than the %d shards", (long long)b, n_shards);
    const size_t nbytes = (size_t)a->input_bytes + (a->with_target ? 8 * (size_t)b : 0);
    int slots = 0;
    size_t stride = 0;
    if (int rc = tsb_ring_geometry(rings[0], &slots, &stride, nullptr)) return rc;
    const int dev = ring_phys_device(rings[local]);
    int sys_fence = 0, n_live_total = 0;
    for (int k = 0; k < n_rings; ++k) {
        int sk = 0;
        size_t st = 0;
        TSB_CHECK(rings[k], "null ring %d", k);
        if (int rc = tsb_ring_geometry(rings[k], &sk, &st, nullptr)) return rc;
        TSB_CHECK(sk == slots && st >= nbytes, "ring %d: %d slots of %zu B (need %d of %zu B)", k,
                  sk, st, slots, nbytes);
        TSB_CHECK(ring_writers(rings[k]) == n_shards, "ring %d has %d writers, not %d shards", k,
                  ring_writers(rings[k]), n_shards);
        TSB_CHECK(ring_has_host_control(rings[k]), "ring %d needs a host control block", k);
        TSB_CHECK(n_live[k] >= 0, "bad live count");
        if (ring_phys_device(rings[k]) != dev) sys_fence = 1;
        n_live_total += n_live[k];
    }
    TSB_CHECK(live || n_live_total == 0, "null live list");
    // shard rows and their byte offsets inside a slot
    const int64_t s0 = shard * b / n_shards, s1 = (shard + 1) * b / n_shards, bs = s1 - s0;
    const int64_t out_sample = a->input_bytes / b;
    TSB_CHECK(out_sample * b == a->input_bytes, "input_bytes is not a whole number of samples");
    auto s = as_stream(stream);
    for (int i = 0; i < n; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        const int slot = (int)((q - 1) % (uint64_t)slots);
        // host flow gate: every ring's live consumers released the slot's previous batch
        if (q > (uint64_t)slots) {
            int off = 0;
            for (int k = 0; k < n_rings; ++k) {
                if (int rc = ring_host_gate(rings[k], live + off, n_live[k], q - (uint64_t)slots))
                    return rc;
                off += n_live[k];
            }
        }
        void *outs[TSB_MAX_DST];
        int64_t *tgts[TSB_MAX_DST];
        uint64_t *readys[TSB_MAX_DST];
        unsigned int *counter = nullptr;
        for (int k = 0; k < n_rings; ++k) {
            void *base = nullptr;
            if (int rc = tsb_ring_slot_ptr(rings[k], slot, &base)) return rc;
            uint8_t *b8 = static_cast<uint8_t *>(base);
            outs[k] = b8 + s0 * out_sample;
            tgts[k] = a->with_target ? reinterpret_cast<int64_t *>(b8 + a->input_bytes) + s0
                                     : nullptr;
            if (int rc = ring_publish_ptrs(rings[k], slot, shard, &readys[k],
                                           k == local ? &counter : nullptr))
                return rc;
        }
        const int64_t *idx = a->d_order + (batch0 + i) * b + s0;
        if (int rc = produce_multi(a->mode, a->src, idx, bs, a->h, a->w, a->c, a->pad, a->flip,
                                   a->seed, a->epoch, a->scale, a->bias, a->out_kind,
                                   a->sample_bytes, outs, tgts, readys, n_rings, counter, q,
                                   i > 0 || a->chain, sys_fence, stream))
            return rc;
    }
    (void)s;
    return TSB_OK;
}

int tsb_produce_group_multi(tsb_ring *const *rings, int n_rings, const tsb_produce_args *args,
                            const int *locals, const int *devices, void *const *streams,
                            int n_writers, uint64_t seq0, int64_t batch0, int n, const int *live,
                            const int *n_live) {
    TSB_CHECK(rings && args && locals && devices && streams && n_live, "null argument");
    TSB_CHECK(n_writers >= 1 && n_writers <= TSB_MAX_DST, "writers must be 1..%d", TSB_MAX_DST);
    int slots = 0;
    if (int rc = tsb_ring_geometry(rings[0], &slots, nullptr, nullptr)) return rc;
    int prev = 0;
    TSB_CUDA(cudaGetDevice(&prev));
    int no_live[TSB_MAX_DST] = {0};
    int rc = TSB_OK;
    for (int i = 0; i < n && rc == TSB_OK; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        if (q > (uint64_t)slots) {  // one host gate for the batch, over every ring
            int off = 0;
            for (int k = 0; k < n_rings && rc == TSB_OK; ++k) {
                rc = ring_host_gate(rings[k], live + off, n_live[k], q - (uint64_t)slots);
                off += n_live[k];
            }
        }
        for (int w = 0; w < n_writers && rc == TSB_OK; ++w) {
            if (cudaSetDevice(devices[w]) != cudaSuccess) {
                cudaGetLastError();
                set_error("cudaSetDevice(%d) failed", devices[w]);
                rc = TSB_ERR_CUDA;
                break;
            }
            tsb_produce_args a = args[w];
            a.chain = args[w].chain || i > 0;  // each writer's stream carries only its kernels
            rc = tsb_produce_group(rings, n_rings, locals[w], &a, w, n_writers, q, batch0 + i, 1,
                                   nullptr, no_live, streams[w]);
        }
    }
    cudaSetDevice(prev);
    return rc;
}

int tsb_restage_collate(tsb_ring *in_ring, int in_consumer, tsb_ring *out_ring,
                        const tsb_produce_args *a, uint64_t seq0, int n, const int *live,
                        int n_live, void *stream) {
    TSB_CHECK(in_ring && out_ring && a && a->ingest, "null argument (tables come from a->ingest)");
    TSB_CHECK(a->mode == TSB_SRC_AUGMENT, "stage 2 collates/augments the staged rows");
    TSB_CHECK(ring_has_host_control(in_ring) && ring_has_host_control(out_ring) &&
                  ring_writers(out_ring) == 1,
              "host-control rings; the output ring has one writer");
    TSB_CHECK(seq0 >= 1 && n >= 0, "bad range");
    const int64_t b = a->batch_size;
    const int64_t sb = a->sample_bytes;
    int in_slots = 0, out_slots = 0;
    size_t in_stride = 0, out_stride = 0;
    if (int rc = tsb_ring_geometry(in_ring, &in_slots, &in_stride, nullptr)) return rc;
    if (int rc = tsb_ring_geometry(out_ring, &out_slots, &out_stride, nullptr)) return rc;
    TSB_CHECK(in_stride >= (size_t)(b * sb + 8 * b), "input slot too small for %lld rows + targets",
              (long long)b);
    const size_t out_bytes = (size_t)a->input_bytes + (a->with_target ? 8 * (size_t)b : 0);
    TSB_CHECK(out_stride >= out_bytes, "output slot too small");
    uint8_t *in_base = nullptr;
    int64_t in_sstride = 0;
    uint64_t *in_ready = nullptr, *in_cursors = nullptr;
    unsigned int *in_counters = nullptr;
    ring_internals(in_ring, &in_base, &in_sstride, &in_ready, &in_cursors, &in_counters);
    for (int i = 0; i < n; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        const int islot = (int)((q - 1) % (uint64_t)in_slots);
        const int oslot = (int)((q - 1) % (uint64_t)out_slots);
        // every writer's shard of batch q is in the input slot (host-side wait,
        // bounded like the flow gate: TSB_GATE_TIMEOUT_S, default 600 s)
        static const int64_t wait_us =
            (int64_t)(1e6 * (getenv("TSB_GATE_TIMEOUT_S") ? atof(getenv("TSB_GATE_TIMEOUT_S"))
                                                          : 600.0));
        if (int rc = tsb_ring_host_wait_ready(in_ring, islot, q, wait_us)) return rc;
        if (q > (uint64_t)out_slots)
            if (int rc = ring_host_gate(out_ring, live, n_live, q - (uint64_t)out_slots)) return rc;
        void *in = nullptr, *out = nullptr;
        if (int rc = tsb_ring_slot_ptr(in_ring, islot, &in)) return rc;
        if (int rc = tsb_ring_slot_ptr(out_ring, oslot, &out)) return rc;
        const int64_t *ridx = reinterpret_cast<const int64_t *>(static_cast<uint8_t *>(in) + b * sb);
        uint64_t *ready = nullptr;
        unsigned int *counter = nullptr;
        if (int rc = ring_publish_ptrs(out_ring, oslot, 0, &ready, &counter)) return rc;
        int64_t *tgt = a->with_target
                           ? reinterpret_cast<int64_t *>(static_cast<uint8_t *>(out) + a->input_bytes)
                           : nullptr;
        // crop/flip keys are the staged target indices (the kernel derives the
        // params itself, no table kernel); the last CTA publishes the output slot
        // and releases the input slot (its cursor := q) once every CTA has read
        // its rows -- so the stream carries only these kernels, PDL-chained
        // with a->d_crc the batch CRC-32 comes from the collate kernel too (in
        // d_crc[oslot], and h_crc[oslot] if given, before the publish); where the
        // fused kernel does not take the geometry the CRC kernel follows the
        // publish, in stream order
        int crc_done = 0;
        if (int rc = collate_augment_publish(
                in, ingest_identity(a->ingest), b, a->h, a->w, a->c, a->pad, a->flip, a->seed,
                a->epoch, a->scale, a->bias, a->out_kind, out, tgt, ready, q, counter,
                (i > 0 || a->chain) ? 1 : 0, stream, nullptr, ridx, in_cursors + in_consumer,
                a->d_crc ? a->d_crc + oslot : nullptr, &crc_done,
                a->d_crc && a->h_crc ? a->h_crc + oslot : nullptr))
            return rc;
        if (a->d_crc && !crc_done)
            if (int rc = tsb_crc32(out, out_bytes, a->d_crc + oslot, nullptr, stream)) return rc;
    }
    return TSB_OK;
}

}  // extern "C"
