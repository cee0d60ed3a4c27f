// The facade producer's per-batch host path behind two native calls.
//
// TensorProducer._publish (sl/producer.py:279-316 in the reference: flow
// gate -> create_segment -> CRC -> Announce to every consumer) costs ~70 us
// of Python per batch, twice the 29 us the fused collate takes on the GPU
// (profiles/r2/facade_rate_*.json).  For the common case -- one GPU, a
// device loader (CollateLoader), host-shared control words -- the steps
// that run per batch move here:
//   tsb_facade_produce:  the reference's flow gate on received wire Acks
//                        (hub acked seqs >= q - buffer_depth), then the fused
//                        producer launch with its slot-reuse gate on the
//                        release cursors (tsb_produce_range).  With a checksum
//                        the collate kernel stores the batch CRC in host-mapped
//                        memory before it publishes the slot (no copy, and the
//                        next launch still chains); where the kernel cannot
//                        (unfused geometries), the CRC's 4-byte read-back + an
//                        event follow the launch;
//   tsb_facade_announce: wait for that batch's CRC (if any: its ready word, or
//                        the event), patch the 80-byte
//                        segment header (epoch, crc, batch_index), base64 it
//                        into the slot name, encode the Announce frame with
//                        the native codec and write it to every consumer
//                        socket (tsb_hub_broadcast).
// The consumer lists (ack-gate ids, live cursors, sockets) are set only when
// they change; Python keeps admission, retention and the ledger.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tsb200.h"

namespace tsb {
void set_error(const char *fmt, ...);
}

struct tsb_facade {
    tsb_hub *hub = nullptr;
    tsb_ring *ring = nullptr;
    tsb_produce_args args{};
    void *stream = nullptr;
    int depth = 2;
    int slots = 1;
    uint64_t ring_id = 0;
    uint8_t header[80] = {0};
    uint64_t nbytes = 0;
    uint32_t *d_crc = nullptr;
    uint32_t *h_crc = nullptr;
    std::vector<cudaEvent_t> events;
    std::vector<uint8_t> fused;  // per slot: the CRC came from the kernel (host-mapped)
    bool tail_kernel = false;    // the stream's last operation is a fused produce kernel
    // TSB_FACADE_STATS=1: time spent in the ack gate, the launch and the CRC wait
    double t_gate = 0, t_launch = 0, t_crc = 0, t_bcast = 0;
    uint64_t n_steps = 0;
    std::vector<uint64_t> ack_ids;
    std::vector<int> live;
    std::vector<int> fds;
};

namespace {
inline double now_us() {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
const char B64[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";

size_t b64_encode(const uint8_t *in, size_t n, char *out) {  // standard alphabet, padded
    size_t o = 0;
    for (size_t i = 0; i < n; i += 3) {
        const uint32_t b0 = in[i], b1 = i + 1 < n ? in[i + 1] : 0, b2 = i + 2 < n ? in[i + 2] : 0;
        const uint32_t v = (b0 << 16) | (b1 << 8) | b2;
        out[o++] = B64[(v >> 18) & 63];
        out[o++] = B64[(v >> 12) & 63];
        out[o++] = i + 1 < n ? B64[(v >> 6) & 63] : '=';
        out[o++] = i + 2 < n ? B64[v & 63] : '=';
    }
    return o;
}
}  // namespace

extern "C" {

int tsb_facade_create(tsb_facade **out) {
    if (!out) return TSB_ERR_INVALID;
    *out = new tsb_facade{};
    return TSB_OK;
}

int tsb_facade_destroy(tsb_facade *f) {
    if (f && getenv("TSB_FACADE_STATS") && f->n_steps)
        fprintf(stderr,
                "facade stats: %llu steps, per step us: gate %.2f launch %.2f crc-wait %.2f "
                "announce %.2f\n",
                (unsigned long long)f->n_steps, f->t_gate / f->n_steps, f->t_launch / f->n_steps,
                f->t_crc / f->n_steps, f->t_bcast / f->n_steps);
    delete f;
    return TSB_OK;
}

int tsb_facade_set_batch(tsb_facade *f, tsb_hub *hub, tsb_ring *ring, const tsb_produce_args *a,
                         void *stream, int depth, uint64_t ring_id, const uint8_t *header80,
                         uint64_t nbytes, uint32_t *d_crc, uint32_t *h_crc, void *const *events,
                         int slots) {
    if (!f || !hub || !ring || !a || !header80 || depth < 1 || slots < 1) {
        tsb::set_error("facade: bad batch setup");
        return TSB_ERR_INVALID;
    }
    f->hub = hub;
    f->ring = ring;
    f->args = *a;
    f->stream = stream;
    f->depth = depth;
    f->ring_id = ring_id;
    memcpy(f->header, header80, 80);
    f->nbytes = nbytes;
    f->d_crc = d_crc;
    f->h_crc = h_crc;
    f->slots = slots;
    f->events.assign(slots, nullptr);
    if (d_crc) {
        if (!h_crc || !events) {
            tsb::set_error("facade: a checksum needs a host mirror and per-slot events");
            return TSB_ERR_INVALID;
        }
        for (int i = 0; i < slots; ++i) f->events[i] = static_cast<cudaEvent_t>(events[i]);
    }
    f->args.d_crc = d_crc;
    f->args.h_crc = d_crc ? h_crc : nullptr;  // pinned: device-accessible under UVA
    f->fused.assign(slots, 0);
    f->tail_kernel = false;
    return TSB_OK;
}

int tsb_facade_set_consumers(tsb_facade *f, const uint64_t *ack_ids, int n_ack, const int *live,
                             int n_live, const int *fds, int n_fds) {
    if (!f || n_ack < 0 || n_live < 0 || n_fds < 0) return TSB_ERR_INVALID;
    f->ack_ids.assign(ack_ids, ack_ids + n_ack);
    f->live.assign(live, live + n_live);
    f->fds.assign(fds, fds + n_fds);
    return TSB_OK;
}

int tsb_facade_produce(tsb_facade *f, uint64_t seq, int64_t index, int chain, int64_t timeout_us) {
    if (!f || !f->ring) return TSB_ERR_INVALID;
    static const bool stats = getenv("TSB_FACADE_STATS") != nullptr;
    const double t0 = stats ? now_us() : 0;
    if (seq > (uint64_t)f->depth) {  // fewer than buffer_depth announced batches await acks
        const int rc = tsb_hub_wait_acked(f->hub, f->ack_ids.data(), (int)f->ack_ids.size(),
                                          seq - (uint64_t)f->depth, timeout_us);
        if (rc) return rc;  // TSB_ERR_STALE: timed out (the caller re-checks for shutdown)
    }
    const double t1 = stats ? now_us() : 0;
    int fused = 0;
    f->args.chain = chain && f->tail_kernel;
    f->args.crc_fused = &fused;
    int rc = tsb_produce_range(f->ring, &f->args, seq, index, 1, f->live.data(),
                               (int)f->live.size(), nullptr, f->stream);
    f->args.crc_fused = nullptr;
    if (stats) {
        const double t2 = now_us();
        f->t_gate += t1 - t0;
        f->t_launch += t2 - t1;
        ++f->n_steps;
    }
    if (rc) return rc;
    f->tail_kernel = !f->d_crc || fused;
    if (f->d_crc) {
        const int slot = (int)((seq - 1) % (uint64_t)f->slots);
        f->fused[slot] = (uint8_t)fused;
        if (fused) return TSB_OK;  // the CRC is in h_crc[slot] when the slot is published
        auto s = static_cast<cudaStream_t>(f->stream);
        cudaError_t e = cudaMemcpyAsync(f->h_crc + slot, f->d_crc + slot, 4,
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(f->events[slot], s);
        if (e != cudaSuccess) {
            tsb::set_error("facade: checksum read-back: %s", cudaGetErrorString(e));
            return TSB_ERR_CUDA;
        }
    }
    return TSB_OK;
}

int tsb_facade_announce(tsb_facade *f, uint64_t seq, uint32_t epoch, uint64_t index,
                        int with_crc, uint32_t *crc_out, int *failed) {
    if (!f || !f->ring) return TSB_ERR_INVALID;
    const int slot = (int)((seq - 1) % (uint64_t)f->slots);
    uint32_t crc = 0;
    static const bool stats = getenv("TSB_FACADE_STATS") != nullptr;
    const double t0 = stats ? now_us() : 0;
    if (with_crc && f->d_crc) {
        if (f->fused[slot]) {  // the kernel stored the CRC before the slot's ready word
            if (int rc = tsb_ring_host_wait_ready(f->ring, slot, seq, 60 * 1000000ll)) return rc;
            crc = reinterpret_cast<volatile uint32_t *>(f->h_crc)[slot];
        } else {
            const cudaError_t e = cudaEventSynchronize(f->events[slot]);
            if (e != cudaSuccess) {
                tsb::set_error("facade: checksum wait: %s", cudaGetErrorString(e));
                return TSB_ERR_CUDA;
            }
            crc = f->h_crc[slot];
        }
    }
    const double t1 = stats ? now_us() : 0;
    // the segment header (payload.py:220-233): epoch u32 @8, crc u32 @12, index u64 @16
    uint8_t hdr[80];
    memcpy(hdr, f->header, 80);
    memcpy(hdr + 8, &epoch, 4);
    memcpy(hdr + 12, &crc, 4);
    memcpy(hdr + 16, &index, 8);
    tsb_msg m{};
    m.kind = TSB_MSG_ANNOUNCE;
    m.epoch = epoch;
    m.batch_index = index;
    int n = snprintf(m.segment_name, sizeof m.segment_name, "tsb1:%llx:%d:",
                     (unsigned long long)f->ring_id, slot);
    n += (int)b64_encode(hdr, 80, m.segment_name + n);
    m.name_len = (uint16_t)n;
    m.byte_len = f->nbytes;
    m.dtype = 0;  // announced as a flat byte blob (sl/producer.py:300-306)
    m.ndim = 1;
    m.shape[0] = f->nbytes;
    m.checksum = crc;
    uint8_t frame[512];
    size_t len = 0;
    if (int rc = tsb_wire_encode(&m, frame, sizeof frame, &len)) return rc;
    if (int rc = tsb_hub_broadcast(f->fds.data(), (int)f->fds.size(), frame, len, failed))
        return rc;
    if (stats) {
        f->t_crc += t1 - t0;
        f->t_bcast += now_us() - t1;
    }
    if (crc_out) *crc_out = crc;
    return TSB_OK;
}

int tsb_facade_step(tsb_facade *f, uint64_t seq, int64_t index, int chain, int64_t timeout_us,
                    uint64_t ann_seq, uint32_t ann_epoch, uint64_t ann_index, int ann_with_crc,
                    uint32_t *crc_out, int *failed) {
    if (int rc = tsb_facade_produce(f, seq, index, chain, timeout_us)) return rc;
    if (!ann_seq) return TSB_OK;
    return tsb_facade_announce(f, ann_seq, ann_epoch, ann_index, ann_with_crc, crc_out, failed);
}

}  // extern "C"
