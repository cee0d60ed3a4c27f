/*
 * tsb200.h -- C ABI of the B200-native shared-loading data plane
 * (TensorSocket, arXiv 2409.18749; reference = /root/reference/pkg).
 *
 * Plain pointers, sizes and integer status codes only: no torch types.  Every
 * device operation is asynchronous on a caller-supplied cudaStream_t passed
 * as `void *stream` (NULL = legacy default stream).  Status: 0 = ok, < 0 =
 * error; tsb_last_error() returns a thread-local message.  The Python facade
 * (paper_2409_18749_b200/_lib.py) maps codes to the reference's exception
 * classes (payload.py:48-61).
 *
 * Which reference interface each entry point replaces is cited per function
 * (paths relative to /root/reference/pkg).
 */
#ifndef TSB200_H
#define TSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSB_OK 0
#define TSB_ERR_INVALID -1   /* ValueError            (payload.py:181-193)   */
#define TSB_ERR_CUDA -2      /* ResourceError         (payload.py:60-61)     */
#define TSB_ERR_STALE -3     /* StaleHandleError      (payload.py:52-53)     */
#define TSB_ERR_CORRUPT -4   /* CorruptSegmentError   (payload.py:56-57)     */
#define TSB_ERR_UNSUPPORTED -5

#define TSB_IPC_HANDLE_BYTES 64
/* max writers per ring (sharded ingest) and max fan-out destinations */
#define TSB_MAX_WRITERS 8
#define TSB_MAX_DST 8
/* cursor value of an evicted consumer / dropped retention (2^62) */
#define TSB_CURSOR_EVICTED 0x4000000000000000ULL

/* collate output kinds (NCHW); PASSTHROUGH keeps the sample bytes as-is */
#define TSB_OUT_U8 0
#define TSB_OUT_F32 1
#define TSB_OUT_BF16 2

/* ---- library / errors ---------------------------------------------------- */
const char *tsb_last_error(void);
int tsb_version(void);
int tsb_device_count(int *n);
int tsb_set_device(int dev);
int tsb_get_device(int *dev);
int tsb_device_info(int dev, int *sm_count, int *cc_major, int *cc_minor, size_t *hbm_bytes);
/* Load every kernel of the library into the current device's context now
 * (no lazy loading: a first launch must never wait for the device to go
 * idle while a stream is parked on a ring wait).  Called per device by the
 * ring constructors. */
int tsb_preload_kernels(void);

/* ---- memory & streams (plumbing; no torch) -------------------------------- */
int tsb_malloc(void **p, size_t bytes);                 /* device HBM */
int tsb_free(void *p);
int tsb_host_alloc(void **p, size_t bytes);             /* pinned + device-mapped */
int tsb_host_free(void *p);
int tsb_host_register(void *p, size_t bytes);           /* pin + map caller memory */
int tsb_host_unregister(void *p);
int tsb_host_device_ptr(void *host, void **dev);        /* device alias of pinned host */
int tsb_memcpy_async(void *dst, const void *src, size_t bytes, void *stream); /* cudaMemcpyDefault */
int tsb_memset_async(void *dst, int value, size_t bytes, void *stream);
int tsb_stream_create(void **stream);
int tsb_stream_destroy(void *stream);
int tsb_stream_sync(void *stream);
int tsb_device_sync(void);
int tsb_event_create(void **ev);
int tsb_event_destroy(void *ev);
int tsb_event_record(void *ev, void *stream);
int tsb_event_sync(void *ev);
int tsb_event_elapsed_ms(void *start, void *end, float *ms);
int tsb_stream_wait_event(void *stream, void *ev);
int tsb_enable_peer(int dev, int peer);                 /* cudaDeviceEnablePeerAccess */
int tsb_can_access_peer(int dev, int peer, int *can);

/* ---- RNG + shuffle (host native; reference kernels.py / pipeline.py) ---- */
/* kernels.py:40-45 */
uint64_t tsb_mix64(uint64_t x);
/* kernels.py:48-53 */
uint64_t tsb_derive_key(uint64_t seed, uint64_t epoch, uint64_t index);
/* kernels.py:170-178 (sequential Fisher-Yates; once per epoch) */
int tsb_permutation(int64_t n, uint64_t key, int64_t *out);
/* pipeline.py:113-123 */
int tsb_epoch_order(int64_t n, uint64_t shuffle_seed, uint64_t epoch, int reshuffle, int64_t *out);

/* ---- batch production kernels (replace pipeline.py:158-213 prepare_batch) */
/* Synthetic source (pipeline.py:183-189, kernels.py:112-121): sample s of the
 * batch = SplitMix64 stream keyed derive_key(seed, epoch, indices[s]).
 * d_indices: device int64[b]. */
int tsb_fill_synthetic(void *out, const int64_t *d_indices, int64_t b, uint64_t seed,
                       uint64_t epoch, int64_t sample_bytes, void *stream);
/* Store materialisation (pipeline.py:139-155 write_directory_dataset):
 * sample i = stream keyed derive_key(seed, 0, first + i). */
int tsb_make_store(void *out, uint64_t seed, int64_t first, int64_t count, int64_t sample_bytes,
                   void *stream);
/* Directory/store source collate (pipeline.py:190-210): out = concat of
 * src[indices[s]] for s < b.  src may be HBM or pinned host (device-mapped). */
int tsb_gather(const void *src, const int64_t *d_indices, int64_t b, int64_t sample_bytes,
               void *out, void *stream);
/* NEW (no reference; SURVEY.md §8a A6'): per-sample crop/flip params from
 * the reference RNG stream.  d_params: device int32[b][3] = (oy, ox, flip). */
int tsb_aug_params(uint64_t aug_seed, uint64_t epoch, const int64_t *d_indices, int64_t b,
                   int pad, int flip, int32_t *d_params, void *stream);
/* NEW fused collate/augment: uint8 HWC samples (HBM or pinned host) ->
 * pad/crop/flip -> normalise -> NCHW u8/f32/bf16 written into `out` (a ring
 * slot).  scale/bias: host float[c] (NULL = identity).  d_params: optional
 * device table from tsb_aug_params (NULL = derive in-kernel). */
int tsb_collate_augment(const void *src, const int64_t *d_indices, int64_t b, int h, int w,
                        int c, int pad, int flip, uint64_t aug_seed, uint64_t epoch,
                        const float *scale, const float *bias, int out_kind,
                        const int32_t *d_params, void *out, void *stream);

/* ---- integrity (wire.py:170-172 checksum; payload.py:218,362-364) ------- */
/* CRC-32/IEEE of n device bytes into *d_out (device uint32).  Needs a
 * device workspace of tsb_crc32_workspace_bytes() bytes. */
size_t tsb_crc32_workspace_bytes(void);
int tsb_crc32(const void *data, size_t n, uint32_t *d_out, void *d_workspace, void *stream);

/* ---- device batch ring (replaces payload.py:165-370 create/map/release
 *      and the producer ledger's release gate, producer.py:169-252) ------- */
typedef struct tsb_ring tsb_ring;
/* One HBM allocation: `slots` payload slots of slot_bytes + a control block
 * (ready word per slot, release cursor per consumer). */
int tsb_ring_create(int dev, int slots, size_t slot_bytes, int max_consumers, tsb_ring **out);
/* CUDA-IPC export for same-GPU consumer processes (64-byte handle). */
int tsb_ring_export(tsb_ring *r, void *handle_out);
int tsb_ring_import(const void *handle, int slots, size_t slot_bytes, int max_consumers,
                    tsb_ring **out);
/* Rings with `writers` > 1 (sharded ingest): slot s is complete when each of
 * the writers published it (one ready word per writer and slot). */
int tsb_ring_create_ex(int dev, int slots, size_t slot_bytes, int max_consumers, int writers,
                       tsb_ring **out);
int tsb_ring_import_ex(const void *handle, int slots, size_t slot_bytes, int max_consumers,
                       int writers, tsb_ring **out);
int tsb_ring_writers(tsb_ring *r, int *writers);
int tsb_ring_destroy(tsb_ring *r);
int tsb_ring_slot_ptr(tsb_ring *r, int slot, void **out);
int tsb_ring_base_ptr(tsb_ring *r, void **out);
int tsb_ring_geometry(tsb_ring *r, int *slots, size_t *slot_bytes, int *max_consumers);
/* Producer: ready[slot] = seq after all prior work on `stream` (release). */
int tsb_ring_publish(tsb_ring *r, int slot, uint64_t seq, void *stream);
/* Writer `writer`'s shard of the slot is complete (sharded ingest). */
int tsb_ring_publish_shard(tsb_ring *r, int slot, int writer, uint64_t seq, void *stream);
/* Consumer: `stream` waits until ready[slot] >= seq for every writer (acquire). */
int tsb_ring_wait_ready(tsb_ring *r, int slot, uint64_t seq, void *stream);
/* Consumer release (device-counted ack): cursor[consumer] = seq after all
 * prior work on `stream` (bs/consumer.py:330 Ack + release_view). */
int tsb_ring_ack(tsb_ring *r, int consumer, uint64_t seq, void *stream);
/* Producer gate before reusing a slot: `stream` waits until every consumer
 * in live[0..n_live) has cursor >= seq (producer.py:230-238 flow gate).
 * seq == 0 is a no-op. */
int tsb_ring_wait_free(tsb_ring *r, const int *live, int n_live, uint64_t seq, void *stream);
/* Host: cursor[consumer] = TSB_CURSOR_EVICTED so no device wait can wedge on
 * an evicted consumer (producer.py:255-269 evict_stale). */
int tsb_ring_evict(tsb_ring *r, int consumer);
/* Host: reset a consumer cursor (admission, producer.py:629-642). */
int tsb_ring_set_cursor(tsb_ring *r, int consumer, uint64_t value);
int tsb_ring_read_cursor(tsb_ring *r, int consumer, uint64_t *out);
int tsb_ring_read_ready(tsb_ring *r, int slot, uint64_t *out);
/* 1 = stream mem-ops (cuStreamWaitValue64), 0 = spin kernels. */
int tsb_ring_sync_mode(void);
/* Host-shared control block: the ready/cursor words move into caller host
 * memory (e.g. a POSIX shm segment every process maps), registered as
 * device-mapped; device memops then target host memory and host-side
 * readers/writers (evict, consumers that only map + ack) never touch a
 * GPU channel -- no cross-process GPU context switch per batch. */
size_t tsb_ring_control_bytes(int slots, int max_consumers);
size_t tsb_ring_control_bytes_ex(int slots, int max_consumers, int writers);
int tsb_ring_attach_host_control(tsb_ring *r, void *host_ctl, size_t bytes, int init);
/* Host flow gate (host control block): block the caller until every live
 * cursor has released `need` (wrap-around GEQ; evicted cursors pass).
 * timeout_us < 0 = forever; TSB_ERR_STALE on timeout.  A producer that gates
 * here keeps device waits out of its streams -- no stream is ever parked on
 * a value another stream of the same process has yet to write. */
int tsb_ring_host_gate(tsb_ring *r, const int *live, int n_live, uint64_t need,
                       int64_t timeout_us);
/* Native map-and-ack consumer loop (bs/cli.py:252-258): for n batches from
 * seq0, spin until the slot is ready, record the fetch time (CLOCK_MONOTONIC
 * us, t_us may be NULL) and release it. */
int tsb_ring_host_consume_range(tsb_ring *r, int consumer, uint64_t seq0, int n, int64_t *t_us);
/* Host consumer: spin until ready[slot] >= seq (timeout_us < 0 = forever). */
int tsb_ring_host_wait_ready(tsb_ring *r, int slot, uint64_t seq, int64_t timeout_us);

/* ---- fan-out + rebatch (NEW) -------------------------- */
/* Copy `bytes` from src into each of dsts[0..n_dst) (device or peer
 * pointers; P2P stores over NVLink/NVSwitch).  dsts: HOST array of n_dst
 * (<= 8) device pointers, passed to the kernel by value. */
int tsb_fanout(const void *src, void *const *dsts, int n_dst, size_t bytes, void *stream);
/* Fused: collate/augment written straight into n_dst (<= 8) destinations
 * (host array of device/peer pointers) -- collate + fan-out in one pass. */
int tsb_collate_augment_fanout(const void *src, const int64_t *d_indices, int64_t b, int h, int w,
                               int c, int pad, int flip, uint64_t aug_seed, uint64_t epoch,
                               const float *scale, const float *bias, int out_kind,
                               void *const *dsts, int n_dst, void *stream);
/* Rebatch gather: copy `count` samples starting at ring sample position
 * `first` (sample-granular ring of ring_samples samples of sample_bytes,
 * wrapping) into out. */
int tsb_rebatch_gather(const void *ring_base, int64_t ring_samples, int64_t sample_bytes,
                       int64_t first, int64_t count, void *out, void *stream);
/* Rebatch window (heterogeneous consumers): a consumer
 * batch = epoch-stream samples [first, first+count) of a producer whose
 * slots hold `per_slot` samples laid out [inputs][targets] (sl/abi.py:27-31
 * pair layout).  slots[0..n_slots) = bases of the producer slots the window
 * touches, in stream order (slot 0 holds sample first).  out = [count
 * inputs][count targets].  Used when the window straddles producer slots;
 * windows inside one slot are zero-copy views. */
int tsb_rebatch_window(const void *const *slots, int n_slots, int64_t first, int64_t count,
                       int64_t per_slot, int64_t in_sample_bytes, int64_t tgt_sample_bytes,
                       void *out, void *stream);

/* ---- native producer/consumer loops (replace the per-batch host work of
 *      Producer._try_announce, producer.py:506-534, and
 *      ConsumerSession.next_batch, consumer.py:286-338) ------------------- */
#define TSB_SRC_AUGMENT 0   /* store -> fused collate/augment            */
#define TSB_SRC_GATHER 1    /* store -> passthrough gather (DirectorySource) */
#define TSB_SRC_SYNTHETIC 2 /* SplitMix64 generator (SyntheticSource)    */
/* Staged PCIe ingest for pinned-host stores (double-buffered
 * HBM staging; one gather kernel per batch reads the mapped pinned rows). */
typedef struct tsb_ingest tsb_ingest;
int tsb_ingest_create(int dev, int64_t max_batch, int64_t sample_bytes, int depth,
                      tsb_ingest **out);
int tsb_ingest_destroy(tsb_ingest *g);
/* 1 if the batched-copy driver API is in use, 0 if per-sample copies. */
int tsb_ingest_batch_api(tsb_ingest *g, int *used);
/* Host->device bytes this ingest has enqueued so far (sample rows + index and
 * parameter uploads).  Augment batches copy only the source rows the crop
 * reads: h - |oy - pad| of the h rows of each sample. */
int tsb_ingest_bytes(tsb_ingest *g, uint64_t *bytes);

/* JPEG sample source (NEW; the paper's decode step, in
 * front of the reference's DirectorySource, pipeline.py:45-54,190-210):
 * nvJPEG batched decode (NVJPG hardware engines when available) of a store
 * of encoded files held in host memory, to interleaved RGB u8 in HBM.
 * libnvjpeg is opened at run time (TSB_ERR_UNSUPPORTED when absent). */
typedef struct tsb_jpeg tsb_jpeg;
int tsb_jpeg_available(int *ok);
/* backend: 0 = hardware (NVJPG) if present, else GPU-assisted Huffman, else
 * default; 1 = default (hybrid); 2 = hardware only */
int tsb_jpeg_create(int dev, int64_t max_batch, int h, int w, int backend, tsb_jpeg **out);
int tsb_jpeg_backend(tsb_jpeg *j, int *backend);  /* 1 = default, 2 = hardware, 3 = GPU Huffman */
/* The store: files[i] / lengths[i] = encoded sample i (host memory the
 * caller keeps alive); every file must decode to h x w. */
int tsb_jpeg_attach_store(tsb_jpeg *j, const uint8_t *const *files, const size_t *lengths,
                          int64_t n);
/* Decode files h_indices[0..b) into out (b x h*w*3 u8 RGB, device) on stream. */
int tsb_jpeg_decode(tsb_jpeg *j, const int64_t *h_indices, int64_t b, void *out, void *stream);
int tsb_jpeg_destroy(tsb_jpeg *j);

typedef struct {
    int mode;                /* TSB_SRC_*                                     */
    const void *src;         /* store base: HBM or pinned host (NULL synthetic) */
    const int64_t *d_order;  /* device int64 epoch order (pipeline.py:113-123) */
    int64_t batch_size;
    int64_t sample_bytes;    /* raw sample bytes                              */
    int h, w, c, pad, flip, out_kind;
    uint64_t seed;           /* augment seed / synthetic source seed         */
    uint64_t epoch;
    float scale[4], bias[4]; /* normalisation (identity: 1, 0)               */
    int with_target;         /* append int64 sample indices after the input  */
    int64_t input_bytes;     /* bytes of the input part of a slot            */
    uint32_t *d_crc;         /* optional device uint32[slots]: batch CRC-32   */
    int wait_stride;         /* device gate: wait on the cursors every k batches
                                (<=1: every batch); effective depth slots - k + 1 */
    int gate;                /* TSB_GATE_DEVICE: the stream waits on the cursors
                                (the calling thread never blocks).  TSB_GATE_HOST
                                (rings with a host control block): the calling
                                thread blocks until the slot is free, the stream
                                carries only kernels and consecutive fused batches
                                chain with programmatic dependent launch */
    tsb_ingest *ingest;      /* non-null (with h_order, src = pinned host store):
                                each batch's sample rows cross PCIe by the copy
                                engine into HBM staging first (augment), or
                                straight into the slot (gather) */
    const int64_t *h_order;  /* host copy of d_order (row addresses for ingest) */
    int persistent;          /* 1 (host-control single-writer ring): the whole
                                range is ONE cooperative persistent launch whose
                                CTAs gate on the release cursors themselves -- no
                                host launch per batch.  Passthrough modes; and the
                                augment mode with d_crc when the fused collate +
                                CRC kernel takes the geometry (each slot's CRC is
                                in d_crc / h_crc before its ready word; other
                                augment geometries run per batch).  Consumers must
                                not need this process's SMs to release slots. */
    int chain;               /* 1: the previous operation on `stream` was a fused
                                produce kernel (so the call's first batch may chain
                                with programmatic dependent launch too) */
    tsb_jpeg *jpeg;          /* non-null (with h_order): samples are JPEG files,
                                decoded per batch into HBM staging (augment) or
                                straight into the slot (gather); src unused */
    uint32_t *h_crc;         /* optional host-mapped (pinned) uint32[slots]: where
                                the batch CRC-32 is computed inside the collate
                                kernel, it is also stored here before the slot's
                                ready word, so a host that sees ready[slot] == q
                                reads it with no copy */
    int *crc_fused;          /* optional out: 1 if every batch of the call got its
                                CRC inside the collate kernel (d_crc / h_crc hold
                                it when the slot is published), else 0 */
    int64_t order_epochs;    /* persistent passthrough only (<= 1 elsewhere): d_order
                                holds this many consecutive epochs' orders
                                (epoch, epoch + 1, ...), order_stride entries
                                apart, and the range may run past the epoch's
                                epoch_len batches into the following epochs --
                                ONE launch across epoch boundaries */
    int64_t epoch_len;       /* batches per epoch (order_epochs > 1)         */
    int64_t order_stride;    /* int64 entries per epoch order (order_epochs > 1) */
} tsb_produce_args;
#define TSB_GATE_DEVICE 0
#define TSB_GATE_HOST 1
/* Enqueue batches batch0..batch0+n-1 of one epoch (global seq seq0..) on
 * `stream`: per batch wait_free(live, q - slots) -> produce into slot ->
 * [crc] -> publish(slot, q).  ev: NULL or 2n events recorded around each
 * batch's production kernel (for per-launch timing). */
int tsb_produce_range(tsb_ring *r, const tsb_produce_args *a, uint64_t seq0, int64_t batch0,
                      int n, const int *live, int n_live, void **ev, void *stream);
/* Consumer: per batch q in seq0..seq0+n-1: wait_ready -> ack (a consumer
 * that maps and releases, bs/cli.py:252-258).  ev: NULL or 2 events recorded
 * after the first and after the last ready wait. */
int tsb_consume_range(tsb_ring *r, int consumer, uint64_t seq0, int n, void **ev, void *stream);

/* Sharded ingest + fused fan-out (NEW, the data "broadcast"
 * of bs/consumer.py:319-321 across GPUs).  Writer `shard` of `n_shards`
 * produces rows [shard*B/n_shards, (shard+1)*B/n_shards) of every batch and
 * stores them straight into the same slot of each of rings[0..n_rings)
 * (<= TSB_MAX_DST): its own device's ring and peer rings opened over CUDA
 * IPC, i.e. P2P stores over NVLink/NVSwitch -- the all-gather is fused into
 * the producing kernel.  The kernel's last CTA publishes ready[slot][shard]
 * in every ring.  rings[local] lives on the launching device (its completion
 * counters are used).  live = the concatenated live-cursor lists of the
 * rings, n_live[i] entries for ring i; the gate is on the host, so every
 * ring needs a host control block.  Each ring must have n_shards writers.
 * n_shards == 1 with several rings is the single-producer star.  Modes:
 * TSB_SRC_AUGMENT (fused collate/augment), TSB_SRC_GATHER, TSB_SRC_SYNTHETIC
 * (sample_bytes a multiple of 16 for the last two).  Consecutive batches
 * are chained with programmatic dependent launch. */
int tsb_produce_group(tsb_ring *const *rings, int n_rings, int local, const tsb_produce_args *a,
                      int shard, int n_shards, uint64_t seq0, int64_t batch0, int n,
                      const int *live, const int *n_live, void *stream);
/* Two-stage multi-GPU production, stage 2 (NEW): stage 1 is
 * tsb_produce_group in TSB_SRC_GATHER mode into per-GPU INPUT rings (the
 * compact u8 rows cross NVLink: 1x the input instead of the 2-4x larger
 * f32/bf16 outputs), target = the real sample indices.  Stage 2, per GPU,
 * for each batch q: host-wait until every writer's shard is in in_ring,
 * host-gate out_ring's slot on its live consumers, then one PDL-chained
 * kernel collates/augments the staged rows into out_ring's slot (crop/flip
 * keyed by the staged target indices, derived in-kernel); its last CTA
 * publishes the output slot and releases the input slot (in_ring cursor
 * in_consumer := q).  a: augment geometry of the OUTPUT, a->ingest for the
 * identity table, a->chain = the stream's previous op was this call's
 * kernel; a->d_crc (optional, [out slots]): the output slot's CRC-32, from
 * the same kernel when it takes the geometry (also into a->h_crc if set),
 * else from a CRC kernel after the publish. */
int tsb_restage_collate(tsb_ring *in_ring, int in_consumer, tsb_ring *out_ring,
                        const tsb_produce_args *a, uint64_t seq0, int n, const int *live,
                        int n_live, void *stream);
/* One process driving every writer (TensorProducer(devices=...)): for each
 * of n batches, one host gate over all rings, then writer w (of n_writers =
 * the shard count) produces its shard on devices[w] / streams[w] with
 * args[w] (its device's order and store pointers) into all rings;
 * rings[locals[w]] is the ring on devices[w].  One call per batch range
 * instead of one per writer and batch. */
int tsb_produce_group_multi(tsb_ring *const *rings, int n_rings, const tsb_produce_args *args,
                            const int *locals, const int *devices, void *const *streams,
                            int n_writers, uint64_t seq0, int64_t batch0, int n, const int *live,
                            const int *n_live);

/* ---- control-plane codec (host; wire.py:1-11,77-156,199-341) ------------
 * The reference's 9-message frame format, byte-identical, plus DType 5 (bf16)
 * and Join v2 (device, batch_size).  One struct carries every kind; unused
 * fields are ignored on encode and zero (device = -1) on decode. */
#define TSB_MSG_JOIN 1
#define TSB_MSG_WELCOME 2
#define TSB_MSG_ANNOUNCE 3
#define TSB_MSG_ACK 4
#define TSB_MSG_HEARTBEAT 5
#define TSB_MSG_EPOCH_START 6
#define TSB_MSG_EPOCH_END 7
#define TSB_MSG_BYE 8
#define TSB_MSG_SHUTDOWN 9
typedef struct {
    uint8_t kind;
    uint64_t consumer_id;
    uint16_t protocol_version;
    int16_t device;              /* Join v2 */
    uint32_t batch_size;         /* Join v2 */
    uint32_t epoch;
    uint64_t epoch_len;
    uint64_t next_batch_index;
    uint16_t buffer_depth;
    uint8_t admitted;
    uint64_t batch_index;
    uint64_t monotonic_millis;
    uint16_t name_len;
    char segment_name[256];
    uint64_t byte_len;
    uint8_t dtype;
    uint8_t ndim;
    uint64_t shape[8];
    uint32_t checksum;
} tsb_msg;
/* Encode one frame into out[0..cap); *len = frame bytes.  TSB_ERR_INVALID on
 * a wire-invariant violation (EncodeError, wire.py:33-38). */
int tsb_wire_encode(const tsb_msg *m, uint8_t *out, size_t cap, size_t *len);
/* Decode exactly one complete frame; TSB_ERR_CORRUPT with *err_off = the
 * failing byte offset (DecodeError(offset, cause), wire.py:41-46). */
int tsb_wire_decode(const uint8_t *frame, size_t len, tsb_msg *m, size_t *err_off);

/* ---- native control-plane hub (bs/producer.py:379-438 readers + broadcast) --
 * One epoll thread reads every admitted consumer's aggregate socket and
 * decodes Ack / Heartbeat / Bye frames natively; the producer drains them
 * in bulk.  tsb_hub_broadcast writes one frame to many sockets.  The caller
 * keeps owning the fds (remove before closing). */
typedef struct tsb_hub tsb_hub;
typedef struct {
    uint8_t kind;          /* TSB_MSG_ACK / _HEARTBEAT / _BYE, or 0 = connection closed */
    uint64_t consumer_id;  /* from the frame (0 for kind 0) */
    uint32_t epoch;
    uint64_t batch_index;
    int64_t t_us;          /* CLOCK_MONOTONIC at receipt */
    int32_t fd;
} tsb_hub_event;
int tsb_hub_create(tsb_hub **out);
/* Start reading fd for consumer_id; `pending` = bytes already read from it. */
int tsb_hub_add(tsb_hub *h, int fd, uint64_t consumer_id, const uint8_t *pending, size_t n);
int tsb_hub_remove(tsb_hub *h, int fd);
int tsb_hub_drain(tsb_hub *h, tsb_hub_event *out, int cap, int *n);
/* Blocking sends of one frame to fds[0..n); failed[i] = 1 on error (peer gone). */
int tsb_hub_broadcast(const int *fds, int n, const uint8_t *frame, size_t len, int *failed);
int tsb_hub_destroy(tsb_hub *h);
/* The reference's flow gate on received wire Acks (bs/producer.py:230-238,
 * sl/producer.py:291-294: announce while fewer than buffer_depth batches await
 * acks).  The hub keeps, per consumer id, the highest acked 1-based global
 * seq (epoch * epoch_len + batch_index + 1) of every Ack it decodes.
 * set_acked assigns (admission baseline, or a sentinel >= 2^61 on drop);
 * wait_acked blocks until every listed consumer acked >= need: TSB_OK, or
 * TSB_ERR_STALE after timeout_us (< 0: no timeout).  read_acked: 0 if unknown. */
int tsb_hub_set_epoch_len(tsb_hub *h, uint64_t epoch_len);
int tsb_hub_set_acked(tsb_hub *h, uint64_t consumer_id, uint64_t seq);
int tsb_hub_read_acked(tsb_hub *h, uint64_t consumer_id, uint64_t *seq);
int tsb_hub_wait_acked(tsb_hub *h, const uint64_t *consumer_ids, int n, uint64_t need,
                       int64_t timeout_us);
/* Largest max - min acked seq seen over the registered consumers (those given
 * a baseline by set_acked, sentinel entries excluded) at any Ack: the
 * reference's drift statistic, sampled at every Ack. */
int tsb_hub_drift_max(tsb_hub *h, uint64_t *drift);

/* ---- the facade producer's per-batch host path (sl/producer.py:279-316) ----
 * For one GPU and a device loader: tsb_facade_produce = the flow gate on the
 * hub's acked seqs (>= seq - depth, TSB_ERR_STALE after timeout_us) +
 * tsb_produce_range(ring, args, seq, index, 1, live) (+ the batch CRC's
 * read-back into h_crc[slot] and events[slot] when d_crc is set);
 * tsb_facade_announce = (wait for the CRC) + the 80-byte segment header with
 * epoch / crc / index patched into `header80`, base64 in the slot name
 * "tsb1:<ring_id hex>:<slot>:<b64>", one Announce frame written to every fd
 * (failed[i] = 1 for a socket that failed). */
typedef struct tsb_facade tsb_facade;
int tsb_facade_create(tsb_facade **out);
int tsb_facade_destroy(tsb_facade *f);
int tsb_facade_set_batch(tsb_facade *f, tsb_hub *hub, tsb_ring *ring, const tsb_produce_args *a,
                         void *stream, int depth, uint64_t ring_id, const uint8_t *header80,
                         uint64_t nbytes, uint32_t *d_crc, uint32_t *h_crc, void *const *events,
                         int slots);
int tsb_facade_set_consumers(tsb_facade *f, const uint64_t *ack_ids, int n_ack, const int *live,
                             int n_live, const int *fds, int n_fds);
int tsb_facade_produce(tsb_facade *f, uint64_t seq, int64_t index, int chain, int64_t timeout_us);
int tsb_facade_announce(tsb_facade *f, uint64_t seq, uint32_t epoch, uint64_t index,
                        int with_crc, uint32_t *crc_out, int *failed);
/* produce(seq) then, if ann_seq != 0, announce(ann_seq): one call per batch. */
int tsb_facade_step(tsb_facade *f, uint64_t seq, int64_t index, int chain, int64_t timeout_us,
                    uint64_t ann_seq, uint32_t ann_epoch, uint64_t ann_index, int ann_with_crc,
                    uint32_t *crc_out, int *failed);

#ifdef __cplusplus
}
#endif
#endif /* TSB200_H */
