// Device batch ring: HBM slots + device-resident ready words and per-consumer
// release cursors ("acks counted on the device").
//
// Replaces the reference transport seam (payload.py:165-370: one POSIX shm
// segment per batch, unlinked on release) and the data-path half of the
// producer ledger (producer.py:169-252: release when every admitted consumer
// acked; announce gate while fewer than buffer_depth are pending).
//
//   producer stream:  wait_free(slot's previous seq) -> collate -> publish(seq)
//   consumer stream:  wait_ready(seq) -> <use the zero-copy view> -> ack(seq)
//
// Synchronisation is entirely on device streams: CUDA stream memory
// operations (cuStreamWaitValue64 / cuStreamWriteValue64, executed by the
// GPU front end without occupying SMs -- they also work across processes
// on the same GPU, where kernels are time-sliced) with spin kernels as the
// device-side alternative.  Host threads only enqueue; eviction writes a
// +inf cursor so no wait can wedge on a dead consumer (producer.py:255-269).
#include <cuda.h>
#include <stdlib.h>
#include <time.h>

#include <mutex>

#include "tsb_common.cuh"

using namespace tsb;

struct tsb_ring {
    int dev;
    int slots;
    size_t slot_bytes;
    size_t slot_stride;
    int max_consumers;
    int writers;       // ready words per slot (sharded ingest: one per writer)
    int phys_dev;      // device whose HBM holds the ring (!= dev for a peer import)
    uint8_t *base;
    uint64_t *ready;   // [slots][writers] device-visible address (memops)
    uint64_t *cursor;  // [max_consumers]  device-visible address (memops)
    uint64_t *h_ctl;   // host view of a host-shared control block (or null)
    unsigned int *counters;  // [slots] device completion counters (fused publish)
    size_t total;
    bool imported;
    cudaStream_t host_stream;  // private non-blocking stream for host pokes
};

namespace {

typedef CUresult (*PFN_wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_devattr)(int *, CUdevice_attribute, CUdevice);

PFN_wait64 g_wait64 = nullptr;
PFN_write64 g_write64 = nullptr;
int g_mode = -1;  // 1 memops, 0 kernels
std::mutex g_mu;

int resolve_mode() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_mode >= 0) return g_mode;
    g_mode = 0;
    const char *env = getenv("TSB_SYNC");
    if (env && env[0] == 'k') return g_mode;  // TSB_SYNC=kernel forces spin kernels
    cudaDriverEntryPointQueryResult q1, q2, q3;
    void *w = nullptr, *wr = nullptr, *da = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWriteValue64", &wr, cudaEnableDefault, &q2) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuDeviceGetAttribute", &da, cudaEnableDefault, &q3) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess ||
        q3 != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return g_mode;
    }
    int dev = 0, ok = 0;
    cudaGetDevice(&dev);
    if (reinterpret_cast<PFN_devattr>(da)(&ok, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS,
                                          (CUdevice)dev) != CUDA_SUCCESS)
        ok = 0;
    if (ok) {
        g_wait64 = reinterpret_cast<PFN_wait64>(w);
        g_write64 = reinterpret_cast<PFN_write64>(wr);
        g_mode = 1;
    }
    return g_mode;
}

// ---- spin-kernel path ------------------------------------------------------
constexpr int MAX_WAIT = 64;
struct WaitSet {
    const uint64_t *addr[MAX_WAIT];
    int n;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void signal_kernel(uint64_t *addr, uint64_t value) {
    __threadfence_system();
    st_release_sys(addr, value);
}

__global__ void wait_kernel(WaitSet set, uint64_t value) {
    const int i = threadIdx.x;
    if (i < set.n) {
        while (ld_acquire_sys(set.addr[i]) < value) __nanosleep(128);
    }
    __syncthreads();
    __threadfence_system();
}

// Driver-API stream memops need a current context on the calling thread;
// runtime calls create it lazily, so bind the ring's device first -- and give
// the caller's current device back afterwards (a multi-GPU producer thread
// must not find its current device switched under it by a ring operation).
struct DeviceGuard {
    int prev = -1;
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
int bind_ctx(int dev, DeviceGuard &guard) {
    static thread_local uint64_t ready_mask = 0;  // devices whose context this thread made current
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) {
        TSB_CUDA(cudaSetDevice(dev));
        guard.prev = cur;
    }
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (!(ready_mask & bit)) {
        TSB_CUDA(cudaFree(nullptr));  // no-op that makes the primary context current
        ready_mask |= bit;
    }
    return TSB_OK;
}

int dev_write(tsb_ring *r, uint64_t *addr, uint64_t v, void *stream) {
    if (resolve_mode() == 1) {
        DeviceGuard guard;
        if (int rc = bind_ctx(r->dev, guard)) return rc;
        CUresult e = g_write64((CUstream)stream, (CUdeviceptr)addr, v, 0);
        if (e != CUDA_SUCCESS) {
            set_error("cuStreamWriteValue64 failed (%d)", (int)e);
            return TSB_ERR_CUDA;
        }
        return TSB_OK;
    }
    (void)r;
    signal_kernel<<<1, 1, 0, as_stream(stream)>>>(addr, v);
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

int dev_wait(tsb_ring *r, const uint64_t *const *addrs, int n, uint64_t v, void *stream) {
    if (n <= 0) return TSB_OK;
    if (resolve_mode() == 1) {
        DeviceGuard guard;
        if (int rc = bind_ctx(r->dev, guard)) return rc;
        for (int i = 0; i < n; ++i) {
            CUresult e = g_wait64((CUstream)stream, (CUdeviceptr)addrs[i], v,
                                  CU_STREAM_WAIT_VALUE_GEQ);
            if (e != CUDA_SUCCESS) {
                set_error("cuStreamWaitValue64 failed (%d)", (int)e);
                return TSB_ERR_CUDA;
            }
        }
        return TSB_OK;
    }
    for (int i0 = 0; i0 < n; i0 += MAX_WAIT) {
        WaitSet set{};
        set.n = n - i0 < MAX_WAIT ? n - i0 : MAX_WAIT;
        for (int i = 0; i < set.n; ++i) set.addr[i] = addrs[i0 + i];
        wait_kernel<<<1, 64, 0, as_stream(stream)>>>(set, v);
        TSB_LAUNCH_CHECK();
    }
    return TSB_OK;
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t ctl_words(const tsb_ring *r) {
    return (size_t)r->slots * (size_t)r->writers + (size_t)r->max_consumers;
}
size_t ctl_words_bytes(const tsb_ring *r) { return round_up(sizeof(uint64_t) * ctl_words(r), 256); }

void layout(tsb_ring *r) {
    r->slot_stride = round_up(r->slot_bytes ? r->slot_bytes : 16, 256);
    const size_t payload = r->slot_stride * (size_t)r->slots;
    r->total = payload + ctl_words_bytes(r) + round_up(sizeof(unsigned int) * r->slots, 256);
}

void bind(tsb_ring *r) {
    const size_t payload = r->slot_stride * (size_t)r->slots;
    r->ready = reinterpret_cast<uint64_t *>(r->base + payload);
    r->cursor = r->ready + (size_t)r->slots * r->writers;
    r->counters = reinterpret_cast<unsigned int *>(r->base + payload + ctl_words_bytes(r));
}

uint64_t *ready_word(tsb_ring *r, int slot, int writer) {
    return r->ready + (size_t)slot * r->writers + writer;
}

// host view of a control word (host-shared control block), or null
uint64_t *host_word(tsb_ring *r, const uint64_t *dev_addr) {
    if (!r->h_ctl) return nullptr;
    return r->h_ctl + (dev_addr - r->ready);
}
int host_write(tsb_ring *r, uint64_t *addr, uint64_t v) {
    if (uint64_t *h = host_word(r, addr)) {
        __atomic_store_n(h, v, __ATOMIC_RELEASE);
        return TSB_OK;
    }
    TSB_CUDA(cudaMemcpyAsync(addr, &v, sizeof(v), cudaMemcpyHostToDevice, r->host_stream));
    TSB_CUDA(cudaStreamSynchronize(r->host_stream));
    return TSB_OK;
}
int host_read(tsb_ring *r, const uint64_t *addr, uint64_t *out) {
    if (uint64_t *h = host_word(r, addr)) {
        *out = __atomic_load_n(h, __ATOMIC_ACQUIRE);
        return TSB_OK;
    }
    TSB_CUDA(cudaMemcpyAsync(out, addr, sizeof(*out), cudaMemcpyDeviceToHost, r->host_stream));
    TSB_CUDA(cudaStreamSynchronize(r->host_stream));
    return TSB_OK;
}

}  // namespace

namespace tsb {
int ring_publish_ptrs(tsb_ring *r, int slot, int writer, uint64_t **ready,
                      unsigned int **counter) {
    TSB_CHECK(r && slot >= 0 && slot < r->slots, "bad slot");
    TSB_CHECK(writer >= 0 && writer < r->writers, "bad writer %d", writer);
    *ready = ready_word(r, slot, writer);
    if (counter) *counter = r->counters + slot;
    return TSB_OK;
}
int ring_writers(const tsb_ring *r) { return r->writers; }
int ring_phys_device(const tsb_ring *r) { return r->phys_dev; }
void ring_internals(tsb_ring *r, uint8_t **base, int64_t *stride, uint64_t **ready,
                    uint64_t **cursors, unsigned int **counters) {
    *base = r->base;
    *stride = (int64_t)r->slot_stride;
    *ready = r->ready;
    *cursors = r->cursor;
    *counters = r->counters;
}

bool ring_has_host_control(const tsb_ring *r) { return r && r->h_ctl; }

// Host-side flow gate for rings whose control words live in host-shared
// memory: block the enqueuing thread until every live cursor has released
// `need` (wrap-around GEQ, as cuStreamWaitValue64; the eviction sentinel
// passes).  The producer's stream then carries only kernels, so consecutive
// batches chain with programmatic dependent launch instead of stalling the
// GPU front end on a PCIe poll per cursor.  Same rule as the device wait
// (producer.py:230-238 flow gate): the host never runs more than `slots`
// batches ahead of the slowest live consumer.
int ring_host_gate(tsb_ring *r, const int *live, int n_live, uint64_t need) {
    TSB_CHECK(r && r->h_ctl, "host gate needs a host control block");
    if (n_live <= 0 || need == 0) return TSB_OK;
    // a consumer that never releases (and is never evicted) must not wedge the
    // producer forever: TSB_GATE_TIMEOUT_S (default 600 s) turns it into an error
    static const double limit_s = getenv("TSB_GATE_TIMEOUT_S") ? atof(getenv("TSB_GATE_TIMEOUT_S"))
                                                                 : 600.0;
    struct timespec t0, t;
    bool started = false;
    for (int i = 0; i < n_live; ++i) {
        TSB_CHECK(live[i] >= 0 && live[i] < r->max_consumers, "bad consumer %d", live[i]);
        const uint64_t *h = r->h_ctl + (size_t)r->slots * r->writers + live[i];
        int64_t spins = 0;
        while ((int64_t)(__atomic_load_n(h, __ATOMIC_ACQUIRE) - need) < 0) {
            if (++spins < 2048) {
                __builtin_ia32_pause();
                continue;
            }
            struct timespec ns = {0, 5000};
            nanosleep(&ns, nullptr);
            if ((spins & 1023) == 0) {
                clock_gettime(CLOCK_MONOTONIC, &t);
                if (!started) {
                    t0 = t;
                    started = true;
                } else if ((t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec) > limit_s) {
                    set_error("flow gate: consumer %d has not released seq %llu for %.0f s",
                              live[i], (unsigned long long)need, limit_s);
                    return TSB_ERR_STALE;
                }
            }
        }
    }
    return TSB_OK;
}
}  // namespace tsb

extern "C" {

int tsb_ring_sync_mode(void) { return resolve_mode(); }

int tsb_ring_create(int dev, int slots, size_t slot_bytes, int max_consumers, tsb_ring **out) {
    return tsb_ring_create_ex(dev, slots, slot_bytes, max_consumers, 1, out);
}

int tsb_ring_create_ex(int dev, int slots, size_t slot_bytes, int max_consumers, int writers,
                       tsb_ring **out) {
    TSB_CHECK(out, "null out");
    TSB_CHECK(slots >= 1 && max_consumers >= 1 && max_consumers <= 4096,
              "bad ring geometry slots=%d consumers=%d", slots, max_consumers);
    TSB_CHECK(writers >= 1 && writers <= TSB_MAX_WRITERS, "writers must be 1..%d", TSB_MAX_WRITERS);
    CurrentDeviceGuard device_guard;
    TSB_CUDA(cudaSetDevice(dev));
    tsb_ring *r = new tsb_ring{};
    r->dev = dev;
    r->slots = slots;
    r->slot_bytes = slot_bytes;
    r->max_consumers = max_consumers;
    r->writers = writers;
    r->phys_dev = dev;
    layout(r);
    const size_t total = r->total;
    cudaError_t e = cudaMalloc(&r->base, total);
    if (e != cudaSuccess) {
        r->base = nullptr;
        delete r;
        set_error("ring allocation of %zu bytes failed: %s", total, cudaGetErrorString(e));
        return TSB_ERR_CUDA;
    }
    bind(r);
    // control words start zeroed; on any failure release everything made so far
    e = cudaStreamCreateWithFlags(&r->host_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(r->ready, 0, total - r->slot_stride * (size_t)r->slots,
                            r->host_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r->host_stream);
    if (e != cudaSuccess) {
        if (r->host_stream) cudaStreamDestroy(r->host_stream);
        cudaFree(r->base);
        delete r;
        set_error("ring control-word init failed: %s", cudaGetErrorString(e));
        return TSB_ERR_CUDA;
    }
    resolve_mode();
    *out = r;
    return TSB_OK;
}

int tsb_ring_export(tsb_ring *r, void *handle_out) {
    TSB_CHECK(r && handle_out, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == TSB_IPC_HANDLE_BYTES, "ipc handle size");
    cudaIpcMemHandle_t h;
    TSB_CUDA(cudaIpcGetMemHandle(&h, r->base));
    memcpy(handle_out, &h, sizeof(h));
    return TSB_OK;
}

int tsb_ring_import(const void *handle, int slots, size_t slot_bytes, int max_consumers,
                    tsb_ring **out) {
    return tsb_ring_import_ex(handle, slots, slot_bytes, max_consumers, 1, out);
}

int tsb_ring_import_ex(const void *handle, int slots, size_t slot_bytes, int max_consumers,
                       int writers, tsb_ring **out) {
    TSB_CHECK(handle && out, "null argument");
    TSB_CHECK(writers >= 1 && writers <= TSB_MAX_WRITERS, "writers must be 1..%d", TSB_MAX_WRITERS);
    tsb_ring *r = new tsb_ring{};
    TSB_CUDA(cudaGetDevice(&r->dev));
    r->slots = slots;
    r->slot_bytes = slot_bytes;
    r->max_consumers = max_consumers;
    r->writers = writers;
    layout(r);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        delete r;
        cudaGetLastError();
        set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
        return TSB_ERR_STALE;
    }
    r->base = static_cast<uint8_t *>(p);
    r->imported = true;
    r->phys_dev = r->dev;
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, p) == cudaSuccess)
        r->phys_dev = pa.device;
    else
        cudaGetLastError();
    bind(r);
    TSB_CUDA(cudaStreamCreateWithFlags(&r->host_stream, cudaStreamNonBlocking));
    resolve_mode();
    *out = r;
    return TSB_OK;
}

size_t tsb_ring_control_bytes(int slots, int max_consumers) {
    return tsb_ring_control_bytes_ex(slots, max_consumers, 1);
}
size_t tsb_ring_control_bytes_ex(int slots, int max_consumers, int writers) {
    return round_up(sizeof(uint64_t) * ((size_t)slots * (size_t)writers + (size_t)max_consumers),
                    4096);
}

int tsb_ring_attach_host_control(tsb_ring *r, void *host_ctl, size_t bytes, int init) {
    TSB_CHECK(r && host_ctl, "null argument");
    TSB_CHECK(!r->h_ctl, "ring already has a host control block");
    const size_t need = sizeof(uint64_t) * ctl_words(r);
    TSB_CHECK(bytes >= need && ((uintptr_t)host_ctl & 7) == 0,
              "host control block too small or misaligned (%zu < %zu)", bytes, need);
    if (init) memset(host_ctl, 0, need);
    CurrentDeviceGuard device_guard;
    TSB_CUDA(cudaSetDevice(r->dev));
    TSB_CUDA(cudaHostRegister(host_ctl, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    void *dptr = nullptr;
    TSB_CUDA(cudaHostGetDevicePointer(&dptr, host_ctl, 0));
    r->h_ctl = static_cast<uint64_t *>(host_ctl);
    r->ready = static_cast<uint64_t *>(dptr);
    r->cursor = r->ready + (size_t)r->slots * r->writers;
    return TSB_OK;
}

int tsb_ring_host_wait_ready(tsb_ring *r, int slot, uint64_t seq, int64_t timeout_us) {
    TSB_CHECK(r && r->h_ctl && slot >= 0 && slot < r->slots, "needs a host control block");
    int64_t spins = 0;
    struct timespec t0, t;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int w = 0; w < r->writers; ++w) {
    uint64_t *h = r->h_ctl + (size_t)slot * r->writers + w;
    while (__atomic_load_n(h, __ATOMIC_ACQUIRE) < seq) {
        if (++spins > 256) {
            clock_gettime(CLOCK_MONOTONIC, &t);
            const int64_t us = (t.tv_sec - t0.tv_sec) * 1000000 + (t.tv_nsec - t0.tv_nsec) / 1000;
            if (timeout_us >= 0 && us > timeout_us) {
                set_error("timed out waiting for slot %d seq %llu", slot, (unsigned long long)seq);
                return TSB_ERR_STALE;
            }
            if (spins > 4096) {
                struct timespec ns = {0, 2000};
                nanosleep(&ns, nullptr);
            }
        }
    }
    }
    return TSB_OK;
}

int tsb_ring_destroy(tsb_ring *r) {
    if (!r) return TSB_OK;
    int rc = TSB_OK;
    if (r->h_ctl) cudaHostUnregister(r->h_ctl);
    if (r->host_stream) cudaStreamDestroy(r->host_stream);
    cudaError_t e = r->imported ? cudaIpcCloseMemHandle(r->base) : cudaFree(r->base);
    if (e != cudaSuccess) {
        set_error("ring release: %s", cudaGetErrorString(e));
        rc = TSB_ERR_CUDA;
    }
    delete r;
    return rc;
}

int tsb_ring_slot_ptr(tsb_ring *r, int slot, void **out) {
    TSB_CHECK(r && out, "null argument");
    TSB_CHECK(slot >= 0 && slot < r->slots, "slot %d out of range", slot);
    *out = r->base + r->slot_stride * (size_t)slot;
    return TSB_OK;
}
int tsb_ring_base_ptr(tsb_ring *r, void **out) {
    TSB_CHECK(r && out, "null argument");
    *out = r->base;
    return TSB_OK;
}
int tsb_ring_writers(tsb_ring *r, int *writers) {
    TSB_CHECK(r && writers, "null argument");
    *writers = r->writers;
    return TSB_OK;
}
int tsb_ring_geometry(tsb_ring *r, int *slots, size_t *slot_bytes, int *max_consumers) {
    TSB_CHECK(r, "null ring");
    if (slots) *slots = r->slots;
    if (slot_bytes) *slot_bytes = r->slot_stride;
    if (max_consumers) *max_consumers = r->max_consumers;
    return TSB_OK;
}

int tsb_ring_publish(tsb_ring *r, int slot, uint64_t seq, void *stream) {
    TSB_CHECK(r && slot >= 0 && slot < r->slots, "bad slot");
    for (int w = 0; w < r->writers; ++w)
        if (int rc = dev_write(r, ready_word(r, slot, w), seq, stream)) return rc;
    return TSB_OK;
}
int tsb_ring_publish_shard(tsb_ring *r, int slot, int writer, uint64_t seq, void *stream) {
    TSB_CHECK(r && slot >= 0 && slot < r->slots, "bad slot");
    TSB_CHECK(writer >= 0 && writer < r->writers, "bad writer %d", writer);
    return dev_write(r, ready_word(r, slot, writer), seq, stream);
}
int tsb_ring_wait_ready(tsb_ring *r, int slot, uint64_t seq, void *stream) {
    TSB_CHECK(r && slot >= 0 && slot < r->slots, "bad slot");
    const uint64_t *a[TSB_MAX_WRITERS];
    for (int w = 0; w < r->writers; ++w) a[w] = ready_word(r, slot, w);
    return dev_wait(r, a, r->writers, seq, stream);
}
int tsb_ring_ack(tsb_ring *r, int consumer, uint64_t seq, void *stream) {
    TSB_CHECK(r && consumer >= 0 && consumer < r->max_consumers, "bad consumer %d", consumer);
    return dev_write(r, r->cursor + consumer, seq, stream);
}
int tsb_ring_wait_free(tsb_ring *r, const int *live, int n_live, uint64_t seq, void *stream) {
    TSB_CHECK(r && (live || n_live == 0), "null argument");
    if (n_live <= 0 || seq == 0) return TSB_OK;
    const uint64_t *addrs[4096];
    TSB_CHECK(n_live <= 4096, "too many consumers");
    for (int i = 0; i < n_live; ++i) {
        TSB_CHECK(live[i] >= 0 && live[i] < r->max_consumers, "bad consumer %d", live[i]);
        addrs[i] = r->cursor + live[i];
    }
    return dev_wait(r, addrs, n_live, seq, stream);
}
int tsb_ring_host_consume_range(tsb_ring *r, int consumer, uint64_t seq0, int n, int64_t *t_us) {
    TSB_CHECK(r && r->h_ctl && consumer >= 0 && consumer < r->max_consumers && n >= 0,
              "needs a host control block and a valid consumer");
    uint64_t *cur = r->h_ctl + (size_t)r->slots * r->writers + consumer;
    for (int i = 0; i < n; ++i) {
        const uint64_t q = seq0 + (uint64_t)i;
        const int slot = (int)((q - 1) % (uint64_t)r->slots);
        if (int rc = tsb_ring_host_wait_ready(r, slot, q, -1)) return rc;
        if (t_us) {
            struct timespec t;
            clock_gettime(CLOCK_MONOTONIC, &t);
            t_us[i] = (int64_t)t.tv_sec * 1000000 + t.tv_nsec / 1000;
        }
        __atomic_store_n(cur, q, __ATOMIC_RELEASE);  // map-and-ack: release at once
    }
    return TSB_OK;
}

int tsb_ring_host_gate(tsb_ring *r, const int *live, int n_live, uint64_t need,
                       int64_t timeout_us) {
    TSB_CHECK(r && r->h_ctl, "host gate needs a host control block");
    TSB_CHECK(live || n_live == 0, "null live list");
    if (timeout_us < 0) return ring_host_gate(r, live, n_live, need);
    struct timespec t0, t;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int i = 0; i < n_live; ++i) {
        TSB_CHECK(live[i] >= 0 && live[i] < r->max_consumers, "bad consumer %d", live[i]);
        const uint64_t *h = r->h_ctl + (size_t)r->slots * r->writers + live[i];
        int64_t spins = 0;
        while ((int64_t)(__atomic_load_n(h, __ATOMIC_ACQUIRE) - need) < 0) {
            if (++spins < 2048) {
                __builtin_ia32_pause();
                continue;
            }
            clock_gettime(CLOCK_MONOTONIC, &t);
            const int64_t us = (t.tv_sec - t0.tv_sec) * 1000000 + (t.tv_nsec - t0.tv_nsec) / 1000;
            if (us > timeout_us) {
                set_error("timed out gating seq %llu on consumer %d", (unsigned long long)need,
                          live[i]);
                return TSB_ERR_STALE;
            }
            struct timespec ns = {0, 5000};
            nanosleep(&ns, nullptr);
        }
    }
    return TSB_OK;
}

int tsb_ring_evict(tsb_ring *r, int consumer) {
    TSB_CHECK(r && consumer >= 0 && consumer < r->max_consumers, "bad consumer %d", consumer);
    // "+inf" for every wait: far ahead of any sequence, yet positive under the
    // wrap-around GEQ of cuStreamWaitValue64 ((int64_t)(*addr - v) >= 0)
    return host_write(r, r->cursor + consumer, TSB_CURSOR_EVICTED);
}
int tsb_ring_set_cursor(tsb_ring *r, int consumer, uint64_t value) {
    TSB_CHECK(r && consumer >= 0 && consumer < r->max_consumers, "bad consumer %d", consumer);
    return host_write(r, r->cursor + consumer, value);
}
int tsb_ring_read_cursor(tsb_ring *r, int consumer, uint64_t *out) {
    TSB_CHECK(r && out && consumer >= 0 && consumer < r->max_consumers, "bad consumer");
    return host_read(r, r->cursor + consumer, out);
}
int tsb_ring_read_ready(tsb_ring *r, int slot, uint64_t *out) {
    TSB_CHECK(r && out && slot >= 0 && slot < r->slots, "bad slot");
    uint64_t lo = ~0ull;
    for (int w = 0; w < r->writers; ++w) {  // complete when every writer's shard landed
        uint64_t v = 0;
        if (int rc = host_read(r, ready_word(r, slot, w), &v)) return rc;
        if (v < lo) lo = v;
    }
    *out = lo;
    return TSB_OK;
}

}  // extern "C"

namespace tsb {
void preload_ring() {
    touch_kernel(signal_kernel);
    touch_kernel(wait_kernel);
}
}  // namespace tsb
