// Library plumbing: errors, memory, streams, events, host RNG + shuffle.
#include <stdarg.h>

#include <vector>

#include "tsb_common.cuh"

namespace tsb {
static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace tsb

using namespace tsb;

extern "C" {

const char *tsb_last_error(void) { return g_err; }
int tsb_version(void) { return 1; }

int tsb_device_count(int *n) {
    TSB_CUDA(cudaGetDeviceCount(n));
    return TSB_OK;
}
int tsb_set_device(int dev) {
    TSB_CUDA(cudaSetDevice(dev));
    return TSB_OK;
}
int tsb_get_device(int *dev) {
    TSB_CUDA(cudaGetDevice(dev));
    return TSB_OK;
}
int tsb_device_info(int dev, int *sm, int *maj, int *min, size_t *hbm) {
    cudaDeviceProp p;
    TSB_CUDA(cudaGetDeviceProperties(&p, dev));
    if (sm) *sm = p.multiProcessorCount;
    if (maj) *maj = p.major;
    if (min) *min = p.minor;
    if (hbm) *hbm = p.totalGlobalMem;
    return TSB_OK;
}

int tsb_malloc(void **p, size_t bytes) {
    TSB_CHECK(p, "null out pointer");
    TSB_CUDA(cudaMalloc(p, bytes ? bytes : 16));
    return TSB_OK;
}
int tsb_free(void *p) {
    TSB_CUDA(cudaFree(p));
    return TSB_OK;
}
int tsb_host_alloc(void **p, size_t bytes) {
    TSB_CUDA(cudaHostAlloc(p, bytes ? bytes : 16, cudaHostAllocMapped | cudaHostAllocPortable));
    return TSB_OK;
}
int tsb_host_free(void *p) {
    TSB_CUDA(cudaFreeHost(p));
    return TSB_OK;
}
int tsb_host_register(void *p, size_t bytes) {
    TSB_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    return TSB_OK;
}
int tsb_host_unregister(void *p) {
    TSB_CUDA(cudaHostUnregister(p));
    return TSB_OK;
}
int tsb_host_device_ptr(void *host, void **dev) {
    TSB_CUDA(cudaHostGetDevicePointer(dev, host, 0));
    return TSB_OK;
}
int tsb_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
    if (!bytes) return TSB_OK;
    TSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
    return TSB_OK;
}
int tsb_memset_async(void *dst, int value, size_t bytes, void *stream) {
    if (!bytes) return TSB_OK;
    TSB_CUDA(cudaMemsetAsync(dst, value, bytes, as_stream(stream)));
    return TSB_OK;
}
int tsb_stream_create(void **stream) {
    cudaStream_t s;
    TSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
    return TSB_OK;
}
int tsb_stream_destroy(void *stream) {
    TSB_CUDA(cudaStreamDestroy(as_stream(stream)));
    return TSB_OK;
}
int tsb_stream_sync(void *stream) {
    TSB_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return TSB_OK;
}
int tsb_device_sync(void) {
    TSB_CUDA(cudaDeviceSynchronize());
    return TSB_OK;
}
int tsb_event_create(void **ev) {
    cudaEvent_t e;
    TSB_CUDA(cudaEventCreate(&e));
    *ev = e;
    return TSB_OK;
}
int tsb_event_destroy(void *ev) {
    TSB_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
    return TSB_OK;
}
int tsb_event_record(void *ev, void *stream) {
    TSB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), as_stream(stream)));
    return TSB_OK;
}
int tsb_event_sync(void *ev) {
    TSB_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(ev)));
    return TSB_OK;
}
int tsb_event_elapsed_ms(void *a, void *b, float *ms) {
    TSB_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(a),
                                  reinterpret_cast<cudaEvent_t>(b)));
    return TSB_OK;
}
int tsb_stream_wait_event(void *stream, void *ev) {
    TSB_CUDA(cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(ev), 0));
    return TSB_OK;
}
int tsb_can_access_peer(int dev, int peer, int *can) {
    TSB_CUDA(cudaDeviceCanAccessPeer(can, dev, peer));
    return TSB_OK;
}
int tsb_enable_peer(int dev, int peer) {
    int prev = 0;
    TSB_CUDA(cudaGetDevice(&prev));
    TSB_CUDA(cudaSetDevice(dev));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(prev);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return TSB_OK;
    }
    if (e != cudaSuccess) {
        set_error("cudaDeviceEnablePeerAccess(%d->%d): %s", dev, peer, cudaGetErrorString(e));
        return TSB_ERR_CUDA;
    }
    return TSB_OK;
}

// ---- host RNG + shuffle ---------------------------------------------------
uint64_t tsb_mix64(uint64_t x) { return mix64(x); }
uint64_t tsb_derive_key(uint64_t s, uint64_t e, uint64_t i) { return derive_key(s, e, i); }

// kernels.py:123-140: Fisher-Yates is a sequential dependency chain (each
// swap reads the previous state), so it stays on the host, once per epoch
// (~15 ms at n = 1.28M); the result is uploaded to HBM by the caller.
int tsb_permutation(int64_t n, uint64_t key, int64_t *out) {
    TSB_CHECK(n >= 0, "n must be >= 0");
    TSB_CHECK(out || n == 0, "null output");
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    uint64_t t = 0;
    for (int64_t i = n - 1; i > 0; --i) {
        uint64_t r = mix64(key + (t + 1) * GAMMA);
        t += 1;
        int64_t j = (int64_t)(r % (uint64_t)(i + 1));
        int64_t tmp = out[i];
        out[i] = out[j];
        out[j] = tmp;
    }
    return TSB_OK;
}

// pipeline.py:113-123
int tsb_epoch_order(int64_t n, uint64_t shuffle_seed, uint64_t epoch, int reshuffle,
                    int64_t *out) {
    uint64_t eff = reshuffle ? epoch : 0;
    return tsb_permutation(n, derive_key(shuffle_seed, eff, SHUFFLE_DOMAIN), out);
}

}  // extern "C"

namespace tsb {
void preload_collate();
void preload_crc32();
void preload_fanout();
void preload_ring();
void preload_ingest();
void preload_jpeg();
}  // namespace tsb

extern "C" int tsb_preload_kernels(void) {
    int dev = -1;
    TSB_CUDA(cudaGetDevice(&dev));
    tsb::preload_collate();
    tsb::preload_crc32();
    tsb::preload_fanout();
    tsb::preload_ring();
    tsb::preload_ingest();
    tsb::preload_jpeg();
    return TSB_OK;
}
