// JPEG sample source: nvJPEG batched decode in front of the collate kernel.
//
// The reference's DirectorySource reads raw sample files (pipeline.py:45-54,
// 190-210); the paper's workloads read JPEGs and decode + augment them on the
// CPU, the cost TensorSocket shares.  Here a store of
// encoded files stays in (pinned) host memory and each batch's files --
// picked by the epoch order -- are decoded by nvJPEG's batched decoder
// (B200 NVJPG hardware engines when available, else the hybrid GPU decoder)
// straight into HBM staging as interleaved RGB u8 (the HWC layout the
// collate kernel reads), then collated (crop/flip/normalise) into the ring
// slot like any other store.  libnvjpeg is opened at run time, so the rest
// of the library works without it and this path fails loudly when absent.
#include <dlfcn.h>
#include <nvjpeg.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "tsb_common.cuh"

using namespace tsb;

namespace {

struct NvJpeg {
    decltype(&nvjpegCreateEx) createEx = nullptr;
    decltype(&nvjpegDestroy) destroy = nullptr;
    decltype(&nvjpegJpegStateCreate) stateCreate = nullptr;
    decltype(&nvjpegJpegStateDestroy) stateDestroy = nullptr;
    decltype(&nvjpegGetImageInfo) imageInfo = nullptr;
    decltype(&nvjpegDecodeBatchedInitialize) batchedInit = nullptr;
    decltype(&nvjpegDecodeBatched) batched = nullptr;
    bool ok = false;
};

NvJpeg &nvjpeg() {
    static NvJpeg f;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnvjpeg.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libnvjpeg.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnvjpeg.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        f.createEx = reinterpret_cast<decltype(f.createEx)>(dlsym(h, "nvjpegCreateEx"));
        f.destroy = reinterpret_cast<decltype(f.destroy)>(dlsym(h, "nvjpegDestroy"));
        f.stateCreate = reinterpret_cast<decltype(f.stateCreate)>(dlsym(h, "nvjpegJpegStateCreate"));
        f.stateDestroy =
            reinterpret_cast<decltype(f.stateDestroy)>(dlsym(h, "nvjpegJpegStateDestroy"));
        f.imageInfo = reinterpret_cast<decltype(f.imageInfo)>(dlsym(h, "nvjpegGetImageInfo"));
        f.batchedInit =
            reinterpret_cast<decltype(f.batchedInit)>(dlsym(h, "nvjpegDecodeBatchedInitialize"));
        f.batched = reinterpret_cast<decltype(f.batched)>(dlsym(h, "nvjpegDecodeBatched"));
        f.ok = f.createEx && f.destroy && f.stateCreate && f.stateDestroy && f.imageInfo &&
               f.batchedInit && f.batched;
    });
    return f;
}

#define NVJ(call)                                                                  \
    do {                                                                           \
        nvjpegStatus_t st_ = (call);                                               \
        if (st_ != NVJPEG_STATUS_SUCCESS) {                                        \
            tsb::set_error("%s failed: nvjpeg status %d", #call, (int)st_);        \
            return TSB_ERR_CUDA;                                                   \
        }                                                                          \
    } while (0)

}  // namespace

struct tsb_jpeg {
    int dev;
    int h, w;
    int64_t max_batch;
    int backend;                 // nvjpegBackend_t in use
    nvjpegHandle_t handle = nullptr;
    nvjpegJpegState_t state = nullptr;
    int init_batch = 0;
    std::vector<const unsigned char *> data;  // the store: one encoded file per sample
    std::vector<size_t> len;
    uint8_t *staging = nullptr;  // [max_batch][h*w*3] HBM (decoded RGB)
    int64_t *d_idx = nullptr;    // [max_batch] the batch's sample indices
    int32_t *d_params = nullptr; // [max_batch][3]
    int64_t *d_identity = nullptr;
    int64_t *h_idx = nullptr;    // pinned upload buffer
    cudaEvent_t idx_done = nullptr;
    bool idx_used = false;
    std::vector<nvjpegImage_t> dst;
    std::vector<const unsigned char *> bdata;
    std::vector<size_t> blen;
};

namespace {
__global__ void jpeg_iota_kernel(int64_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = i;
}
}  // namespace

namespace tsb {
void preload_jpeg() { touch_kernel(jpeg_iota_kernel); }

// Decode store files h_idx[0..b) into out (b x h*w*3 RGB u8, device) on `stream`.
int jpeg_decode(tsb_jpeg *j, const int64_t *h_idx, int64_t b, void *out, void *stream) {
    TSB_CHECK(j && h_idx && out, "null argument");
    TSB_CHECK(b >= 1 && b <= j->max_batch, "batch %lld exceeds the decoder capacity %lld",
              (long long)b, (long long)j->max_batch);
    TSB_CHECK(!j->data.empty(), "no JPEG store attached");
    NvJpeg &f = nvjpeg();
    if (j->init_batch != (int)b) {
        NVJ(f.batchedInit(j->handle, j->state, (int)b, 1, NVJPEG_OUTPUT_RGBI));
        j->init_batch = (int)b;
    }
    const size_t sb = (size_t)j->h * j->w * 3;
    for (int64_t i = 0; i < b; ++i) {
        const int64_t k = h_idx[i];
        TSB_CHECK(k >= 0 && k < (int64_t)j->data.size(), "sample %lld outside the store",
                  (long long)k);
        j->bdata[i] = j->data[k];
        j->blen[i] = j->len[k];
        memset(&j->dst[i], 0, sizeof(nvjpegImage_t));
        j->dst[i].channel[0] = static_cast<unsigned char *>(out) + (size_t)i * sb;
        j->dst[i].pitch[0] = (size_t)j->w * 3;
    }
    NVJ(f.batched(j->handle, j->state, j->bdata.data(), j->blen.data(), j->dst.data(),
                  as_stream(stream)));
    return TSB_OK;
}

// Upload the batch's indices (for the augment params and the target) into d_idx.
int jpeg_upload_indices(tsb_jpeg *j, const int64_t *h_idx, int64_t b, void *stream) {
    if (j->idx_used) TSB_CUDA(cudaEventSynchronize(j->idx_done));  // pinned buffer reuse
    memcpy(j->h_idx, h_idx, sizeof(int64_t) * (size_t)b);
    TSB_CUDA(cudaMemcpyAsync(j->d_idx, j->h_idx, sizeof(int64_t) * (size_t)b,
                             cudaMemcpyHostToDevice, as_stream(stream)));
    TSB_CUDA(cudaEventRecord(j->idx_done, as_stream(stream)));
    j->idx_used = true;
    return TSB_OK;
}
uint8_t *jpeg_staging(tsb_jpeg *j) { return j->staging; }
int64_t *jpeg_indices(tsb_jpeg *j) { return j->d_idx; }
int32_t *jpeg_params(tsb_jpeg *j) { return j->d_params; }
int64_t *jpeg_identity(tsb_jpeg *j) { return j->d_identity; }
int64_t jpeg_sample_bytes(tsb_jpeg *j) { return (int64_t)j->h * j->w * 3; }
}  // namespace tsb

extern "C" {

int tsb_jpeg_available(int *ok) {
    TSB_CHECK(ok, "null argument");
    *ok = nvjpeg().ok ? 1 : 0;
    return TSB_OK;
}

int tsb_jpeg_create(int dev, int64_t max_batch, int h, int w, int backend, tsb_jpeg **out) {
    TSB_CHECK(out && max_batch >= 1 && h > 0 && w > 0, "bad decoder geometry");
    NvJpeg &f = nvjpeg();
    if (!f.ok) {
        set_error("libnvjpeg.so.12 not found: the JPEG source needs nvJPEG");
        return TSB_ERR_UNSUPPORTED;
    }
    CurrentDeviceGuard device_guard;
    TSB_CUDA(cudaSetDevice(dev));
    tsb_jpeg *j = new tsb_jpeg{};
    j->dev = dev;
    j->h = h;
    j->w = w;
    j->max_batch = max_batch;
    // backend: 0 = NVJPG hardware if present, else GPU-assisted Huffman (batches
    // > 50), else the default hybrid decoder; 1 = default; 2 = hardware only
    nvjpegStatus_t st = NVJPEG_STATUS_IMPLEMENTATION_NOT_SUPPORTED;
    const nvjpegBackend_t order0[] = {NVJPEG_BACKEND_HARDWARE, NVJPEG_BACKEND_GPU_HYBRID,
                                      NVJPEG_BACKEND_DEFAULT};
    const nvjpegBackend_t order1[] = {NVJPEG_BACKEND_DEFAULT};
    const nvjpegBackend_t order2[] = {NVJPEG_BACKEND_HARDWARE};
    const nvjpegBackend_t *order = backend == 1 ? order1 : backend == 2 ? order2 : order0;
    const int n_order = backend == 0 ? 3 : 1;
    for (int i = 0; i < n_order && st != NVJPEG_STATUS_SUCCESS; ++i) {
        j->handle = nullptr;
        st = f.createEx(order[i], nullptr, nullptr, 0, &j->handle);
        j->backend = order[i];
    }
    if (st != NVJPEG_STATUS_SUCCESS && backend == 2) {
        delete j;
        set_error("nvJPEG hardware backend unavailable (status %d)", (int)st);
        return TSB_ERR_UNSUPPORTED;
    }
    if (st != NVJPEG_STATUS_SUCCESS || f.stateCreate(j->handle, &j->state) != NVJPEG_STATUS_SUCCESS) {
        if (j->handle) f.destroy(j->handle);
        delete j;
        set_error("nvjpegCreateEx failed (status %d)", (int)st);
        return TSB_ERR_CUDA;
    }
    const size_t sb = (size_t)h * w * 3;
    cudaError_t e = cudaMalloc(&j->staging, sb * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&j->d_idx, sizeof(int64_t) * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&j->d_params, sizeof(int32_t) * 3 * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&j->d_identity, sizeof(int64_t) * max_batch);
    if (e == cudaSuccess) e = cudaHostAlloc(&j->h_idx, sizeof(int64_t) * max_batch, 0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&j->idx_done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_error("decoder allocation: %s", cudaGetErrorString(e));
        tsb_jpeg_destroy(j);
        return TSB_ERR_CUDA;
    }
    jpeg_iota_kernel<<<(unsigned)((max_batch + 255) / 256), 256>>>(j->d_identity, max_batch);
    TSB_LAUNCH_CHECK();
    TSB_CUDA(cudaDeviceSynchronize());
    j->dst.resize(max_batch);
    j->bdata.resize(max_batch);
    j->blen.resize(max_batch);
    *out = j;
    return TSB_OK;
}

int tsb_jpeg_backend(tsb_jpeg *j, int *backend) {
    TSB_CHECK(j && backend, "null argument");
    *backend = j->backend == NVJPEG_BACKEND_HARDWARE     ? 2
               : j->backend == NVJPEG_BACKEND_GPU_HYBRID ? 3
                                                         : 1;
    return TSB_OK;
}

int tsb_jpeg_attach_store(tsb_jpeg *j, const uint8_t *const *files, const size_t *lengths,
                          int64_t n) {
    TSB_CHECK(j && files && lengths && n >= 1, "bad store");
    NvJpeg &f = nvjpeg();
    j->data.assign(files, files + n);
    j->len.assign(lengths, lengths + n);
    for (int64_t i = 0; i < n; ++i) {  // every file must decode to the store's h x w RGB
        int nc = 0, ws[NVJPEG_MAX_COMPONENT] = {0}, hs[NVJPEG_MAX_COMPONENT] = {0};
        nvjpegChromaSubsampling_t ss;
        NVJ(f.imageInfo(j->handle, files[i], lengths[i], &nc, &ss, ws, hs));
        TSB_CHECK(ws[0] == j->w && hs[0] == j->h && (nc == 3 || nc == 1),
                  "file %lld is %dx%d with %d components, the store is %dx%d RGB", (long long)i,
                  ws[0], hs[0], nc, j->w, j->h);
    }
    return TSB_OK;
}

int tsb_jpeg_decode(tsb_jpeg *j, const int64_t *h_indices, int64_t b, void *out, void *stream) {
    return jpeg_decode(j, h_indices, b, out, stream);
}

int tsb_jpeg_destroy(tsb_jpeg *j) {
    if (!j) return TSB_OK;
    cudaDeviceSynchronize();
    NvJpeg &f = nvjpeg();
    if (j->state) f.stateDestroy(j->state);
    if (j->handle) f.destroy(j->handle);
    cudaFree(j->staging);
    cudaFree(j->d_idx);
    cudaFree(j->d_params);
    cudaFree(j->d_identity);
    if (j->h_idx) cudaFreeHost(j->h_idx);
    if (j->idx_done) cudaEventDestroy(j->idx_done);
    delete j;
    return TSB_OK;
}

}  // extern "C"
