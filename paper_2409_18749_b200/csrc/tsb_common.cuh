// Shared helpers for the tsb200 C-ABI library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/tsb200.h"

namespace tsb {

void set_error(const char *fmt, ...);

#define TSB_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            ::tsb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                             cudaGetErrorString(e_));                               \
            return TSB_ERR_CUDA;                                                    \
        }                                                                           \
    } while (0)

#define TSB_CHECK(cond, ...)                                                        \
    do {                                                                            \
        if (!(cond)) {                                                              \
            ::tsb::set_error(__VA_ARGS__);                                          \
            return TSB_ERR_INVALID;                                                 \
        }                                                                           \
    } while (0)

#define TSB_LAUNCH_CHECK()                                                          \
    do {                                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess) {                                                    \
            ::tsb::set_error("%s:%d launch: %s", __FILE__, __LINE__,                \
                             cudaGetErrorString(e_));                               \
            return TSB_ERR_CUDA;                                                    \
        }                                                                           \
    } while (0)

constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;
constexpr uint64_t SHUFFLE_DOMAIN = 0x53485546ULL;  // pipeline.py:25
constexpr uint64_t AUG_DOMAIN = 0x41554731ULL;      // "AUG1" (SURVEY.md §8a A6')

// kernels.py:40-45 SplitMix64 finalizer (u64 wrap-around)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

// kernels.py:48-53
__host__ __device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t epoch,
                                                        uint64_t index) {
    uint64_t h = mix64(seed + GAMMA);
    h = mix64((h ^ epoch) + GAMMA);
    h = mix64((h ^ index) + GAMMA);
    return h;
}

// Augment params of one sample (SURVEY.md §8a A6'), host and device:
//   ka = derive_key(mix64(aug_seed ^ AUG_DOMAIN), epoch, idx)
//   oy = mix64(ka+1G) % (2P+1), ox = mix64(ka+2G) % (2P+1), flip = mix64(ka+3G) & 1
__host__ __device__ __forceinline__ void derive_aug_host(uint64_t aug_mixed, uint64_t epoch,
                                                         int64_t index, int pad, int flip_en,
                                                         int &oy, int &ox, int &fl) {
    const uint64_t ka = derive_key(aug_mixed, epoch, (uint64_t)index);
    const uint64_t m = (uint64_t)(2 * pad + 1);
    oy = (int)(mix64(ka + GAMMA) % m);
    ox = (int)(mix64(ka + 2 * GAMMA) % m);
    fl = flip_en ? (int)(mix64(ka + 3 * GAMMA) & 1) : 0;
}

// Crop geometry for a crop-aware ingest (tsb_ingest.cu): which source rows of
// each staged sample the collate kernel will read.
struct IngestCrop {
    uint64_t aug_mixed;  // mix64(aug_seed ^ AUG_DOMAIN)
    uint64_t epoch;
    int h, w, row_bytes, pad, flip;
};

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Restores the calling thread's current device on scope exit: an entry point
// that works on a given device leaves the caller's device as it found it.
struct CurrentDeviceGuard {
    int prev = -1;
    CurrentDeviceGuard() { cudaGetDevice(&prev); }
    ~CurrentDeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

inline int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

// 128-bit streaming global accesses (guide G13/G14)
__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_cs_v4(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

}  // namespace tsb

namespace tsb {
// ---- mbarrier + TMA 1D bulk copy (cp.async.bulk, SASS UBLKCP) ------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// same, with an L2 eviction-priority policy (createpolicy) for streamed sources
__device__ __forceinline__ void tma_load_1d_hint(void *smem_dst, const void *gsrc, uint32_t bytes,
                                                 uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gsrc, uint32_t bytes,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
}  // namespace tsb

namespace tsb {
// Force eager loading of this file's kernels in the current context: a lazily
// loaded kernel's first launch can wait for the device to go idle, which
// deadlocks when a stream is parked on a ring wait that this very launch
// would satisfy (e.g. an in-process consumer's first rebatch gather).
template <typename F>
inline void touch_kernel(F f) {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(f)) != cudaSuccess)
        cudaGetLastError();
}
}  // namespace tsb
