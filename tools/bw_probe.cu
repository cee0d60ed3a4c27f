// HBM bandwidth probe for the traffic mixes of the hot kernels (write-heavy streams).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write_k(uint4 *out, size_t n16, uint32_t v) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride)
        out[i] = make_uint4(v, v, v, v);
}
__global__ void read_k(const uint4 *in, size_t n16, uint32_t *sink) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        uint4 x = __ldg(in + i);
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345678) *sink = acc;
}
// read n16 from in, write ratio x n16 to out (each input vector written `ratio` times)
__global__ void mix_k(const uint4 *in, uint4 *out, size_t n16, int ratio) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        uint4 x = __ldg(in + i);
        for (int r = 0; r < ratio; ++r) out[r * n16 + i] = x;
    }
}

__global__ void write_cs_k(uint4 *out, size_t n16, uint32_t v) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride)
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(out + i), "r"(v) : "memory");
}
// TMA bulk stores: each CTA streams `chunk`-byte pieces of its smem buffer to
// global, grid-strided; lane 0 of each warp owns every 8th chunk.
__global__ void tma_write_k(uint8_t *out, size_t bytes, int chunk) {
    extern __shared__ __align__(128) uint8_t sm[];
    for (int i = threadIdx.x; i < chunk * 8 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(7, 7, 7, 7);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nchunks = bytes / chunk;
    if (lane == 0) {
        int issued = 0;
        for (size_t c = (size_t)blockIdx.x * 8 + warp; c < nchunks; c += (size_t)gridDim.x * 8) {
            const uint8_t *src = sm + (size_t)warp * chunk;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * chunk),
                         "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(chunk)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++issued >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// phased 1:ratio mix: each CTA loads a CHUNK-byte tile into smem with one
// TMA bulk copy, then writes it `ratio` times with 16 B stores (reads and
// writes of a CTA are separated in time, not interleaved per thread)
template <int CHUNK>
__global__ void phased_mix_k(const uint8_t *in, uint8_t *out, size_t n, int ratio) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const size_t nchunks = n / CHUNK;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(CHUNK) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((uint32_t)__cvta_generic_to_shared(sm)), "l"(in + c * CHUNK), "r"(CHUNK),
                         "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(phase) : "memory");
        phase ^= 1;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(sm);
        for (int r = 0; r < ratio; ++r) {
            uint4 *o = reinterpret_cast<uint4 *>(out + ((size_t)r * n) + c * CHUNK);
            for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) o[i] = s4[i];
        }
        __syncthreads();
    }
}

int main() {
    const size_t N = 38535168;  // bytes of one u8 batch (256 x 150528)
    uint4 *a, *b;
    uint32_t *sink;
    cudaMalloc(&a, 8 * N);
    cudaMalloc(&b, 8 * N);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 1, 8 * N);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](const char *name, double bytes, auto fn) {
        for (int i = 0; i < 5; ++i) fn();
        cudaEventRecord(e0);
        const int it = 30;
        for (int i = 0; i < it; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.1f GB/s  (%.1f us)\n", name, bytes / (ms / it) / 1e6, 1000 * ms / it);
    };
    const int g = sms * 8, t = 256;
    time("write_only 154MB", 4.0 * N, [&] { write_k<<<g, t>>>(b, 4 * N / 16, 7); });
    time("write_only 616MB", 16.0 * N, [&] { write_k<<<g, t>>>(b, 8 * N / 16, 7); write_k<<<g, t>>>(a, 8 * N / 16, 7); });
    time("read_only 308MB", 8.0 * N, [&] { read_k<<<g, t>>>(a, 8 * N / 16, sink); });
    time("copy 1:1 154MB+154MB", 8.0 * N, [&] { mix_k<<<g, t>>>(a, b, 4 * N / 16, 1); });
    time("mix 1:4 (u8->f32) 192MB", 5.0 * N, [&] { mix_k<<<g, t>>>(a, b, N / 16, 4); });
    time("mix 1:2 (u8->bf16) 115MB", 3.0 * N, [&] { mix_k<<<g, t>>>(a, b, N / 16, 2); });
    time("mix 1:1 (u8->u8) 77MB", 2.0 * N, [&] { mix_k<<<g, t>>>(a, b, N / 16, 1); });
    time("memset 154MB", 4.0 * N, [&] { cudaMemsetAsync(b, 0, 4 * N); });
    time("write_only st.cs 154MB", 4.0 * N, [&] { write_cs_k<<<g, t>>>(b, 4 * N / 16, 7); });
    cudaFuncSetAttribute(phased_mix_k<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(phased_mix_k<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int per : {4, 8}) {
        char nm[80];
        snprintf(nm, sizeof nm, "phased 1:4 16KB x%d/SM", per);
        time(nm, 5.0 * N, [&] { phased_mix_k<16384><<<sms * per, 256, 16384>>>(reinterpret_cast<const uint8_t *>(a), reinterpret_cast<uint8_t *>(b), N, 4); });
        snprintf(nm, sizeof nm, "phased 1:2 16KB x%d/SM", per);
        time(nm, 3.0 * N, [&] { phased_mix_k<16384><<<sms * per, 256, 16384>>>(reinterpret_cast<const uint8_t *>(a), reinterpret_cast<uint8_t *>(b), N, 2); });
    }
    for (int per : {2, 3}) {
        char nm[80];
        snprintf(nm, sizeof nm, "phased 1:4 64KB x%d/SM", per);
        time(nm, 5.0 * N, [&] { phased_mix_k<65536><<<sms * per, 512, 65536>>>(reinterpret_cast<const uint8_t *>(a), reinterpret_cast<uint8_t *>(b), N, 4); });
    }
    for (int chunk : {4096, 8192, 16384}) {
        cudaFuncSetAttribute(tma_write_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * chunk);
        char name[64];
        snprintf(name, sizeof name, "tma_write %dB chunks 154MB", chunk);
        for (int ctas : {1, 2}) {
            char nm[80];
            snprintf(nm, sizeof nm, "%s x%d/SM", name, ctas);
            time(nm, 4.0 * N, [&] {
                tma_write_k<<<sms * ctas, 256, 8 * chunk>>>(reinterpret_cast<uint8_t *>(b), 4 * N, chunk);
            });
        }
    }
    return 0;
}
