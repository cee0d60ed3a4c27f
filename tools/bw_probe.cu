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
    return 0;
}
