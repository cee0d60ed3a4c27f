// Batch production kernels: synthetic fill, store gather, fused collate/augment.
//
// Replaces the reference's CPU collate, pipeline.py:158-213 (prepare_batch)
// and kernels.py:112-121 (fill_batch), and adds the NEW crop/flip/normalise
// augment of SURVEY.md §8a A6'.  All of them are HBM-bound byte movers
// (no contraction -> no tensor cores): 128-bit coalesced accesses, source rows
// staged through shared memory, grids of thousands of CTAs.
#include "tsb_common.cuh"

using namespace tsb;

namespace {

// ---------------------------------------------------------------------------
// SplitMix64 fill: out[s*W + w] = mix64(key_s + (w+1)*GAMMA)
// key_mode 0: key_s = derive_key(seed, epoch, idx[s])   (SyntheticSource)
// key_mode 1: key_s = derive_key(seed, 0, first + s)    (store / DirectorySource)
constexpr int FILL_THREADS = 256;
constexpr int FILL_WORDS_PER_CTA = 8192;  // 64 KB of output per CTA

__global__ void __launch_bounds__(FILL_THREADS)
    fill_kernel(uint64_t *__restrict__ out, const int64_t *__restrict__ idx, uint64_t seed,
                uint64_t epoch, int64_t wps, int key_mode, int64_t first) {
    const int64_t s = blockIdx.y;
    const uint64_t key = key_mode == 0 ? derive_key(seed, epoch, (uint64_t)idx[s])
                                       : derive_key(seed, 0, (uint64_t)(first + s));
    uint64_t *dst = out + s * wps;
    const int64_t w0 = (int64_t)blockIdx.x * FILL_WORDS_PER_CTA;
    const int64_t w1 = min(w0 + FILL_WORDS_PER_CTA, wps);
    if ((wps & 1) == 0) {
        // pairs of words -> 16-byte stores; sample base is 16B aligned
        for (int64_t w = w0 + 2 * threadIdx.x; w < w1; w += 2 * FILL_THREADS) {
            uint64_t a = mix64(key + (uint64_t)(w + 1) * GAMMA);
            uint64_t b = mix64(key + (uint64_t)(w + 2) * GAMMA);
            uint4 v = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
            st_v4(dst + w, v);
        }
    } else {
        for (int64_t w = w0 + threadIdx.x; w < w1; w += FILL_THREADS)
            dst[w] = mix64(key + (uint64_t)(w + 1) * GAMMA);
    }
}

// ---------------------------------------------------------------------------
// Gather (passthrough collate): out[s] = src[idx[s]] for whole samples.
constexpr int GATHER_THREADS = 256;
constexpr int GATHER_UNROLL = 4;
constexpr int64_t GATHER_BYTES_PER_CTA = GATHER_THREADS * GATHER_UNROLL * 16 * 4;  // 64 KB

__global__ void __launch_bounds__(GATHER_THREADS)
    gather_v16_kernel(const uint8_t *__restrict__ src, const int64_t *__restrict__ idx,
                      int64_t sb, uint8_t *__restrict__ out) {
    const int64_t s = blockIdx.y;
    const uint4 *in = reinterpret_cast<const uint4 *>(src + idx[s] * sb);
    uint4 *o = reinterpret_cast<uint4 *>(out + s * sb);
    const int64_t n16 = sb >> 4;
    const int64_t v0 = (int64_t)blockIdx.x * (GATHER_BYTES_PER_CTA >> 4);
    const int64_t v1 = min(v0 + (GATHER_BYTES_PER_CTA >> 4), n16);
    for (int64_t v = v0 + threadIdx.x; v < v1; v += GATHER_THREADS * GATHER_UNROLL) {
        uint4 r[GATHER_UNROLL];
#pragma unroll
        for (int u = 0; u < GATHER_UNROLL; ++u) {
            int64_t k = v + (int64_t)u * GATHER_THREADS;
            if (k < v1) r[u] = ld_nc_v4(in + k);
        }
#pragma unroll
        for (int u = 0; u < GATHER_UNROLL; ++u) {
            int64_t k = v + (int64_t)u * GATHER_THREADS;
            if (k < v1) st_v4(o + k, r[u]);
        }
    }
}

__global__ void gather_v1_kernel(const uint8_t *__restrict__ src, const int64_t *__restrict__ idx,
                                 int64_t sb, uint8_t *__restrict__ out) {
    const int64_t s = blockIdx.y;
    const uint8_t *in = src + idx[s] * sb;
    uint8_t *o = out + s * sb;
    const int64_t b0 = (int64_t)blockIdx.x * GATHER_BYTES_PER_CTA;
    const int64_t b1 = min(b0 + GATHER_BYTES_PER_CTA, sb);
    for (int64_t k = b0 + threadIdx.x; k < b1; k += blockDim.x) o[k] = in[k];
}

// ---------------------------------------------------------------------------
// Augment params (SURVEY.md §8a A6'):
//   ka = derive_key(mix64(aug_seed ^ AUG_DOMAIN), epoch, idx)
//   oy = mix64(ka+1G) % (2P+1), ox = mix64(ka+2G) % (2P+1), flip = mix64(ka+3G) & 1
__device__ __forceinline__ void derive_aug(uint64_t aug_mixed, uint64_t epoch, int64_t index,
                                           int pad, int flip_en, int &oy, int &ox, int &fl) {
    const uint64_t ka = derive_key(aug_mixed, epoch, (uint64_t)index);
    const uint64_t m = (uint64_t)(2 * pad + 1);
    oy = (int)(mix64(ka + GAMMA) % m);
    ox = (int)(mix64(ka + 2 * GAMMA) % m);
    fl = flip_en ? (int)(mix64(ka + 3 * GAMMA) & 1) : 0;
}

__global__ void aug_params_kernel(uint64_t aug_mixed, uint64_t epoch,
                                  const int64_t *__restrict__ idx, int64_t b, int pad, int flip_en,
                                  int32_t *__restrict__ params) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b) return;
    int oy, ox, fl;
    derive_aug(aug_mixed, epoch, idx[i], pad, flip_en, oy, ox, fl);
    params[3 * i] = oy;
    params[3 * i + 1] = ox;
    params[3 * i + 2] = fl;
}

// ---------------------------------------------------------------------------
// Fused collate/augment: uint8 HWC -> pad/crop/flip -> normalise -> NCHW.
//
// CTA = (sample, block of ROWS output rows).  The crop shifts whole rows, so
// the source rows of a row block are one contiguous byte range: it is
// staged into shared memory with 16-byte loads (coalesced, read once), then
// every thread emits 16-byte stores of VEC consecutive x of one channel row
// -- NCHW channel planes are written as fully coalesced streams.
// Normalisation is fl(fl(u*scale)+bias) (no FMA), bit-exact with the oracle.
constexpr int CA_THREADS = 256;
constexpr int CA_ROWS = 8;
constexpr int MAX_DST = 8;

struct Norm {
    float scale[4];
    float bias[4];
};
struct Dsts {
    void *p[MAX_DST];
    int n;
};

template <int OUT_KIND>
struct OutTraits;
template <>
struct OutTraits<TSB_OUT_U8> {
    static constexpr int VEC = 16;
    static constexpr int ELEM = 1;
};
template <>
struct OutTraits<TSB_OUT_F32> {
    static constexpr int VEC = 4;
    static constexpr int ELEM = 4;
};
template <>
struct OutTraits<TSB_OUT_BF16> {
    static constexpr int VEC = 8;
    static constexpr int ELEM = 2;
};

__device__ __forceinline__ uint32_t bf16_rne_bits(float f) {
    uint32_t u = __float_as_uint(f);
    // inputs are finite (u8 * finite scale + finite bias); RNE on the top half
    u += 0x7FFFu + ((u >> 16) & 1u);
    return u >> 16;
}

template <int OUT_KIND>
__global__ void __launch_bounds__(CA_THREADS)
    collate_augment_kernel(const uint8_t *__restrict__ src, const int64_t *__restrict__ idx,
                           int h, int w, int c, int pad, int flip_en, uint64_t aug_mixed,
                           uint64_t epoch, Norm norm, const int32_t *__restrict__ params,
                           Dsts dsts, int vec_src) {
    using T = OutTraits<OUT_KIND>;
    extern __shared__ __align__(16) uint8_t rows[];
    __shared__ int s_par[3];

    const int s = blockIdx.y;
    const int y0 = blockIdx.x * CA_ROWS;
    const int nrows = min(CA_ROWS, h - y0);
    const int row_bytes = w * c;
    const int64_t sample_bytes = (int64_t)h * row_bytes;

    if (threadIdx.x == 0) {
        int oy, ox, fl;
        if (params) {
            oy = params[3 * s];
            ox = params[3 * s + 1];
            fl = params[3 * s + 2];
        } else {
            derive_aug(aug_mixed, epoch, idx[s], pad, flip_en, oy, ox, fl);
        }
        s_par[0] = oy;
        s_par[1] = ox;
        s_par[2] = fl;
    }
    __syncthreads();
    const int oy = s_par[0], ox = s_par[1], fl = s_par[2];

    // contiguous source row range for this row block
    const int sy_first = y0 + oy - pad;  // source row of output row y0
    const int lo = max(sy_first, 0);
    const int hi = min(sy_first + nrows, h);  // exclusive
    const uint8_t *sample = src + idx[s] * sample_bytes;
    if (hi > lo) {
        const uint8_t *g = sample + (int64_t)lo * row_bytes;
        uint8_t *sm = rows + (lo - sy_first) * row_bytes;
        const int nbytes = (hi - lo) * row_bytes;
        if (vec_src) {
            const int n16 = nbytes >> 4;
            for (int v = threadIdx.x; v < n16; v += CA_THREADS)
                reinterpret_cast<uint4 *>(sm)[v] = ld_nc_v4(g + 16 * v);
        } else {
            for (int v = threadIdx.x; v < nbytes; v += CA_THREADS) sm[v] = g[v];
        }
    }
    __syncthreads();

    const int xg_per_row = w / T::VEC;
    const int items = c * nrows * xg_per_row;
    const int64_t plane = (int64_t)h * w;
    for (int it = threadIdx.x; it < items; it += CA_THREADS) {
        const int xg = it % xg_per_row;
        const int rc = it / xg_per_row;
        const int r = rc % nrows;
        const int ch = rc / nrows;
        const int sy = sy_first + r;
        const bool row_ok = (sy >= 0) && (sy < h);
        const uint8_t *srow = rows + r * row_bytes + ch;
        const int x0 = xg * T::VEC;
        uint8_t u[T::VEC];
#pragma unroll
        for (int k = 0; k < T::VEC; ++k) {
            const int x = x0 + k;
            const int sx = (fl ? (w - 1 - x) : x) + ox - pad;
            u[k] = (row_ok && sx >= 0 && sx < w) ? srow[sx * c] : (uint8_t)0;
        }
        uint4 v;
        if constexpr (OUT_KIND == TSB_OUT_U8) {
            uint32_t wv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wv[q] = (uint32_t)u[4 * q] | ((uint32_t)u[4 * q + 1] << 8) |
                        ((uint32_t)u[4 * q + 2] << 16) | ((uint32_t)u[4 * q + 3] << 24);
            v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        } else {
            // static indexing only (dynamic param-array indexing spills to local)
            float sc = norm.scale[0], bi = norm.bias[0];
            if (ch == 1) { sc = norm.scale[1]; bi = norm.bias[1]; }
            else if (ch == 2) { sc = norm.scale[2]; bi = norm.bias[2]; }
            else if (ch == 3) { sc = norm.scale[3]; bi = norm.bias[3]; }
            float f[T::VEC];
#pragma unroll
            for (int k = 0; k < T::VEC; ++k) f[k] = __fadd_rn(__fmul_rn((float)u[k], sc), bi);
            if constexpr (OUT_KIND == TSB_OUT_F32) {
                v = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                               __float_as_uint(f[2]), __float_as_uint(f[3]));
            } else {
                uint32_t wv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    wv[q] = bf16_rne_bits(f[2 * q]) | (bf16_rne_bits(f[2 * q + 1]) << 16);
                v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
        }
        const int64_t off =
            (((int64_t)s * c + ch) * plane + (int64_t)(y0 + r) * w + x0) * T::ELEM;
#pragma unroll
        for (int d = 0; d < MAX_DST; ++d)
            if (d < dsts.n) st_v4(static_cast<uint8_t *>(dsts.p[d]) + off, v);
    }
}

int launch_collate(const void *src, const int64_t *d_indices, int64_t b, int h, int w, int c,
                   int pad, int flip, uint64_t aug_seed, uint64_t epoch, const float *scale,
                   const float *bias, int out_kind, const int32_t *d_params, const Dsts &dsts,
                   void *stream) {
    TSB_CHECK(src && d_indices, "null src/indices");
    TSB_CHECK(b >= 0 && h > 0 && w > 0 && c > 0 && c <= 4, "bad shape b=%lld h=%d w=%d c=%d",
              (long long)b, h, w, c);
    TSB_CHECK(pad >= 0 && pad <= 1 << 20, "bad pad %d", pad);
    TSB_CHECK(out_kind >= TSB_OUT_U8 && out_kind <= TSB_OUT_BF16, "bad out_kind %d", out_kind);
    TSB_CHECK(b <= 65535, "batch %lld exceeds grid.y limit", (long long)b);
    if (b == 0) return TSB_OK;
    const int vec = out_kind == TSB_OUT_U8 ? 16 : out_kind == TSB_OUT_F32 ? 4 : 8;
    const int elem = out_kind == TSB_OUT_U8 ? 1 : out_kind == TSB_OUT_F32 ? 4 : 2;
    TSB_CHECK(w % vec == 0, "width %d must be a multiple of %d for this output kind", w, vec);
    for (int d = 0; d < dsts.n; ++d)
        TSB_CHECK(((uintptr_t)dsts.p[d] & 15) == 0, "output must be 16-byte aligned");
    (void)elem;
    Norm norm;
    for (int i = 0; i < 4; ++i) {
        norm.scale[i] = (scale && i < c) ? scale[i] : 1.0f;
        norm.bias[i] = (bias && i < c) ? bias[i] : 0.0f;
    }
    const int row_bytes = w * c;
    const int vec_src = ((row_bytes & 15) == 0) && (((uintptr_t)src & 15) == 0);
    const size_t smem = (size_t)CA_ROWS * row_bytes;
    TSB_CHECK(smem <= 200 * 1024, "row too wide for shared staging (%zu B)", smem);
    const uint64_t aug_mixed = mix64(aug_seed ^ AUG_DOMAIN);
    dim3 grid((h + CA_ROWS - 1) / CA_ROWS, (unsigned)b);
    auto s = as_stream(stream);
#define TSB_LAUNCH_CA(K)                                                                   \
    do {                                                                                   \
        if (smem > 48 * 1024)                                                              \
            TSB_CUDA(cudaFuncSetAttribute(collate_augment_kernel<K>,                       \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                          (int)smem));                                     \
        collate_augment_kernel<K><<<grid, CA_THREADS, smem, s>>>(                          \
            static_cast<const uint8_t *>(src), d_indices, h, w, c, pad, flip, aug_mixed,   \
            epoch, norm, d_params, dsts, vec_src);                                         \
    } while (0)
    if (out_kind == TSB_OUT_U8)
        TSB_LAUNCH_CA(TSB_OUT_U8);
    else if (out_kind == TSB_OUT_F32)
        TSB_LAUNCH_CA(TSB_OUT_F32);
    else
        TSB_LAUNCH_CA(TSB_OUT_BF16);
#undef TSB_LAUNCH_CA
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

}  // namespace

extern "C" {

int tsb_fill_synthetic(void *out, const int64_t *d_indices, int64_t b, uint64_t seed,
                       uint64_t epoch, int64_t sample_bytes, void *stream) {
    TSB_CHECK(out && d_indices, "null pointer");
    TSB_CHECK(sample_bytes > 0 && sample_bytes % 8 == 0,
              "synthetic sample size must be a multiple of 8 bytes (got %lld)",
              (long long)sample_bytes);
    TSB_CHECK(((uintptr_t)out & 15) == 0, "output must be 16-byte aligned");
    TSB_CHECK(b >= 0 && b <= 65535, "bad batch %lld", (long long)b);
    if (b == 0) return TSB_OK;
    const int64_t wps = sample_bytes / 8;
    dim3 grid((unsigned)((wps + FILL_WORDS_PER_CTA - 1) / FILL_WORDS_PER_CTA), (unsigned)b);
    fill_kernel<<<grid, FILL_THREADS, 0, as_stream(stream)>>>(static_cast<uint64_t *>(out),
                                                              d_indices, seed, epoch, wps, 0, 0);
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

int tsb_make_store(void *out, uint64_t seed, int64_t first, int64_t count, int64_t sample_bytes,
                   void *stream) {
    TSB_CHECK(out, "null pointer");
    TSB_CHECK(sample_bytes > 0 && sample_bytes % 8 == 0, "sample_bytes must be a multiple of 8");
    TSB_CHECK(((uintptr_t)out & 15) == 0, "output must be 16-byte aligned");
    const int64_t wps = sample_bytes / 8;
    // grid.y is limited to 65535: chunk over samples
    for (int64_t s0 = 0; s0 < count; s0 += 65535) {
        const int64_t n = (count - s0) < 65535 ? (count - s0) : 65535;
        dim3 grid((unsigned)((wps + FILL_WORDS_PER_CTA - 1) / FILL_WORDS_PER_CTA), (unsigned)n);
        fill_kernel<<<grid, FILL_THREADS, 0, as_stream(stream)>>>(
            static_cast<uint64_t *>(out) + s0 * wps, nullptr, seed, 0, wps, 1, first + s0);
        TSB_LAUNCH_CHECK();
    }
    return TSB_OK;
}

int tsb_gather(const void *src, const int64_t *d_indices, int64_t b, int64_t sample_bytes,
               void *out, void *stream) {
    TSB_CHECK(src && out && d_indices, "null pointer");
    TSB_CHECK(sample_bytes > 0, "bad sample_bytes");
    TSB_CHECK(b >= 0 && b <= 65535, "bad batch %lld", (long long)b);
    if (b == 0) return TSB_OK;
    dim3 grid((unsigned)((sample_bytes + GATHER_BYTES_PER_CTA - 1) / GATHER_BYTES_PER_CTA),
              (unsigned)b);
    const bool v16 = (sample_bytes % 16 == 0) && (((uintptr_t)src & 15) == 0) &&
                     (((uintptr_t)out & 15) == 0);
    if (v16)
        gather_v16_kernel<<<grid, GATHER_THREADS, 0, as_stream(stream)>>>(
            static_cast<const uint8_t *>(src), d_indices, sample_bytes, static_cast<uint8_t *>(out));
    else
        gather_v1_kernel<<<grid, GATHER_THREADS, 0, as_stream(stream)>>>(
            static_cast<const uint8_t *>(src), d_indices, sample_bytes, static_cast<uint8_t *>(out));
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

int tsb_aug_params(uint64_t aug_seed, uint64_t epoch, const int64_t *d_indices, int64_t b, int pad,
                   int flip, int32_t *d_params, void *stream) {
    TSB_CHECK(d_indices && d_params, "null pointer");
    TSB_CHECK(pad >= 0, "bad pad");
    if (b <= 0) return TSB_OK;
    const int t = 256;
    aug_params_kernel<<<(unsigned)((b + t - 1) / t), t, 0, as_stream(stream)>>>(
        mix64(aug_seed ^ AUG_DOMAIN), epoch, d_indices, b, pad, flip, d_params);
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

int tsb_collate_augment(const void *src, const int64_t *d_indices, int64_t b, int h, int w, int c,
                        int pad, int flip, uint64_t aug_seed, uint64_t epoch, const float *scale,
                        const float *bias, int out_kind, const int32_t *d_params, void *out,
                        void *stream) {
    TSB_CHECK(out, "null output");
    Dsts d{};
    d.p[0] = out;
    d.n = 1;
    return launch_collate(src, d_indices, b, h, w, c, pad, flip, aug_seed, epoch, scale, bias,
                          out_kind, d_params, d, stream);
}

int tsb_collate_augment_fanout(const void *src, const int64_t *d_indices, int64_t b, int h, int w,
                               int c, int pad, int flip, uint64_t aug_seed, uint64_t epoch,
                               const float *scale, const float *bias, int out_kind,
                               void *const *dsts, int n_dst, void *stream) {
    TSB_CHECK(dsts && n_dst >= 1 && n_dst <= MAX_DST, "n_dst must be 1..%d", MAX_DST);
    Dsts d{};
    for (int i = 0; i < n_dst; ++i) {
        TSB_CHECK(dsts[i], "null destination %d", i);
        d.p[i] = dsts[i];
    }
    d.n = n_dst;
    return launch_collate(src, d_indices, b, h, w, c, pad, flip, aug_seed, epoch, scale, bias,
                          out_kind, nullptr, d, stream);
}

}  // extern "C"
