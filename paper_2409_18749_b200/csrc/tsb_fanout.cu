// Fan-out (one slot -> N destination slots, local or peer GPUs over
// NVLink/NVSwitch with P2P stores) and the per-consumer rebatch gather.
//
// NEW subsystems (no reference code): the reference's
// "broadcast" is every consumer mapping the same shm name
// (bs/consumer.py:319-321); across GPUs the bytes must move.  Each source
// 16-byte vector is loaded once and stored to every destination, so the
// producer reads HBM once and its egress is (N-1) x bytes on NVLink.
#include "tsb_common.cuh"

using namespace tsb;

namespace {

constexpr int FO_THREADS = 512;
constexpr int FO_MAX = 8;
struct DstList {
    void *p[FO_MAX];
    int n;
};

__global__ void __launch_bounds__(FO_THREADS)
    fanout_v16_kernel(const uint4 *__restrict__ src, DstList d, uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * FO_THREADS;
    uint64_t i = (uint64_t)blockIdx.x * FO_THREADS + threadIdx.x;
    constexpr int U = 4;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_nc_v4(src + i + u * stride);
#pragma unroll
        for (int k = 0; k < FO_MAX; ++k) {
            if (k < d.n) {
                uint4 *o = static_cast<uint4 *>(d.p[k]);
#pragma unroll
                for (int u = 0; u < U; ++u) st_v4(o + i + u * stride, v[u]);
            }
        }
    }
    for (; i < n16; i += stride) {
        uint4 v = ld_nc_v4(src + i);
#pragma unroll
        for (int k = 0; k < FO_MAX; ++k)
            if (k < d.n) st_v4(static_cast<uint4 *>(d.p[k]) + i, v);
    }
}

__global__ void fanout_tail_kernel(const uint8_t *__restrict__ src, DstList d, uint64_t from,
                                   uint64_t n) {
    for (uint64_t i = from + threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
        for (int k = 0; k < FO_MAX; ++k)
            if (k < d.n) static_cast<uint8_t *>(d.p[k])[i] = src[i];
}

// Rebatch: out[j] = ring[(first + j) mod ring_samples], whole samples.
constexpr int RB_THREADS = 256;
constexpr int64_t RB_BYTES_PER_CTA = 64 * 1024;

__global__ void __launch_bounds__(RB_THREADS)
    rebatch_kernel(const uint8_t *__restrict__ ring, int64_t ring_samples, int64_t sb,
                   int64_t first, uint8_t *__restrict__ out, int vec) {
    const int64_t j = blockIdx.y;
    const int64_t pos = (first + j) % ring_samples;
    const uint8_t *in = ring + pos * sb;
    uint8_t *o = out + j * sb;
    const int64_t b0 = (int64_t)blockIdx.x * RB_BYTES_PER_CTA;
    const int64_t b1 = min(b0 + RB_BYTES_PER_CTA, sb);
    if (vec) {
        for (int64_t k = b0 + 16 * threadIdx.x; k < b1; k += 16 * RB_THREADS)
            st_v4(o + k, ld_nc_v4(in + k));
    } else {
        for (int64_t k = b0 + threadIdx.x; k < b1; k += RB_THREADS) o[k] = in[k];
    }
}

// Rebatch window: consumer batch = stream samples [first, first+count) of a
// producer whose slots hold `per_slot` samples laid out [inputs][targets]
// (the pair layout of sl/abi.py:27-31).  slots[k] = base of the k-th
// producer slot the window touches (first / per_slot is slot 0).  Output:
// [count inputs][count targets].  One CTA row per window sample; each part
// moves in 16 B vectors when its offsets allow (vec bit 0: inputs, bit 1:
// targets, bit 2: aligned 8-byte int64 targets; the int64 target alone used
// to force the byte loop on the inputs too -- 241 us for a 115 MB window,
// profiles/r2/ncu_full_rebatch_v1.txt).
constexpr int RW_MAX_SLOTS = 32;
struct SlotList {
    const uint8_t *p[RW_MAX_SLOTS];
};

__global__ void __launch_bounds__(RB_THREADS)
    rebatch_window_kernel(SlotList sl, int64_t first, int64_t per_slot, int64_t in_sb,
                          int64_t tg_sb, int64_t count, uint8_t *__restrict__ out, int vec) {
    const int64_t j = blockIdx.y;
    const int64_t pos = first + j;
    const int64_t k = pos / per_slot - first / per_slot, i = pos % per_slot;
    const uint8_t *slot = sl.p[k];
    // input part, then target part of sample j
    for (int part = 0; part < 2; ++part) {
        const int64_t sb = part ? tg_sb : in_sb;
        if (!sb) continue;
        const uint8_t *in = part ? slot + per_slot * in_sb + i * tg_sb : slot + i * in_sb;
        uint8_t *o = part ? out + count * in_sb + j * tg_sb : out + j * in_sb;
        const int64_t b0 = (int64_t)blockIdx.x * RB_BYTES_PER_CTA;
        const int64_t b1 = min(b0 + RB_BYTES_PER_CTA, sb);
        if ((vec >> part) & 1) {  // 4 independent 16 B loads in flight per thread
            constexpr int U = 4;
            for (int64_t q = b0 + 16 * threadIdx.x; q < b1; q += 16 * RB_THREADS * U) {
                uint4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t qq = q + (int64_t)u * 16 * RB_THREADS;
                    if (qq < b1) v[u] = ld_nc_v4(in + qq);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t qq = q + (int64_t)u * 16 * RB_THREADS;
                    if (qq < b1) st_v4(o + qq, v[u]);
                }
            }
        } else if (part && sb == 8 && (vec & 4)) {  // one aligned int64 target per sample
            if (blockIdx.x == 0 && threadIdx.x == 0)
                *reinterpret_cast<int64_t *>(o) = *reinterpret_cast<const int64_t *>(in);
        } else {
            for (int64_t q = b0 + threadIdx.x; q < b1; q += RB_THREADS) o[q] = in[q];
        }
    }
}

}  // namespace

extern "C" {

int tsb_rebatch_window(const void *const *slots, int n_slots, int64_t first, int64_t count,
                       int64_t per_slot, int64_t in_sample_bytes, int64_t tgt_sample_bytes,
                       void *out, void *stream) {
    TSB_CHECK(slots && out, "null pointer");
    TSB_CHECK(per_slot > 0 && first >= 0 && count >= 0 && count <= 65535 && in_sample_bytes > 0 &&
                  tgt_sample_bytes >= 0,
              "bad rebatch window");
    if (!count) return TSB_OK;
    const int64_t need = (first + count - 1) / per_slot - first / per_slot + 1;
    TSB_CHECK(n_slots >= need && n_slots <= RW_MAX_SLOTS, "window needs %lld slots, got %d (max %d)",
              (long long)need, n_slots, RW_MAX_SLOTS);
    SlotList sl{};
    bool aligned = ((uintptr_t)out & 15) == 0;
    for (int k = 0; k < n_slots; ++k) {
        TSB_CHECK(slots[k], "null slot %d", k);
        sl.p[k] = static_cast<const uint8_t *>(slots[k]);
        aligned = aligned && (((uintptr_t)slots[k] & 15) == 0);
    }
    // inputs: every sample offset 16-byte aligned; targets: their region's
    // start in the slot and in the output too
    const bool vec_in = aligned && in_sample_bytes % 16 == 0;
    const bool vec_tg = aligned && tgt_sample_bytes % 16 == 0 &&
                        (per_slot * in_sample_bytes) % 16 == 0 && (count * in_sample_bytes) % 16 == 0;
    const bool tg8 = tgt_sample_bytes == 8 && (per_slot * in_sample_bytes) % 8 == 0 &&
                     (((uintptr_t)out + (uintptr_t)(count * in_sample_bytes)) & 7) == 0 && aligned;
    const int vec = (vec_in ? 1 : 0) | (vec_tg ? 2 : 0) | (tg8 ? 4 : 0);
    const int64_t mx = in_sample_bytes > tgt_sample_bytes ? in_sample_bytes : tgt_sample_bytes;
    dim3 grid((unsigned)((mx + RB_BYTES_PER_CTA - 1) / RB_BYTES_PER_CTA), (unsigned)count);
    rebatch_window_kernel<<<grid, RB_THREADS, 0, as_stream(stream)>>>(
        sl, first, per_slot, in_sample_bytes, tgt_sample_bytes, count, static_cast<uint8_t *>(out),
        vec ? 1 : 0);
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

int tsb_fanout(const void *src, void *const *dsts, int n_dst, size_t bytes, void *stream) {
    TSB_CHECK(src && dsts && n_dst >= 1 && n_dst <= FO_MAX, "n_dst must be 1..%d", FO_MAX);
    DstList d{};
    d.n = n_dst;
    bool aligned = ((uintptr_t)src & 15) == 0;
    for (int i = 0; i < n_dst; ++i) {
        TSB_CHECK(dsts[i], "null destination %d", i);
        d.p[i] = dsts[i];
        aligned = aligned && (((uintptr_t)dsts[i] & 15) == 0);
    }
    if (!bytes) return TSB_OK;
    auto s = as_stream(stream);
    uint64_t n16 = aligned ? bytes / 16 : 0;
    if (n16) {
        uint64_t blocks = (n16 + FO_THREADS * 4 - 1) / (FO_THREADS * 4);
        const uint64_t cap = (uint64_t)sm_count() * 4;
        if (blocks > cap) blocks = cap;
        fanout_v16_kernel<<<(unsigned)blocks, FO_THREADS, 0, s>>>(
            static_cast<const uint4 *>(src), d, n16);
        TSB_LAUNCH_CHECK();
    }
    if (n16 * 16 < bytes) {
        fanout_tail_kernel<<<1, 256, 0, s>>>(static_cast<const uint8_t *>(src), d, n16 * 16, bytes);
        TSB_LAUNCH_CHECK();
    }
    return TSB_OK;
}

int tsb_rebatch_gather(const void *ring_base, int64_t ring_samples, int64_t sample_bytes,
                       int64_t first, int64_t count, void *out, void *stream) {
    TSB_CHECK(ring_base && out, "null pointer");
    TSB_CHECK(ring_samples > 0 && sample_bytes > 0 && first >= 0 && count >= 0 &&
                  count <= 65535,
              "bad rebatch geometry");
    if (!count) return TSB_OK;
    const int vec = (sample_bytes % 16 == 0) && (((uintptr_t)ring_base & 15) == 0) &&
                    (((uintptr_t)out & 15) == 0);
    dim3 grid((unsigned)((sample_bytes + RB_BYTES_PER_CTA - 1) / RB_BYTES_PER_CTA), (unsigned)count);
    rebatch_kernel<<<grid, RB_THREADS, 0, as_stream(stream)>>>(
        static_cast<const uint8_t *>(ring_base), ring_samples, sample_bytes, first % ring_samples,
        static_cast<uint8_t *>(out), vec);
    TSB_LAUNCH_CHECK();
    return TSB_OK;
}

}  // extern "C"

namespace tsb {
void preload_fanout() {
    touch_kernel(fanout_v16_kernel);
    touch_kernel(fanout_tail_kernel);
    touch_kernel(rebatch_kernel);
    touch_kernel(rebatch_window_kernel);
}
}  // namespace tsb
