/*
 * ts_oracle.c -- CPU ORACLE for the shared-loading hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path
 * (paper_2409_18749_b200/) never links, imports or calls anything here.
 *
 * It restates, in plain C, the reference algorithm of the path
 * (reference = /root/reference, paths relative to pkg/):
 *
 *   mix64            src/batchsocket/kernels.py:40-45   (SplitMix64 finalizer)
 *   derive_key       src/batchsocket/kernels.py:48-53
 *   fill_batch       src/batchsocket/kernels.py:112-121 (numba) / :64-67 (numpy)
 *   permutation      src/batchsocket/kernels.py:123-140 (Fisher-Yates)
 *   epoch_order      src/batchsocket/pipeline.py:113-123 (_SHUFFLE_DOMAIN :25)
 *   prepare_batch    src/batchsocket/pipeline.py:158-213 (synthetic :183-189,
 *                    directory/store gather :190-210)
 *   checksum         src/batchsocket/wire.py:170-172 (zlib CRC-32/IEEE)
 *
 * and the NEW crop/flip/normalise augment spec (SURVEY.md §8a row A6'),
 * which has no reference implementation: "parity unpinned" for that part --
 * it is pinned only by this restatement and the independent numpy
 * restatement in oracle/oracle.py (tests cross-check the two).
 *
 * Everything except the augment is pinned against golden vectors generated
 * by running the reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GAMMA 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL
#define SHUFFLE_DOMAIN 0x53485546ULL /* pipeline.py:25 */
#define AUG_DOMAIN 0x41554731ULL     /* "AUG1", SURVEY.md §8a A6' */

/* kernels.py:40-45 */
uint64_t tso_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

/* kernels.py:48-53 */
uint64_t tso_derive_key(uint64_t seed, uint64_t epoch, uint64_t index) {
    uint64_t h = tso_mix64(seed + GAMMA);
    h = tso_mix64((h ^ epoch) + GAMMA);
    h = tso_mix64((h ^ index) + GAMMA);
    return h;
}

/* kernels.py:123-140 -- sequential Fisher-Yates driven by the key stream. */
void tso_permutation(int64_t n, uint64_t key, int64_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    uint64_t t = 0;
    for (int64_t i = n - 1; i > 0; --i) {
        uint64_t r = tso_mix64(key + (t + 1) * GAMMA);
        t += 1;
        int64_t j = (int64_t)(r % (uint64_t)(i + 1));
        int64_t tmp = out[i];
        out[i] = out[j];
        out[j] = tmp;
    }
}

/* pipeline.py:113-123 */
void tso_epoch_order(int64_t n, uint64_t shuffle_seed, uint64_t epoch, int reshuffle,
                     int64_t *out) {
    uint64_t eff = reshuffle ? epoch : 0;
    tso_permutation(n, tso_derive_key(shuffle_seed, eff, SHUFFLE_DOMAIN), out);
}

/* kernels.py:112-121: out[s*W + w] = mix64(key_s + (w+1)*GAMMA), little-endian words */
void tso_fill_batch(uint64_t *out, const uint64_t *keys, int64_t nkeys, int64_t wps) {
    for (int64_t s = 0; s < nkeys; ++s)
        for (int64_t w = 0; w < wps; ++w)
            out[s * wps + w] = tso_mix64(keys[s] + (uint64_t)(w + 1) * GAMMA);
}

/* pipeline.py:183-189: synthetic source, key per sample = derive_key(seed, epoch, idx). */
void tso_prepare_synthetic(uint64_t seed, uint64_t epoch, const int64_t *indices, int64_t b,
                           int64_t sample_bytes, uint8_t *out, int nthreads) {
    int64_t wps = sample_bytes / 8;
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
    for (int64_t s = 0; s < b; ++s) {
        uint64_t k = tso_derive_key(seed, epoch, (uint64_t)indices[s]);
        uint64_t *dst = (uint64_t *)(out + s * sample_bytes);
        for (int64_t w = 0; w < wps; ++w) dst[w] = tso_mix64(k + (uint64_t)(w + 1) * GAMMA);
    }
}

/* pipeline.py:139-155: directory dataset file i = fill(derive_key(seed, 0, i)).
 * Materialises samples [first, first+count) of such a store. */
void tso_make_store(uint64_t seed, int64_t first, int64_t count, int64_t sample_bytes,
                    uint8_t *out, int nthreads) {
    int64_t wps = sample_bytes / 8;
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
    for (int64_t s = 0; s < count; ++s) {
        uint64_t k = tso_derive_key(seed, 0, (uint64_t)(first + s));
        uint64_t *dst = (uint64_t *)(out + s * sample_bytes);
        for (int64_t w = 0; w < wps; ++w) dst[w] = tso_mix64(k + (uint64_t)(w + 1) * GAMMA);
    }
}

/* pipeline.py:190-210: batch bytes = concatenation of store samples in order. */
void tso_gather(const uint8_t *store, const int64_t *indices, int64_t b, int64_t sample_bytes,
                uint8_t *out, int nthreads) {
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
    for (int64_t s = 0; s < b; ++s)
        memcpy(out + s * sample_bytes, store + indices[s] * sample_bytes, (size_t)sample_bytes);
}

/* ---- augment spec (NEW; SURVEY.md §8a A6') -------------------------------
 * ka = derive_key(mix64(aug_seed ^ AUG_DOMAIN), epoch, sample_idx)
 * r_w = mix64(ka + (w+1)*GAMMA)           (same word convention as fill_batch)
 * oy = r0 % (2P+1), ox = r1 % (2P+1), flip = flip_enable ? (r2 & 1) : 0
 */
void tso_aug_params(uint64_t aug_seed, uint64_t epoch, const int64_t *indices, int64_t b,
                    int pad, int flip_enable, int32_t *params /* b x 3: oy, ox, flip */) {
    uint64_t s = tso_mix64(aug_seed ^ AUG_DOMAIN);
    uint64_t m = (uint64_t)(2 * pad + 1);
    for (int64_t i = 0; i < b; ++i) {
        uint64_t ka = tso_derive_key(s, epoch, (uint64_t)indices[i]);
        params[3 * i + 0] = (int32_t)(tso_mix64(ka + 1 * GAMMA) % m);
        params[3 * i + 1] = (int32_t)(tso_mix64(ka + 2 * GAMMA) % m);
        params[3 * i + 2] = flip_enable ? (int32_t)(tso_mix64(ka + 3 * GAMMA) & 1) : 0;
    }
}

/* fp32 normalisation constants: scale = f32(1/(255*std)), bias = f32(-mean/std),
 * both computed in double and rounded once. */
void tso_norm_consts(const double *mean, const double *stdv, int c, float *scale, float *bias) {
    for (int i = 0; i < c; ++i) {
        scale[i] = (float)(1.0 / (255.0 * stdv[i]));
        bias[i] = (float)(-mean[i] / stdv[i]);
    }
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

/* out_kind: 0 = u8 NCHW (crop/flip only), 1 = f32 NCHW, 2 = bf16 NCHW.
 * Output pixel (c, y, x) of sample i:
 *   sy = y + oy - P;  sx = (flip ? W-1-x : x) + ox - P
 *   u  = (0 <= sy < H && 0 <= sx < W) ? src[(sy*W + sx)*C + c] : 0   (pad-then-crop)
 *   v  = fl(fl(float(u) * scale[c]) + bias[c])                        (no FMA)
 * params: optional b x 3 table (oy, ox, flip); NULL = derive from the RNG. */
void tso_collate_augment(const uint8_t *store, const int64_t *indices, int64_t b, int h, int w,
                         int c, int pad, int flip_enable, uint64_t aug_seed, uint64_t epoch,
                         const float *scale, const float *bias, int out_kind,
                         const int32_t *params, void *out, int nthreads) {
    (void)nthreads;
    int64_t sample_bytes = (int64_t)h * w * c;
    int64_t plane = (int64_t)h * w;
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
    for (int64_t i = 0; i < b; ++i) {
        int32_t p3[3];
        if (params) {
            p3[0] = params[3 * i];
            p3[1] = params[3 * i + 1];
            p3[2] = params[3 * i + 2];
        } else {
            tso_aug_params(aug_seed, epoch, &indices[i], 1, pad, flip_enable, p3);
        }
        const uint8_t *src = store + indices[i] * sample_bytes;
        for (int ch = 0; ch < c; ++ch) {
            float sc = scale ? scale[ch] : 1.0f, bi = bias ? bias[ch] : 0.0f;
            for (int y = 0; y < h; ++y) {
                int sy = y + p3[0] - pad;
                int64_t obase = ((i * c + ch) * plane) + (int64_t)y * w;
                for (int x = 0; x < w; ++x) {
                    int sx = (p3[2] ? (w - 1 - x) : x) + p3[1] - pad;
                    uint8_t u = (sy >= 0 && sy < h && sx >= 0 && sx < w)
                                    ? src[((int64_t)sy * w + sx) * c + ch]
                                    : 0;
                    if (out_kind == 0) {
                        ((uint8_t *)out)[obase + x] = u;
                    } else {
                        /* two roundings: built with -ffp-contract=off (no FMA) */
                        float v = (float)u * sc + bi;
                        if (out_kind == 1)
                            ((float *)out)[obase + x] = v;
                        else
                            ((uint16_t *)out)[obase + x] = f32_to_bf16_rne(v);
                    }
                }
            }
        }
    }
}

/* ---- CRC-32/IEEE (reflected 0xEDB88320, init/xorout 0xFFFFFFFF) ----------
 * wire.py:170-172 uses zlib.crc32; tests/test_wire.py:27-34 is the bitwise
 * oracle it is pinned to.  Slice-by-8 for speed; running form like zlib:
 * crc32(data, n, prev) with prev = 0 for a fresh checksum. */
static uint32_t crc_tab[8][256];
static int crc_ready = 0;

static void crc_init(void) {
    if (crc_ready) return;
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t r = i;
        for (int k = 0; k < 8; ++k) r = (r >> 1) ^ (0xEDB88320u & (0u - (r & 1u)));
        crc_tab[0][i] = r;
    }
    for (uint32_t i = 0; i < 256; ++i)
        for (int t = 1; t < 8; ++t)
            crc_tab[t][i] = (crc_tab[t - 1][i] >> 8) ^ crc_tab[0][crc_tab[t - 1][i] & 0xFF];
    crc_ready = 1;
}

uint32_t tso_crc32(const uint8_t *p, size_t n, uint32_t prev) {
    crc_init();
    uint32_t crc = ~prev;
    while (n && ((uintptr_t)p & 7)) {
        crc = crc_tab[0][(crc ^ *p++) & 0xFF] ^ (crc >> 8);
        --n;
    }
    while (n >= 8) {
        uint64_t v;
        memcpy(&v, p, 8);
        uint32_t lo = (uint32_t)v ^ crc, hi = (uint32_t)(v >> 32);
        crc = crc_tab[7][lo & 0xFF] ^ crc_tab[6][(lo >> 8) & 0xFF] ^ crc_tab[5][(lo >> 16) & 0xFF] ^
              crc_tab[4][lo >> 24] ^ crc_tab[3][hi & 0xFF] ^ crc_tab[2][(hi >> 8) & 0xFF] ^
              crc_tab[1][(hi >> 16) & 0xFF] ^ crc_tab[0][hi >> 24];
        p += 8;
        n -= 8;
    }
    while (n--) crc = crc_tab[0][(crc ^ *p++) & 0xFF] ^ (crc >> 8);
    return ~crc;
}

/* Bitwise CRC (tests/test_wire.py:27-34 restated), for cross-checking. */
uint32_t tso_crc32_bitwise(const uint8_t *p, size_t n) {
    uint32_t crc = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) {
        crc ^= p[i];
        for (int k = 0; k < 8; ++k) crc = (crc >> 1) ^ (0xEDB88320u * (crc & 1u));
    }
    return crc ^ 0xFFFFFFFFu;
}

/* GF(2) polynomial arithmetic mod the reflected CRC polynomial: the standard
 * CRC combination identity crc(A||B) = x^(8|B|)*crc(A) + crc(B). */
static uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}

static uint32_t x8nmodp(uint64_t n) { /* x^(8n) mod p */
    uint32_t p = 1u << 31, sq = 1u << 30; /* x^0, x^1 */
    for (int i = 0; i < 3; ++i) sq = multmodp(sq, sq); /* x^8 */
    while (n) {
        if (n & 1) p = multmodp(sq, p);
        n >>= 1;
        sq = multmodp(sq, sq);
    }
    return p;
}

uint32_t tso_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
    return multmodp(x8nmodp(len2), crc1) ^ crc2;
}

/* Rebatch: consumer with batch size bsz, batch j of epoch -> samples
 * order[j*bsz : (j+1)*bsz] (pipeline.py:178-180 with batch_size = bsz;
 * the epoch order does not depend on the batch size, pipeline.py:113-123). */
int64_t tso_epoch_len(int64_t samples_per_epoch, int64_t bsz) { return samples_per_epoch / bsz; }

int tso_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
