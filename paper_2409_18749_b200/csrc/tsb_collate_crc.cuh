// Collate/augment with the batch CRC-32 fused in (included by tsb_collate.cu,
// inside its anonymous namespace: uses CaGeom, Norm, Dsts, Epi, ItemPar,
// OutTraits, make_vec, item_par, write_targets).
//
// Replaces create_segment's crc32 over the whole segment (payload.py:218,
// called per batch by the producer, bs/producer.py and sl/producer.py:311-314).
// The separate pass (tsb_crc32 after the collate) re-read the 154 MB slot
// from HBM at one table lookup per output BYTE; here the checksum costs one
// conflict-free shared-memory lookup per output ELEMENT, done by the warps
// that already hold the element's source byte in a register, and no HBM
// traffic at all.
//
// The output element of channel c for source byte v is F_c(v) (f32 / bf16 /
// u8), so by linearity of the raw (zero-init) CRC over GF(2) the checksum of
// a run of 32 consecutive output elements is
//     raw(run) = XOR_p G_c[v_p][p],   G_c[v][p] = x^(8 E (31-p)) * raw(F_c(v))
// (a table of 256 x 32 words per channel).  G_c[v][p] sits at shared address
// R1 + c_off | v << 8 | p << 2: ONE PRMT puts the data byte into address byte
// 1 next to the lane's position bits, and the word lands in bank p.
//
// Emit warps (14): thread t owns one column group (P elements of every
// channel) of rows t / groups + k*dr of each staged item.  Besides the
// normalised stores it looks up its P elements per channel; the lanes of a
// warp cover P column runs, and each lane visits its elements in an order
// rotated by its run index (register and byte rotations), so every lookup
// instruction reads 32 distinct positions p -- 32 banks, no conflicts.  The
// 32/P lanes of a run XOR-reduce (shuffles) and one writes raw(row, run) of
// each channel to a small per-stage buffer.
//
// Combiner warps (one per column run): lane r takes row r, shifts raw(row r,
// run) to the end of the item's segment (a lane-specific constant multiply,
// lane-replicated nibble tables), the warp XOR-reduces the rows, and the run
// offset and the segment's place in the slot are applied by bit expansion
// (W[m][i] = x^(8 (SEGB m + tail)) * e_i: bit i of the value selects lane i's
// word; one table per column run folds in the run's offset), accumulated per
// lane -- no per-segment reduction.  Block 0's first
// combiner also folds in the int64 target that follows the input.  At the
// end each combiner reduces its accumulator into one device word
// (atomicXor), and the CTA that completes the batch turns it into the zlib
// CRC-32 of the slot (input + target) before it releases the ready word.
//
// Shared memory: two 64 KB-aligned table regions (R1: G_0 | G_1 in the two
// 128-byte halves of each 256-byte row, R2: G_2 | the row-shift nibble
// tables), and first-fit around them the item stages, zero row, barriers,
// params and the run buffers.
constexpr int CC_EMIT = 448;       // 14 emit warps (8 / 16 / 32 rows apart for f32 / bf16 / u8)
constexpr int CC_MAX_RUNS = 9;     // combiner warps: 32-element column runs per row (w <= 288)
constexpr int CC_MAX_C = 3;
constexpr int CC_SMEM = 232448;    // the 227 KB opt-in maximum
constexpr int CC_MAX_STAGES = 8;  // item stages: as many as fit next to the tables (3 at 32 rows of 224x3)
constexpr uint32_t CC_META_STRIDE = 48;  // range kernel: per-stage item record
constexpr int CC_BCNT = 16;       // range kernel: per-batch completion counters (ring > stages)
constexpr uint32_t CC_IMG_WORDS = 2 * 256 * 64;  // the two table regions (128 KB)
constexpr int CC_ACC_POOL = 1024;
constexpr int CC_MAX_PLANS = 64;   // table sets per process (never freed: kernels may be in flight)
__device__ uint32_t g_cc_acc[CC_ACC_POOL];     // per-launch accumulators (zero at rest)
__device__ unsigned int g_cc_cnt[CC_ACC_POOL]; // per-launch CTA completion counters (zero at rest)

struct CrcFuse {
    const uint32_t *img;    // CC_IMG_WORDS: the shared image of the two table regions
    const uint32_t *slice;  // zlib slice-by-4 tables T0..T3 (target checksum)
    const uint32_t *wtab;   // [runs][nseg][32]: run -> row end, segment -> slot end
    uint32_t tgt_k[5];      // x^(8 * 8 nl 2^k): the target lanes' tree
    uint32_t init;          // x^(8 total) * ~0 ^ ~0: the init/xorout term of the slot
    int nseg;
    int with_tgt;
    int tab_c;              // 1: every channel uses table 0 (u8 output: F_c(v) = v)
    uint32_t *acc;          // this launch's accumulator (the completing CTA resets it)
    unsigned int *count;    // this launch's CTA completion counter (same)
    uint32_t *out;          // the slot's CRC-32
    uint32_t *out_host;     // optional host-mapped copy (written before the ready word)
    int ne;                 // emit threads: groups x dr (dr rows apart, dr divides R)
    int fold;               // shuffle levels before the run's atomic XOR fold (TSB_CC_FOLD)
};

// Shuffle levels before the atomic fold: the 32/P lanes of a column run XOR
// k shuffle levels first, so 32/P >> k of them (not all) fold into the run's
// word -- fewer same-address shared atomics, each an N-way bank conflict
// (118 M of the 123 M excess shared wavefronts of an f32 range).  Measured per
// output kind (range kernel, us per B=256 batch, k = 0/1/2/3):
// f32 32.5 / 30.65 / 33.5 / 35.9, bf16 24.0 / 25.5 / 26.5 / 26.5, u8 30.8 /
// 32.0 / 31.7 / 31.8 (profiles/r2/range/fold_ab.jsonl, no consumers): one
// level for f32 (8 lanes per run), none for bf16 / u8.  Inside bench.py (4
// consumers, 8-slot gate) f32 runs 31.9-32.3 us either way (fold_bench_ab.jsonl):
// the kernel is then held elsewhere.  TSB_CC_FOLD=k overrides (A/B).
inline int cc_fold_knob(int out_kind) {
    static const int k = getenv("TSB_CC_FOLD") ? atoi(getenv("TSB_CC_FOLD")) : -1;
    if (k >= 0) return k;
    return out_kind == TSB_OUT_F32 ? 1 : 0;
}

__device__ __forceinline__ uint32_t cc_lds(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
template <uint32_t OFF>
__device__ __forceinline__ uint32_t cc_lds_off(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ uint32_t cc_prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
// product with a lane-replicated nibble table: t = table base + lane*4 (entry
// e of lane l at t + e*256)
__device__ __forceinline__ uint32_t cc_mul_nib(uint32_t v, uint32_t t) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= cc_lds(t + ((uint32_t)(j * 16) << 8) + (((v >> (4 * j)) & 15u) << 8));
    return r;
}
// a * b mod P (reflected; x^0 = bit 31), 32 branch-free steps
__device__ __forceinline__ uint32_t cc_multmodp(uint32_t a, uint32_t b) {
    uint32_t p = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        p ^= b & (0u - ((a >> (31 - i)) & 1u));
        b = (b >> 1) ^ (0xEDB88320u & (0u - (b & 1u)));
    }
    return p;
}
__device__ __forceinline__ uint32_t cc_crc_word(const uint32_t *__restrict__ t, uint32_t c,
                                                uint32_t w) {
    const uint32_t x = c ^ w;
    return __ldg(t + 3 * 256 + (x & 0xFFu)) ^ __ldg(t + 2 * 256 + ((x >> 8) & 0xFFu)) ^
           __ldg(t + 256 + ((x >> 16) & 0xFFu)) ^ __ldg(t + (x >> 24));
}
// mbarrier wait that sleeps until the phase completes (suspend-time hint)
__device__ __forceinline__ void cc_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "CCW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra CCW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x100000u)
        : "memory");
}
// bytes K0..K3 (compile-time indices into the realigned window words wv[0..NWV))
// packed into one word, byte t = window byte K_t
template <int NWV, int K0, int K1, int K2, int K3>
__device__ __forceinline__ uint32_t cc_gather4(const uint32_t *wv) {
    constexpr int KMIN = K0 < K1 ? (K0 < K2 ? (K0 < K3 ? K0 : K3) : (K2 < K3 ? K2 : K3))
                                 : (K1 < K2 ? (K1 < K3 ? K1 : K3) : (K2 < K3 ? K2 : K3));
    constexpr int LO = KMIN >> 2;
    constexpr int k[4] = {K0 - 4 * LO, K1 - 4 * LO, K2 - 4 * LO, K3 - 4 * LO};
    constexpr uint32_t sa = (uint32_t)((k[0] < 8 ? k[0] : 0) | (k[1] < 8 ? k[1] : 0) << 4 |
                                       (k[2] < 8 ? k[2] : 0) << 8 | (k[3] < 8 ? k[3] : 0) << 12);
    constexpr bool need_b = k[0] >= 8 || k[1] >= 8 || k[2] >= 8 || k[3] >= 8;
    constexpr int W1 = LO + 1 < NWV ? LO + 1 : NWV - 1;
    const uint32_t a = cc_prmt(wv[LO], wv[W1], sa);
    if constexpr (!need_b) {
        return a;
    } else {
        constexpr uint32_t sb = (uint32_t)((k[0] >= 8 ? k[0] - 8 : 0) | (k[1] >= 8 ? k[1] - 8 : 0) << 4 |
                                           (k[2] >= 8 ? k[2] - 8 : 0) << 8 |
                                           (k[3] >= 8 ? k[3] - 8 : 0) << 12);
        constexpr int W2 = LO + 2 < NWV ? LO + 2 : NWV - 1;
        constexpr int W3 = LO + 3 < NWV ? LO + 3 : NWV - 1;
        const uint32_t b = cc_prmt(wv[W2], wv[W3], sb);
        constexpr uint32_t sm = (uint32_t)((k[0] < 8 ? 0 : 4) | (k[1] < 8 ? 1 : 5) << 4 |
                                           (k[2] < 8 ? 2 : 6) << 8 | (k[3] < 8 ? 3 : 7) << 12);
        return cc_prmt(a, b, sm);
    }
}

// Shared layout, identical in every CTA (offsets from the dynamic base).
struct CcLayout {
    uint32_t r1, r2;        // shared addresses of the two table regions
    uint32_t lo_stage, n_lo, hi_stage;  // stages: n_lo at lo_stage, the rest at hi_stage
    uint32_t zero, bars, par, part, meta;  // offsets
};
__host__ __device__ inline bool cc_layout(uint32_t sbase, uint32_t stage_bytes, uint32_t rs,
                                          uint32_t part_bytes, int nstage, CcLayout &L) {
    L.r1 = (sbase + 0xFFFFu) & ~0xFFFFu;
    L.r2 = L.r1 + 0x10000u;
    uint32_t lo = 0, lo_end = L.r1 - sbase;
    uint32_t hi = L.r2 + 0x10000u - sbase, hi_end = (uint32_t)CC_SMEM;
    if (hi > hi_end) return false;
    auto take = [&](uint32_t bytes, uint32_t align, uint32_t &out) {
        uint32_t a = (lo + align - 1) & ~(align - 1);
        if (a + bytes <= lo_end) { out = a; lo = a + bytes; return true; }
        a = (hi + align - 1) & ~(align - 1);
        if (a + bytes <= hi_end) { out = a; hi = a + bytes; return true; }
        return false;
    };
    bool ok = take((3 * nstage + 1) * 8, 8, L.bars) &&
              take(META_CAP * (uint32_t)sizeof(ItemPar), 16, L.par) && take(rs, 128, L.zero) &&
              take(part_bytes * nstage, 16, L.part) &&
              take(CC_META_STRIDE * nstage + 4u * CC_BCNT, 16, L.meta);
    // stages: as many as fit below region 1, the rest above region 2
    L.lo_stage = (lo + 127) & ~127u;
    const uint32_t below = lo_end > L.lo_stage ? (lo_end - L.lo_stage) / stage_bytes : 0;
    L.n_lo = below < (uint32_t)nstage ? below : (uint32_t)nstage;
    L.hi_stage = (hi + 127) & ~127u;
    const uint32_t need_hi = (uint32_t)nstage - L.n_lo;
    if (need_hi && L.hi_stage + need_hi * stage_bytes > hi_end) return false;
    return ok;
}

// One slot of an emit thread: P elements x C channels of output row r -- the
// normalised stores, and raw(row r, the lane's run) of each channel into the
// run buffer (after the 32/P lanes of the run XOR-reduced their lookups).
template <int OUT_KIND, int C, bool FLIP, int CH>
__device__ __forceinline__ void cc_emit_channel(const uint32_t *wv, const Norm &norm, uint8_t *out,
                                                int64_t plane_bytes, int lane,
                                                const uint32_t *A, const uint32_t *B, int ra,
                                                int rb, uint32_t *part_c, int fold) {
    using T = OutTraits<OUT_KIND>;
    constexpr int P = T::P;
    constexpr int NS = P / 4;          // 4-element sub-words per lane
    constexpr int LPR = 32 / P;        // lanes per column run
    constexpr int NWV = (P * C + 3) / 4;
    const uint4 v = make_vec<OUT_KIND, C, FLIP, CH>(wv, norm.scale[CH], norm.bias[CH],
                                                    std::make_integer_sequence<int, P>{});
    st_cs_v4(out + CH * plane_bytes, v);
    // the channel's P source bytes in output order, 4 per word
    uint32_t V[NS];
    if constexpr (OUT_KIND == TSB_OUT_U8) {
        V[0] = v.x;
        V[1] = v.y;
        V[2] = v.z;
        V[3] = v.w;
    } else {
        constexpr auto kx = [](int q) { return (FLIP ? P - 1 - q : q) * C + CH; };
        V[0] = cc_gather4<NWV, kx(0), kx(1), kx(2), kx(3)>(wv);
        if constexpr (NS > 1) V[1] = cc_gather4<NWV, kx(4), kx(5), kx(6), kx(7)>(wv);
    }
    // rotate: word s <- V[(s + ra) % NS], then bytes by rb (lane's run index = ra*4 + rb)
    uint32_t R[NS];
    if constexpr (NS == 1) {
        R[0] = V[0];
    } else if constexpr (NS == 2) {
        R[0] = ra ? V[1] : V[0];
        R[1] = ra ? V[0] : V[1];
    } else {
        uint32_t t1[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) t1[s] = (ra & 1) ? V[(s + 1) & 3] : V[s];
#pragma unroll
        for (int s = 0; s < 4; ++s) R[s] = (ra & 2) ? t1[(s + 2) & 3] : t1[s];
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) R[s] = __funnelshift_r(R[s], R[s], 8 * rb);
    constexpr uint32_t COFF = OUT_KIND == TSB_OUT_U8 ? 0u : (CH == 0 ? 0u : CH == 1 ? 128u : 65536u);
    uint32_t acc = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int t = 0; t < 4; ++t)
            acc ^= cc_lds_off<COFF>(cc_prmt(R[s], A[s] | B[t], 0x7604u | (t << 4)));
    // the run's lanes fold their lookups into its word (zeroed by the combiner);
    // the run's lanes are the aligned group of LPR consecutive lanes
    int writers = LPR;
#pragma unroll
    for (int d = LPR / 2; d >= 1; d >>= 1) {
        if (fold <= 0) break;
        acc ^= __shfl_xor_sync(0xffffffffu, acc, d);
        writers = d;
        --fold;
    }
    if ((lane & (LPR - 1)) < writers) atomicXor(part_c, acc);
}

template <int OUT_KIND, int C, bool FLIP, int... CHs>
__device__ __forceinline__ void cc_emit_slot(const uint32_t *smem_words, uint32_t ws,
                                             const Norm &norm, uint8_t *out, int64_t plane_bytes,
                                             int lane, const uint32_t *A,
                                             const uint32_t *B, int ra, int rb, uint32_t *part,
                                             int part_cstride, int fold,
                                             std::integer_sequence<int, CHs...>) {
    constexpr int P = OutTraits<OUT_KIND>::P;
    constexpr int NB = P * C;
    constexpr int NW = (NB + 3) / 4 + 1;
    const uint32_t *wp = smem_words + (ws >> 2);
    const int shift = 8 * (int)(ws & 3);
    uint32_t raw[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) raw[i] = wp[i];
    uint32_t wv[NW - 1];
#pragma unroll
    for (int i = 0; i < NW - 1; ++i) wv[i] = __funnelshift_r(raw[i], raw[i + 1], shift);
    (cc_emit_channel<OUT_KIND, C, FLIP, CHs>(wv, norm, out, plane_bytes, lane, A, B, ra, rb,
                                             part + CHs * part_cstride, fold),
     ...);
}

template <int OUT_KIND, int C>
__global__ void __launch_bounds__(CC_EMIT + 32 + 32 * CC_MAX_RUNS, 1)
    collate_crc_kernel(const uint8_t *__restrict__ src, const int64_t *__restrict__ idx, CaGeom g,
                       int flip_en, uint64_t aug_mixed, uint64_t epoch, Norm norm,
                       const int32_t *__restrict__ params, Dsts dsts, Epi ep, CrcFuse cf) {
    using T = OutTraits<OUT_KIND>;
    constexpr int P = T::P;
    constexpr int E = T::ELEM;
    constexpr int NS = P / 4;
    const int NT = cf.ne;
    const int NCW = NT >> 5;             // emit warps; warp NCW = producer; then the combiners
    const int NST = g.nstage;
    const int runs = g.w >> 5;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const uint32_t stage_bytes = (uint32_t)(g.R * g.rs);
    const int part_words = C * g.R * runs;  // per stage: [c][row][run]
    CcLayout L;
    if (!cc_layout(sbase, stage_bytes, (uint32_t)g.rs, 4u * part_words, NST, L)) __trap();
    auto soff = [&](int st) -> uint32_t {
        return (uint32_t)st < L.n_lo ? L.lo_stage + (uint32_t)st * stage_bytes
                                      : L.hi_stage + ((uint32_t)st - L.n_lo) * stage_bytes;
    };
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *empty = full + NST;
    uint64_t *pfull = empty + NST;
    uint64_t *tab_bar = pfull + NST;
    ItemPar *par = reinterpret_cast<ItemPar *>(smem + L.par);
    uint32_t *part = reinterpret_cast<uint32_t *>(smem + L.part);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t *kidx = ep.tgt_idx ? ep.tgt_idx : idx;
    pdl_launch_dependents();  // the next batch may launch now (it waits for this SM's smem)
    const int nk = (g.items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int i0 = (int)blockIdx.x, istep = (int)gridDim.x;

    // zero the stages and the zero row once: borders are never overwritten
    for (int st = 0; st < NST; ++st) {
        uint4 *z = reinterpret_cast<uint4 *>(smem + soff(st));
        for (int i = tid; i < (int)(stage_bytes >> 4); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    }
    {
        uint4 *z = reinterpret_cast<uint4 *>(smem + L.zero);
        for (int i = tid; i < (g.rs >> 4); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    }
    for (int i = tid; i < NST * part_words; i += blockDim.x) part[i] = 0u;
    for (int k = tid; k < min(nk, META_CAP); k += blockDim.x)
        par[k] = item_par(g, i0 + k * istep, idx, kidx, params, aug_mixed, epoch, flip_en);
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW + runs);
            mbar_init(&pfull[i], NT);
        }
        mbar_init(tab_bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto get_par = [&](int k) -> ItemPar {
        return k < META_CAP ? par[k]
                            : item_par(g, i0 + k * istep, idx, kidx, params, aug_mixed, epoch,
                                       flip_en);
    };

    if (warp == NCW) {
        // ---------------- producer warp: the tables, then the items' source rows ----
        if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(tab_bar, CC_IMG_WORDS * 4u);
            tma_load_1d(smem + (L.r1 - sbase), cf.img, 65536u, tab_bar);
            tma_load_1d(smem + (L.r2 - sbase), cf.img + CC_IMG_WORDS / 2, 65536u, tab_bar);
        }
        for (int k = 0, st = 0, ph = 0; k < nk; ++k) {
            if (k >= NST) cc_wait(&empty[st], ph ^ 1);
            const int item = i0 + k * istep;
            const ItemPar p = get_par(k);
            const int y0 = (item - p.s * g.nrb) * g.R;
            const int sy_first = y0 + p.oy - g.pad;
            const int lo = max(sy_first, 0), hi = min(sy_first + g.R, g.h);
            const uint8_t *sample = src + p.src_off;
            uint8_t *dst = smem + soff(st) + g.io;
            // one lane per row: the row copies are issued in parallel
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&full[st], (uint32_t)max(0, hi - lo) * (uint32_t)g.row_bytes);
            }
            __syncwarp();
            const uint64_t pol = l2_evict_first_policy();
            for (int r = lo + lane; r < hi; r += 32)
                tma_load_1d_hint(dst + (r - sy_first) * g.rs, sample + (int64_t)r * g.row_bytes,
                                 (uint32_t)g.row_bytes, &full[st], pol);
            if (++st == NST) st = 0, ph ^= 1;
        }
        return;
    }

    if (warp < NCW) {
        // ------- emit warps: normalised NCHW + per-element checksum lookups -----------
        const uint32_t *smem_words = reinterpret_cast<const uint32_t *>(smem);
        if (blockIdx.x == 0) write_targets(ep, idx, g.b, tid, NT);
        const int64_t plane_bytes = g.plane * E;
        const int xg = tid % g.groups, r_first = tid / g.groups, dr = NT / g.groups;
        const int x0 = xg * P, run = x0 >> 5;
        const int ridx = lane / (32 / P), ra = ridx >> 2, rb = ridx & 3;
        uint32_t A[NS], B[4];  // position bits: p = (x0 & 31) + 4*((s + ra) % NS) + ((t + rb) & 3)
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2)
            A[s2] = L.r1 | ((uint32_t)((x0 & 31) + 4 * ((s2 + ra) % NS)) << 2);
#pragma unroll
        for (int t = 0; t < 4; ++t) B[t] = (uint32_t)((t + rb) & 3) << 2;
        const int n_iter = g.R / dr;  // cc_fusable: dr divides R, every slot is a real row
        cc_wait(tab_bar, 0);          // the lookup tables have landed
        for (int k = 0, st = 0, ph = 0; k < nk; ++k) {
            const int item = i0 + k * istep;
            const ItemPar p = get_par(k);
            const int y0 = (item - p.s * g.nrb) * g.R;
            const int sy_first = y0 + p.oy - g.pad;
            const int lo = max(sy_first, 0), hi = min(sy_first + g.R, g.h);
            uint8_t *out_item = static_cast<uint8_t *>(dsts.p[0]) +
                                ((int64_t)p.s * C * g.plane + (int64_t)y0 * g.w + x0) * E;
            const uint32_t so = soff(st);
            uint32_t *pst = part + st * part_words + run;
            cc_wait(&full[st], ph);
#pragma unroll 1
            for (int j = 0; j < n_iter; ++j) {
                const int r = r_first + j * dr;
                const int sy = sy_first + r;
                const uint32_t row_off = (sy >= lo && sy < hi) ? so + (uint32_t)(r * g.rs) : L.zero;
                uint8_t *o = out_item + (int64_t)r * g.w * E;
                uint32_t *pr = pst + r * runs;
                if (!p.fl)
                    cc_emit_slot<OUT_KIND, C, false>(smem_words, row_off + g.rdoff + (x0 + p.ox) * C,
                                                     norm, o, plane_bytes, lane, A, B, ra, rb,
                                                     pr, g.R * runs, cf.fold, std::make_integer_sequence<int, C>{});
                else
                    cc_emit_slot<OUT_KIND, C, true>(smem_words,
                                                    row_off + g.rdoff + (g.w - P - x0 + p.ox) * C,
                                                    norm, o, plane_bytes, lane, A, B, ra, rb,
                                                    pr, g.R * runs, cf.fold, std::make_integer_sequence<int, C>{});
            }
            mbar_arrive(&pfull[st]);  // this thread's run values are in the buffer
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == NST) st = 0, ph ^= 1;
        }
    } else {
        // ------- combiner warps: one column run, lane = row of the item ---------------
        const int run = warp - NCW - 1;
        const uint32_t rowsh = L.r2 + 128u + 4u * (uint32_t)lane + (128u << 8);  // x^(8 wE (R-1-lane))
        const uint32_t *wrun_tab = cf.wtab + (int64_t)run * cf.nseg * 32 + lane;
        uint32_t wacc = 0;
        if (blockIdx.x == 0 && run == 0 && cf.with_tgt) {
            // raw CRC of the int64 target (b entries after the input): lane l takes
            // nl entries of the front-zero-padded run, then a 5-level tree
            const int nl = (g.b + 31) >> 5, z = 32 * nl - g.b;
            uint32_t cr = 0;
            for (int e = 0; e < nl; ++e) {
                const int v = lane * nl + e - z;
                if (v >= 0) {
                    const uint64_t x = (uint64_t)kidx[v];
                    cr = cc_crc_word(cf.slice, cr, (uint32_t)x);
                    cr = cc_crc_word(cf.slice, cr, (uint32_t)(x >> 32));
                }
            }
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, cr, 1 << k);
                cr = (lane & (1 << k)) ? cc_multmodp(cf.tgt_k[k], other) ^ cr
                                       : cc_multmodp(cf.tgt_k[k], cr) ^ other;
            }
            if (lane == 0) wacc = cr;
        }
        cc_wait(tab_bar, 0);
        for (int k = 0, st = 0, ph = 0; k < nk; ++k) {
            const int item = i0 + k * istep;
            const ItemPar p = get_par(k);
            const int rb = item - p.s * g.nrb;
            uint32_t wv[C];
#pragma unroll
            for (int c = 0; c < C; ++c)
                wv[c] = __ldg(wrun_tab + (int64_t)(cf.nseg - 1 - ((p.s * C + c) * g.nrb + rb)) * 32);
            cc_wait(&pfull[st], ph);
            uint32_t S[C];
#pragma unroll
            for (int c = 0; c < C; ++c)
            {
                uint32_t *w = part + st * part_words + (c * g.R + lane) * runs + run;
                S[c] = lane < g.R ? *w : 0u;
                if (lane < g.R) *w = 0u;  // ready for the stage's next item
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);  // the run buffer is read
            if (++st == NST) st = 0, ph ^= 1;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                uint32_t x = lane < g.R ? cc_mul_nib(S[c], rowsh) : 0u;  // row -> segment's last row
#pragma unroll
                for (int k2 = 16; k2 >= 1; k2 >>= 1) x ^= __shfl_xor_sync(0xFFFFFFFFu, x, k2);
                // the run's column -> the row's end and the segment -> the slot's end
                wacc ^= ((x >> lane) & 1u) ? wv[c] : 0u;
            }
        }
#pragma unroll
        for (int k2 = 16; k2 >= 1; k2 >>= 1) wacc ^= __shfl_xor_sync(0xFFFFFFFFu, wacc, k2);
        if (lane == 0 && wacc) atomicXor(cf.acc, wacc);
    }
    // the completing CTA finishes the checksum, then publishes the slot (each
    // warp reconverges first: a named barrier counts whole warps)
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(NT + 32 * runs) : "memory");
    if (tid == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(cf.count, 1u);
        if (prev == gridDim.x - 1) {
            *cf.count = 0u;
            __threadfence();
            const uint32_t v = atomicExch(cf.acc, 0u);
            *cf.out = v ^ cf.init;
            if (cf.out_host) *cf.out_host = v ^ cf.init;
            __threadfence_system();
            for (int d = 0; d < ep.n; ++d)
                if (ep.ready[d])
                    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ep.ready[d]),
                                 "l"(ep.seq)
                                 : "memory");
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent range kernel (tsb_produce_range with persistent=1 and a CRC):
// ONE cooperative launch produces n consecutive batches, one CTA per SM for
// the whole range.  The per-batch kernel pays, per batch and SM, the CTA
// start, the 128 KB table load, the stage zeroing and the pipeline fill --
// the 6 us intercept of per-batch time against B (21.6 / 36.3 / 66.5 us at
// B = 128 / 256 / 512, profiles/r2/crc_fused_bscaling.jsonl).  Here the work
// items of all n batches form one stream (CTA b takes b, b + grid, ...), so a
// CTA's stages run across batch boundaries.
//   * the slot gate moves to the device: before the first item of batch q the
//     producer warp waits until every live consumer released q - slots (CTA 0
//     reads the host-shared cursors and raises a gate word the others poll in
//     L2; the reference's gate is bs/producer.py:230-238);
//   * the producer derives the next item's crop before it waits for a stage,
//     and writes each staged item's params into the stage record;
//   * completion without a CTA-wide barrier and off the emit path: each
//     consumer warp, after its last item of a batch, counts itself in a
//     per-CTA shared counter (CTA-scope release); a publisher warp waits for
//     the CTA's count, fences at GPU scope (cumulative over what it observed,
//     the cooperative-groups grid-barrier pattern) and counts the CTA into the
//     slot's global counter; the CTA that completes the batch writes its
//     CRC-32 and publishes the slot.  The emit warps never wait on a fence.
constexpr int CC_MAX_LIVE = 16;
struct CcRange {
    uint8_t *ring_base;
    int64_t slot_stride;
    int slots;
    uint64_t *ready;             // [slots] (single writer)
    const uint64_t *cursors;     // release cursors (host-shared, device-mapped)
    unsigned int *counters;      // [slots] completion counters (zero at rest)
    unsigned long long *gate;    // device word: every live cursor has released this much
    int live[CC_MAX_LIVE];
    int n_live;
    uint64_t seq0;
    int n;
    int64_t input_bytes;
    int with_target;
    uint32_t *d_crc;             // [slots]: each batch's CRC-32, written before its publish
    uint32_t *h_crc;             // optional host-mapped [slots] copy
    uint32_t *acc_pool;          // g_cc_acc
    unsigned acc_base;           // batch i accumulates into acc_pool[(acc_base + i) % POOL]
    int refresh;                 // CTA 0 re-polls while its level is < refresh batches ahead
};
struct CcItem {                  // per stage: the staged item (written by the producer)
    ItemPar p;
    int batch, j, slot, last;    // last: the CTA's last item of this batch
};
static_assert(sizeof(CcItem) <= CC_META_STRIDE, "stage record");

__device__ __forceinline__ uint64_t cc_ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// min over the live release cursors (host-shared, PCIe reads), wrap-around order
__device__ __forceinline__ uint64_t cc_min_live(const CcRange &rg, uint64_t need) {
    uint64_t lo = need + (1ull << 61);
    for (int j = 0; j < rg.n_live; ++j) {
        const uint64_t c = cc_ld_acquire_sys(rg.cursors + rg.live[j]);
        if ((int64_t)(c - lo) < 0) lo = c;
    }
    return lo;
}

template <int OUT_KIND, int C>
__global__ void __launch_bounds__(CC_EMIT + 64 + 32 * CC_MAX_RUNS, 1)
    collate_crc_range_kernel(const uint8_t *__restrict__ src, const int64_t *__restrict__ order0,
                             CaGeom g, int flip_en, uint64_t aug_mixed, uint64_t epoch, Norm norm,
                             CrcFuse cf, CcRange rg) {
    using T = OutTraits<OUT_KIND>;
    constexpr int P = T::P;
    constexpr int E = T::ELEM;
    constexpr int NS = P / 4;
    const int NT = cf.ne;
    const int NCW = NT >> 5;
    const int NST = g.nstage;
    const int runs = g.w >> 5;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const uint32_t stage_bytes = (uint32_t)(g.R * g.rs);
    const int part_words = C * g.R * runs;
    CcLayout L;
    if (!cc_layout(sbase, stage_bytes, (uint32_t)g.rs, 4u * part_words, NST, L)) __trap();
    auto soff = [&](int st) -> uint32_t {
        return (uint32_t)st < L.n_lo ? L.lo_stage + (uint32_t)st * stage_bytes
                                      : L.hi_stage + ((uint32_t)st - L.n_lo) * stage_bytes;
    };
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *empty = full + NST;
    uint64_t *pfull = empty + NST;
    uint64_t *tab_bar = pfull + NST;
    uint32_t *part = reinterpret_cast<uint32_t *>(smem + L.part);
    CcItem *meta = reinterpret_cast<CcItem *>(smem + L.meta);
    unsigned int *bcnt =
        reinterpret_cast<unsigned int *>(smem + L.meta + CC_META_STRIDE * NST);  // [CC_BCNT]
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int items = g.items;  // per batch
    const int64_t total = (int64_t)items * rg.n;
    const int grid = (int)gridDim.x;
    const int nk = (int)((total - (int64_t)blockIdx.x + grid - 1) / grid);
    // CTAs that take part in each batch (a window of `items` consecutive items)
    const unsigned int ctas_per_batch = (unsigned int)(items < grid ? items : grid);

    for (int st = 0; st < NST; ++st) {
        uint4 *z = reinterpret_cast<uint4 *>(smem + soff(st));
        for (int i = tid; i < (int)(stage_bytes >> 4); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    }
    {
        uint4 *z = reinterpret_cast<uint4 *>(smem + L.zero);
        for (int i = tid; i < (g.rs >> 4); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    }
    for (int i = tid; i < NST * part_words; i += blockDim.x) part[i] = 0u;
    if (tid < CC_BCNT) bcnt[tid] = 0u;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW + runs);
            mbar_init(&pfull[i], NT);
        }
        mbar_init(tab_bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // this CTA's items b, b + grid, ... as (batch, item-in-batch), stepped
    // without divisions; is_last: the CTA's last item of that batch
    const int bi0 = (int)blockIdx.x / items, j0 = (int)blockIdx.x - bi0 * items;
    auto step = [&](int &bi, int &j) {
        j += grid;
        while (j >= items) j -= items, ++bi;
    };
    auto is_last = [&](int k, int j) { return k + 1 >= nk || j + grid >= items; };
    const int slot0 = (int)((rg.seq0 - 1) % (uint64_t)rg.slots);
    // a consumer warp is done with batch bi (its stores and checksum share
    // issued): count it for the publisher warp, CTA-scope release
    auto warp_done = [&](int bi) {
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            atomicAdd(bcnt + (bi & (CC_BCNT - 1)), 1u);
        }
    };

    if (warp == NCW + 1 + runs) {
        // ---------------- publisher warp: the CTA's share of each batch -------------
        // Consumer warps stay within NST items of each other (they share the
        // stages), so a ring of CC_BCNT > NST monotonic counters cannot alias.
        if (lane == 0) {
            unsigned int want[CC_BCNT];
            for (int x = 0; x < CC_BCNT; ++x) want[x] = 0u;
            const unsigned int W = (unsigned int)(NCW + runs);
            for (int k = 0, bi = bi0, j = j0; k < nk; ++k, step(bi, j)) {
                if (!is_last(k, j)) continue;
                const int x = bi & (CC_BCNT - 1);
                want[x] += W;
                while ((int)(*(volatile unsigned int *)(bcnt + x) - want[x]) < 0) __nanosleep(64);
                __threadfence();  // the consumers' stores and checksum shares, GPU-wide
                const uint64_t q = rg.seq0 + (uint64_t)bi;
                const int slot = (slot0 + bi) % rg.slots;
                const unsigned int gp = atomicAdd(rg.counters + slot, 1u);
                if (gp == ctas_per_batch - 1u) {  // the batch is complete
                    rg.counters[slot] = 0u;
                    __threadfence();
                    uint32_t *acc = rg.acc_pool + (rg.acc_base + (unsigned)bi) % CC_ACC_POOL;
                    const uint32_t v = atomicExch(acc, 0u) ^ cf.init;
                    rg.d_crc[slot] = v;
                    if (rg.h_crc) rg.h_crc[slot] = v;
                    __threadfence_system();
                    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(rg.ready + slot),
                                 "l"(q)
                                 : "memory");
                }
            }
        }
        return;
    }

    if (warp == NCW) {
        // ---------------- producer warp: tables, the device slot gate, the items ----
        if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(tab_bar, CC_IMG_WORDS * 4u);
            tma_load_1d(smem + (L.r1 - sbase), cf.img, 65536u, tab_bar);
            tma_load_1d(smem + (L.r2 - sbase), cf.img + CC_IMG_WORDS / 2, 65536u, tab_bar);
        }
        // item params (sample, crop, flip) one 32-item chunk ahead, one item
        // per lane, into a 64-entry ring: the dependent order/sample loads stay
        // off the per-item path (the per-batch kernel caches them in its prologue)
        ItemPar *par = reinterpret_cast<ItemPar *>(smem + L.par);
        auto fill = [&](int k0) {  // items k0 .. k0 + 31
            const int k = k0 + lane;
            if (k < nk) {
                const int64_t gi = (int64_t)blockIdx.x + (int64_t)k * grid;
                const int bi = (int)(gi / items), j = (int)(gi - (int64_t)bi * items);
                ItemPar p;
                p.s = j / g.nrb;
                const int64_t sample = order0[(int64_t)bi * g.b + p.s];
                p.src_off = sample * g.sample_bytes;
                derive_aug(aug_mixed, epoch, sample, g.pad, flip_en, p.oy, p.ox, p.fl);
                par[k & 63] = p;
            }
        };
        fill(0);
        fill(32);
        __syncwarp();
        uint64_t known = 0;  // (every lane) every live cursor is known to have released this level
        int gated = -1;
        for (int k = 0, st = 0, ph = 0, bi = bi0, j = j0; k < nk; ++k, step(bi, j)) {
            if ((k & 31) == 0 && k >= 32) {  // items k .. k+31 were filled; fill k+32 ..
                fill(k + 32);
                __syncwarp();
            }
            const ItemPar p = par[k & 63];
            if (k >= NST) cc_wait(&empty[st], ph ^ 1);
            const uint64_t q = rg.seq0 + (uint64_t)bi;
            if (bi != gated) {  // first item of a batch: its slot must be free
                gated = bi;
                if (q > (uint64_t)rg.slots) {  // (warp-uniform: every lane steps bi alike)
                    const uint64_t need = q - (uint64_t)rg.slots;
                    if (lane == 0) {
                        // the slot's previous batch is published: its completion counter
                        // is free again (without live consumers nothing else orders it)
                        const uint64_t *rw = rg.ready + (slot0 + bi) % rg.slots;
                        uint64_t pub;
                        for (;;) {
                            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(pub)
                                         : "l"(rw) : "memory");
                            if ((int64_t)(pub - need) >= 0) break;
                            __nanosleep(64);
                        }
                    }
                    __syncwarp();
                    while ((int64_t)(known - need) < 0) {  // `known` is warp-uniform
                        uint64_t gw = 0;
                        if (lane == 0)
                            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(gw)
                                         : "l"(rg.gate) : "memory");
                        gw = __shfl_sync(0xffffffffu, gw, 0);
                        if ((int64_t)(gw - known) > 0) known = gw;
                        if ((int64_t)(known - need) >= 0) break;
                        if (blockIdx.x == 0) {
                            // CTA 0 alone reads the host-shared cursors, one lane per
                            // consumer: the PCIe acquire loads are in flight together
                            uint64_t lo = need + (1ull << 61);
                            for (int jl = lane; jl < rg.n_live; jl += 32) {
                                const uint64_t cv = cc_ld_acquire_sys(rg.cursors + rg.live[jl]);
                                if ((int64_t)(cv - lo) < 0) lo = cv;
                            }
#pragma unroll
                            for (int o = 16; o; o >>= 1) {
                                const uint64_t other = __shfl_xor_sync(0xffffffffu, lo, o);
                                if ((int64_t)(other - lo) < 0) lo = other;
                            }
                            __syncwarp();  // every lane's acquire before lane 0 raises the gate
                            if ((int64_t)(lo - known) > 0) {
                                known = lo;
                                if (lane == 0) atomicMax(rg.gate, (unsigned long long)lo);
                            }
                        }
                        if ((int64_t)(known - need) < 0) __nanosleep(blockIdx.x == 0 ? 200 : 100);
                    }
                    // (TSB_CC_REFRESH=k) CTA 0 polls ahead while its level covers fewer
                    // than k more batches, so the other CTAs rarely find the gate word
                    // behind them and wait for CTA 0 to reach the same batch
                    if (blockIdx.x == 0 && rg.refresh > 0 &&
                        (int64_t)(known - need) < (int64_t)rg.refresh) {
                        uint64_t lo = need + (1ull << 61);
                        for (int jl = lane; jl < rg.n_live; jl += 32) {
                            const uint64_t cv = cc_ld_acquire_sys(rg.cursors + rg.live[jl]);
                            if ((int64_t)(cv - lo) < 0) lo = cv;
                        }
#pragma unroll
                        for (int o = 16; o; o >>= 1) {
                            const uint64_t other = __shfl_xor_sync(0xffffffffu, lo, o);
                            if ((int64_t)(other - lo) < 0) lo = other;
                        }
                        __syncwarp();
                        if ((int64_t)(lo - known) > 0) {
                            known = lo;
                            if (lane == 0) atomicMax(rg.gate, (unsigned long long)lo);
                        }
                    }
                }
                __syncwarp();
            }
            const int y0 = (j - p.s * g.nrb) * g.R;
            const int sy_first = y0 + p.oy - g.pad;
            const int lo = max(sy_first, 0), hi = min(sy_first + g.R, g.h);
            const uint8_t *sample = src + p.src_off;
            uint8_t *dst = smem + soff(st) + g.io;
            if (lane == 0) {
                meta[st].p = p;
                meta[st].batch = bi;
                meta[st].j = j;
                meta[st].slot = (slot0 + bi) % rg.slots;
                meta[st].last = is_last(k, j);
                fence_proxy_async();
                mbar_arrive_expect_tx(&full[st], (uint32_t)max(0, hi - lo) * (uint32_t)g.row_bytes);
            }
            __syncwarp();
            const uint64_t pol = l2_evict_first_policy();
            for (int r = lo + lane; r < hi; r += 32)
                tma_load_1d_hint(dst + (r - sy_first) * g.rs, sample + (int64_t)r * g.row_bytes,
                                 (uint32_t)g.row_bytes, &full[st], pol);
            if (++st == NST) st = 0, ph ^= 1;
        }
        // CTA 0 keeps the gate level moving until the range's last batch is out:
        // other CTAs may still wait on it after CTA 0 ran out of items
        if (blockIdx.x == 0 && lane == 0 && rg.n > 0) {
            const uint64_t q_last = rg.seq0 + (uint64_t)rg.n - 1;
            const int last_slot = (int)((q_last - 1) % (uint64_t)rg.slots);
            while (cc_ld_acquire_sys(rg.ready + last_slot) != q_last) {
                const uint64_t need = q_last > (uint64_t)rg.slots ? q_last - (uint64_t)rg.slots : 0;
                const uint64_t lo = cc_min_live(rg, need);
                if ((int64_t)(lo - known) > 0) {
                    known = lo;
                    atomicMax(rg.gate, (unsigned long long)lo);
                }
                __nanosleep(500);
            }
        }
        return;
    }

    if (warp < NCW) {
        // ------- emit warps: normalised NCHW + per-element checksum lookups -----------
        const uint32_t *smem_words = reinterpret_cast<const uint32_t *>(smem);
        const int64_t plane_bytes = g.plane * E;
        const int xg = tid % g.groups, r_first = tid / g.groups, dr = NT / g.groups;
        const int x0 = xg * P, run = x0 >> 5;
        const int ridx = lane / (32 / P), ra = ridx >> 2, rb = ridx & 3;
        uint32_t A[NS], B[4];
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2)
            A[s2] = L.r1 | ((uint32_t)((x0 & 31) + 4 * ((s2 + ra) % NS)) << 2);
#pragma unroll
        for (int t = 0; t < 4; ++t) B[t] = (uint32_t)((t + rb) & 3) << 2;
        const int n_iter = g.R / dr;
        cc_wait(tab_bar, 0);
        for (int k = 0, st = 0, ph = 0; k < nk; ++k) {
            cc_wait(&full[st], ph);
            const CcItem it = meta[st];
            const ItemPar p = it.p;
            uint8_t *slot_base = rg.ring_base + (int64_t)it.slot * rg.slot_stride;
            if (it.j == 0 && rg.with_target) {  // the batch's target: its sample indices
                const int64_t *idx = order0 + (int64_t)it.batch * g.b;
                int64_t *tgt = reinterpret_cast<int64_t *>(slot_base + rg.input_bytes);
                for (int t = tid; t < g.b; t += NT) tgt[t] = idx[t];
            }
            const int y0 = (it.j - p.s * g.nrb) * g.R;
            const int sy_first = y0 + p.oy - g.pad;
            const int lo = max(sy_first, 0), hi = min(sy_first + g.R, g.h);
            uint8_t *out_item = slot_base + ((int64_t)p.s * C * g.plane + (int64_t)y0 * g.w + x0) * E;
            const uint32_t so = soff(st);
            uint32_t *pst = part + st * part_words + run;
#pragma unroll 1
            for (int jj = 0; jj < n_iter; ++jj) {
                const int r = r_first + jj * dr;
                const int sy = sy_first + r;
                const uint32_t row_off = (sy >= lo && sy < hi) ? so + (uint32_t)(r * g.rs) : L.zero;
                uint8_t *o = out_item + (int64_t)r * g.w * E;
                uint32_t *pr = pst + r * runs;
                if (!p.fl)
                    cc_emit_slot<OUT_KIND, C, false>(smem_words, row_off + g.rdoff + (x0 + p.ox) * C,
                                                     norm, o, plane_bytes, lane, A, B, ra, rb, pr,
                                                     g.R * runs, cf.fold, std::make_integer_sequence<int, C>{});
                else
                    cc_emit_slot<OUT_KIND, C, true>(smem_words,
                                                    row_off + g.rdoff + (g.w - P - x0 + p.ox) * C,
                                                    norm, o, plane_bytes, lane, A, B, ra, rb, pr,
                                                    g.R * runs, cf.fold, std::make_integer_sequence<int, C>{});
            }
            mbar_arrive(&pfull[st]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == NST) st = 0, ph ^= 1;
            if (it.last) warp_done(it.batch);
        }
    } else {
        // ------- combiner warps: one column run, lane = row of the item ---------------
        const int run = warp - NCW - 1;
        const uint32_t rowsh = L.r2 + 128u + 4u * (uint32_t)lane + (128u << 8);
        const uint32_t *wrun_tab = cf.wtab + (int64_t)run * cf.nseg * 32 + lane;
        uint32_t wacc = 0;
        cc_wait(tab_bar, 0);
        for (int k = 0, st = 0, ph = 0, bi = bi0, j = j0; k < nk; ++k, step(bi, j)) {
            const int s_ = j / g.nrb, rb = j - s_ * g.nrb;
            uint32_t wv[C];
#pragma unroll
            for (int c = 0; c < C; ++c)
                wv[c] = __ldg(wrun_tab + (int64_t)(cf.nseg - 1 - ((s_ * C + c) * g.nrb + rb)) * 32);
            if (j == 0 && run == 0 && cf.with_tgt) {  // raw CRC of the batch's int64 target
                const int64_t *idx = order0 + (int64_t)bi * g.b;
                const int nl = (g.b + 31) >> 5, z = 32 * nl - g.b;
                uint32_t cr = 0;
                for (int e = 0; e < nl; ++e) {
                    const int v = lane * nl + e - z;
                    if (v >= 0) {
                        const uint64_t x = (uint64_t)idx[v];
                        cr = cc_crc_word(cf.slice, cr, (uint32_t)x);
                        cr = cc_crc_word(cf.slice, cr, (uint32_t)(x >> 32));
                    }
                }
#pragma unroll
                for (int k2 = 0; k2 < 5; ++k2) {
                    const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, cr, 1 << k2);
                    cr = (lane & (1 << k2)) ? cc_multmodp(cf.tgt_k[k2], other) ^ cr
                                            : cc_multmodp(cf.tgt_k[k2], cr) ^ other;
                }
                if (lane == 0) wacc ^= cr;
            }
            cc_wait(&pfull[st], ph);
            uint32_t S[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                uint32_t *w = part + st * part_words + (c * g.R + lane) * runs + run;
                S[c] = lane < g.R ? *w : 0u;
                if (lane < g.R) *w = 0u;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == NST) st = 0, ph ^= 1;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                uint32_t x = lane < g.R ? cc_mul_nib(S[c], rowsh) : 0u;
#pragma unroll
                for (int k2 = 16; k2 >= 1; k2 >>= 1) x ^= __shfl_xor_sync(0xFFFFFFFFu, x, k2);
                wacc ^= ((x >> lane) & 1u) ? wv[c] : 0u;
            }
            if (is_last(k, j)) {  // this warp's share of the batch's checksum
#pragma unroll
                for (int k2 = 16; k2 >= 1; k2 >>= 1) wacc ^= __shfl_xor_sync(0xFFFFFFFFu, wacc, k2);
                if (lane == 0 && wacc)
                    atomicXor(rg.acc_pool + (rg.acc_base + (unsigned)bi) % CC_ACC_POOL, wacc);
                wacc = 0;
                warp_done(bi);
            }
        }
    }
}

// ---- host: tables (cached per configuration) and the launch ---------------
constexpr uint32_t CC_POLY = 0xEDB88320u;
inline uint32_t cc_h_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ CC_POLY : b >> 1;
    }
    return p;
}
inline uint32_t cc_h_x8n(uint64_t n) {  // x^(8n) mod P
    uint32_t p = 1u << 31, sq = 1u << 30;  // sq = x^1
    for (int i = 0; i < 3; ++i) sq = cc_h_multmodp(sq, sq);  // x^8
    while (n) {
        if (n & 1) p = cc_h_multmodp(sq, p);
        n >>= 1;
        sq = cc_h_multmodp(sq, sq);
    }
    return p;
}
inline void cc_h_tables(uint32_t t[4 * 256]) {
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t r = i;
        for (int k = 0; k < 8; ++k) r = (r >> 1) ^ (CC_POLY & (0u - (r & 1u)));
        t[i] = r;
    }
    for (int s = 1; s < 4; ++s)
        for (uint32_t i = 0; i < 256; ++i)
            t[s * 256 + i] = (t[(s - 1) * 256 + i] >> 8) ^ t[t[(s - 1) * 256 + i] & 0xFFu];
}
// the output element F_c(v) as the emit path computes it (two IEEE roundings;
// bf16 by round-to-nearest-even of that f32)
inline void cc_h_element(int out_kind, const Norm &n, int c, int v, uint8_t *b) {
    if (out_kind == TSB_OUT_U8) {
        b[0] = (uint8_t)v;
        return;
    }
    volatile float prod = (float)v * n.scale[c];
    volatile float sum = prod + n.bias[c];
    const float f = sum;
    uint32_t bits;
    memcpy(&bits, &f, 4);
    if (out_kind == TSB_OUT_F32) {
        memcpy(b, &bits, 4);
        return;
    }
    const uint16_t h = (uint16_t)((bits + 0x7FFFu + ((bits >> 16) & 1u)) >> 16);
    memcpy(b, &h, 2);
}

struct CcKey {
    int dev, out_kind, c, w, h, R, b, with_tgt;
    float scale[4], bias[4];
};
struct CcPlan {
    CcKey key;
    uint32_t *d_img = nullptr, *d_slice = nullptr, *d_w = nullptr;
    uint32_t tgt_k[5];
    uint32_t init;
    int nseg;
};

int cc_plan(const CcKey &key, cudaStream_t s, const CcPlan **out) {
    static std::mutex mu;
    static CcPlan plans[CC_MAX_PLANS];
    static int n_plans = 0;
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n_plans; ++i)
        if (memcmp(&plans[i].key, &key, sizeof(CcKey)) == 0) {
            *out = &plans[i];
            return TSB_OK;
        }
    if (n_plans >= CC_MAX_PLANS) {  // the caller takes the unfused path (collate, then tsb_crc32)
        *out = nullptr;
        return TSB_OK;
    }
    const int E = key.out_kind == TSB_OUT_U8 ? 1 : key.out_kind == TSB_OUT_F32 ? 4 : 2;
    Norm nm{};
    memcpy(nm.scale, key.scale, sizeof(nm.scale));
    memcpy(nm.bias, key.bias, sizeof(nm.bias));
    std::vector<uint32_t> img(CC_IMG_WORDS, 0u), slice(4 * 256);
    cc_h_tables(slice.data());
    uint32_t kp[32];
    for (int p = 0; p < 32; ++p) kp[p] = cc_h_x8n((uint64_t)E * (31 - p));
    const int ntab = key.out_kind == TSB_OUT_U8 ? 1 : key.c;
    for (int tc = 0; tc < ntab; ++tc) {
        const int region = tc >> 1, half = tc & 1;
        for (int v = 0; v < 256; ++v) {
            uint8_t el[4];
            cc_h_element(key.out_kind, nm, tc, v, el);
            uint32_t raw = 0;
            for (int i = 0; i < E; ++i) raw = slice[(raw ^ el[i]) & 0xFFu] ^ (raw >> 8);
            for (int p = 0; p < 32; ++p)
                img[(size_t)(region * 256 + v) * 64 + half * 32 + p] = cc_h_multmodp(kp[p], raw);
        }
    }
    // region 2, upper halves: entries 128..255 the lane-specific row shift
    for (int l = 0; l < 32; ++l) {
        const uint32_t kr = l < key.R ? cc_h_x8n((uint64_t)key.w * E * (key.R - 1 - l)) : 0u;
        for (int j = 0; j < 8; ++j)
            for (uint32_t q = 0; q < 16; ++q)
                img[(size_t)(256 + 128 + j * 16 + q) * 64 + 32 + l] =
                    l < key.R ? cc_h_multmodp(kr, q << (4 * j)) : 0u;
    }
    const int runs = key.w / 32;
    const int nrb = key.h / key.R;
    const int64_t nseg = (int64_t)key.b * key.c * nrb;
    const uint64_t segb = (uint64_t)key.R * key.w * E;
    const uint64_t tail = key.with_tgt ? 8ull * (uint64_t)key.b : 0ull;
    // W[run][m][i] = x^(8 (SEGB m + tail + 32E (runs-1-run))) * e_i: the column
    // run's value -> the end of its row, and segment m -> the slot's end.  Bit i
    // is x^(31-i), so W[..][31] = K and each step down multiplies by x.
    std::vector<uint32_t> wt((size_t)runs * nseg * 32);
    const uint32_t k_seg = cc_h_x8n(segb);
    for (int r = 0; r < runs; ++r) {
        uint32_t km = cc_h_multmodp(cc_h_x8n(tail), cc_h_x8n((uint64_t)32 * E * (runs - 1 - r)));
        for (int64_t m = 0; m < nseg; ++m) {
            uint32_t v = km;
            for (int i = 31; i >= 0; --i) {
                wt[((size_t)r * nseg + m) * 32 + i] = v;
                v = (v & 1) ? (v >> 1) ^ CC_POLY : v >> 1;
            }
            km = cc_h_multmodp(k_seg, km);
        }
    }
    CcPlan &pl = plans[n_plans];
    pl.key = key;
    const int nl = (key.b + 31) >> 5;
    for (int k = 0; k < 5; ++k) pl.tgt_k[k] = cc_h_x8n((uint64_t)8 * nl << k);
    pl.init = cc_h_multmodp(cc_h_x8n((uint64_t)nseg * segb + tail), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
    pl.nseg = (int)nseg;
    TSB_CUDA(cudaMalloc(&pl.d_img, img.size() * 4));
    TSB_CUDA(cudaMalloc(&pl.d_slice, slice.size() * 4));
    TSB_CUDA(cudaMalloc(&pl.d_w, wt.size() * 4));
    // stream-ordered before the launch; synchronous on the host side so the
    // staging vectors may go (pageable sources are staged before return)
    TSB_CUDA(cudaMemcpyAsync(pl.d_img, img.data(), img.size() * 4, cudaMemcpyHostToDevice, s));
    TSB_CUDA(cudaMemcpyAsync(pl.d_slice, slice.data(), slice.size() * 4, cudaMemcpyHostToDevice, s));
    TSB_CUDA(cudaMemcpyAsync(pl.d_w, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice, s));
    TSB_CUDA(cudaStreamSynchronize(s));
    ++n_plans;
    *out = &pl;
    return TSB_OK;
}

// TSB_CRC_FUSED: 1 (default) the fused kernel, 0 the output-side CRC
// (tsb_crc32) after the collate (A/B).
int cc_mode_knob() {
    static const int v = getenv("TSB_CRC_FUSED") ? atoi(getenv("TSB_CRC_FUSED")) : 1;
    return v;
}

// Item stages that fit next to the tables for any dynamic shared base the
// runtime may pick (TSB_CC_STAGES caps it, A/B); < 2: the kernel does not fit.
int cc_stages(const CaGeom &g, int c) {
    static const int cap = getenv("TSB_CC_STAGES") ? atoi(getenv("TSB_CC_STAGES")) : CC_MAX_STAGES;
    const uint32_t part = 4u * (uint32_t)(c * g.R * (g.w / 32));
    for (int n = cap < CC_MAX_STAGES ? cap : CC_MAX_STAGES; n >= 2; --n) {
        bool ok = true;
        CcLayout L;
        for (uint32_t sb : {0u, 1024u, 2048u})
            ok = ok && cc_layout(sb, (uint32_t)(g.R * g.rs), (uint32_t)g.rs, part, n, L);
        if (ok) return n;
    }
    return 0;
}

// Can this batch take the fused kernel?  Returns its emit thread count
// (groups x dr, a whole number of warps, dr dividing the item's rows) or 0:
// collate, then tsb_crc32.
int cc_fusable(const CaGeom &g, int c, int out_kind, const Dsts &dsts, bool publishes) {
    if (!cc_mode_knob() || !publishes || dsts.n != 1 || c > CC_MAX_C || !g.use_tma ||
        g.use_direct)
        return 0;
    const int P = out_kind == TSB_OUT_U8 ? 16 : out_kind == TSB_OUT_F32 ? 4 : 8;
    if (g.w % 32 || g.w / 32 > CC_MAX_RUNS || g.R > 32 || g.h % g.R || g.nrb * g.R != g.h) return 0;
    const int groups = g.w / P;
    int ne = 0;
    for (int dr = g.R; dr >= 1 && !ne; --dr)
        if (g.R % dr == 0 && groups * dr <= CC_EMIT && (groups * dr) % 32 == 0) ne = groups * dr;
    if (!ne) return 0;
    if (cc_stages(g, c) < 2) return 0;
    return ne;
}

template <int K, int C>
int launch_cc(const uint8_t *src, const int64_t *idx, CaGeom g, int flip, uint64_t aug_mixed,
              uint64_t epoch, const Norm &norm, const int32_t *params, const Dsts &dsts,
              cudaStream_t s, const Epi &ep, const CrcFuse &cf) {
    auto kern = collate_crc_kernel<K, C>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64) dev = 63;
    if (!attr_set[dev]) {
        TSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CC_SMEM));
        attr_set[dev] = true;
    }
    const int grid = g.items < sm_count() ? g.items : sm_count();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(cf.ne + 32 + 32 * (g.w / 32));
    cfg.dynamicSmemBytes = CC_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ep.pdl ? 1 : 0;
    TSB_CUDA(cudaLaunchKernelEx(&cfg, kern, src, idx, g, flip, aug_mixed, epoch, norm, params, dsts,
                                ep, cf));
    return TSB_OK;
}

template <int K>
int launch_cc_c(int c, const uint8_t *src, const int64_t *idx, const CaGeom &g, int flip,
                uint64_t aug_mixed, uint64_t epoch, const Norm &norm, const int32_t *params,
                const Dsts &dsts, cudaStream_t s, const Epi &ep, const CrcFuse &cf) {
    switch (c) {
        case 1: return launch_cc<K, 1>(src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
        case 2: return launch_cc<K, 2>(src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
        default: return launch_cc<K, 3>(src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
    }
}

// Fused collate + batch checksum into a ring slot (the caller checked
// cc_fusable).  crc_out receives the zlib CRC-32 of input + target before
// the slot is published.
int launch_collate_crc(const uint8_t *src, const int64_t *idx, CaGeom g, int c, int flip,
                       uint64_t aug_mixed, uint64_t epoch, const Norm &norm, int out_kind,
                       const int32_t *params, const Dsts &dsts, cudaStream_t s, const Epi &ep,
                       uint32_t *crc_out, int ne, uint32_t *crc_host) {
    int dev = 0;
    TSB_CUDA(cudaGetDevice(&dev));
    CcKey key{};
    key.dev = dev;
    key.out_kind = out_kind == OUT_BF16_FMA ? TSB_OUT_BF16 : out_kind;
    key.c = c;
    key.w = g.w;
    key.h = g.h;
    key.R = g.R;
    key.b = g.b;
    key.with_tgt = ep.tgt[0] != nullptr;
    if (key.out_kind != TSB_OUT_U8) {
        memcpy(key.scale, norm.scale, sizeof(key.scale));
        memcpy(key.bias, norm.bias, sizeof(key.bias));
    }
    const CcPlan *pl = nullptr;
    if (int rc = cc_plan(key, s, &pl)) return rc;
    if (!pl) return TSB_ERR_STALE;  // plan table full: unfused path
    static uint32_t *acc_base[64] = {nullptr};
    static unsigned int *cnt_base[64] = {nullptr};
    static std::atomic<unsigned> acc_next{0};
    if (!acc_base[dev]) {
        void *p = nullptr, *q = nullptr;
        TSB_CUDA(cudaGetSymbolAddress(&p, g_cc_acc));
        TSB_CUDA(cudaGetSymbolAddress(&q, g_cc_cnt));
        acc_base[dev] = static_cast<uint32_t *>(p);
        cnt_base[dev] = static_cast<unsigned int *>(q);
    }
    const unsigned slot = acc_next.fetch_add(1, std::memory_order_relaxed) % CC_ACC_POOL;
    CrcFuse cf{};
    cf.img = pl->d_img;
    cf.slice = pl->d_slice;
    cf.wtab = pl->d_w;
    memcpy(cf.tgt_k, pl->tgt_k, sizeof(cf.tgt_k));
    cf.init = pl->init;
    cf.nseg = pl->nseg;
    cf.with_tgt = key.with_tgt;
    cf.tab_c = key.out_kind == TSB_OUT_U8;
    cf.acc = acc_base[dev] + slot;
    cf.count = cnt_base[dev] + slot;
    cf.out = crc_out;
    cf.out_host = crc_host;
    cf.ne = ne;
    cf.fold = cc_fold_knob(key.out_kind);
    g.nstage = cc_stages(g, c);
    if (out_kind == TSB_OUT_U8)
        return launch_cc_c<TSB_OUT_U8>(c, src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
    if (out_kind == TSB_OUT_F32)
        return launch_cc_c<TSB_OUT_F32>(c, src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
    if (out_kind == OUT_BF16_FMA)
        return launch_cc_c<OUT_BF16_FMA>(c, src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
    return launch_cc_c<TSB_OUT_BF16>(c, src, idx, g, flip, aug_mixed, epoch, norm, params, dsts, s, ep, cf);
}

template <int K, int C>
int launch_ccr(const uint8_t *src, const int64_t *order0, const CaGeom &g, int flip,
               uint64_t aug_mixed, uint64_t epoch, const Norm &norm, cudaStream_t s,
               const CrcFuse &cf, const CcRange &rg) {
    auto kern = collate_crc_range_kernel<K, C>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64) dev = 63;
    if (!attr_set[dev]) {
        TSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CC_SMEM));
        attr_set[dev] = true;
    }
    const int64_t total = (int64_t)g.items * rg.n;
    // SMs the range leaves free for other kernels (TSB_CC_RANGE_FREE_SMS,
    // default 0): the launch holds one CTA per SM for the whole range.  Alone,
    // f32 runs faster on 136 SMs (31.0 vs 32.4 us per C2 batch), but inside the
    // bench with its consumers and the device gate all 148 are best (32.2 vs
    // 33.4 us); bf16/u8 lose 9% with 12 free (profiles/r2/range/
    // range_free_sms.jsonl, bench_free_sms.txt)
    static const int free_sms = getenv("TSB_CC_RANGE_FREE_SMS")
                                    ? atoi(getenv("TSB_CC_RANGE_FREE_SMS")) : 0;
    int sms = sm_count() - (free_sms > 0 ? free_sms : 0);
    if (sms < 1) sms = 1;
    const int grid = (int)(total < sms ? total : sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(cf.ne + 64 + 32 * (g.w / 32));  // emit, producer, combiners, publisher
    cfg.dynamicSmemBytes = CC_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: CTAs gate independently
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TSB_CUDA(cudaLaunchKernelEx(&cfg, kern, src, order0, g, flip, aug_mixed, epoch, norm, cf, rg));
    return TSB_OK;
}

// n batches of the fused collate + checksum in one persistent launch (the
// caller checked cc_fusable); TSB_ERR_STALE: take the per-batch path.
int launch_collate_crc_range(const uint8_t *src, const int64_t *order0, CaGeom g, int c, int flip,
                             uint64_t aug_mixed, uint64_t epoch, const Norm &norm, int out_kind,
                             cudaStream_t s, CcRange rg, int ne) {
    int dev = 0;
    TSB_CUDA(cudaGetDevice(&dev));
    CcKey key{};
    key.dev = dev;
    key.out_kind = out_kind == OUT_BF16_FMA ? TSB_OUT_BF16 : out_kind;
    key.c = c;
    key.w = g.w;
    key.h = g.h;
    key.R = g.R;
    key.b = g.b;
    key.with_tgt = rg.with_target;
    if (key.out_kind != TSB_OUT_U8) {
        memcpy(key.scale, norm.scale, sizeof(key.scale));
        memcpy(key.bias, norm.bias, sizeof(key.bias));
    }
    const CcPlan *pl = nullptr;
    if (int rc = cc_plan(key, s, &pl)) return rc;
    if (!pl) return TSB_ERR_STALE;
    static uint32_t *acc_base[64] = {nullptr};
    static unsigned long long *gate_words[64] = {nullptr};
    static std::atomic<unsigned> acc_next{0};
    if (!acc_base[dev]) {
        void *p = nullptr;
        TSB_CUDA(cudaGetSymbolAddress(&p, g_cc_acc));
        acc_base[dev] = static_cast<uint32_t *>(p);
        TSB_CUDA(cudaMalloc(&gate_words[dev], 256));
    }
    CrcFuse cf{};
    cf.img = pl->d_img;
    cf.slice = pl->d_slice;
    cf.wtab = pl->d_w;
    memcpy(cf.tgt_k, pl->tgt_k, sizeof(cf.tgt_k));
    cf.init = pl->init;
    cf.nseg = pl->nseg;
    cf.with_tgt = key.with_tgt;
    cf.tab_c = key.out_kind == TSB_OUT_U8;
    cf.ne = ne;
    cf.fold = cc_fold_knob(key.out_kind);
    rg.acc_pool = acc_base[dev];
    rg.acc_base = acc_next.fetch_add((unsigned)rg.n, std::memory_order_relaxed) % CC_ACC_POOL;
    rg.gate = gate_words[dev];
    // bench A/B (profiles/r2/range/refresh_ab.jsonl, refresh_sweep.jsonl): 0 ->
    // 32.4-32.5 us per f32 batch, 2 -> 32.1-35.3, 3 -> 32.6, 4 -> 31.9-32.1,
    // 5 -> 32.1, 6 -> 32.5
    static const int refresh = getenv("TSB_CC_REFRESH") ? atoi(getenv("TSB_CC_REFRESH")) : 4;
    rg.refresh = refresh;
    TSB_CUDA(cudaMemsetAsync(rg.gate, 0, sizeof(unsigned long long), s));
    g.nstage = cc_stages(g, c);
#define TSB_CCR(KK)                                                                                \
    switch (c) {                                                                                   \
        case 1: return launch_ccr<KK, 1>(src, order0, g, flip, aug_mixed, epoch, norm, s, cf, rg); \
        case 2: return launch_ccr<KK, 2>(src, order0, g, flip, aug_mixed, epoch, norm, s, cf, rg); \
        default: return launch_ccr<KK, 3>(src, order0, g, flip, aug_mixed, epoch, norm, s, cf, rg); \
    }
    if (out_kind == TSB_OUT_U8) TSB_CCR(TSB_OUT_U8)
    if (out_kind == TSB_OUT_F32) TSB_CCR(TSB_OUT_F32)
    if (out_kind == OUT_BF16_FMA) TSB_CCR(OUT_BF16_FMA)
    TSB_CCR(TSB_OUT_BF16)
#undef TSB_CCR
}

template <int K>
void preload_cc() {
    touch_kernel(collate_crc_kernel<K, 1>);
    touch_kernel(collate_crc_kernel<K, 2>);
    touch_kernel(collate_crc_kernel<K, 3>);
    touch_kernel(collate_crc_range_kernel<K, 1>);
    touch_kernel(collate_crc_range_kernel<K, 2>);
    touch_kernel(collate_crc_range_kernel<K, 3>);
}
