// vr_warp_rows.cuh -- warp voting (strategies.py:173-232) for static batches, tile kernel.
// Included by vr_run.cu inside namespace vr (uses RunCtx, report_error, finish_stats, lds_*/sts_*).
//
// A TILE is 64 consecutive static batches (batching.py:76-84): one contiguous 64 * batch_size *
// 4-byte piece of the index buffer.  The grid is PERSISTENT (one CTA per shared-memory slot of the
// GPU, 4 per SM); a CTA has 2 dedup warps (one thread per batch) and 4 helper warps and draws
// tickets in a loop.  With ticket i it works on TWO tiles at once -- software pipelining across tiles:
//
//   dedup warps, tile i
//     A  stage   every row (batch) arrives by ONE bulk asynchronous copy (cp.async.bulk, the 1-D
//                TMA path, completion on an mbarrier) into its own shared-memory row: the tile is
//                read from HBM as whole 128-byte lines, no register staging.  The copies of tile
//                i were issued during the post phase of the CTA's previous tile.
//     B  dedup   one THREAD per batch runs the closed form of Algorithm 1 over its row as a
//                per-lane state machine (see below).  Claims are appended IN PLACE at the front of
//                the row, local indices are bytes in a rank row.
//     C  post    all six warps: the rows' claims are copied, compacted, into the tile's slot of an
//                L2-resident scratch list together with the per-row round records; the next
//                ticket's rows are staged; local indices leave as coalesced 16-byte stores
//                (8 x uint16); then the tile's (rounds, claims) AGGREGATE is published.  The CTA
//                never waits for the tile's output offsets.
//   helper warps, tile j = i - K  (K = 1.5 x the number of CTAs: tile j was published half a round ago)
//     D  offsets two-level scan: j's exclusive prefix = inclusive prefix of the previous 32-tile GROUP
//                (decoupled look-back over group sums that the tiles accumulate when they publish)
//                + the aggregates of the earlier tiles of j's own group; one L2 round trip;
//     E  shade   the tile's flat claim list is streamed from the scratch (L2 hits): coalesced id
//                store, 16-byte position gather, FP32 4x4 transform + w-divide (strategies.py:53-67),
//                coalesced 16-byte stores; round tables from the round records.
//                This memory-bound work runs UNDER the compute-bound dedup of tile i.
//     F  (optional, VR_PREFETCH=1) the vertices of tile i are prefetched into L2.
//
// The K tickets after the last tile only shade (their dedup warps idle).
// Debug / tuning knobs (environment, read at launch): VR_LAG=<K>, VR_PREFETCH=1, VR_NO_PDL=1.
#pragma once

constexpr int kRowGroup = 32;    // tiles per group of the two-level offset scan
constexpr int kRowThreads = 64;      // batches per tile = dedup threads
constexpr int kRowCtaThreads = 192;  // + 4 helper warps

struct RowsGeom {
    int row_words;   // shared-memory row stride in 32-bit words (odd multiple of 4)
    int slack;       // words in front of the indices that absorb the tail re-claims
    int rk_stride;   // bytes per rank row (an odd number of words)
    int max_rounds;  // upper bound of rounds per batch
    int row_cap;     // upper bound of claims per batch
    int tile_words;  // scratch words per tile: meta[2][64] | rounds[64][max_rounds] | claims[64 * row_cap]
    int lag;         // K: the helpers of the CTA with ticket i shade tile i - K
    int n_tiles;
    int n_groups;  // groups of kRowGroup tiles (two-level offset scan)
    uint32_t cpr_magic;  // ceil(2^32 / (batch_size / 8)): chunk -> row by multiply-high
    size_t smem;
};

// every round but the last consumes at least 3 * floor(W / 3) indices (SURVEY 7-3 / DESIGN 4)
static inline bool rows_geometry(int W, int bs, RowsGeom& g) {
    if (bs % 24 != 0 || bs > 384) return false;  // whole 16-byte quads, whole 8-slot chunks
    const int per_round = 3 * (W / 3);
    g.max_rounds = (bs + per_round - 1) / per_round;
    g.slack = (2 * g.max_rounds + 2) & ~3;  // >= 2 * max_rounds - 1: see the claim-list store in the dedup loop
    int rw = bs + g.slack + 4;  // >= 4 pad words after the indices: the dedup loop's read-ahead stays inside the row
    while ((rw & 7) != 4) rw += 4;
    g.row_words = rw;
    g.rk_stride = bs + 4;  // odd number of words: same-slot byte stores of a warp are conflict-free
    g.row_cap = bs + 2 * g.max_rounds;
    g.tile_words = kRowThreads * (2 + g.max_rounds + g.row_cap);
    const int cpr = bs / 8;
    g.cpr_magic = (uint32_t)(((1ull << 32) + cpr - 1) / cpr);  // exact for chunk * cpr < 2^32
    const int S = 2 * W;
    g.smem = (size_t)kRowThreads * ((size_t)rw * 4 + (size_t)S * 4 + (size_t)g.rk_stride + (size_t)g.max_rounds * 4 + 4);
    return g.smem <= 100 * 1024;
}
// scratch words needed by the tile kernel for nb batches (aliases the staging area of the other kernels)
static inline size_t rows_scratch_words(int W, int bs, int64_t nb) {
    RowsGeom g;
    if (!rows_geometry(W, bs, g)) return 0;
    return (size_t)ceil_div(nb, kRowThreads) * (size_t)g.tile_words;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}
// 1-D bulk copy global -> shared (UBLKCP): dst/src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifdef VR_TIMELINE
// debugging aid: per-tile phase time stamps (ns, %globaltimer) of dedup warp 0 and helper warp 2
constexpr int kTimelineMarks = 12, kTimelineTiles = 8192;
__device__ unsigned long long g_timeline[kTimelineMarks * 2 * kTimelineTiles];
__device__ __forceinline__ unsigned long long timeline_now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define VR_MARK_AT(k, value)                                                                   \
    do {                                                                                       \
        if ((t & 31) == 0 && ((t >> 5) == 0 || (t >> 5) == 2) && tile < kTimelineTiles)        \
            g_timeline[((k) * 2 + ((t >> 5) ? 1 : 0)) * kTimelineTiles + tile] = (value);      \
    } while (0)
#define VR_MARK(k) VR_MARK_AT(k, timeline_now())
#else
#define VR_MARK_AT(k, value) do {} while (0)
#define VR_MARK(k) do {} while (0)
#endif

// ---- D/E: shading of one finished tile by 128 threads (4 warps; `ht` = 0..127).  Used by the helper
// warps of the tile kernel (tile = ticket - K).
template <int DUMMY>
__device__ __forceinline__ void rows_shade_tile(const RunCtx& c, const RowsGeom& g, const ShaderParams& sp, int stile, int ht,
                                                int2* s_base_ptr) {
    constexpr int T = kRowThreads, NH = kRowCtaThreads - kRowThreads;
    const int lane = ht & 31;
    const bool lb_warp = ht < 32;
    int2& s_base = *s_base_ptr;
#ifdef VR_TIMELINE
    const int t = ht + 64, tile = stile + g.lag;  // marks are filed under the CTA's own tile
#endif
    // Every helper warp waits for the tile's aggregate (normally published long ago: K tiles
    // back) -- it carries the claim count, and acquiring it makes the tile's scratch visible.
    unsigned long long mine = 0;
    bool lost = false;
    {
        int spins = 0;
        for (;;) {
            mine = ld_acquire_gpu_u64(c.tile_state + stile);  // every thread acquires: the scratch is visible to it
            if (__all_sync(0xffffffffu, (mine >> 62) != 0)) break;
            // (forward progress is guaranteed by ticket order; the bound only turns a broken launch into an error
            // instead of a hang, and backs off so that a preempted / time-sliced producer is not mistaken for one:
            // 2^12 polls at full rate, then ~2^20 x 0.5 us)
            if (++spins > (1 << 12)) __nanosleep(500);
            if (spins > (1 << 20) + (1 << 12)) { lost = true; break; }
        }
    }
    VR_MARK(8);
    // (the claim count is taken from the scratch, not from the state word: the first helper warp
    // may already have replaced the aggregate by the tile's inclusive prefix when a later warp polls)
    const uint32_t* __restrict__ sc = c.stage_uid + (size_t)stile * (size_t)g.tile_words;
    const uint32_t mlast = lost ? 0u : __ldcg(sc + T - 1);
    const int tot = (int)(mlast & 0xFFFFu) + (int)(mlast >> 16);  // prefix + claims of the last row
    const uint32_t* __restrict__ claims = sc + T * (2 + g.max_rounds);
    const bool want_uid = c.out.d_unique_ids != nullptr;
    const bool want_pos = sp.kind == VR_SHADER_POSITION;
    uint32_t m0 = 0, m1 = 0;  // round-table metadata of row ht, in flight with everything else
    constexpr int RW = 4;     // round records fetched up front (a 96-index batch at W = 32 has at most 4 rounds)
    uint32_t rw[RW];
    if (ht < T) {
        m0 = __ldcg(sc + ht);
        m1 = __ldcg(sc + T + ht);
#pragma unroll
        for (int q = 0; q < RW; q++) rw[q] = q < g.max_rounds ? __ldcg(sc + 2 * T + q * T + ht) : 0u;
    }
    // ---- E (part 1): the first U8 claims of every thread are gathered and shaded while the
    // first helper warp is still resolving the tile's output offsets
#ifndef VR_U8
#define VR_U8 4
#endif
#ifndef VR_TRIP_UNROLL
#define VR_TRIP_UNROLL 4  // dedup trips between two votes on "any lane still has slots"
#endif
#ifndef VR_HELPER_PREFETCH
#define VR_HELPER_PREFETCH 1
#endif
    constexpr int U8 = VR_U8;
    uint32_t uid[U8], nxt[U8];
    float4 pv[U8];
#pragma unroll
    for (int u = 0; u < U8; u++) uid[u] = ht + NH * u < tot ? __ldcg(claims + ht + NH * u) : 0u;
#pragma unroll
    for (int u = 0; u < U8; u++) nxt[u] = ht + NH * (U8 + u) < tot ? __ldcg(claims + ht + NH * (U8 + u)) : 0u;
    if (want_pos) {
#pragma unroll
        for (int u = 0; u < U8; u++)
            if (ht + NH * u < tot) pv[u] = __ldg(sp.pos4 + uid[u]);
#pragma unroll
        for (int u = 0; u < U8; u++)  // the next step's vertices: on their way to L2 while this step is shaded
            if (VR_HELPER_PREFETCH && ht + NH * (U8 + u) < tot) prefetch_l2(sp.pos4 + nxt[u]);
    }
    // ---- D: output offsets of tile stile (first helper warp).  All ~600 tiles in flight reach this
    // point together, so a tile-by-tile look-back would have to walk ~600 aggregates (five dependent
    // round trips to L2).  Two levels instead: every tile adds its aggregate to its GROUP's sum when
    // it publishes; a tile's exclusive prefix is (inclusive prefix of the previous group, found by a
    // decoupled look-back over groups: 64 groups = 2048 tiles per step) + (aggregates of the earlier
    // tiles of its own group).  All loads of both levels are in flight together: one round trip.
    if (lb_warp) {
        const long long ar = (long long)((mine >> 32) & 0x3FFFFFFFull), au = (long long)(mine & 0xFFFFFFFFull);
        unsigned long long* __restrict__ grp_sum = c.tile_state + g.n_tiles + 1;   // count<<58 | rounds<<34 | claims
        unsigned long long* __restrict__ grp_incl = grp_sum + g.n_groups + 1;      // flag<<62 | rounds<<32 | claims
        const int grp = stile / kRowGroup, pos = stile % kRowGroup;
        long long pr = 0, pu = 0;  // this lane's share of the exclusive prefix of the tile
        bool found = grp == 0;
#ifndef VR_LB
#define VR_LB 2
#endif
        constexpr int LB = VR_LB;
        bool first = true;
        for (int pz = grp - 1; (first || (pz >= 0 && !found)) && !lost; pz -= 32 * LB) {
            unsigned long long word[LB], sum[LB], tw = 0;
            int spins = 0;
            for (;;) {
                bool pending = false;
                if (first && lane < pos) tw = ld_relaxed_gpu_u64(c.tile_state + grp * kRowGroup + lane);
#pragma unroll
                for (int k = 0; k < LB; k++) {
                    const int idx = pz - lane - 32 * k;
                    word[k] = found ? 0ull : ld_relaxed_gpu_u64(grp_incl + (idx >= 0 ? idx : 0));
                    sum[k] = found ? 0ull : ld_relaxed_gpu_u64(grp_sum + (idx >= 0 ? idx : 0));
                }
                if (first && lane < pos) pending |= (tw >> 62) == 0;
#pragma unroll
                for (int k = 0; k < LB; k++) {
                    if (pz - lane - 32 * k < 0) word[k] = kStateInclusive + 0ull;  // before the first group: inclusive zero
                    // (every group before the last one holds kRowGroup tiles)
                    pending |= !found && (word[k] >> 62) == 0 && (sum[k] >> 58) != (unsigned long long)kRowGroup;
                }
                if (!__any_sync(0xffffffffu, pending)) break;
                if (++spins > (1 << 12)) __nanosleep(500);
                if (spins > (1 << 20) + (1 << 12)) { lost = true; break; }
            }
            if (lost) break;
            if (first && lane < pos) {
                pr += (long long)((tw >> 32) & 0x3FFFFFFFull);
                pu += (long long)(tw & 0xFFFFFFFFull);
            }
#pragma unroll
            for (int k = 0; k < LB; k++) {
                const uint32_t incl = __ballot_sync(0xffffffffu, !found && (word[k] >> 62) == 2);
                const int upto = found ? -1 : (incl ? __ffs(incl) - 1 : 31);
                if (lane < upto) {  // nearer groups: their complete sums
                    pr += (long long)((sum[k] >> 34) & 0xFFFFFFull);
                    pu += (long long)(sum[k] & 0x3FFFFFFFFull);
                } else if (lane == upto && incl) {  // the nearest group that knows its inclusive prefix
                    pr += (long long)((word[k] >> 32) & 0x3FFFFFFFull);
                    pu += (long long)(word[k] & 0xFFFFFFFFull);
                } else if (lane == upto) {
                    pr += (long long)((sum[k] >> 34) & 0xFFFFFFull);
                    pu += (long long)(sum[k] & 0x3FFFFFFFFull);
                }
                found |= incl != 0;
            }
            first = false;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            pr += __shfl_xor_sync(0xffffffffu, pr, d);
            pu += __shfl_xor_sync(0xffffffffu, pu, d);
        }
        if (lane == 0 && !lost) {
            // the last tile of a group knows the group's inclusive prefix: later groups stop there
            if (pos == kRowGroup - 1)
                st_relaxed_gpu_u64(grp_incl + grp, kStateInclusive | ((unsigned long long)((pr + ar) & 0x3FFFFFFF) << 32) | (unsigned long long)((pu + au) & 0xFFFFFFFFll));
        }
        const long long er = pr, eu = pu;
        if (lane == 0) {
            if (lost) report_error(c, (int64_t)stile * T, VR_ERR_CUDA);
            const long long R = er + ar, U = eu + au;
            const bool fits = U <= c.out.cap_unique && R <= c.out.cap_rounds && U <= 0x7fffffffLL && !lost;
            if (!fits) report_error(c, (int64_t)stile * T, VR_ERR_CAPACITY);
            s_base = fits ? make_int2((int)er, (int)eu) : make_int2(-1, -1);
            if (stile == g.n_tiles - 1) { __threadfence(); finish_stats(c, R, U); }
        }
    }
    VR_MARK(9);
    asm volatile("bar.sync 1, %0;" ::"n"(NH) : "memory");  // helpers: offsets known
    const int2 off = s_base;
    if (off.x >= 0) {
        // ---- E (part 2): stores; further claims U8 at a time, their ids loaded one step ahead
        for (int j0 = ht;; j0 += NH * U8) {
#pragma unroll
            for (int u = 0; u < U8; u++) {
                const int j = j0 + NH * u;
                if (j < tot) {
                    if (want_uid) c.out.d_unique_ids[(int64_t)off.y + j] = uid[u];
                    if (want_pos) reinterpret_cast<float4*>(c.out.d_shaded4)[(int64_t)off.y + j] = transform_position(sp, pv[u]);
                }
            }
            if (j0 + NH * U8 - ht >= tot) break;  // warp-uniform: no claim left for any thread
#pragma unroll
            for (int u = 0; u < U8; u++) uid[u] = nxt[u];
            if (want_pos) {
#pragma unroll
                for (int u = 0; u < U8; u++)
                    if (j0 + NH * (U8 + u) < tot) pv[u] = __ldg(sp.pos4 + uid[u]);
            }
#pragma unroll
            for (int u = 0; u < U8; u++) nxt[u] = j0 + NH * (2 * U8 + u) < tot ? __ldcg(claims + j0 + NH * (2 * U8 + u)) : 0u;
            if (want_pos) {
#pragma unroll
                for (int u = 0; u < U8; u++)
                    if (VR_HELPER_PREFETCH && j0 + NH * (2 * U8 + u) < tot) prefetch_l2(sp.pos4 + nxt[u]);
            }
        }
        VR_MARK(10);
        // attribute pass-through and per-vertex tally (strategies.py:485-489): one compact loop
        if ((sp.attr_words && c.out.d_shaded_attr) || c.out.d_shade_counts) {
#pragma unroll 1
            for (int j = ht; j < tot; j += NH) {
                const uint32_t id = __ldcg(claims + j);
                if (sp.attr_words && c.out.d_shaded_attr) {
#pragma unroll 1
                    for (int w = 0; w < sp.attr_words; w++)
                        c.out.d_shaded_attr[((int64_t)off.y + j) * sp.attr_words + w] = __ldg(sp.attr + (int64_t)id * sp.attr_words + w);
                }
                if (c.out.d_shade_counts) atomicAdd(&c.out.d_shade_counts[id], 1);
            }
        }
        // round tables (strategies.py:114-129, flattened): one thread per row
        if (ht < T) {
            const int sb = stile * T + ht;
            const int nr = (int)(m1 >> 16);
            if (sb < c.n_batches) {
                const int r0w = off.x + (int)(m1 & 0xFFFFu);
                int run = off.y + (int)(m0 & 0xFFFFu);
                if (c.out.d_batch_round_off) c.out.d_batch_round_off[sb] = r0w;
#pragma unroll
                for (int q = 0; q < RW; q++) {
                    if (q < nr) {
                        if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0w + q] = run;
                        if (c.out.d_round_prims) c.out.d_round_prims[r0w + q] = (int)(rw[q] >> 8);
                        run += (int)(rw[q] & 0xFFu);
                    }
                }
#pragma unroll 1
                for (int q = RW; q < nr; q++) {
                    const uint32_t wv = __ldcg(sc + 2 * T + q * T + ht);
                    if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0w + q] = run;
                    if (c.out.d_round_prims) c.out.d_round_prims[r0w + q] = (int)(wv >> 8);
                    run += (int)(wv & 0xFFu);
                }
            }
        }
    }
}

template <int W, bool PREFETCH>
__global__ void __launch_bounds__(kRowCtaThreads, 4) warp_rows_kernel(RunCtx c, int bs, RowsGeom g, ShaderParams sp) {
    constexpr int S = 2 * W;
    constexpr int LOG2W = W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
    constexpr int LOG2S = LOG2W + 1;
    constexpr int T = kRowThreads, NT = kRowCtaThreads, NH = NT - T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_tile[2];            // this iteration's ticket and the next one's
    __shared__ int2 s_warp_tot[T / 32];  // (rounds, claims) of each dedup warp
    __shared__ int2 s_base;              // output offsets of the tile being shaded (look-back result)
    __shared__ int s_cnt[T], s_ex[T];    // claims of each row, exclusive prefix inside the row's dedup warp
    __shared__ int s_rnd[T], s_rex[T];   // rounds of each row, exclusive prefix inside the row's dedup warp
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    const int lane = t & 31, wid = t >> 5;
    const bool dedup_thread = t < T;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t row_bytes = 4u * (uint32_t)g.row_words;
    const uint32_t a_row = sbase + row_bytes * t;                          // claims from word 0
    const uint32_t a_ids = a_row + 4u * (uint32_t)g.slack;                 // indices of the batch
    const uint32_t a_tab0 = sbase + row_bytes * T;                         // table
    const uint32_t a_idtab = a_tab0 + 4u * t;                              // + 4*T*slot
    const uint32_t a_ranks0 = a_tab0 + 4u * T * S;                         // rank rows
    uint32_t a_ranks = a_ranks0 + (uint32_t)g.rk_stride * t;
    const uint32_t a_rounds0 = a_ranks0 + (uint32_t)g.rk_stride * T;       // round records [round][thread]
    const uint32_t a_rounds = a_rounds0 + 4u * t;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    // static batching (batching.py:76-84): batch b = [first + b * bs, min(.. + bs, last_end)); the
    // caller's claim is verified off the critical path below
    const int first = __ldg(c.bbegin), last_end = __ldg(c.bend + (c.n_batches - 1));
    auto zero_table = [&]() {  // tag 0 = never used
        for (uint32_t o = 16u * t; o < (uint32_t)(4 * S * T); o += 16u * NT)
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a_tab0 + o), "r"(0u) : "memory");
    };
    // ---- A: stage the rows of a tile.  Row r is issued by lane r / 6 of warp r % 6 (a bulk copy is a
    // uniform-datapath instruction, so a warp issues its copies one after the other: 11 per warp
    // instead of 32).  Memory safety of the copy does not depend on the caller's batch arrays.  A
    // ticket past the last tile still makes its 64 arrivals, so that the barrier's phases stay in step.
    auto stage = [&](int tile_) {
        if (lane * (NT / 32) + wid < T) {
            const int r = lane * (NT / 32) + wid;
            const int rb = tile_ * T + r;
            const int rbegin = first + rb * bs;
            int rn = tile_ < g.n_tiles && rb < c.n_batches ? min(bs, last_end - rbegin) : 0;
            if (rn != 0 && (first < 0 || (first & 3) || rn < 0 || (int64_t)rbegin + rn > c.n_idx || rn % 3 != 0 || rn > c.max_span)) rn = 0;  // reported by the row's dedup thread
            const uint32_t dst = sbase + row_bytes * (uint32_t)r + 4u * (uint32_t)g.slack;
            const uint32_t bytes = (rn & 3) == 0 ? 4u * (uint32_t)rn : 0u;
            if (!bytes) {
#pragma unroll 1
                for (int i = 0; i < rn; i++) sts_u32(dst + 4 * i, __ldg(c.idx + rbegin + i));  // short last batch
            }
            mbar_arrive_expect_tx(bar, bytes);
            if (bytes) bulk_g2s(dst, c.idx + rbegin, bytes, bar);
        }
    };
    zero_table();
    // the rows start as zeros: whatever the dedup loop reads past a row's last index (its read-ahead, a
    // finished lane's current slot) is then a valid id: zero, a stale index or claim of an earlier tile
    for (uint32_t o = 16u * t; o < row_bytes * T; o += 16u * NT)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(sbase + o), "r"(0u) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ordered before the bulk copies into the rows
    // launched as a programmatic dependent of init_kernel: everything above overlapped its tail
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t == 0) {
        s_tile[0] = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);  // tiles in ticket order
        mbar_init(bar, T);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int tile = s_tile[0];
    stage(tile);
    uint32_t parity = 0;
    int cur = 0;

    // The CTA is PERSISTENT: it draws tickets until the tiles and the K trailing shade-only tickets
    // are used up.  The next ticket is drawn while the current tile is deduplicated, and the next
    // tile's rows are staged as soon as the current tile's claims have left them, under the rest of
    // the post phase: a tile pays neither a CTA launch nor its staging latency.
    for (;;) {
        if (tile >= g.n_tiles + g.lag) break;
        const int stile = tile - g.lag;          // the helpers shade tile `stile`
        const bool has_tile = tile < g.n_tiles;
        const bool has_stile = stile >= 0 && stile < g.n_tiles;
        VR_MARK(1);
        uint32_t* __restrict__ my_scratch = c.stage_uid + (size_t)tile * (size_t)g.tile_words;
        if (t == NT - 1) s_tile[cur ^ 1] = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);

        if (dedup_thread) {
            const int b = tile * T + t;
            bool active = has_tile && b < c.n_batches;
            const int begin = first + b * bs;
            int n = active ? min(bs, last_end - begin) : 0;
            if (active && (first < 0 || (first & 3) || n <= 0 || (int64_t)begin + n > c.n_idx || n % 3 != 0 || n > c.max_span)) {
                report_error(c, b, first < 0 || (first & 3) || n <= 0 || (int64_t)begin + n > c.n_idx || n % 3 != 0 ? VR_ERR_BAD_BATCH : VR_ERR_UNSUPPORTED);
                active = false;
                n = 0;
            }
            const int claimed_begin = active ? __ldg(c.bbegin + b) : 0, claimed_end = active ? __ldg(c.bend + b) : 0;

            mbar_wait(bar, parity);
            VR_MARK(2);

        // ---- B: dedup as a per-lane STATE MACHINE: every trip of the loop does one table probe for
        // the lane's current slot p.  A probe that collides moves the lane to the next table slot; one
        // that resolves (hit, or free slot = new claim) stores the local index and moves the lane to
        // slot p + 1; a round end (strategies.py:220-231) records the round and REWINDS the lane to
        // the first unconsumed slot, so the discarded tail is re-claimed by the ordinary path.  Lanes
        // never wait for each other's extra probes or round ends: the loop runs
        // max-over-lanes(slots + collisions + replays) trips, not the sum of per-slot maxima.
        //   table: entry[slot][thread] = id << 8 | round tag << LOG2W | rank, one 32-bit shared load
        //   per probe; a slot is occupied iff its tag is the current round's, so a new round clears
        //   nothing (tag 0 = never used; ids must fit 24 bits: the helper warps check every index).
        // The trip is software-pipelined by hand: the probe and the next slot's id for trip i+1 are
        // loaded as soon as the lane's next state is known, and the side effects of trip i issue
        // under that latency.  The table store goes to a per-thread dummy word when the lane does
        // not claim, so the only branches are the loop and the (rare) round end.
        constexpr uint32_t kTagInc = 1u << LOG2W;
        constexpr uint32_t kTagMask = 0xFFu & ~(uint32_t)(W - 1);
        uint32_t a_dummy = a_rounds + 4u * T * (uint32_t)g.max_rounds;  // one spare word per thread
        // opaque from here on: otherwise the compiler recomputes both from the shared-memory base inside
        // the loop (~10 instructions per four trips) to save two registers
        a_dummy = __shfl_sync(0xffffffffu, a_dummy, lane);  // (ptxas rematerialises anything it can see through)
        a_ranks = __shfl_sync(0xffffffffu, a_ranks, lane);
        int p = 0, fill = 0, cursor = 0, rounds = 0;
        uint32_t cl = a_row;  // next claim slot of the row
        uint32_t tagw = kTagInc;
        uint32_t ax = a_ids;  // address of slot p
        uint32_t x = lds_u32(ax);
        // every index is range-checked as it becomes the lane's current slot: the packed table entry
        // holds 24 bits (vertex_count <= 2^24 on this path) and the gather must stay inside the buffer
        const uint32_t vcount = (uint32_t)sp.vertex_count;
        uint32_t mx = x;  // largest id seen; slots past the row's end hold valid ids (see the zeroing above)
        uint32_t ai = a_idtab + 4u * T * ((x * 0x9E3779B1u) >> (32 - LOG2S));  // address of the probed table slot
        const uint32_t a_tab_end = a_idtab + 4u * T * S;
        uint32_t v = lds_u32(ai), cand = lds_u32(ax + 4);
        for (;;) {
#pragma unroll
            for (int u = 0; u < VR_TRIP_UNROLL; u++) {
                const bool live = p < n;
                // off the critical path (known before the probe v arrives): the slot a collision moves
                // to, the slot the next id hashes to, and the part of the round-end test that does not
                // depend on the probe
                uint32_t a_coll = ai + 4u * T;
                a_coll -= a_coll >= a_tab_end ? 4u * T * S : 0u;
                const uint32_t a_cand = a_idtab + 4u * T * ((cand * 0x9E3779B1u) >> (32 - LOG2S));
                const bool full = fill == W;
                const bool full_edge = full & (((p - cursor) & (W - 1)) == 0);
                const uint32_t xk = x * 256u + tagw;              // id << 8 | tag: one IMAD
                const uint32_t tq = v ^ xk;                       // == rank (< W) iff the slot holds x in this round
                const bool hit = tq < (uint32_t)W;
                const bool fre = (tq & kTagMask) != 0;            // slot not used in this round
                // The round ends before slot p once all W lanes are claimed and either x is the first id
                // that cannot be assigned (free slot reached), or the W-wide fetch in which the last
                // claim was made is exhausted: fetches start at cursor, cursor + W, ... and a new one
                // starts only while a lane is free (strategies.py:201, :220).
                const bool ends = full_edge | (full & fre);
                const bool adv = live & (hit | fre) & !ends;
                const bool clm = adv & fre;  // strategies.py:207-212: new id -> lowest free lane
                sts_u32(clm ? ai : a_dummy, xk | (uint32_t)fill);  // before the next probe is loaded
                const uint32_t xn = adv ? cand : x;
                const uint32_t ain = adv ? a_cand : a_coll;  // (a resolved probe that does not advance is a round end or a finished lane)
                const uint32_t axn = ax + (adv ? 4u : 0u);
                uint32_t vn = lds_u32(ain), candn = lds_u32(axn + 4);
                // claim list and local index: written unconditionally, a lane that does not resolve slot
                // p here overwrites both when it does (the addresses only move on adv / clm)
                sts_u32(cl, x);
                sts_u8(a_ranks + (uint32_t)p, min(tq, (uint32_t)fill));  // hit: tq = rank < fill; new claim: tq >= W >= fill
                cl += clm ? 4u : 0u;
                fill += clm ? 1 : 0;
                p += adv ? 1 : 0;
                mx = max(mx, xn);
                ax = axn; x = xn; ai = ain;
                if (ends) {
                    const int d = p - cursor;
                    const int emitted = (int)(((uint32_t)d * 43691u) >> 17);  // d / 3 for d < 2^16
                    sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)emitted << 8) | (uint32_t)fill);
                    rounds++;
                    fill = 0;
                    cursor += 3 * emitted;
                    p = cursor;  // re-open at the first unconsumed slot (the row still holds it: see slack)
                    ax = a_ids + 4u * (uint32_t)p;
                    x = lds_u32(ax);
                    ai = a_idtab + 4u * T * ((x * 0x9E3779B1u) >> (32 - LOG2S));
                    if (tagw == kTagMask) {  // tag space exhausted: wipe this thread's column
#pragma unroll 1
                        for (int k = 0; k < S; k++) sts_u32(a_idtab + 4u * T * k, 0u);
                        tagw = 0;
                    }
                    tagw += kTagInc;
                    vn = lds_u32(ai);
                    candn = lds_u32(ax + 4);
                }
                v = vn; cand = candn;
            }
            if (!__any_sync(0xffffffffu, p < n)) break;
        }
            VR_MARK(3);
            if (active && mx >= vcount) {
                report_error(c, b, VR_ERR_VERTEX_RANGE);  // index outside the vertex buffer
                active = false;
            }
            if (active && (claimed_begin != begin || claimed_end != begin + n)) {
                report_error(c, b, VR_ERR_BAD_BATCH);  // not the static batching this path was promised
                active = false;
            }
            // the batch end closes the last round; nothing is discarded.  (`ends` does not look at `live`: a
            // finished lane with all W lanes claimed may already have recorded exactly this round, from
            // whatever id follows the row: then cursor == n.)
            if (active && cursor < n) {
                sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)((n - cursor) / 3) << 8) | (uint32_t)fill);
                rounds++;
            }
            const int my_r = active ? rounds : 0, my_u = active ? (int)((cl - a_row) >> 2) : 0;
            const int inc_r = warp_incl_scan(my_r, lane), inc_u = warp_incl_scan(my_u, lane);
            if (lane == 31) s_warp_tot[wid] = make_int2(inc_r, inc_u);
            s_cnt[t] = my_u;
            s_ex[t] = inc_u - my_u;  // + s_warp_tot[0].y for rows of warp 1
            s_rnd[t] = my_r;
            s_rex[t] = inc_r - my_r;
        } else {
            // ================= helper warps: tile `stile` =================
            const int ht = t - T;  // 0..127
            if (has_stile) prefetch_l2(c.stage_uid + (size_t)stile * (size_t)g.tile_words + 32 * ht);  // its scratch: 16 KB
            // ---- F (optional): the vertices of tile `tile` are prefetched into L2; they are gathered ~K
            // tiles later.  One request per distinct 32-byte sector among the 32 indices of a step.
            if (PREFETCH && has_tile) {
                const uint32_t vcount_h = (uint32_t)sp.vertex_count;
                const int64_t tb = (int64_t)first + (int64_t)tile * T * bs;
                const int tn = (int)max((int64_t)0, min((int64_t)T * bs, (int64_t)last_end - tb));
                constexpr int HU = 4;
                for (int j0 = ht; j0 - lane < tn; j0 += HU * NH) {  // warp-uniform trip count
                    uint32_t id[HU];
#pragma unroll
                    for (int u = 0; u < HU; u++) id[u] = j0 + u * NH < tn ? __ldg(c.idx + tb + j0 + u * NH) : 0xFFFFFFFFu;
#pragma unroll
                    for (int u = 0; u < HU; u++) {
                        const bool ok = id[u] < vcount_h;
                        const uint32_t same = __match_any_sync(0xffffffffu, ok ? (id[u] >> 1) : 0xFFFFFFFFu);
                        if (ok && (uint32_t)lane == (uint32_t)(__ffs(same) - 1)) prefetch_l2(sp.pos4 + id[u]);
                    }
                }
            }
            VR_MARK(7);
            if (has_stile) rows_shade_tile<0>(c, g, sp, stile, ht, &s_base);
            VR_MARK(6);
        }
        __syncthreads();  // the tile's dedup is done, the helpers are back, the next ticket is known
        VR_MARK(4);
        const int next = s_tile[cur ^ 1];
        const unsigned long long aggregate = kStateAggregate | ((unsigned long long)(uint32_t)(s_warp_tot[0].x + s_warp_tot[1].x) << 32) |
                                             (uint32_t)(s_warp_tot[0].y + s_warp_tot[1].y);

        // ---- C: post.  First everything that reads the rows: per-row prefixes, round records and the
        // compacted claims go to the tile's scratch slot.
        // Scratch: meta0[r] = claim prefix | claims << 16, meta1[r] = round prefix | rounds << 16 (both
        // tile-wide), round records [q][r], then the rows' claims back to back.
        if (has_tile) {
        const int w0r = s_warp_tot[0].x, w0u = s_warp_tot[0].y;
        if (t < T) {
            const int exu = s_ex[t] + (t >= 32 ? w0u : 0), exr = s_rex[t] + (t >= 32 ? w0r : 0);
            my_scratch[t] = (uint32_t)exu | ((uint32_t)s_cnt[t] << 16);
            my_scratch[T + t] = (uint32_t)exr | ((uint32_t)s_rnd[t] << 16);
        }
        for (int k = t; k < T * g.max_rounds; k += NT)  // [round][row] in shared memory and in the scratch
            my_scratch[2 * T + k] = lds_u32(a_rounds0 + 4u * (uint32_t)k);
        {
            uint32_t* __restrict__ claims = my_scratch + T * (2 + g.max_rounds);
            constexpr int CG = 4;  // rows per warp and step: independent load -> store chains
#pragma unroll 1
            for (int r0 = wid; r0 < T; r0 += CG * (NT / 32)) {
                int cnt[CG], e[CG];
#pragma unroll
                for (int i = 0; i < CG; i++) {
                    const int r = r0 + i * (NT / 32);
                    cnt[i] = r < T ? s_cnt[r] : 0;
                    e[i] = r < T ? s_ex[r] + (r >= 32 ? w0u : 0) : 0;
                }
                int most = 0;
#pragma unroll
                for (int i = 0; i < CG; i++) most = max(most, cnt[i]);
                for (int k = lane; k < most; k += 32) {
                    uint32_t v[CG];
#pragma unroll
                    for (int i = 0; i < CG; i++)  // reading past a row's claims stays inside shared memory
                        v[i] = lds_u32(sbase + row_bytes * (uint32_t)min(r0 + i * (NT / 32), T - 1) + 4u * (uint32_t)k);
#pragma unroll
                    for (int i = 0; i < CG; i++)
                        if (k < cnt[i]) claims[e[i] + k] = v[i];
                }
            }
        }
        }
        __syncthreads();  // the rows are free
        stage(next);      // the next tile's indices arrive under the rest of the post phase
        // Local indices: chunk = 8 slots of one row -> one 16-byte store; consecutive threads write
        // consecutive chunks of the tile's contiguous piece of the assembly map.
        if (has_tile) {
        if (c.out.d_assembly_map) {
            const int cpr = bs >> 3;
            uint16_t* __restrict__ amap = c.out.d_assembly_map + (int64_t)tile * T * bs;
            const int64_t slots_left = (int64_t)last_end - first - (int64_t)tile * T * bs;
            const int chunks = (int)min((int64_t)T * cpr, (slots_left + 7) >> 3);
            for (int ch = t; ch < chunks; ch += NT) {
                const int row = (int)__umulhi((uint32_t)ch, g.cpr_magic);
                const int qo = ch - row * cpr;
                const uint32_t ra = a_ranks0 + (uint32_t)g.rk_stride * row + 8u * qo;
                const uint32_t lo = lds_u32(ra), hi = lds_u32(ra + 4);
                uint4 o;
                o.x = __byte_perm(lo, 0, 0x4140);
                o.y = __byte_perm(lo, 0, 0x4342);
                o.z = __byte_perm(hi, 0, 0x4140);
                o.w = __byte_perm(hi, 0, 0x4342);
                if ((int64_t)8 * ch + 8 <= slots_left) {
                    *reinterpret_cast<uint4*>(amap + 8 * (int64_t)ch) = o;
                } else {
                    const uint32_t w4[4] = {o.x, o.y, o.z, o.w};
#pragma unroll 1
                    for (int k = 0; k < 8 && (int64_t)8 * ch + k < slots_left; k++)
                        amap[8 * (int64_t)ch + k] = (uint16_t)(w4[k >> 1] >> (16 * (k & 1)));
                }
            }
        }
        }
        zero_table();
        // release: the barrier orders every thread's writes (and reported errors) before thread 0's
        // cumulative gpu-scope fence, which orders them before the aggregate
        __syncthreads();
        if (t == 0 && has_tile) {
            __threadfence();
            st_relaxed_gpu_u64(c.tile_state + tile, aggregate);
            // ... and into the tile's group: count << 58 | rounds << 34 | claims (the value is the message:
            // a reader that sees count == kRowGroup has the complete sum)
            atomicAdd(c.tile_state + g.n_tiles + 1 + tile / kRowGroup,
                      (1ull << 58) | (((aggregate >> 32) & 0x3FFFFFFFull) << 34) | (aggregate & 0xFFFFFFFFull));
        }
        VR_MARK(5);
        tile = next;
        cur ^= 1;
        parity ^= 1;
    }
}

template <int W>
static int launch_warp_rows(const RunCtx& c, int bs, const RowsGeom& g_in, const ShaderParams& sp, cudaStream_t stream) {
    // Optional: prefetch the vertices of a tile into L2 when it is deduplicated (VR_PREFETCH=1).  Off by
    // default: on the B200 the gathers ~K tiles later are L2 hits or overlap the next tile's dedup
    // anyway, and the extra L2 requests cost more than they save (profiles/README.md).
    const DebugKnobs& knobs = debug_knobs();
    const bool prefetch = sp.kind == VR_SHADER_POSITION && knobs.rows_prefetch == 1;
    auto kernel = prefetch ? warp_rows_kernel<W, true> : warp_rows_kernel<W, false>;
    RowsGeom g = g_in;
    VR_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kRowCtaThreads, g.smem);
    g.n_tiles = (int)ceil_div(c.n_batches, kRowThreads);
    g.n_groups = (int)ceil_div(g.n_tiles, kRowGroup);
    const int resident = sms * (per_sm > 0 ? per_sm : 1);
    // Tickets go round the persistent CTAs, so tile i - resident is the CTA's own previous tile and its
    // predecessors are being published by the other CTAs just now: with K = 1.5 x resident every
    // aggregate the look-back needs is half a round old and nothing waits.  A longer lag only
    // lengthens the shade-only tail (measured: 0.138 / 0.131 / 0.128 / 0.134 ms at 1.0 / 1.25 / 1.5 / 2.0).
    g.lag = knobs.rows_lag > 0 ? knobs.rows_lag : resident + resident / 2;
    if (g.lag > g.n_tiles) g.lag = g.n_tiles;
    if (g.lag < 1) g.lag = 1;
    const int tickets = g.n_tiles + g.lag;  // the last `lag` tickets only shade
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(tickets < resident ? tickets : resident));  // persistent CTAs
    cfg.blockDim = dim3(kRowCtaThreads);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap init_kernel's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = knobs.no_pdl ? 0 : 1;
    VR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, c, bs, g, sp));
    return VR_OK;
}
