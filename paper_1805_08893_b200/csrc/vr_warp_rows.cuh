// vr_warp_rows.cuh -- warp voting (strategies.py:173-232) for static batches, tile kernel.
// Included by vr_run.cu inside namespace vr (uses RunCtx, report_error, finish_stats, lds_*/sts_*).
//
// One CTA owns a TILE of 64 consecutive static batches (batching.py:76-84), i.e. one contiguous
// 64 * batch_size * 4-byte piece of the index buffer, and takes it through the whole stage.  The
// CTA has 2 dedup warps (one thread per batch) and 4 helper warps: shared memory, not registers,
// limits the tiles in flight per SM, so the helpers are free parallelism for every phase that is
// not the per-batch dedup chain (look-back, local-index write-out, claim compaction, shading).
//
//   A  stage    every dedup thread issues ONE bulk asynchronous copy (cp.async.bulk, the 1-D TMA
//               path, completion on an mbarrier) of its batch's indices into its own shared-memory
//               ROW.  The tile is read from HBM as whole 128-byte lines, no register staging.
//   B  dedup    one THREAD per batch runs the closed form of Algorithm 1 over its row as a per-lane
//               state machine (see below): claimed ids of the current round live in a private
//               open-addressing table entry[slot][thread]; claims are appended IN PLACE at the
//               front of the row (a claim never overtakes the read cursor: claims so far <= slots
//               read + 2 per finished round, and the row starts with that much slack), so the
//               unique ids never leave the SM before they are shaded; local indices are bytes in
//               a rank row.
//   C  place    the CTA's (rounds, ids) aggregate enters a decoupled look-back over tiles (ticket
//               order) run by one helper warp, while the other warps write the local indices as
//               coalesced 16-byte stores (8 x uint16) and compact the rows' claims into one flat
//               list (in the table's shared memory, which is dead by then);
//   D  shade    all 6 warps stream the flat list: coalesced id store, 16-byte position gather
//               (prefetched into L2 when the id was claimed), FP32 4x4 transform + w-divide
//               (strategies.py:53-67), coalesced 16-byte stores, 4 gathers in flight per thread.
#pragma once

constexpr int kRowThreads = 64;      // batches per tile = dedup threads
constexpr int kRowCtaThreads = 192;  // + 4 helper warps

struct RowsGeom {
    int row_words;   // shared-memory row stride in 32-bit words (odd multiple of 4)
    int slack;       // words in front of the indices that absorb the tail re-claims
    int rk_stride;   // bytes per rank row (an odd number of words)
    int max_rounds;  // upper bound of rounds per batch
    uint32_t cpr_magic;  // ceil(2^32 / (batch_size / 8)): chunk -> row by multiply-high
    size_t smem;
};

// every round but the last consumes at least 3 * floor(W / 3) indices (SURVEY 7-3 / DESIGN 4)
static inline bool rows_geometry(int W, int bs, RowsGeom& g) {
    if (bs % 24 != 0 || bs > 384) return false;  // whole 16-byte quads, whole 8-slot chunks
    const int per_round = 3 * (W / 3);
    g.max_rounds = (bs + per_round - 1) / per_round;
    g.slack = (2 * (g.max_rounds - 1) + 3) & ~3;
    int rw = bs + g.slack;
    while ((rw & 7) != 4) rw += 4;
    g.row_words = rw;
    g.rk_stride = bs + 4;  // odd number of words: same-slot byte stores of a warp are conflict-free
    const int cpr = bs / 8;
    g.cpr_magic = (uint32_t)(((1ull << 32) + cpr - 1) / cpr);  // exact for chunk * cpr < 2^32
    const int S = 2 * W;
    if (bs + 2 * g.max_rounds > S * kRowThreads) return false;  // one row's claims fit the flat list
    g.smem = (size_t)kRowThreads * ((size_t)rw * 4 + (size_t)S * 4 + (size_t)g.rk_stride + (size_t)g.max_rounds * 4 + 4);
    return g.smem <= 100 * 1024;
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

#ifdef VR_TIMELINE
// debugging aid: per-tile phase time stamps (ns, %globaltimer) of dedup warps 0/1; vr_debug_timeline() reads them
constexpr int kTimelineMarks = 6, kTimelineTiles = 4096;
__device__ unsigned long long g_timeline[kTimelineMarks * 2 * kTimelineTiles];
__device__ __forceinline__ unsigned long long timeline_now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define VR_MARK_AT(k, value)                                                                   \
    do {                                                                                       \
        if ((t & 31) == 0 && t < 64 && tile < kTimelineTiles)                                  \
            g_timeline[((k) * 2 + (t >> 5)) * kTimelineTiles + tile] = (value);                \
    } while (0)
#define VR_MARK(k) VR_MARK_AT(k, timeline_now())
#else
#define VR_MARK_AT(k, value) do {} while (0)
#define VR_MARK(k) do {} while (0)
#endif

template <int W, bool PREFETCH>
__global__ void __launch_bounds__(kRowCtaThreads, 4) warp_rows_kernel(RunCtx c, int bs, RowsGeom g, ShaderParams sp) {
    constexpr int S = 2 * W;
    constexpr int LOG2W = W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
    constexpr int LOG2S = LOG2W + 1;
    constexpr int T = kRowThreads, NT = kRowCtaThreads;
    constexpr int kLookbackWarp = T / 32;  // first helper warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_tile;
    __shared__ int2 s_warp_tot[T / 32];  // (rounds, claims) of each dedup warp
    __shared__ int2 s_base;              // output offsets of the tile (look-back result)
    __shared__ int s_cnt[T], s_ex[T + 1];  // claims of each row, exclusive prefix over the tile
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t row_bytes = 4u * (uint32_t)g.row_words;
    const uint32_t a_tab0 = sbase + row_bytes * T;                         // table, later the flat claim list
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
#ifdef VR_TIMELINE
    const unsigned long long t_entry = timeline_now();
#endif
    // static batching (batching.py:76-84): batch b = [first + b * bs, min(.. + bs, last_end)); the two
    // uniform loads overlap the ticket; the caller's claim is verified off the critical path below
    const int first = __ldg(c.bbegin), last_end = __ldg(c.bend + (c.n_batches - 1));
    for (uint32_t o = 16u * threadIdx.x; o < (uint32_t)(4 * S * T); o += 16u * NT)  // tag 0 = never used
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a_tab0 + o), "r"(0u) : "memory");
    if (threadIdx.x == 0) {
        s_tile = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);  // tiles in ticket order
        mbar_init(bar, T);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tile = s_tile;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    const bool dedup_thread = t < T;
    const uint32_t a_row = sbase + row_bytes * t;                          // claims from word 0
    const uint32_t a_ids = a_row + 4u * (uint32_t)g.slack;                 // indices of the batch
    const uint32_t a_idtab = a_tab0 + 4u * t;                              // + 4*T*slot
    const uint32_t a_ranks0 = a_tab0 + 4u * T * S;                         // rank rows
    const uint32_t a_ranks = a_ranks0 + (uint32_t)g.rk_stride * t;
    const uint32_t a_rounds = a_ranks0 + (uint32_t)g.rk_stride * T + 4u * t;  // + 4*T*round
#ifdef VR_TIMELINE
    VR_MARK_AT(0, t_entry);
#endif
    VR_MARK(1);
    const int b = tile * T + t;
    bool active = false;
    int rt_prefix = 0, rt_rounds = 0;  // this row's rounds: exclusive prefix inside its warp, count

    if (dedup_thread) {
        active = b < c.n_batches;
        const int begin = first + b * bs;
        int n = active ? min(bs, last_end - begin) : 0;
        // memory safety of the staged copy does not depend on the batch arrays
        if (active && (first < 0 || (first & 3) || n <= 0 || (int64_t)begin + n > c.n_idx || n % 3 != 0 || bs > c.max_span)) {
            report_error(c, b, first < 0 || (first & 3) || n <= 0 || (int64_t)begin + n > c.n_idx || n % 3 != 0 ? VR_ERR_BAD_BATCH : VR_ERR_UNSUPPORTED);
            active = false;
            n = 0;
        }
        const int claimed_begin = active ? __ldg(c.bbegin + b) : 0, claimed_end = active ? __ldg(c.bend + b) : 0;

        // ---- A: stage the row
        {
            const uint32_t bytes = (n & 3) == 0 ? 4u * (uint32_t)n : 0u;
            mbar_arrive_expect_tx(bar, bytes);
            if (bytes) {
                bulk_g2s(a_ids, c.idx + begin, bytes, bar);
            } else {
                for (int i = 0; i < n; i++) sts_u32(a_ids + 4 * i, __ldg(c.idx + begin + i));  // short last batch
            }
        }
        mbar_wait(bar, 0);
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
        //   nothing (tag 0 = never used; ids must fit 24 bits, checked below).
        // The trip is software-pipelined by hand: the probe and the next slot's id for trip i+1 are
        // loaded as soon as the lane's next state is known, and the side effects of trip i (claim
        // list, local index, counters, L2 prefetch of the claimed vertex) issue under that latency.
        // Side-effect stores go to a per-thread dummy word when the lane does not take them, so the
        // only branches are the loop and the (rare) round end.
        constexpr uint32_t kTagInc = 1u << LOG2W;
        constexpr uint32_t kTagMask = 0xFFu & ~(uint32_t)(W - 1);
        const uint32_t a_dummy = a_rounds + 4u * T * (uint32_t)g.max_rounds;  // one spare word per thread
        int p = 0, fill = 0, cursor = 0, stop = n, rounds = 0;
        uint32_t cl = a_row;  // next claim slot of the row
        uint32_t tagw = kTagInc;
        uint32_t ax = a_ids;  // address of slot p
        uint32_t x = lds_u32(ax);
        uint32_t bad = n > 0 ? (x >> 24) : 0u;
        uint32_t h = (x * 0x9E3779B1u) >> (32 - LOG2S);
        uint32_t v = lds_u32(a_idtab + 4u * T * h), cand = lds_u32(ax + 4);
        for (;;) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool live = p < n;
                const uint32_t ai = a_idtab + 4u * T * h;
                const uint32_t xk = (x << 8) | tagw;
                const uint32_t tq = v ^ xk;                       // == rank (< W) iff the slot holds x in this round
                const bool hit = tq < (uint32_t)W;
                const bool fre = (tq & kTagMask) != 0;            // slot not used in this round
                // round end before slot p: the fetch that filled the warp is exhausted (p >= stop), or x is
                // the first id that cannot be assigned (free slot reached with all W lanes claimed)
                const bool ends = live & ((p >= stop) | (fre & (fill == W)));
                const bool adv = live & (hit | fre) & !ends;
                const bool clm = adv & fre;  // strategies.py:207-212: new id -> lowest free lane
                sts_u32(clm ? ai : a_dummy, xk | (uint32_t)fill);  // before the next probe is loaded
                const uint32_t xn = adv ? cand : x;
                const uint32_t hx = (xn * 0x9E3779B1u) >> (32 - LOG2S);
                const uint32_t hn = (hit | fre) ? hx : ((h + 1) & (S - 1));
                const int pn = p + (adv ? 1 : 0);
                const uint32_t axn = ax + (adv ? 4u : 0u);
                uint32_t vn = lds_u32(a_idtab + 4u * T * hn), candn = lds_u32(axn + 4);
                const uint32_t r = hit ? tq : (uint32_t)fill;
                sts_u32(clm ? cl : a_dummy, x);
                sts_u8(adv ? a_ranks + (uint32_t)p : a_dummy, r);
                if (PREFETCH && clm) prefetch_l2(sp.pos4 + x);
                cl += clm ? 4u : 0u;
                fill += clm ? 1 : 0;
                if (clm && fill == W) stop = min(n, cursor + (((p - cursor) >> LOG2W) + 1) * W);  // end of this fetch
                if (pn < n) bad |= xn >> 24;
                p = pn; ax = axn; x = xn; h = hn;
                if (ends) {
                    const int d = p - cursor;
                    const int emitted = (int)(((uint32_t)d * 43691u) >> 17);  // d / 3 for d < 2^16
                    sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)emitted << 8) | (uint32_t)fill);
                    rounds++;
                    fill = 0;
                    cursor += 3 * emitted;
                    stop = n;
                    p = cursor;  // re-open at the first unconsumed slot (the row still holds it: see slack)
                    ax = a_ids + 4u * (uint32_t)p;
                    x = lds_u32(ax);
                    h = (x * 0x9E3779B1u) >> (32 - LOG2S);
                    if (tagw == kTagMask) {  // tag space exhausted: wipe this thread's column
                        for (int k = 0; k < S; k++) sts_u32(a_idtab + 4u * T * k, 0u);
                        tagw = 0;
                    }
                    tagw += kTagInc;
                    vn = lds_u32(a_idtab + 4u * T * h);
                    candn = lds_u32(ax + 4);
                }
                v = vn; cand = candn;
            }
            if (!__any_sync(0xffffffffu, p < n)) break;
        }
        VR_MARK(3);
        if (active && bad) {  // an id does not fit the packed table entry
            report_error(c, b, VR_ERR_UNSUPPORTED);
            active = false;
        }
        if (active && (claimed_begin != begin || claimed_end != begin + n)) {
            report_error(c, b, VR_ERR_BAD_BATCH);  // not the static batching this path was promised
            active = false;
        }
        if (active) {  // the batch end closes the last round; nothing is discarded
            sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)((n - cursor) / 3) << 8) | (uint32_t)fill);
            rounds++;
        }
        const int my_r = active ? rounds : 0, my_u = active ? (int)((cl - a_row) >> 2) : 0;
        const int inc_r = warp_incl_scan(my_r, lane), inc_u = warp_incl_scan(my_u, lane);
        if (lane == 31) s_warp_tot[wid] = make_int2(inc_r, inc_u);
        s_cnt[t] = my_u;
        s_ex[t] = inc_u - my_u;  // exclusive inside the warp; made tile-wide after the barrier
        rt_prefix = inc_r - my_r;
        rt_rounds = my_r;
        __syncthreads();  // the tile's dedup is done
        if (wid == 1) s_ex[t] += s_warp_tot[0].y;
        if (t == T - 1) s_ex[T] = s_warp_tot[0].y + s_warp_tot[1].y;
    } else {
        __syncthreads();  // the tile's dedup is done
    }

    if (wid == kLookbackWarp) {
        // ---- C (first helper warp): output offsets by decoupled look-back over tiles
        const int ar = s_warp_tot[0].x + s_warp_tot[1].x, au = s_warp_tot[0].y + s_warp_tot[1].y;
        volatile unsigned long long* state = c.tile_state;
        if (lane == 0) {
            __threadfence();  // errors reported by this tile are visible before its state
            state[tile] = kStateAggregate | ((unsigned long long)(uint32_t)ar << 32) | (uint32_t)au;
        }
        long long er = 0, eu = 0;  // exclusive prefix of this tile
        bool lost = false;
        for (int pz = tile - 1; pz >= 0; pz -= 32) {
            const int idx = pz - lane;
            unsigned long long word = kStateInclusive;  // tiles before the first one: inclusive zero
            int spins = 0;
            for (;;) {
                if (idx >= 0) word = state[idx];
                if (!__any_sync(0xffffffffu, (word >> 62) == 0)) break;
                if (++spins > (1 << 20)) { lost = true; break; }
                __nanosleep(20);
            }
            if (lost) break;
            const uint32_t incl = __ballot_sync(0xffffffffu, (word >> 62) == 2);
            const int upto = incl ? __ffs(incl) - 1 : 31;  // nearest predecessor holding an inclusive prefix
            long long vr = lane <= upto ? (long long)((word >> 32) & 0x3FFFFFFFull) : 0;
            long long vu = lane <= upto ? (long long)(word & 0xFFFFFFFFull) : 0;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                vr += __shfl_xor_sync(0xffffffffu, vr, d);
                vu += __shfl_xor_sync(0xffffffffu, vu, d);
            }
            er += vr;
            eu += vu;
            if (incl) break;
        }
        if (lane == 0) {
            if (lost) report_error(c, (int64_t)tile * T, VR_ERR_CUDA);
            const long long R = er + ar, U = eu + au;
            state[tile] = kStateInclusive | ((unsigned long long)(R & 0x3FFFFFFF) << 32) | (unsigned long long)(U & 0xFFFFFFFFll);
            const bool fits = U <= c.out.cap_unique && R <= c.out.cap_rounds && U <= 0x7fffffffLL && !lost;
            if (!fits) report_error(c, (int64_t)tile * T, VR_ERR_CAPACITY);
            s_base = fits ? make_int2((int)er, (int)eu) : make_int2(-1, -1);
            if (tile == c.n_fused_tiles - 1) { __threadfence(); finish_stats(c, R, U); }
        }
    } else {
        asm volatile("bar.sync 1, %0;" ::"n"(kRowCtaThreads - 32) : "memory");  // s_ex is tile-wide now (5 warps)
    }
    if (wid != kLookbackWarp && c.out.d_assembly_map) {
        // ---- C (other warps): local indices.  chunk = 8 slots of one row -> one 16-byte store;
        // consecutive threads write consecutive chunks of the tile's contiguous piece of the map
        const int pt = t < T ? t : t - 32;
        constexpr int NP = NT - 32;
        const int cpr = bs >> 3;
        uint16_t* __restrict__ amap = c.out.d_assembly_map + (int64_t)tile * T * bs;
        const int64_t slots_left = (int64_t)last_end - first - (int64_t)tile * T * bs;
        const int chunks = (int)min((int64_t)T * cpr, (slots_left + 7) >> 3);
        for (int ch = pt; ch < chunks; ch += NP) {
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
                for (int k = 0; k < 8 && (int64_t)8 * ch + k < slots_left; k++)
                    amap[8 * (int64_t)ch + k] = (uint16_t)(w4[k >> 1] >> (16 * (k & 1)));
            }
        }
    }

    // ---- C/D: compaction of the rows' claims into a flat list, then shading by all warps.  The flat
    // list lives in the table's shared memory (S * T words); tiles whose claims do not fit (every
    // index unique, e.g. a shuffled mesh) are taken in several groups of rows.
    const bool want_uid = c.out.d_unique_ids != nullptr;
    const bool want_pos = sp.kind == VR_SHADER_POSITION;
    const bool want_attr = sp.attr_words && c.out.d_shaded_attr;
    const bool want_cnt = c.out.d_shade_counts != nullptr;
    constexpr int kCap = S * T;
    int2 off = make_int2(0, 0);
    for (int r0 = 0, pass = 0; r0 < T; pass++) {
        if (pass > 0) __syncthreads();  // the flat list of the previous group was consumed
        const int base = s_ex[r0];
        int r1 = r0 + 1;
        if (s_ex[T] - base <= kCap) r1 = T;
        else while (r1 < T && s_ex[r1 + 1] - base <= kCap) r1++;
        // the look-back warp of pass 0 is still busy: the other five warps copy, one row per warp
        if (pass > 0 || wid != kLookbackWarp) {
            const int cw = pass > 0 ? wid : (wid < kLookbackWarp ? wid : wid - 1);
            const int ncw = pass > 0 ? NT / 32 : NT / 32 - 1;
            for (int r = r0 + cw; r < r1; r += ncw) {
                const int cnt = s_cnt[r];
                const uint32_t src = sbase + row_bytes * (uint32_t)r, dst = a_tab0 + 4u * (uint32_t)(s_ex[r] - base);
                for (int k = lane; k < cnt; k += 32) sts_u32(dst + 4u * k, lds_u32(src + 4u * k));
            }
        }
        __syncthreads();
        if (pass == 0) {
            VR_MARK(4);
            off = s_base;
            if (off.x < 0) return;  // offsets unknown or outputs too small: leave the outputs untouched
            if (dedup_thread && active) {  // round tables (strategies.py:114-129, flattened)
                const int r0w = off.x + rt_prefix + (wid == 1 ? s_warp_tot[0].x : 0);
                int run = off.y + s_ex[t];
                if (c.out.d_batch_round_off) c.out.d_batch_round_off[b] = r0w;
                for (int q = 0; q < rt_rounds; q++) {
                    const uint32_t wv = lds_u32(a_rounds + 4u * T * q);
                    if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0w + q] = run;
                    if (c.out.d_round_prims) c.out.d_round_prims[r0w + q] = (int)(wv >> 8);
                    run += (int)(wv & 0xFFu);
                }
            }
        }
        const int tot = s_ex[r1] - base;
        const int64_t o0 = (int64_t)off.y + base;
        uint32_t* __restrict__ out_uid = c.out.d_unique_ids + o0;
        float4* __restrict__ shaded = reinterpret_cast<float4*>(c.out.d_shaded4) + o0;
        constexpr int U4 = 4;
        for (int j0 = t; j0 < tot; j0 += NT * U4) {
            uint32_t uid[U4];
            float4 pv[U4];
#pragma unroll
            for (int u = 0; u < U4; u++) {
                const int j = j0 + NT * u;
                uid[u] = j < tot ? lds_u32(a_tab0 + 4u * (uint32_t)j) : 0u;
            }
            if (want_pos) {
#pragma unroll
                for (int u = 0; u < U4; u++)
                    if (j0 + NT * u < tot) pv[u] = __ldg(sp.pos4 + uid[u]);
            }
#pragma unroll
            for (int u = 0; u < U4; u++) {
                const int j = j0 + NT * u;
                if (j >= tot) continue;
                if (want_uid) out_uid[j] = uid[u];
                if (want_pos) shaded[j] = transform_position(sp, pv[u]);
                if (want_attr)
                    for (int q = 0; q < sp.attr_words; q++)
                        c.out.d_shaded_attr[(o0 + j) * sp.attr_words + q] = __ldg(sp.attr + (int64_t)uid[u] * sp.attr_words + q);
                if (want_cnt) atomicAdd(&c.out.d_shade_counts[uid[u]], 1);
            }
        }
        r0 = r1;
    }
    VR_MARK(5);
}

template <int W>
static int launch_warp_rows(const RunCtx& c, int bs, const RowsGeom& g, const ShaderParams& sp, cudaStream_t stream) {
    const int blocks = (int)ceil_div(c.n_batches, kRowThreads);
    if (sp.kind == VR_SHADER_POSITION) {  // claims prefetch their vertex into L2 for the shading phase
        VR_CUDA_CHECK(cudaFuncSetAttribute(warp_rows_kernel<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
        warp_rows_kernel<W, true><<<blocks, kRowCtaThreads, g.smem, stream>>>(c, bs, g, sp);
    } else {
        VR_CUDA_CHECK(cudaFuncSetAttribute(warp_rows_kernel<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
        warp_rows_kernel<W, false><<<blocks, kRowCtaThreads, g.smem, stream>>>(c, bs, g, sp);
    }
    return VR_OK;
}
