// vr_warp_rows.cuh -- warp voting (strategies.py:173-232) for static batches, tile kernel.
// Included by vr_run.cu (uses RunCtx, report_error, validate_batch, finish_stats).
//
// One CTA of 64 threads owns a TILE of 64 consecutive static batches (batching.py:76-84), i.e.
// one contiguous 64 * batch_size * 4-byte piece of the index buffer, and takes it through the
// whole stage:
//
//   A  stage    every thread issues ONE bulk asynchronous copy (cp.async.bulk, the 1-D TMA path,
//               completion on an mbarrier) of its batch's indices into its own shared-memory ROW.
//               The tile is read from HBM as whole 128-byte lines, no register staging.
//   B  dedup    one THREAD per batch runs the closed form of Algorithm 1 over its row (16-byte
//               shared loads, conflict-free because the row stride is an odd multiple of 16 bytes):
//                 * the claimed ids of the current round live in a private open-addressing table
//                   id[slot][thread] (one 32-bit compare per probe) whose occupancy bits are a
//                   REGISTER mask -- a new round clears the table by zeroing that mask;
//                 * claims are appended IN PLACE at the front of the row (a claim never overtakes
//                   the read cursor: claims so far <= slots read + 2 per finished round, and the
//                   row starts with that much slack), so the unique ids never leave the SM
//                   before they are shaded;
//                 * local indices are bytes in a rank row; the <= 2 slots of a round's discarded
//                   tail are re-claimed in closed form from registers (strategies.py:225-231).
//   C  place    local indices leave as coalesced 16-byte stores (8 x uint16); the CTA's
//               (rounds, ids) aggregate enters a decoupled look-back over tiles (ticket order)
//               that yields the tile's output offsets without a second kernel;
//   D  shade    each warp streams the claims of its 32 rows out of shared memory: coalesced id
//               store, 16-byte position gather, FP32 4x4 transform + w-divide
//               (strategies.py:53-67), coalesced 16-byte stores, 8 gathers in flight per lane.
#pragma once
// (included inside namespace vr)

constexpr int kRowThreads = 64;

struct RowsGeom {
    int row_words;   // shared-memory row stride in 32-bit words (odd multiple of 4)
    int slack;       // words in front of the indices that absorb the tail re-claims
    int rk_stride;   // bytes per rank row (an odd number of words)
    int max_rounds;  // upper bound of rounds per batch
    uint32_t cpr_magic;  // ceil(2^32 / (batch_size / 8)): chunk -> row by multiply-high
    size_t smem;
};

// every round but the last consumes at least 3 * floor(W / 3) indices (see SURVEY 7-3 / DESIGN)
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
    g.smem = (size_t)kRowThreads * ((size_t)rw * 4 + (size_t)S * 4 + (size_t)S + (size_t)g.rk_stride + (size_t)g.max_rounds * 4 + 4);
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
// debugging aid: per-tile, per-warp phase time stamps (ns, %globaltimer); vr_debug_timeline() reads them
constexpr int kTimelineMarks = 6, kTimelineTiles = 4096;
__device__ unsigned long long g_timeline[kTimelineMarks * 2 * kTimelineTiles];
__device__ __forceinline__ unsigned long long timeline_now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define VR_MARK_AT(k, value)                                                                   \
    do {                                                                                       \
        if ((threadIdx.x & 31) == 0 && tile < kTimelineTiles)                                  \
            g_timeline[((k) * 2 + (threadIdx.x >> 5)) * kTimelineTiles + tile] = (value);      \
    } while (0)
#define VR_MARK(k) VR_MARK_AT(k, timeline_now())
#else
#define VR_MARK_AT(k, value) do {} while (0)
#define VR_MARK(k) do {} while (0)
#endif

template <int W, bool PREFETCH>
__global__ void __launch_bounds__(kRowThreads) warp_rows_kernel(RunCtx c, int bs, RowsGeom g, ShaderParams sp) {
    constexpr int S = 2 * W;
    constexpr int LOG2W = W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
    constexpr int LOG2S = LOG2W + 1;
    constexpr int T = kRowThreads;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_tile;
    __shared__ int2 s_warp_tot[T / 32];
    __shared__ int2 s_base;
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    const int lane = t & 31, wid = t >> 5;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t row_bytes = 4u * (uint32_t)g.row_words;
    const uint32_t a_row = sbase + row_bytes * t;                          // claims from word 0
    const uint32_t a_ids = a_row + 4u * (uint32_t)g.slack;                 // indices of the batch
    const uint32_t a_idtab = sbase + row_bytes * T + 4u * t;               // + 4*T*slot
    const uint32_t a_rktab = sbase + row_bytes * T + 4u * T * S + t;       // + T*slot
    const uint32_t a_ranks0 = sbase + row_bytes * T + 5u * T * S;          // rank rows
    const uint32_t a_ranks = a_ranks0 + (uint32_t)g.rk_stride * t;
    const uint32_t a_rounds = a_ranks0 + (uint32_t)g.rk_stride * T + 4u * t;  // + 4*T*round
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);

    // static batching (batching.py:76-84): batch b = [first + b * bs, min(.. + bs, last_end)); the two
    // uniform loads overlap the ticket; the caller's claim is verified off the critical path below
#ifdef VR_TIMELINE
    const unsigned long long t_entry = timeline_now();
#endif
    const int first = __ldg(c.bbegin), last_end = __ldg(c.bend + (c.n_batches - 1));
    for (uint32_t o = 16u * t; o < (uint32_t)(S * T); o += 16u * T)  // tag 0 = never used
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(sbase + row_bytes * T + 4u * T * S + o), "r"(0u) : "memory");
    if (t == 0) {
        s_tile = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);  // tiles in ticket order
        mbar_init(bar, T);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tile = s_tile;
#ifdef VR_TIMELINE
    VR_MARK_AT(0, t_entry);
#endif
    VR_MARK(1);
    const int b = tile * T + t;
    bool active = b < c.n_batches;
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

    // ---- B: dedup, one thread per batch, as a per-lane STATE MACHINE: every trip of the loop
    // does one table probe for the lane's current slot p.  A probe that collides moves the lane to
    // the next table slot; one that resolves (hit, or free slot = new claim) stores the local
    // index and moves the lane to slot p + 1; a round end (strategies.py:220-231) records the
    // round and REWINDS the lane to the first unconsumed slot, so the discarded tail is re-claimed
    // by the ordinary path.  Lanes never wait for each other's extra probes or round ends: the
    // loop runs max-over-lanes(slots + collisions + replays) trips, not the sum of per-slot maxima.
    // The trip body is straight-line: side effects are stores whose address is redirected to a
    // per-thread dummy word when the lane does not take them, so the only branches are the loop
    // and the (rare) round end, and the recurrence is probe -> compare -> select -> next hash.
    //   table: id[slot][thread] (32-bit ids) and rk[slot][thread] (byte: round tag << LOG2W | rank);
    //   a slot is occupied iff its tag is the current round's, so a new round clears nothing.
    constexpr int TAGBITS = 8 - LOG2W;
    constexpr uint32_t kTagMax = (1u << TAGBITS) - 1;
    const uint32_t a_dummy = a_rounds + 4u * T * (uint32_t)g.max_rounds;  // one spare word per thread
    int p = 0, fill = 0, cursor = 0, stop = n, rounds = 0;
    uint32_t cl = a_row;  // next claim slot of the row
    uint32_t tagw = 1u << LOG2W;
    uint32_t x = lds_u32(a_ids);
    uint32_t h = (x * 0x9E3779B1u) >> (32 - LOG2S);
    while (__any_sync(0xffffffffu, p < n)) {
        const bool live = p < n;
        const uint32_t cand = lds_u32(a_ids + 4u * (uint32_t)p + 4);  // the next slot, in flight with the probe
        const uint32_t ai = a_idtab + 4u * T * h, ar = a_rktab + (uint32_t)T * h;
        const uint32_t idv = lds_u32(ai);
        const uint32_t tq = lds_u8(ar) ^ tagw;       // == rank (< W) iff the slot belongs to this round
        const bool occb = tq < (uint32_t)W;
        const bool coll = occb && idv != x;
        // round end before slot p: the fetch that filled the warp is exhausted (p >= stop), or x is
        // the first id that cannot be assigned (free slot reached with all W lanes claimed)
        const bool ends = live && (p >= stop || (!occb && fill == W));
        const bool adv = live && !coll && !ends;
        const bool clm = adv && !occb;  // strategies.py:207-212: new id -> lowest free lane
        const uint32_t r = occb ? tq : (uint32_t)fill;
        sts_u32(clm ? ai : a_dummy, x);
        sts_u8(clm ? ar : a_dummy, tagw | r);
        sts_u32(clm ? cl : a_dummy, x);
        sts_u8(adv ? a_ranks + (uint32_t)p : a_dummy, r);
        if (PREFETCH && clm) prefetch_l2(sp.pos4 + x);
        cl += clm ? 4u : 0u;
        fill += clm ? 1 : 0;
        if (clm && fill == W) stop = min(n, cursor + (((p - cursor) >> LOG2W) + 1) * W);  // end of this fetch
        p += adv ? 1 : 0;
        x = adv ? cand : x;
        h = (coll && !ends) ? ((h + 1) & (S - 1)) : ((x * 0x9E3779B1u) >> (32 - LOG2S));
        if (ends) {
            const int d = p - cursor;
            const int emitted = (int)(((uint32_t)d * 43691u) >> 17);  // d / 3 for d < 2^16
            sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)emitted << 8) | (uint32_t)fill);
            rounds++;
            fill = 0;
            cursor += 3 * emitted;
            stop = n;
            p = cursor;  // re-open at the first unconsumed slot (the row still holds it: see slack)
            x = lds_u32(a_ids + 4u * (uint32_t)p);
            h = (x * 0x9E3779B1u) >> (32 - LOG2S);
            if ((tagw >> LOG2W) == kTagMax) {  // tag space exhausted: wipe this thread's column
                for (int k = 0; k < S; k++) sts_u8(a_rktab + (uint32_t)T * k, 0u);
                tagw = 0;
            }
            tagw += 1u << LOG2W;
        }
    }
    VR_MARK(3);
    if (active && (claimed_begin != begin || claimed_end != begin + n)) {
        report_error(c, b, VR_ERR_BAD_BATCH);  // not the static batching this path was promised
        active = false;
    }
    if (active) {  // the batch end closes the last round; nothing is discarded
        sts_u32(a_rounds + 4u * T * rounds, ((uint32_t)((n - cursor) / 3) << 8) | (uint32_t)fill);
        rounds++;
    }
    const int inv = (int)((cl - a_row) >> 2);
    const int my_r = active ? rounds : 0, my_u = active ? inv : 0;
    const int inc_r = warp_incl_scan(my_r, lane), inc_u = warp_incl_scan(my_u, lane);
    if (lane == 31) s_warp_tot[wid] = make_int2(inc_r, inc_u);
    __syncthreads();

    // ---- C: output offsets by decoupled look-back (warp 0), local indices meanwhile (warp 1..)
    if (wid == 0) {
        int ar = 0, au = 0;
#pragma unroll
        for (int w = 0; w < T / 32; w++) { ar += s_warp_tot[w].x; au += s_warp_tot[w].y; }
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
    }
    // local indices: chunk = 8 slots of one row -> one 16-byte store; consecutive threads write
    // consecutive chunks of the tile's contiguous piece of the assembly map
    if (c.out.d_assembly_map) {
        const int cpr = bs >> 3;
        uint16_t* __restrict__ amap = c.out.d_assembly_map + (int64_t)tile * T * bs;
        const int64_t slots_left = (int64_t)c.bend[c.n_batches - 1] - c.bbegin[0] - (int64_t)tile * T * bs;
        const int chunks = (int)min((int64_t)T * cpr, (slots_left + 7) >> 3);
        for (int ch = t; ch < chunks; ch += T) {
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
    __syncthreads();
    VR_MARK(4);
    int2 off = s_base;
    if (off.x < 0) return;  // offsets unknown or outputs too small: leave them untouched
    for (int w = 0; w < wid; w++) { off.x += s_warp_tot[w].x; off.y += s_warp_tot[w].y; }

    // ---- D: round tables, then unique ids + shading for the 32 rows of this warp
    const int ex = inc_u - my_u;
    if (active) {
        const int r0 = off.x + inc_r - my_r;
        int run = off.y + ex;
        if (c.out.d_batch_round_off) c.out.d_batch_round_off[b] = r0;
        for (int q = 0; q < my_r; q++) {
            const uint32_t wv = lds_u32(a_rounds + 4u * T * q);
            if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0 + q] = run;
            if (c.out.d_round_prims) c.out.d_round_prims[r0 + q] = (int)(wv >> 8);
            run += (int)(wv & 0xFFu);
        }
    }
    const int tot = __shfl_sync(0xffffffffu, inc_u, 31);
    const bool want_uid = c.out.d_unique_ids != nullptr;
    const bool want_pos = sp.kind == VR_SHADER_POSITION;
    const bool want_attr = sp.attr_words && c.out.d_shaded_attr;
    const bool want_cnt = c.out.d_shade_counts != nullptr;
    uint32_t* __restrict__ out_uid = c.out.d_unique_ids + off.y;
    float4* __restrict__ shaded = reinterpret_cast<float4*>(c.out.d_shaded4) + off.y;
    const uint32_t lt = (1u << lane) - 1;
    int first_owner = 0;
    constexpr int U8 = 8;
    for (int j0 = 0; j0 < tot; j0 += 32 * U8) {
        uint32_t uid[U8];
        float4 pv[U8];
#pragma unroll
        for (int u = 0; u < U8; u++) {
            // owner row of output j: one warp-wide OR marks the last output of every row that ends
            // inside this 32-window; owner = first owner of the window + row ends before the lane
            const int jb = j0 + 32 * u;
            const int d = inc_u - jb - 1;
            const uint32_t ends = __reduce_or_sync(0xffffffffu, (my_u > 0 && d >= 0 && d < 32) ? (1u << d) : 0u);
            const int owner = (first_owner + __popc(ends & lt)) & 31;
            first_owner += __popc(ends);
            const int oex = __shfl_sync(0xffffffffu, ex, owner);
            const int j = jb + lane;
            uid[u] = j < tot ? lds_u32(sbase + row_bytes * (uint32_t)(32 * wid + owner) + 4u * (uint32_t)(j - oex)) : 0u;
        }
        if (want_pos) {
#pragma unroll
            for (int u = 0; u < U8; u++)
                if (j0 + 32 * u + lane < tot) pv[u] = __ldg(sp.pos4 + uid[u]);
        }
#pragma unroll
        for (int u = 0; u < U8; u++) {
            const int j = j0 + 32 * u + lane;
            if (j >= tot) continue;
            if (want_uid) out_uid[j] = uid[u];
            if (want_pos) shaded[j] = transform_position(sp, pv[u]);
            if (want_attr)
                for (int q = 0; q < sp.attr_words; q++)
                    c.out.d_shaded_attr[((int64_t)off.y + j) * sp.attr_words + q] = __ldg(sp.attr + (int64_t)uid[u] * sp.attr_words + q);
            if (want_cnt) atomicAdd(&c.out.d_shade_counts[uid[u]], 1);
        }
    }
    VR_MARK(5);
}

template <int W>
static int launch_warp_rows(const RunCtx& c, int bs, const RowsGeom& g, const ShaderParams& sp, cudaStream_t stream) {
    const int blocks = (int)ceil_div(c.n_batches, kRowThreads);
    if (sp.kind == VR_SHADER_POSITION) {  // claims prefetch their vertex into L2 for the shading phase
        VR_CUDA_CHECK(cudaFuncSetAttribute(warp_rows_kernel<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
        warp_rows_kernel<W, true><<<blocks, kRowThreads, g.smem, stream>>>(c, bs, g, sp);
    } else {
        VR_CUDA_CHECK(cudaFuncSetAttribute(warp_rows_kernel<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
        warp_rows_kernel<W, false><<<blocks, kRowThreads, g.smem, stream>>>(c, bs, g, sp);
    }
    return VR_OK;
}

