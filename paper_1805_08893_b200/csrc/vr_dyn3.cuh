// vr_dyn3.cuh -- sort / hash / phash dedup for budgeted (dynamic) batches in three kernels.
// Included by vr_run.cu inside namespace vr (uses RunCtx, report_error, finish_stats, shade_stream).
//
// The paper's dynamic batches hold <= max_unique (256) distinct ids in <= max_indices (1023) slots.
// The three strategies differ only in WHERE a distinct id ends up in the round's unique list:
//   sort   strategies.py:235-260   ascending by id
//   hash   strategies.py:263-298   table order of linear probing, ids inserted in batch order
//   phash  strategies.py:301-367   table order of the two-tier insertion (groups of warp_width)
// so the work is split by what parallelises how:
//   A  one WARP per batch: the batch's distinct ids by insertion into a private open-addressing set
//      (shared memory, CAS), numbered d = 0.. -- in first-occurrence order for hash/phash, which is the
//      reference's insertion order.  Leaves d of every element in the assembly map (rewritten by C), the
//      distinct ids and (hash/phash) their home slots in the workspace, (rounds, uniques) per batch, the batch's
//      output offset inside its 32-batch tile and the tile's totals; the last tile to finish scans the totals.
//   B  hash/phash only, one THREAD per batch: the reference's sequential table construction replayed
//      on the DISTINCT ids only.  Duplicates never change the table, and "probe until the slot is free"
//      is a find-next-zero on an occupancy bitmap, so a batch costs <= 256 short steps; all batches of
//      the run are resident at once.  For phash the fast pass is "first free slot within max_fast_probes
//      of the home slot, else deferred to the end of the element's group, then first free slot from
//      home + max_fast_probes" -- the w-slot windows of strategies.py:345-363 only matter for the
//      statistics, which follow in closed form from the final distance (kernel C).
//   C  one warp per batch: position of every distinct id in the unique list (bitonic sort of
//      id << 8 | d in registers / rank of its table slot), local indices = position of the element's d,
//      ProbeStats from the circular distance home -> slot, round tables, and the vertex shader straight
//      from the list in shared memory (no staging of unique ids in global memory).
// Limits of this path (vr_run falls back to the general kernels otherwise): <= 256 distinct ids per
// batch and table_size <= 256 (d, slots and ranks are bytes), ids < 2^24 for sort (packed sort key).
#pragma once

constexpr int kDyn3Warps = 8;          // warps per CTA of kernels A and C
constexpr int kDyn3Tile = 32;          // most batches per CTA of kernel A (a TILE: one entry of the first level of offset sums); Dyn3Geom.tile_shift
constexpr int kDyn3InsertThreads = 128;  // batches per CTA of kernel B (hash); phash keeps more per batch: half of that

struct Dyn3Geom {
    int q;               // slots of the private set (power of two)
    int u_bound;         // distinct ids a batch may hold before it fails
    int over_status;     // status reported when u_bound is exceeded
    int per_warp_bytes;  // shared memory per warp of kernel A
    int w, mfp;          // phash: group width, fast probes
    int strategy;
    int slot_ids;        // distinct ids a batch's scratch slot holds (dyn3_slot_ids: a multiple of 16, <= 256)
    int tile_shift;      // log2 of the batches per tile: 5, or 4 / 3 for short runs (more CTAs than 1 per 32 batches)
    int prefetch;        // kernel C: L2 prefetch of the distinct vertices before they are put in order
    unsigned char* aux;  // hash/phash: per batch occupancy bitmap[32 B] | home[span'] | slot[span'] | grp u16[span']
    float* queue;        // vr_outputs.d_stream_xyz (kernel C with QUEUE)
    const int64_t* nb_dev;  // vr_run_counted: device int64[2] = {batch count, vr_status} of vr_dynamic_batches, or NULL
};

// vr_run_counted: the batch count lives on the device (the output of vr_dynamic_batches, no host round trip); the
// launch was sized for an upper bound.  A failed batch formation leaves no batches.
__device__ __forceinline__ int dyn3_batch_count(const RunCtx& c, const Dyn3Geom& g) {
    if (!g.nb_dev) return c.n_batches;
    if (__ldg(g.nb_dev + 1) != 0) return 0;
    const long long n = __ldg(g.nb_dev);
    return (int)(n < 0 ? 0 : n > c.n_batches ? c.n_batches : n);
}

// Scratch of a batch at a FIXED stride by batch number (not by its place in the index buffer): kernel C issues the loads
// of the distinct ids / slots together with the batch's header instead of behind it (one dependent round trip less in
// a warp's life).  slot_ids = U distinct ids per batch (the configuration's largest span, at most 256, rounded up to 16):
//   distinct ids   stage_uid + b * U                      (32-bit words)
//   aux            aux + b * (32 + 4 U):  occupancy bitmap[32 B] | home[U] | slot[U] | grp u16[U]
static inline int dyn3_slot_ids(const vr_batch_config* cfg) {
    int m = cfg->max_indices > cfg->batch_size ? cfg->max_indices : cfg->batch_size;
    if (m > 256) m = 256;
    if (m < 16) m = 16;
    return (m + 15) & ~15;
}
static inline size_t dyn3_dist_words(int64_t nb, const vr_batch_config* cfg) { return (size_t)nb * dyn3_slot_ids(cfg) + 256; }  // (+ the read-ahead of C's 8-per-lane load)
static inline size_t dyn3_aux_bytes(int64_t nb, const vr_batch_config* cfg) { return (size_t)nb * (32 + 4 * (size_t)dyn3_slot_ids(cfg)) + 1024; }
constexpr int kDyn3AuxHome = 32;  // byte offset of home[] behind the bitmap
__device__ __forceinline__ int64_t dyn3_dist_base(const Dyn3Geom& g, int b) { return (int64_t)b * g.slot_ids; }
__device__ __forceinline__ int64_t dyn3_aux_base(const Dyn3Geom& g, int b) { return (int64_t)b * (kDyn3AuxHome + 4 * g.slot_ids); }

// Output offsets without a scan pass and without any tile waiting for another: kernel A leaves, per batch, the
// (rounds, ids) of the batches before it in its TILE (32 batches), per tile its totals, and adds the tile's totals to
// its GROUP (32 tiles) and its SUPERGROUP (32 groups = 32768 batches).  Kernel C adds up, per batch, the supergroups
// before its own, the groups of its supergroup before its own, the tiles of its group before its own (one word per
// lane each) and the batch's offset in its tile.  Words are rounds << 32 | ids; ids sum to <= the index count < 2^31
// and rounds to <= the batch count < 2^30, so the halves never carry.
constexpr int kDyn3Group = 32;
struct Dyn3Levels {
    unsigned long long* tiles;   // [n_tiles]
    unsigned long long* groups;  // [n_groups]
    unsigned long long* supers;  // [n_supers]
    int n_supers;
};
__host__ __device__ __forceinline__ int dyn3_state_words(int n_tiles) {
    const int n_groups = (n_tiles + kDyn3Group - 1) / kDyn3Group;
    return n_tiles + 1 + n_groups + 1 + (n_groups + kDyn3Group - 1) / kDyn3Group + 1;
}
__device__ __forceinline__ Dyn3Levels dyn3_levels(const RunCtx& c) {
    const int n_tiles = c.n_fused_tiles, n_groups = (n_tiles + kDyn3Group - 1) / kDyn3Group;
    Dyn3Levels l;
    l.tiles = c.tile_state;
    l.groups = l.tiles + n_tiles + 1;
    l.supers = l.groups + n_groups + 1;
    l.n_supers = (n_groups + kDyn3Group - 1) / kDyn3Group;
    return l;
}
__device__ __forceinline__ int2 dyn3_offsets(const RunCtx& c, int tile_shift, int b, int lane) {
    const Dyn3Levels l = dyn3_levels(c);
    const int tile = b >> tile_shift, grp = tile / kDyn3Group, sup = grp / kDyn3Group;
    unsigned long long w = lane < tile % kDyn3Group ? __ldcg(l.tiles + grp * kDyn3Group + lane) : 0ull;
    w += lane < grp % kDyn3Group ? __ldcg(l.groups + sup * kDyn3Group + lane) : 0ull;
    for (int k = lane; k < sup; k += 32) w += __ldcg(l.supers + k);
    const int2 in_tile = c.seg_off[b];
    return make_int2(in_tile.x + (int)__reduce_add_sync(0xffffffffu, (unsigned)(w >> 32)),
                     in_tile.y + (int)__reduce_add_sync(0xffffffffu, (unsigned)(w & 0xFFFFFFFFull)));
}
// (rounds, ids) of the whole run: one thread, after every tile of kernel A has finished
__device__ __forceinline__ int2 dyn3_totals(const RunCtx& c) {
    const Dyn3Levels l = dyn3_levels(c);
    unsigned long long w = 0;
    for (int k = 0; k < l.n_supers; k++) w += __ldcg(l.supers + k);
    return make_int2((int)(w >> 32), (int)(w & 0xFFFFFFFFull));
}

__device__ __forceinline__ uint32_t atomicCAS_shared(uint32_t saddr, uint32_t cmp, uint32_t val) {
    uint32_t r;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(r) : "r"(saddr), "r"(cmp), "r"(val) : "memory");
    return r;
}

// ---- A ------------------------------------------------------------------------------------------
// WIDE: 64 elements per step, two per lane, their two probe chains interleaved -- for LONG batches (a strip-ordered mesh:
// ~760 indices per batch): the second chain hides the first one's shared-memory atomic latency.  On the short batches of
// a shuffled mesh (~255 indices) the 40+ registers cost more resident warps than that saves (measured), so vr_run picks
// the variant by the average batch length.
template <bool ORDERED, bool PHASH, bool WIDE>
__global__ void __launch_bounds__(kDyn3Warps * 32, WIDE ? 6 : 0) dyn3_dedup_kernel(RunCtx c_in, Dyn3Geom g) {
    RunCtx c = c_in;
    c.n_batches = dyn3_batch_count(c_in, g);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int2 s_cnt[kDyn3Tile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid == 0) s_cnt[lane] = make_int2(0, 0);  // (slots past a short tile stay empty)
    __syncthreads();
    const int tile = (int)blockIdx.x;
    if (g.nb_dev && tile == 0 && threadIdx.x == 0) {  // what the host would have checked before the launch
        const long long fst = __ldg(g.nb_dev + 1), fnb = __ldg(g.nb_dev);
        if (fst != 0) report_error(c, 0, (int)fst);
        else if (fnb > c_in.n_batches) report_error(c, 0, VR_ERR_CAPACITY);
    }
    const bool abort = c.acc[ACC_ABORT] != 0;
    unsigned char* base = smem_raw + (size_t)wid * g.per_warp_bytes;
    uint32_t* kkey = reinterpret_cast<uint32_t*>(base);  // [q] the set
    // ORDERED: [q] smallest position of the id while its first step is open, its number d afterwards (d <= every
    // position of the id, so later atomicMin's leave it alone); else u16 [q] number d of the id
    uint32_t* kpos = kkey + g.q;
    uint16_t* kidx = reinterpret_cast<uint16_t*>(kpos);
    const uint32_t a_keys = (uint32_t)__cvta_generic_to_shared(kkey);
    const uint32_t a_dummy = (uint32_t)__cvta_generic_to_shared(base + g.per_warp_bytes - 128 + 4 * lane);  // one spare word per lane
    const uint32_t qmask = (uint32_t)g.q - 1;
    const int qshift = 32 - ilog2((uint32_t)g.q);
    const uint32_t lt = (1u << lane) - 1;
    const int wshift = PHASH ? ilog2((uint32_t)g.w) : 0;
#pragma unroll 1
    for (int k = 0; k < (1 << g.tile_shift) / kDyn3Warps; k++) {
        const int slot_in_tile = k * kDyn3Warps + wid;
        const int b = (tile << g.tile_shift) + slot_in_tile;
        int rounds = 0, nu = 0;
        int begin, n;
        if (b < c.n_batches && !abort && validate_batch(c, b, begin, n)) {
            const int mo = batch_map_off(c, b, begin);
            const uint32_t* __restrict__ ids = c.idx + begin;
            uint16_t* __restrict__ dmap = c.out.d_assembly_map + mo;
            uint32_t* __restrict__ dist = c.stage_uid + dyn3_dist_base(g, b);
            asm volatile("" : "+l"(dist));  // (opaque: ptxas otherwise recomputes it from the kernel parameters at every store)
            if (!WIDE) { asm volatile("" : "+l"(ids)); asm volatile("" : "+l"(dmap)); }
            unsigned char* __restrict__ home = nullptr;
            uint16_t* __restrict__ grp = nullptr;
            if (ORDERED) {
                home = g.aux + dyn3_aux_base(g, b) + kDyn3AuxHome;
                grp = reinterpret_cast<uint16_t*>(home + 2 * g.slot_ids);
            }
            uint32_t id_next = lane < n ? __ldg(ids + lane) : 0u;
            __syncwarp();
            for (int i = 4 * lane; i < g.q; i += 128) {
                *reinterpret_cast<uint4*>(kkey + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
                if (ORDERED) *reinterpret_cast<uint4*>(kpos + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            }
            __syncwarp();
            bool overflow = false;
            if (WIDE) {
                uint32_t next_b = lane + 32 < n ? __ldg(ids + lane + 32) : 0u;
                for (int i0 = 0; i0 < n; i0 += 64) {
                    const int ia = i0 + lane, ib = ia + 32;
                    const bool va = ia < n, vb = ib < n;
                    const uint32_t id_a = id_next, id_b = next_b;
                    if (ia + 64 < n) id_next = __ldg(ids + ia + 64);
                    if (ib + 64 < n) next_b = __ldg(ids + ib + 64);
                    uint32_t ha = (id_a * 0x9E3779B1u) >> qshift, hb = (id_b * 0x9E3779B1u) >> qshift;
                    bool first_a = false, first_b = false;
                    bool pa = va, pb = vb;
                    auto probe2 = [&]() {  // (branch-free, see the one-element loop below)
                        uint32_t ra = atomicCAS_shared(pa ? a_keys + 4u * ha : a_dummy, kEmpty, id_a);
                        uint32_t rb = atomicCAS_shared(pb ? a_keys + 4u * hb : a_dummy, kEmpty, id_b);
                        ra = pa ? ra : id_a;
                        rb = pb ? rb : id_b;
                        first_a |= ra == kEmpty;
                        first_b |= rb == kEmpty;
                        pa = ra != kEmpty && ra != id_a;
                        pb = rb != kEmpty && rb != id_b;
                        ha = pa ? (ha + 1) & qmask : ha;
                        hb = pb ? (hb + 1) & qmask : hb;
                    };
                    probe2();
                    while (__any_sync(0xffffffffu, pa || pb)) {
                        probe2();
                        probe2();
                    }
                    if (ORDERED) {
                        if (va) atomicMin(&kpos[ha], (uint32_t)ia);
                        if (vb) atomicMin(&kpos[hb], (uint32_t)ib);
                        __syncwarp();
                        first_a = va && kpos[ha] == (uint32_t)ia;
                        first_b = vb && kpos[hb] == (uint32_t)ib;
                    }
                    const uint32_t ma = __ballot_sync(0xffffffffu, first_a), mb = __ballot_sync(0xffffffffu, first_b);
                    const int da = nu + __popc(ma & lt), db = nu + __popc(ma) + __popc(mb & lt);
                    nu += __popc(ma) + __popc(mb);
                    if (nu > g.u_bound) { overflow = true; break; }  // uniform
                    if (ORDERED) __syncwarp();
                    if (first_a) {
                        if (ORDERED) kpos[ha] = (uint32_t)da; else kidx[ha] = (uint16_t)da;
                        dist[da] = id_a;
                        if (ORDERED) home[da] = (unsigned char)hash_slot(id_a, c.multiplier, c.table_bits);
                        if (PHASH) grp[da] = (uint16_t)(ia >> wshift);
                    }
                    if (first_b) {
                        if (ORDERED) kpos[hb] = (uint32_t)db; else kidx[hb] = (uint16_t)db;
                        dist[db] = id_b;
                        if (ORDERED) home[db] = (unsigned char)hash_slot(id_b, c.multiplier, c.table_bits);
                        if (PHASH) grp[db] = (uint16_t)(ib >> wshift);
                    }
                    __syncwarp();
                    if (va) dmap[ia] = ORDERED ? (uint16_t)kpos[ha] : kidx[ha];
                    if (vb) dmap[ib] = ORDERED ? (uint16_t)kpos[hb] : kidx[hb];
                }
            } else {
                for (int i0 = 0; i0 < n; i0 += 32) {
                    const int i = i0 + lane;
                    const bool valid = i < n;
                    const uint32_t id = id_next;
                    if (i + 32 < n) id_next = __ldg(ids + i + 32);
                    uint32_t h = (id * 0x9E3779B1u) >> qshift;
                    bool first = false;
                    {
                        // up to four probes per trip of a warp-uniform loop, each a PREDICATED atomic (no divergent branch per
                        // probe: at a load of 1/4..1/2 some lane of the warp needs a third probe in most steps, and ncu showed
                        // the warps of this kernel waiting on branches more than on the atomics).  A lane that is done -- or
                        // has no element -- gets its own id back: "found".
                        bool open = valid;
                        auto probe = [&]() {
                            uint32_t prev = atomicCAS_shared(open ? a_keys + 4u * h : a_dummy, kEmpty, id);
                            prev = open ? prev : id;
                            first |= prev == kEmpty;
                            open = prev != kEmpty && prev != id;
                            h = open ? (h + 1) & qmask : h;
                        };
                        probe();  // (a stream with much reuse mostly ends here: the id is in its home slot)
                        while (__any_sync(0xffffffffu, open)) {
                            probe();
                            probe();
                        }
                        if (ORDERED && valid) atomicMin(&kpos[h], (uint32_t)i);
                    }
                    if (ORDERED) {
                        // the reference inserts in batch order: among equal ids of this step the lowest position is the
                        // first occurrence (ids of earlier steps hold their d, which is below every later position)
                        __syncwarp();
                        first = valid && kpos[h] == (uint32_t)i;
                    }
                    const uint32_t m = __ballot_sync(0xffffffffu, first);
                    const int d = nu + __popc(m & lt);
                    nu += __popc(m);
                    if (nu > g.u_bound) { overflow = true; break; }  // uniform
                    // (every lane's read of kpos above feeds the ballot, so it is complete here; the barrier states it)
                    if (ORDERED) __syncwarp();
                    if (first) {
                        if (ORDERED) kpos[h] = (uint32_t)d; else kidx[h] = (uint16_t)d;
                        dist[d] = id;
                        if (ORDERED) home[d] = (unsigned char)hash_slot(id, c.multiplier, c.table_bits);
                        if (PHASH) grp[d] = (uint16_t)(i >> wshift);
                    }
                    __syncwarp();
                    if (valid) dmap[i] = ORDERED ? (uint16_t)kpos[h] : kidx[h];
                }
            }
            rounds = 1;
            if (overflow) {  // strategies.py:451-455 / :283-284
                if (lane == 0) report_error(c, b, g.over_status);
                rounds = 0;
                nu = 0;
            } else if (c.enforce_budget && nu > c.max_unique) {
                if (lane == 0) report_error(c, b, VR_ERR_OVER_BUDGET);
            }
        }
        if (lane == 0) {
            s_cnt[slot_in_tile] = make_int2(rounds, nu);
            if (b < c.n_batches) c.counts[b] = make_int2(rounds, nu);
        }
    }
    __syncthreads();
    // ---- output offsets: see dyn3_offsets.  (A decoupled look-back here kept the CTA's shared memory and warp slots
    // occupied while one warp polled its predecessors: measured ~1/3 of a CTA's residency when the grid runs in waves.)
    if (wid == 0) {
        const int2 v = s_cnt[lane];
        const int ir = warp_incl_scan(v.x, lane), iu = warp_incl_scan(v.y, lane);
        const int bl = (tile << g.tile_shift) + lane;
        if (lane < (1 << g.tile_shift) && bl < c.n_batches) c.seg_off[bl] = make_int2(ir - v.x, iu - v.y);
        if (lane == 31) {
            const Dyn3Levels l = dyn3_levels(c);
            const unsigned long long total = ((unsigned long long)(uint32_t)ir << 32) | (unsigned long long)(uint32_t)iu;
            l.tiles[tile] = total;
            atomicAdd(l.groups + tile / kDyn3Group, total);
            atomicAdd(l.supers + tile / (kDyn3Group * kDyn3Group), total);
        }
    }
}

// ---- B ------------------------------------------------------------------------------------------
// Occupancy bitmap of one batch's table: words [w][thread] in shared memory (bank == lane); which words are
// full is kept in a register, so a probe reads at most two words however full the table is.
template <int NT>
struct Dyn3Bitmap {
    uint32_t* bm;  // + w * NT
    uint32_t all;  // one bit per word
    uint32_t full;
    // first free slot at or after h, circular; `held` = the word that holds it (take does not read it again)
    __device__ __forceinline__ uint32_t next_free(uint32_t h, uint32_t& held) const {
        uint32_t w = h >> 5;
        held = bm[w * NT];
        uint32_t bits = ~held & (0xFFFFFFFFu << (h & 31));
        if (bits == 0) {  // next word with a free slot, circular (w itself again last: its slots below h)
            const uint32_t open = ~full & all;
            const uint32_t above = open & ~((2u << w) - 1u);
            w = (uint32_t)__ffs((int)(above ? above : open)) - 1;
            held = bm[w * NT];
            bits = ~held;
        }
        return (w << 5) + (uint32_t)__ffs((int)bits) - 1;
    }
    __device__ __forceinline__ void take(uint32_t s, uint32_t held) {
        const uint32_t w = s >> 5;
        const uint32_t v = held | (1u << (s & 31));
        bm[w * NT] = v;
        if (v == 0xFFFFFFFFu) full |= 1u << w;
    }
};

template <bool PHASH>
__global__ void __launch_bounds__(PHASH ? kDyn3InsertThreads / 2 : kDyn3InsertThreads) dyn3_insert_kernel(RunCtx c_in, Dyn3Geom g) {
    RunCtx c = c_in;
    c.n_batches = dyn3_batch_count(c_in, g);
    constexpr int NT = PHASH ? kDyn3InsertThreads / 2 : kDyn3InsertThreads;
    __shared__ uint32_t s_bm[8 * NT];
    // phash: deferred ids of the open group (d) and their home slots, [w][NT] each -- dynamic, so that a narrower group
    // width leaves room for more resident batches (w = 32: 10 CTAs/SM instead of 8)
    extern __shared__ unsigned char s_deferred[];
    unsigned char* s_dd = s_deferred;
    unsigned char* s_dh = s_deferred + (PHASH ? g.w * NT : 0);
    __shared__ unsigned char s_slot[PHASH ? 256 * NT : 1];  // slot of every d (written out of order)
    const int t = threadIdx.x;
    const int b = blockIdx.x * NT + t;
    if (b >= c.n_batches) return;
    const int2 cnt = c.counts[b];
    if (cnt.x == 0 || cnt.y == 0) return;
    const int nu = cnt.y;
    const uint32_t tsize = c.table_size, tmask = tsize - 1;
    const int n_words = tsize >= 32 ? (int)(tsize >> 5) : 1;
    Dyn3Bitmap<NT> B{s_bm + t, (1u << n_words) - 1u, 0u};
    for (int w = 0; w < n_words; w++) s_bm[w * NT + t] = tsize >= 32 ? 0u : ~((1u << tsize) - 1u);
    const int begin = __ldg(c.bbegin + b), n = __ldg(c.bend + b) - begin;
    const int mo = batch_map_off(c, b, begin);
    const int stride = g.slot_ids;
    unsigned char* __restrict__ aux = g.aux + dyn3_aux_base(g, b);
    const unsigned char* __restrict__ home = aux + kDyn3AuxHome;
    unsigned char* __restrict__ slot = aux + kDyn3AuxHome + stride;
    const uint16_t* __restrict__ grp = reinterpret_cast<const uint16_t*>(home + 2 * stride);
    if (!PHASH) {
        // strategies.py:277-294 on the distinct ids: next free slot at or after the home slot
        uint4 hv = *reinterpret_cast<const uint4*>(home);
        auto group = [&](int d0, auto whole_tag) {  // 16 ids; a whole group needs no "d < nu" per id
            constexpr bool WHOLE = decltype(whole_tag)::value;
            const uint4 cur = hv;
            if (d0 + 16 < nu) hv = *reinterpret_cast<const uint4*>(home + d0 + 16);
            const uint32_t hw[4] = {cur.x, cur.y, cur.z, cur.w};
            uint32_t ow[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (WHOLE || d0 + k < nu) {
                    const uint32_t h = (hw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                    uint32_t held;
                    const uint32_t s = B.next_free(h, held);
                    B.take(s, held);
                    ow[k >> 2] |= s << (8 * (k & 3));
                }
            }
            *reinterpret_cast<uint4*>(slot + d0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        };
        int d0 = 0;
        for (; d0 + 16 <= nu; d0 += 16) group(d0, std::true_type{});
        if (d0 < nu) group(d0, std::false_type{});
    } else {
        // strategies.py:321-363 on the distinct ids
        const uint32_t mfp = (uint32_t)g.mfp;
        int nd = 0, open_grp = -1;
        auto flush = [&]() {  // :345: the deferred ids one at a time, from where fast probing stopped
            for (int k = 0; k < nd; k++) {
                const uint32_t d = s_dd[k * NT + t], h = s_dh[k * NT + t];
                uint32_t held;
                const uint32_t s = B.next_free((h + mfp) & tmask, held);
                B.take(s, held);
                s_slot[d * NT + t] = (unsigned char)s;
            }
            nd = 0;
        };
        uint4 hv = *reinterpret_cast<const uint4*>(home);
        uint4 g0 = *reinterpret_cast<const uint4*>(grp), g1 = *reinterpret_cast<const uint4*>(grp + 8);
        for (int d0 = 0; d0 < nu; d0 += 16) {
            const uint4 cur = hv, cg0 = g0, cg1 = g1;
            if (d0 + 16 < nu) {
                hv = *reinterpret_cast<const uint4*>(home + d0 + 16);
                g0 = *reinterpret_cast<const uint4*>(grp + d0 + 16);
                g1 = *reinterpret_cast<const uint4*>(grp + d0 + 24);
            }
            const uint32_t hw[4] = {cur.x, cur.y, cur.z, cur.w};
            const uint32_t gw[8] = {cg0.x, cg0.y, cg0.z, cg0.w, cg1.x, cg1.y, cg1.z, cg1.w};
#pragma unroll
            for (int k = 0; k < 16; k++) {
                const int d = d0 + k;
                if (d < nu) {
                    const int gd = (int)((gw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);
                    if (gd != open_grp) { flush(); open_grp = gd; }
                    const uint32_t h = (hw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                    uint32_t held;
                    const uint32_t s = B.next_free(h, held);
                    if (((s - h) & tmask) < mfp) {  // :328-339 resolved by the fast pass
                        B.take(s, held);
                        s_slot[d * NT + t] = (unsigned char)s;
                    } else {
                        s_dd[nd * NT + t] = (unsigned char)d;
                        s_dh[nd * NT + t] = (unsigned char)h;
                        nd++;
                    }
                }
            }
        }
        flush();
        for (int d0 = 0; d0 < nu; d0 += 16) {
            uint32_t ow[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 16; k++) ow[k >> 2] |= (uint32_t)s_slot[(d0 + k) * NT + t] << (8 * (k & 3));
            *reinterpret_cast<uint4*>(slot + d0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
    }
    // the table's occupancy for kernel C (ranks in table order, strategies.py:370-380)
    uint32_t bw[8];
#pragma unroll
    for (int w = 0; w < 8; w++) bw[w] = w < n_words ? s_bm[w * NT + t] : 0u;
    if (tsize < 32) bw[0] &= (1u << tsize) - 1u;
    *reinterpret_cast<uint4*>(aux) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
    *reinterpret_cast<uint4*>(aux + 16) = make_uint4(bw[4], bw[5], bw[6], bw[7]);
}

// ---- C ------------------------------------------------------------------------------------------
// Bitonic sort of 32 * R keys held R per lane, key index = lane * R + r ("blocked": the 3 innermost steps of
// every merge stay inside a thread), every comparator ascending: a merge of size k first pairs i with
// i ^ (k - 1), then i with i ^ j for j = k/4 .. 1, the lower index keeps the smaller key.
template <int R>
__device__ __forceinline__ void warp_bitonic_blocked(uint32_t (&v)[R], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int mask = (j == (k >> 1)) ? k - 1 : j;  // partner = i ^ mask
            const int lmask = mask / R, rmask = mask % R;
            if (lmask == 0) {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    if ((r ^ rmask) > r) {
                        const uint32_t a = v[r], d = v[r ^ rmask];
                        v[r] = min(a, d);
                        v[r ^ rmask] = max(a, d);
                    }
                }
            } else {
                int top = lmask;  // highest set bit of the lane part decides who is the lower index
                top |= top >> 1; top |= top >> 2; top |= top >> 4;
                top = (top + 1) >> 1;
                const bool lower = (lane & top) == 0;
                uint32_t o[R];
#pragma unroll
                for (int r = 0; r < R; r++) o[r] = __shfl_xor_sync(0xffffffffu, v[r ^ rmask], lmask);
#pragma unroll
                for (int r = 0; r < R; r++) v[r] = lower ? min(v[r], o[r]) : max(v[r], o[r]);
            }
        }
    }
}

// QUEUE: also write the stage's output queue (vr_outputs.d_stream_xyz) -- a separate instantiation, so that the
// default kernel's register allocation does not pay for it
template <int STRATEGY, bool QUEUE>
__global__ void __launch_bounds__(kDyn3Warps * 32, 5) dyn3_finish_kernel(RunCtx c_in, ShaderParams sp, Dyn3Geom g) {
    RunCtx c = c_in;
    c.n_batches = dyn3_batch_count(c_in, g);
    __shared__ __align__(16) uint32_t s_list[kDyn3Warps][256];  // the round's unique ids, in output order
    __shared__ __align__(16) uint16_t s_of_d[kDyn3Warps][256];  // per distinct id d: distance home -> slot << 8 | position in the list
    __shared__ uint32_t s_bm[kDyn3Warps][16];                   // hash: occupancy words, their exclusive popcount prefix
    extern __shared__ __align__(16) unsigned char smem_raw[];   // the batch's shaded records [warp][256] when the queue is wanted
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float* __restrict__ queue = QUEUE ? g.queue : nullptr;
    float4* kept = QUEUE ? reinterpret_cast<float4*>(smem_raw) + 256 * wid : nullptr;
    float* qstage = QUEUE ? reinterpret_cast<float*>(smem_raw) + 4 * 256 * kDyn3Warps + 96 * wid : nullptr;  // one row of records
    __shared__ unsigned int s_fast[kDyn3Warps], s_slow[kDyn3Warps], s_cmax[kDyn3Warps];  // the warps' probe statistics
    if (lane == 0) { s_fast[wid] = 0; s_slow[wid] = 0; s_cmax[wid] = 0; }
    const int b = blockIdx.x * kDyn3Warps + wid;
    if (b < c.n_batches && !c.acc[ACC_ABORT]) {
        // the batch's distinct ids in the 8-per-lane layout of a full batch: their slot depends on b alone, so the loads
        // travel with the header's instead of behind them (smaller batches reload in their own layout below)
        const uint4* __restrict__ dist8 = reinterpret_cast<const uint4*>(c.stage_uid + dyn3_dist_base(g, b) + 8 * lane);
        uint4 pre0 = make_uint4(0, 0, 0, 0), pre1 = pre0;
        if (c.max_span > 128) { pre0 = __ldcg(dist8); pre1 = __ldcg(dist8 + 1); }  // (only such batch lists have batches of > 128 ids)
        const int2 cnt = c.counts[b];
        const int2 off = dyn3_offsets(c, g.tile_shift, b, lane);
        const int begin = __ldg(c.bbegin + b), n = __ldg(c.bend + b) - begin;
        const int vbase = sp.batch_base ? __ldg(sp.batch_base + b) : 0;
        if (lane == 0 && c.out.d_batch_round_off) c.out.d_batch_round_off[b] = off.x;
        const int nu = cnt.y;
        const bool fits = (int64_t)off.y + nu <= c.out.cap_unique && (int64_t)off.x + cnt.x <= c.out.cap_rounds;
        if (cnt.x != 0 && fits) {
            const int mo = batch_map_off(c, b, begin);
            uint32_t* list = s_list[wid];
            uint16_t* of_d = s_of_d[wid];
            const uint32_t* __restrict__ dist = c.stage_uid + dyn3_dist_base(g, b);
            const bool want_pos = sp.kind == VR_SHADER_POSITION;
            if (lane == 0) {
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[off.x] = off.y;
                if (c.out.d_round_prims) c.out.d_round_prims[off.x] = n / c.ps;
            }
            // the first 256 elements' numbers d are loaded before the list is put in order (their latency hides there)
            uint16_t* __restrict__ amap = c.out.d_assembly_map + mo;
            constexpr int EA = 8;
            uint32_t early[EA];
#pragma unroll
            for (int k = 0; k < EA; k++) early[k] = lane + 32 * k < n ? (uint32_t)__ldcg(amap + lane + 32 * k) : 0u;
            // R distinct ids per lane, d = lane * R + r (16-byte loads; words past nu stay inside the batch's area)
            auto run = [&](auto rtag) {
                constexpr int R = decltype(rtag)::value;
                uint32_t v[R];
                if (R == 8) {
                    const uint32_t w8[8] = {pre0.x, pre0.y, pre0.z, pre0.w, pre1.x, pre1.y, pre1.z, pre1.w};
#pragma unroll
                    for (int r = 0; r < R; r++) v[r] = lane * R + r < nu ? w8[r % 8] : 0u;
                } else if (R >= 4) {
#pragma unroll
                    for (int r = 0; r < R; r += 4) {
                        uint4 x = make_uint4(0, 0, 0, 0);
                        if (lane * R + r < nu) x = __ldcg(reinterpret_cast<const uint4*>(dist + lane * R + r));
                        v[r] = x.x; v[r + 1 < R ? r + 1 : r] = x.y; v[r + 2 < R ? r + 2 : r] = x.z; v[r + 3 < R ? r + 3 : r] = x.w;
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < R; r++) v[r] = lane * R + r < nu ? __ldcg(dist + lane * R + r) : 0u;
                }
                if (want_pos && g.prefetch) {  // the vertices on their way to L2 while the list is put in order
#pragma unroll
                    for (int r = 0; r < R; r++)
                        if (lane * R + r < nu && vertex_in_range(sp, (uint32_t)vbase + v[r])) prefetch_l2(sp.pos4 + vbase + v[r]);
                }
                if (STRATEGY == VR_SORT) {
                    // ascending ids: sort id << 8 | d; position j holds the j-th smallest id and says which d it was
#pragma unroll
                    for (int r = 0; r < R; r++) v[r] = lane * R + r < nu ? ((v[r] << 8) | (uint32_t)(lane * R + r)) : kEmpty;
                    warp_bitonic_blocked<R>(v, lane);
                    // (the list leaves the registers as 16-byte stores: word stores at a stride of R words would be
                    // R-way bank conflicts; entries past nu are never read)
                    if (R >= 4) {
#pragma unroll
                        for (int r = 0; r < R; r += 4)
                            *reinterpret_cast<uint4*>(list + lane * R + r) =
                                make_uint4(v[r] >> 8, v[r + 1 < R ? r + 1 : r] >> 8, v[r + 2 < R ? r + 2 : r] >> 8, v[r + 3 < R ? r + 3 : r] >> 8);
                    } else {
#pragma unroll
                        for (int r = 0; r < R; r++) list[lane * R + r] = v[r] >> 8;
                    }
#pragma unroll
                    for (int r = 0; r < R; r++)
                        if (lane * R + r < nu) of_d[v[r] & 0xFFu] = (uint16_t)(lane * R + r);
                } else {
                    const int stride = g.slot_ids;
                    const unsigned char* __restrict__ aux = g.aux + dyn3_aux_base(g, b);
                    const unsigned char* __restrict__ home = aux + kDyn3AuxHome;
                    const unsigned char* __restrict__ slot = home + stride;
                    uint32_t* bm = s_bm[wid];
                    {  // occupancy words of the table and their exclusive popcount prefix
                        const uint32_t wv = lane < 8 ? __ldcg(reinterpret_cast<const uint32_t*>(aux) + lane) : 0u;
                        const int inc = warp_incl_scan(__popc(wv), lane);
                        if (lane < 8) { bm[lane] = wv; bm[8 + lane] = (uint32_t)(inc - __popc(wv)); }
                    }
                    uint32_t sl[R], hm[R];
                    if (R == 8) {  // 8 slots / home slots of a lane: one 8-byte load each (rows past nu stay inside the batch's area)
                        const uint2 sv = lane * R < nu ? __ldcg(reinterpret_cast<const uint2*>(slot + lane * R)) : make_uint2(0, 0);
                        const uint2 hv = lane * R < nu ? __ldcg(reinterpret_cast<const uint2*>(home + lane * R)) : make_uint2(0, 0);
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            sl[r] = ((r < 4 ? sv.x : sv.y) >> (8 * (r & 3))) & 0xFFu;
                            hm[r] = ((r < 4 ? hv.x : hv.y) >> (8 * (r & 3))) & 0xFFu;
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            const int d = lane * R + r;
                            sl[r] = d < nu ? (uint32_t)__ldcg(slot + d) : 0u;
                            hm[r] = d < nu ? (uint32_t)__ldcg(home + d) : 0u;
                        }
                    }
                    __syncwarp();
                    const uint32_t tmask = c.table_size - 1;
                    uint32_t e[R];
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        const int d = lane * R + r;
                        e[r] = 0;
                        if (d < nu) {  // strategies.py:370-380: rank of the slot among the occupied ones
                            const uint32_t wi = sl[r] >> 5;
                            const uint32_t j = bm[8 + wi] + (uint32_t)__popc(bm[wi] & ((1u << (sl[r] & 31)) - 1u));
                            list[j] = v[r];
                            e[r] = (((sl[r] - hm[r]) & tmask) << 8) | j;
                        }
                    }
                    if (R == 8) {
                        *reinterpret_cast<uint4*>(of_d + lane * R) =
                            make_uint4(e[0] | (e[1] << 16), e[2 % R] | (e[3 % R] << 16), e[4 % R] | (e[5 % R] << 16), e[6 % R] | (e[7 % R] << 16));
                    } else {
#pragma unroll
                        for (int r = 0; r < R; r++) of_d[lane * R + r] = (uint16_t)e[r];
                    }
                }
            };
            if (nu <= 32) run(std::integral_constant<int, 1>{});
            else if (nu <= 64) run(std::integral_constant<int, 2>{});
            else if (nu <= 128) run(std::integral_constant<int, 4>{});
            else run(std::integral_constant<int, 8>{});
            __syncwarp();
            // local indices (and the probe statistics of every element, duplicates included)
            unsigned int fast = 0, slow = 0, cmax = 0;
            const int wshift = ilog2((uint32_t)g.w);
            // with the output queue (strategies.py:456-463) the records are shaded first and kept in shared memory:
            // a corner's record is then one more shared-memory read next to its local index
            if (QUEUE) {
                shade_stream<VR_SORT>(c, sp, list, nu, off.y, lane, 32, mo, vbase, b, kept);
                __syncwarp();
            }
            auto element = [&](int i, uint32_t dnum) {
                const uint32_t e = of_d[dnum & 0xFFu];
                amap[i] = (uint16_t)(e & 0xFFu);
                if (QUEUE) {  // the corner's record, on its way out through the warp's staging row (see queue_row)
                    const float4 rec = kept[e & 0xFFu];
                    qstage[3 * lane + 0] = rec.x; qstage[3 * lane + 1] = rec.y; qstage[3 * lane + 2] = rec.z;
                }
                if (STRATEGY != VR_SORT) {
                    const uint32_t dd = e >> 8;  // chain - 1 (strategies.py:277-297)
                    if (STRATEGY == VR_HASH || dd < (uint32_t)g.mfp) {
                        fast += dd + 1;
                    } else {  // :341-363: max_fast_probes fast probes, then w-slot windows up to the one that holds the slot
                        fast += (uint32_t)g.mfp;
                        slow += (((dd - (uint32_t)g.mfp) >> wshift) + 1u) << wshift;
                    }
                    cmax = max(cmax, dd + 1);
                }
            };
            // The 32 records of a step are 96 consecutive floats of the queue: written as three fully coalesced 4-byte
            // stores per lane (word l, l + 32, l + 64 of the row) after a transposition through shared memory -- a
            // lane storing its own 12-byte record would touch 12 sectors per instruction instead of 4.
            auto queue_row = [&](int i0) {
                __syncwarp();
                const int words = 3 * min(32, n - i0);
                float* q = queue + 3 * ((int64_t)mo + i0);
#pragma unroll
                for (int k = 0; k < 3; k++)
                    if (lane + 32 * k < words) q[lane + 32 * k] = qstage[lane + 32 * k];
                __syncwarp();
            };
#pragma unroll
            for (int k = 0; k < EA; k++) {
                if (lane + 32 * k < n) element(lane + 32 * k, early[k]);
                if (QUEUE && 32 * k < n) queue_row(32 * k);
            }
            // longer batches: EA steps' numbers in flight together (a load per step would be a dependent L2 round trip per
            // step: the stores to the same array keep the compiler from hoisting it)
            for (int c0 = 32 * EA; c0 < n; c0 += 32 * EA) {
#pragma unroll
                for (int k = 0; k < EA; k++) early[k] = c0 + lane + 32 * k < n ? (uint32_t)__ldcg(amap + c0 + lane + 32 * k) : 0u;
#pragma unroll
                for (int k = 0; k < EA; k++) {
                    if (c0 + 32 * k >= n) break;  // uniform
                    if (c0 + lane + 32 * k < n) element(c0 + lane + 32 * k, early[k]);
                    if (QUEUE) queue_row(c0 + 32 * k);
                }
            }
            if (STRATEGY != VR_SORT) {
                fast = __reduce_add_sync(0xffffffffu, fast);
                slow = __reduce_add_sync(0xffffffffu, slow);
                cmax = __reduce_max_sync(0xffffffffu, cmax);
                if (lane == 0) {  // (added up per CTA below: an atomic per batch on the same three addresses serialises in L2)
                    s_fast[wid] = fast;
                    s_slow[wid] = slow;
                    s_cmax[wid] = cmax;
                }
            }
            if (!QUEUE) shade_stream<VR_SORT>(c, sp, list, nu, off.y, lane, 32, mo, vbase, b);
        }
    }
    // the last CTA to finish writes the statistics block (every CTA's probe counts are in by then)
    __syncthreads();
    if (threadIdx.x == 0) {
        if (STRATEGY != VR_SORT) {
            unsigned long long fast = 0, slow = 0;
            unsigned int cmax = 0;
            for (int k = 0; k < kDyn3Warps; k++) {
                fast += s_fast[k];
                slow += s_slow[k];
                cmax = max(cmax, s_cmax[k]);
            }
            if (fast) atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_FAST], fast);
            if (slow) atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_SLOW], slow);
            if (cmax) atomicMax(&c.acc[ACC_MAX_CHAIN], (long long)cmax);
        }
        __threadfence();
        const unsigned long long done = atomicAdd((unsigned long long*)&c.acc[ACC_DONE], 1ull);
        if (done == (unsigned long long)gridDim.x - 1) {
            __threadfence();
            const int2 tot = dyn3_totals(c);
            finish_stats(c, tot.x, tot.y);
        }
    }
}

struct Dyn3Plan { bool ok; Dyn3Geom g; size_t smem_a; };

// Whether the three-kernel path takes this run, and its geometry.
static Dyn3Plan dyn3_plan(int strategy, const vr_batch_config* cfg, const vr_hash_config& hc, int max_span, bool enforce_budget,
                          const vr_shader* shader, const vr_outputs* out) {
    Dyn3Plan p{};
    if (strategy != VR_SORT && strategy != VR_HASH && strategy != VR_PHASH) return p;
    if (!out->d_assembly_map || max_span > 65535) return p;
    Dyn3Geom& g = p.g;
    g.strategy = strategy;
    g.w = cfg->warp_width;
    g.mfp = (int)hc.max_fast_probes;
    if (strategy == VR_SORT) {
        g.u_bound = enforce_budget && cfg->max_unique < max_span ? cfg->max_unique : max_span;
        g.over_status = VR_ERR_OVER_BUDGET;
        if (!shader || shader->vertex_count <= 0 || shader->vertex_count > (1 << 24)) return p;  // packed sort key
    } else {
        g.u_bound = (uint32_t)max_span < hc.table_size ? max_span : (int)hc.table_size;
        g.over_status = VR_ERR_HASH_FULL;
        if (hc.table_size > 256) return p;
        if (strategy == VR_PHASH && (max_span >> ilog2((uint32_t)cfg->warp_width)) > 65535) return p;
    }
    if (g.u_bound > 256) return p;
    g.q = (int)next_pow2((uint32_t)((g.u_bound + 64) * 3 / 2 + 2));  // the set holds <= u_bound + 64 ids: load <= 2/3
    if (g.q < 128) g.q = 128;
    g.tile_shift = 5;
    g.slot_ids = dyn3_slot_ids(cfg);
    if (g.u_bound > g.slot_ids) return p;  // (a batch list with longer spans than the configuration's: the general kernels)
    g.per_warp_bytes = g.q * (strategy == VR_SORT ? 4 + 2 : 4 + 4) + 128;  // + one spare word per lane
    p.smem_a = (size_t)kDyn3Warps * g.per_warp_bytes;
    p.ok = true;
    return p;
}
