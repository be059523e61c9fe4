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
//      distinct ids and (hash/phash) their home slots in the workspace, (rounds, uniques) per batch; the
//      CTA's tail turns these into output offsets with a decoupled look-back over CTA tiles.
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

constexpr int kDyn3Warps = 8;          // batches per CTA of kernels A and C
constexpr int kDyn3InsertThreads = 128;

struct Dyn3Geom {
    int q;               // slots of the private set (power of two)
    int u_bound;         // distinct ids a batch may hold before it fails
    int over_status;     // status reported when u_bound is exceeded
    int per_warp_bytes;  // shared memory per warp of kernel A
    int w, mfp;          // phash: group width, fast probes
    int strategy;
    unsigned char* aux;  // hash/phash: per batch home[span'] | slot[span'] | grp u16[span']
};

__device__ __forceinline__ int64_t dyn3_aux_base(const RunCtx& c, int b, int mo) { return ((int64_t)mo * 4 + (int64_t)b * 128) & ~15LL; }
__device__ __forceinline__ int dyn3_aux_stride(int span) { return (span + 15) & ~15; }

// ---- A ------------------------------------------------------------------------------------------
template <bool ORDERED, bool PHASH>
__global__ void __launch_bounds__(kDyn3Warps * 32) dyn3_dedup_kernel(RunCtx c, Dyn3Geom g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_tile;
    __shared__ int2 s_cnt[kDyn3Warps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);  // tiles in ticket order
    __syncthreads();
    const int tile = s_tile;
    const int b = tile * kDyn3Warps + wid;
    int rounds = 0, nu = 0;
    if (b < c.n_batches && !c.acc[ACC_ABORT]) {
        unsigned char* base = smem_raw + (size_t)wid * g.per_warp_bytes;
        uint32_t* kkey = reinterpret_cast<uint32_t*>(base);           // [q] the set
        uint32_t* kpos = kkey + g.q;                                  // [q] smallest position of the id (ORDERED)
        uint16_t* kidx = reinterpret_cast<uint16_t*>(ORDERED ? kpos + g.q : kpos);  // [q] number d of the id
        int begin, n;
        if (validate_batch(c, b, begin, n)) {
            const int mo = batch_map_off(c, b, begin);
            const uint32_t qmask = (uint32_t)g.q - 1;
            const int qshift = 32 - ilog2((uint32_t)g.q);
            const uint32_t* __restrict__ ids = c.idx + begin;
            uint16_t* __restrict__ dmap = c.out.d_assembly_map + mo;
            uint32_t* __restrict__ dist = c.stage_uid + stage_uid_base(c, b, mo);
            unsigned char* __restrict__ home = nullptr;
            uint16_t* __restrict__ grp = nullptr;
            if (ORDERED) {
                home = g.aux + dyn3_aux_base(c, b, mo);
                grp = reinterpret_cast<uint16_t*>(home + 2 * dyn3_aux_stride(n));
            }
            for (int i = 4 * lane; i < g.q; i += 128) {
                *reinterpret_cast<uint4*>(kkey + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
                if (ORDERED) *reinterpret_cast<uint4*>(kpos + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            }
            __syncwarp();
            const uint32_t lt = (1u << lane) - 1;
            const int wshift = PHASH ? ilog2((uint32_t)g.w) : 0;
            bool overflow = false;
            uint32_t id_next = lane < n ? __ldg(ids + lane) : 0u;
            for (int i0 = 0; i0 < n; i0 += 32) {
                const int i = i0 + lane;
                const bool valid = i < n;
                const uint32_t id = id_next;
                if (i + 32 < n) id_next = __ldg(ids + i + 32);
                uint32_t h = (id * 0x9E3779B1u) >> qshift;
                bool first = false;
                if (valid) {
                    for (;;) {
                        const uint32_t prev = atomicCAS(&kkey[h], kEmpty, id);
                        if (prev == kEmpty) first = true;
                        if (prev == kEmpty || prev == id) break;
                        h = (h + 1) & qmask;
                    }
                    if (ORDERED) atomicMin(&kpos[h], (uint32_t)i);
                }
                if (ORDERED) {
                    // the reference inserts in batch order: among equal ids of this step the lowest position is the
                    // first occurrence (earlier steps hold smaller positions already)
                    __syncwarp();
                    first = valid && kpos[h] == (uint32_t)i;
                }
                const uint32_t m = __ballot_sync(0xffffffffu, first);
                const int d = nu + __popc(m & lt);
                nu += __popc(m);
                if (nu > g.u_bound) { overflow = true; break; }  // uniform
                if (first) {
                    kidx[h] = (uint16_t)d;
                    dist[d] = id;
                    if (ORDERED) home[d] = (unsigned char)hash_slot(id, c.multiplier, c.table_bits);
                    if (PHASH) grp[d] = (uint16_t)(i >> wshift);
                }
                __syncwarp();
                if (valid) dmap[i] = kidx[h];
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
    }
    if (lane == 0) {
        s_cnt[wid] = make_int2(rounds, nu);
        if (b < c.n_batches) c.counts[b] = make_int2(rounds, nu);
    }
    __syncthreads();
    // ---- output offsets: decoupled look-back over tiles (every predecessor holds an earlier ticket, so it is
    // resident or finished)
    if (wid == 0) {
        const int2 v = lane < kDyn3Warps ? s_cnt[lane] : make_int2(0, 0);
        const int ir = warp_incl_scan(v.x, lane), iu = warp_incl_scan(v.y, lane);
        const long long ar = __shfl_sync(0xffffffffu, ir, 31), au = __shfl_sync(0xffffffffu, iu, 31);
        unsigned long long* __restrict__ state = c.tile_state;
        if (lane == 0)
            st_relaxed_gpu_u64(state + tile, (tile == 0 ? kStateInclusive : kStateAggregate) | ((unsigned long long)ar << 32) | (unsigned long long)au);
        long long er = 0, eu = 0;
        bool lost = false;
        if (tile > 0) {
            for (int pz = tile - 1;; pz -= 32) {
                const int idx = pz - lane;
                unsigned long long word = kStateInclusive;  // before the first tile: inclusive zero
                int spins = 0;
                for (;;) {
                    if (idx >= 0) word = ld_relaxed_gpu_u64(state + idx);
                    if (__all_sync(0xffffffffu, (word >> 62) != 0)) break;
                    if (++spins > (1 << 12)) __nanosleep(100);
                    if (spins > (1 << 22)) { lost = true; break; }
                }
                if (lost) break;
                const uint32_t incl = __ballot_sync(0xffffffffu, (word >> 62) == 2);
                const int upto = incl ? __ffs((int)incl) - 1 : 31;
                if (lane <= upto) {
                    er += (long long)((word >> 32) & 0x3FFFFFFFull);
                    eu += (long long)(word & 0xFFFFFFFFull);
                }
                if (incl) break;
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                er += __shfl_xor_sync(0xffffffffu, er, d);
                eu += __shfl_xor_sync(0xffffffffu, eu, d);
            }
            if (lane == 0) {
                if (lost) report_error(c, (int64_t)tile * kDyn3Warps, VR_ERR_CUDA);
                st_relaxed_gpu_u64(state + tile, kStateInclusive | ((unsigned long long)((er + ar) & 0x3FFFFFFF) << 32) | (unsigned long long)((eu + au) & 0xFFFFFFFFll));
            }
        }
        const int bl = tile * kDyn3Warps + lane;
        if (lane < kDyn3Warps && bl < c.n_batches)
            c.seg_off[bl] = make_int2((int)min(er + ir - v.x, 0x7fffffffLL), (int)min(eu + iu - v.y, 0x7fffffffLL));
        if (lane == 0 && (tile + 1) * kDyn3Warps >= c.n_batches)
            c.seg_off[c.n_batches] = make_int2((int)min(er + ar, 0x7fffffffLL), (int)min(eu + au, 0x7fffffffLL));
    }
}

// ---- B ------------------------------------------------------------------------------------------
// Occupancy bitmap of one batch's table: words [w][thread] in shared memory (bank == lane).
struct Dyn3Bitmap {
    uint32_t* bm;  // + w * kDyn3InsertThreads
    uint32_t wmask;
    __device__ __forceinline__ uint32_t next_free(uint32_t h) const {  // first free slot at or after h, circular
        uint32_t w = h >> 5;
        uint32_t bits = ~bm[w * kDyn3InsertThreads] & (0xFFFFFFFFu << (h & 31));
        while (bits == 0) {
            w = (w + 1) & wmask;
            bits = ~bm[w * kDyn3InsertThreads];
        }
        return (w << 5) + (uint32_t)__ffs((int)bits) - 1;
    }
    __device__ __forceinline__ void take(uint32_t s) { bm[(s >> 5) * kDyn3InsertThreads] |= 1u << (s & 31); }
};

template <bool PHASH>
__global__ void __launch_bounds__(kDyn3InsertThreads) dyn3_insert_kernel(RunCtx c, Dyn3Geom g) {
    __shared__ uint32_t s_bm[8 * kDyn3InsertThreads];
    __shared__ unsigned char s_dd[PHASH ? 64 * kDyn3InsertThreads : 1];  // deferred ids of the open group (d)
    __shared__ unsigned char s_dh[PHASH ? 64 * kDyn3InsertThreads : 1];  //   and their home slots
    const int t = threadIdx.x;
    const int b = blockIdx.x * kDyn3InsertThreads + t;
    if (b >= c.n_batches) return;
    const int2 cnt = c.counts[b];
    if (cnt.x == 0 || cnt.y == 0) return;
    const int nu = cnt.y;
    const uint32_t tsize = c.table_size, tmask = tsize - 1;
    const int n_words = tsize >= 32 ? (int)(tsize >> 5) : 1;
    Dyn3Bitmap B{s_bm + t, (uint32_t)n_words - 1};
    for (int w = 0; w < n_words; w++) s_bm[w * kDyn3InsertThreads + t] = tsize >= 32 ? 0u : ~((1u << tsize) - 1u);
    const int begin = __ldg(c.bbegin + b), n = __ldg(c.bend + b) - begin;
    const int mo = batch_map_off(c, b, begin);
    const int stride = dyn3_aux_stride(n);
    const unsigned char* __restrict__ home = g.aux + dyn3_aux_base(c, b, mo);
    unsigned char* __restrict__ slot = g.aux + dyn3_aux_base(c, b, mo) + stride;
    const uint16_t* __restrict__ grp = reinterpret_cast<const uint16_t*>(home + 2 * stride);
    if (!PHASH) {
        // strategies.py:277-294 on the distinct ids: next free slot at or after the home slot
        uint4 hv = *reinterpret_cast<const uint4*>(home);
        for (int d0 = 0; d0 < nu; d0 += 16) {
            const uint4 cur = hv;
            if (d0 + 16 < nu) hv = *reinterpret_cast<const uint4*>(home + d0 + 16);
            const uint32_t hw[4] = {cur.x, cur.y, cur.z, cur.w};
            uint32_t ow[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (d0 + k < nu) {
                    const uint32_t h = (hw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                    const uint32_t s = B.next_free(h);
                    B.take(s);
                    ow[k >> 2] |= s << (8 * (k & 3));
                }
            }
            *reinterpret_cast<uint4*>(slot + d0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
    } else {
        // strategies.py:321-363 on the distinct ids
        const uint32_t mfp = (uint32_t)g.mfp;
        int nd = 0, open_grp = -1;
        auto flush = [&]() {  // :345: the deferred ids one at a time, from where fast probing stopped
            for (int k = 0; k < nd; k++) {
                const uint32_t d = s_dd[k * kDyn3InsertThreads + t], h = s_dh[k * kDyn3InsertThreads + t];
                const uint32_t s = B.next_free((h + mfp) & tmask);
                B.take(s);
                slot[d] = (unsigned char)s;
            }
            nd = 0;
        };
        for (int d = 0; d < nu; d++) {
            const int gd = grp[d];
            if (gd != open_grp) { flush(); open_grp = gd; }
            const uint32_t h = home[d];
            const uint32_t s = B.next_free(h);
            if (((s - h) & tmask) < mfp) {  // :328-339 resolved by the fast pass
                B.take(s);
                slot[d] = (unsigned char)s;
            } else {
                s_dd[nd * kDyn3InsertThreads + t] = (unsigned char)d;
                s_dh[nd * kDyn3InsertThreads + t] = (unsigned char)h;
                nd++;
            }
        }
        flush();
    }
}

// ---- C ------------------------------------------------------------------------------------------
template <int STRATEGY>
__global__ void __launch_bounds__(kDyn3Warps * 32) dyn3_finish_kernel(RunCtx c, ShaderParams sp, Dyn3Geom g) {
    __shared__ uint32_t s_list[kDyn3Warps][256];   // the round's unique ids, in output order
    __shared__ uint16_t s_of_d[kDyn3Warps][256];   // per distinct id d: distance home -> slot << 8 | position in the list
    __shared__ uint32_t s_bm[kDyn3Warps][16];      // hash: occupancy words, then their exclusive popcount prefix
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int b = blockIdx.x * kDyn3Warps + wid;
    if (b < c.n_batches && !c.acc[ACC_ABORT]) {
        const int2 cnt = c.counts[b];
        const int2 off = c.seg_off[b];
        const int begin = __ldg(c.bbegin + b), n = __ldg(c.bend + b) - begin;
        if (lane == 0 && c.out.d_batch_round_off) c.out.d_batch_round_off[b] = off.x;
        const int nu = cnt.y;
        const bool fits = (int64_t)off.y + nu <= c.out.cap_unique && (int64_t)off.x + cnt.x <= c.out.cap_rounds;
        if (cnt.x != 0 && fits) {
            const int mo = batch_map_off(c, b, begin);
            uint32_t* list = s_list[wid];
            uint16_t* of_d = s_of_d[wid];
            const uint32_t* __restrict__ dist = c.stage_uid + stage_uid_base(c, b, mo);
            if (lane == 0) {
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[off.x] = off.y;
                if (c.out.d_round_prims) c.out.d_round_prims[off.x] = n / c.ps;
            }
            if (STRATEGY == VR_SORT) {
                // ascending ids: sort id << 8 | d in registers; position j holds the j-th smallest id and says which d it was
                auto run = [&](auto rtag) {
                    constexpr int R = decltype(rtag)::value;
                    uint32_t v[R];
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        const int d = r * 32 + lane;
                        v[r] = d < nu ? ((__ldcg(dist + d) << 8) | (uint32_t)d) : kEmpty;
                    }
                    warp_bitonic_regs<R>(v, lane);
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        const int j = r * 32 + lane;
                        if (j < nu) {
                            list[j] = v[r] >> 8;
                            of_d[v[r] & 0xFFu] = (uint16_t)j;
                        }
                    }
                };
                if (nu <= 32) run(std::integral_constant<int, 1>{});
                else if (nu <= 64) run(std::integral_constant<int, 2>{});
                else if (nu <= 128) run(std::integral_constant<int, 4>{});
                else run(std::integral_constant<int, 8>{});
            } else {
                const int stride = dyn3_aux_stride(n);
                const unsigned char* __restrict__ home = g.aux + dyn3_aux_base(c, b, mo);
                const unsigned char* __restrict__ slot = home + stride;
                uint32_t* bm = s_bm[wid];
                if (lane < 16) bm[lane] = 0;
                __syncwarp();
                uint32_t sl[8], hm[8], idv[8];
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int d = r * 32 + lane;
                    sl[r] = d < nu ? (uint32_t)__ldcg(slot + d) : 0u;
                    hm[r] = d < nu ? (uint32_t)__ldcg(home + d) : 0u;
                    idv[r] = d < nu ? __ldcg(dist + d) : 0u;
                    if (d < nu) atomicOr(&bm[sl[r] >> 5], 1u << (sl[r] & 31));
                }
                __syncwarp();
                {  // exclusive popcount prefix of the 8 occupancy words -> bm[8..16)
                    const uint32_t wv = lane < 8 ? bm[lane] : 0u;
                    const int inc = warp_incl_scan(__popc(wv), lane);
                    if (lane < 8) bm[8 + lane] = (uint32_t)(inc - __popc(wv));
                }
                __syncwarp();
                const uint32_t tmask = c.table_size - 1;
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int d = r * 32 + lane;
                    if (d < nu) {  // strategies.py:370-380: rank of the slot among the occupied ones
                        const uint32_t wi = sl[r] >> 5;
                        const uint32_t j = bm[8 + wi] + (uint32_t)__popc(bm[wi] & ((1u << (sl[r] & 31)) - 1u));
                        list[j] = idv[r];
                        of_d[d] = (uint16_t)((((sl[r] - hm[r]) & tmask) << 8) | j);
                    }
                }
            }
            __syncwarp();
            // local indices (and the probe statistics of every element, duplicates included)
            uint16_t* __restrict__ amap = c.out.d_assembly_map + mo;
            unsigned int fast = 0, slow = 0, cmax = 0;
            const int wshift = ilog2((uint32_t)g.w);
            for (int i = lane; i < n; i += 32) {
                const uint32_t e = of_d[amap[i] & 0xFFu];
                amap[i] = (uint16_t)(e & 0xFFu);
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
            }
            if (STRATEGY != VR_SORT) {
                fast = __reduce_add_sync(0xffffffffu, fast);
                slow = __reduce_add_sync(0xffffffffu, slow);
                cmax = __reduce_max_sync(0xffffffffu, cmax);
                if (lane == 0) {
                    atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_FAST], (unsigned long long)fast);
                    if (STRATEGY == VR_PHASH) atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_SLOW], (unsigned long long)slow);
                    atomicMax(&c.acc[ACC_MAX_CHAIN], (long long)cmax);
                }
            }
            shade_stream<VR_SORT>(c, sp, list, nu, off.y, lane, 32, mo, sp.batch_base ? __ldg(sp.batch_base + b) : 0, b);
        }
    }
    // the last CTA to finish writes the statistics block (every CTA's probe counts are in by then)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long done = atomicAdd((unsigned long long*)&c.acc[ACC_DONE], 1ull);
        if (done == (unsigned long long)gridDim.x - 1) {
            __threadfence();
            const int2 tot = __ldcg(c.seg_off + c.n_batches);
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
    g.q = (int)next_pow2((uint32_t)((g.u_bound + 32) * 3 / 2 + 2));  // the set holds <= u_bound + 32 ids: load <= 2/3
    if (g.q < 128) g.q = 128;
    g.per_warp_bytes = g.q * (strategy == VR_SORT ? 4 + 2 : 4 + 4 + 2);
    p.smem_a = (size_t)kDyn3Warps * g.per_warp_bytes;
    p.ok = true;
    return p;
}
