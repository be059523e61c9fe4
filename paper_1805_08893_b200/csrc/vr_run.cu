// vr_run.cu -- per-batch dedup kernels, shading/assembly and the vr_run entry point.
//
// Pipeline of one vr_run call (all on the caller's stream, no host sync):
//   K0 span_scan     exclusive scan of batch spans -> position of every batch in the
//                    concatenated assembly map; validates the ranges
//                    (strategies.py:426-428)
//   K1 dedup_*       one thread group per batch: the strategy's dedup
//                    (strategies.py:159-298) -> assembly map (final), unique ids and
//                    round records (staged), per-batch (rounds, invocations)
//   K2 count_scan    exclusive scan of (rounds, invocations) -> output offsets, totals,
//                    statistics (strategies.py:472-483)
//   K3 finalize      unique ids to their final place + vertex shader once per unique id
//                    (strategies.py:456-463) + per-vertex tally (strategies.py:485-489)
#include "vr_common.cuh"

namespace vr {

struct RunCtx {
    const uint32_t* __restrict__ idx;
    int64_t n_idx;
    const int32_t* __restrict__ bbegin;
    const int32_t* __restrict__ bend;
    int n_batches;
    int max_span;
    int ps;
    int max_unique;
    int warp_width;
    uint32_t table_size;
    uint32_t multiplier;
    int table_bits;
    int enforce_budget;  // strategies.py:451-455 applies to sort/hash/phash
    int stage_factor;    // staged unique ids per batch <= span * stage_factor + ps
    // workspace
    int32_t* map_off;      // [n_batches+1]
    int2* counts;          // [n_batches] (rounds, invocations)
    int32_t* uid_off;      // [n_batches+1]
    int32_t* round_off;    // [n_batches+1]
    int64_t span_cap;      // caller's bound on the sum of batch spans
    uint32_t* stage_uid;   // staged unique ids
    int32_t* stage_rn;     // staged per-round claim counts (warp)
    int32_t* stage_rp;     // staged per-round primitives (warp)
    int32_t* flags;        // [0] abort
    // outputs
    vr_outputs out;
};

__device__ __forceinline__ int64_t stage_uid_base(const RunCtx& c, int b, int mo) {
    return (int64_t)mo * c.stage_factor + (int64_t)b * c.ps;
}
__device__ __forceinline__ int64_t stage_round_base(const RunCtx& c, int b, int mo) {
    return (int64_t)mo / c.ps + b;
}

// ---------------------------------------------------------------------------------
// K0: spans -> map_off (single CTA, strided chunks).  Also initialises the statistics.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) span_scan_kernel(RunCtx c) {
    __shared__ int scratch[40];
    __shared__ int chunk[1024];
    __shared__ long long carry;
    const int tid = threadIdx.x;
    if (tid == 0) {
        carry = 0;
        for (int i = 0; i < VR_STATS_WORDS; i++) c.out.d_stats[i] = 0;
        c.out.d_stats[VR_STAT_ERROR] = 0x7fffffffffffffffLL;
        c.flags[0] = 0;
    }
    __syncthreads();
    for (int base = 0; base < c.n_batches; base += 1024) {
        int b = base + tid;
        int span = 0;
        if (b < c.n_batches) {
            int bg = c.bbegin[b], en = c.bend[b];
            // strategies.py:427: 0 <= begin < end <= len(idx) and span % ps == 0
            bool ok = bg >= 0 && bg < en && (int64_t)en <= c.n_idx && ((en - bg) % c.ps) == 0;
            if (!ok) report_error(c.out.d_stats, b, VR_ERR_BAD_BATCH);
            else if (en - bg > c.max_span) report_error(c.out.d_stats, b, VR_ERR_UNSUPPORTED);
            else span = en - bg;
        }
        chunk[tid] = span;
        __syncthreads();
        int total = block_exclusive_scan(chunk, 1024, scratch);
        long long cbase = carry;
        if (b < c.n_batches) {
            long long off = cbase + chunk[tid];
            c.map_off[b] = (int32_t)off;
        }
        __syncthreads();
        if (tid == 0) carry = cbase + total;
        __syncthreads();
    }
    if (tid == 0) {
        c.map_off[c.n_batches] = (int32_t)carry;
        if (carry > 0x7fffffffLL) report_error(c.out.d_stats, 0, VR_ERR_UNSUPPORTED);
        else if (carry > c.span_cap) report_error(c.out.d_stats, 0, VR_ERR_CAPACITY);
        if (c.out.d_stats[VR_STAT_ERROR] != 0x7fffffffffffffffLL) c.flags[0] = 1;  // abort K1..K3
    }
}

// ---------------------------------------------------------------------------------
// K1 (naive): strategies.py:159-170 -- one round per primitive, no reuse.  Closed form:
// nothing to stage, the finalize kernel reads the index buffer directly.
// ---------------------------------------------------------------------------------
__global__ void naive_counts_kernel(RunCtx c) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= c.n_batches || c.flags[0]) return;
    int span = c.map_off[b + 1] - c.map_off[b];
    c.counts[b] = make_int2(span / c.ps, span);
}

// ---------------------------------------------------------------------------------
// K1 (warp voting), generic path: strategies.py:173-232 in closed form, one thread per
// batch, any warp_width in {4,8,16,32,64} and any batch size.
//
// Per round over the not yet consumed ids v[cursor..n):
//   claims   = distinct values in first-occurrence order (Algorithm 1 assigns each new id
//              to the lowest free lane, strategies.py:207-212), at most w of them;
//   the round stops at the first value that would be the (w+1)-th distinct one
//   (outgoing == 0, strategies.py:220), or at the end of the w-wide fetch in which the
//   w-th claim was made (loop condition fill < w, strategies.py:201), or at the batch end
//   (sentinel lanes, strategies.py:202,220);
//   primitives emitted = done // ps, cursor += emitted * ps (strategies.py:225-231);
//   every claim is shaded, including those only referenced by the discarded tail.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) warp_generic_kernel(RunCtx c) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= c.n_batches || c.flags[0]) return;
    const int begin = c.bbegin[b];
    const int mo = c.map_off[b];
    const int n = c.map_off[b + 1] - mo;
    const int w = c.warp_width, ps = c.ps;
    const uint32_t* __restrict__ ids = c.idx + begin;
    uint16_t* __restrict__ amap = c.out.d_assembly_map ? c.out.d_assembly_map + mo : nullptr;
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    int32_t* __restrict__ srn = c.stage_rn + stage_round_base(c, b, mo);
    int32_t* __restrict__ srp = c.stage_rp + stage_round_base(c, b, mo);
    uint32_t claims[64];
    int cursor = 0, rounds = 0, inv = 0;
    while (cursor < n) {
        int fill = 0, stop = n, done;
        int i = cursor;
        for (;; i++) {
            if (i >= stop) { done = stop; break; }
            uint32_t x = ids[i];
            int r = -1;
            for (int k = 0; k < fill; k++)
                if (claims[k] == x) { r = k; break; }
            if (r < 0) {
                if (fill >= w) { done = i; break; }  // first unassignable slot
                claims[fill] = x;
                suid[inv + fill] = x;
                r = fill++;
                if (fill == w) stop = min(n, cursor + ((i - cursor) / w + 1) * w);
            }
            if (amap) amap[i] = (uint16_t)r;
        }
        int emitted = (done - cursor) / ps;
        if (emitted == 0) {  // strategies.py:226-227 (unreachable for w >= ps)
            report_error(c.out.d_stats, b, VR_ERR_WARP_NO_PROGRESS);
            break;
        }
        srn[rounds] = fill;
        srp[rounds] = emitted;
        rounds++;
        inv += fill;
        cursor += emitted * ps;
    }
    c.counts[b] = make_int2(rounds, inv);
}

// ---------------------------------------------------------------------------------
// K1 (sort): strategies.py:235-260 -- Algorithm 2.  One CTA per batch: bitonic sort of
// (id << 32 | slot) keys in shared memory (the slot in the low half makes it the stable
// sort the reference asks for), run-head marks, CTA exclusive scan -> ranks, unique ids in
// ascending order, assembly_map[slot] = rank.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sort_batch_kernel(RunCtx c, int pmax) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
    int* heads = reinterpret_cast<int*>(keys + pmax);
    uint16_t* maps = reinterpret_cast<uint16_t*>(heads + pmax);
    __shared__ int scratch[40];
    const int b = blockIdx.x;
    if (c.flags[0]) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int begin = c.bbegin[b];
    const int mo = c.map_off[b];
    const int n = c.map_off[b + 1] - mo;
    const int P = (int)next_pow2((uint32_t)max(n, 2));
    const uint32_t* __restrict__ ids = c.idx + begin;
    for (int i = tid; i < P; i += nt)
        keys[i] = i < n ? (((unsigned long long)ids[i] << 32) | (unsigned)i) : ~0ull;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = tid; t < (P >> 1); t += nt) {
                int lo = 2 * t - (t & (j - 1));
                int hi = lo + j;
                bool asc = (lo & k) == 0;
                unsigned long long a = keys[lo], d = keys[hi];
                if ((a > d) == asc) { keys[lo] = d; keys[hi] = a; }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < P; i += nt)
        heads[i] = (i < n && (i == 0 || (uint32_t)(keys[i] >> 32) != (uint32_t)(keys[i - 1] >> 32))) ? 1 : 0;
    __syncthreads();
    const int nu = block_exclusive_scan(heads, P, scratch);
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    for (int i = tid; i < n; i += nt) {
        unsigned long long kv = keys[i];
        uint32_t id = (uint32_t)(kv >> 32);
        bool head = (i == 0) || id != (uint32_t)(keys[i - 1] >> 32);
        int rank = head ? heads[i] : heads[i] - 1;
        maps[(uint32_t)kv] = (uint16_t)rank;
        if (head) suid[rank] = id;
    }
    __syncthreads();
    if (c.out.d_assembly_map)
        for (int i = tid; i < n; i += nt) c.out.d_assembly_map[mo + i] = maps[i];
    if (tid == 0) {
        c.counts[b] = make_int2(1, nu);
        if (c.enforce_budget && nu > c.max_unique) report_error(c.out.d_stats, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K1 (hash): strategies.py:263-298 -- Algorithm 3, bit-exact with the reference's
// sequential insertion order for any thread schedule:
//   phase 1  first occurrence of every id (set insert into a private table with CAS,
//            min position per id);
//   phase 2  only first occurrences enter the reference table (multiplicative hash
//            strategies.py:88-91, linear probing).  A slot stores the inserting element's
//            POSITION in the batch; insertion is atomicMin with displacement, so the entry
//            that the sequential loop would have inserted earlier always wins the slot and
//            the loser keeps probing.  The final layout equals lane-0-first insertion.
//   phase 3  every element (duplicates too) walks from its home slot to its id: chain
//            length = distance + 1 gives ProbeStats.fast / max_chain (strategies.py:292-297);
//            occupied slots are ranked in table order (strategies.py:370-380).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) hash_batch_kernel(RunCtx c, int nmax, int q) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* ids = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* kkey = ids + nmax;
    uint32_t* kpos = kkey + q;
    uint32_t* tpos = kpos + q;
    uint32_t* tid_ = tpos + c.table_size;
    int* occ = reinterpret_cast<int*>(tid_ + c.table_size);
    uint16_t* maps = reinterpret_cast<uint16_t*>(occ + c.table_size);
    uint8_t* first = reinterpret_cast<uint8_t*>(maps + nmax);
    __shared__ int scratch[40];
    __shared__ int s_unique, s_chain_max;
    __shared__ unsigned long long s_chain_sum;
    const int b = blockIdx.x;
    if (c.flags[0]) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int begin = c.bbegin[b];
    const int mo = c.map_off[b];
    const int n = c.map_off[b + 1] - mo;
    const uint32_t tsize = c.table_size, tmask = tsize - 1;
    const uint32_t qmask = (uint32_t)q - 1;
    const int qbits = ilog2((uint32_t)q);
    for (int i = tid; i < n; i += nt) ids[i] = c.idx[begin + i];
    for (int i = tid; i < q; i += nt) { kkey[i] = kEmpty; kpos[i] = kEmpty; }
    for (int i = tid; i < (int)tsize; i += nt) tpos[i] = kEmpty;
    if (tid == 0) { s_unique = 0; s_chain_max = 0; s_chain_sum = 0; }
    __syncthreads();
    // phase 1
    for (int i = tid; i < n; i += nt) {
        uint32_t id = ids[i];
        uint32_t h = qbits ? (id * 0x9E3779B1u) >> (32 - qbits) : 0;
        for (;;) {
            uint32_t prev = atomicCAS(&kkey[h], kEmpty, id);
            if (prev == kEmpty || prev == id) break;
            h = (h + 1) & qmask;
        }
        atomicMin(&kpos[h], (uint32_t)i);
        maps[i] = (uint16_t)h;
    }
    __syncthreads();
    int mine = 0;
    for (int i = tid; i < n; i += nt) {
        bool f = kpos[maps[i]] == (uint32_t)i;
        first[i] = f;
        mine += f;
    }
    if (mine) atomicAdd(&s_unique, mine);
    __syncthreads();
    const int nu = s_unique;
    if (nu > (int)tsize) {  // strategies.py:283-284: chain would exceed table_size
        if (tid == 0) {
            report_error(c.out.d_stats, b, VR_ERR_HASH_FULL);
            c.counts[b] = make_int2(1, 0);
        }
        return;
    }
    // phase 2
    volatile uint32_t* vt = tpos;
    for (int i = tid; i < n; i += nt) {
        if (!first[i]) continue;
        uint32_t cur = (uint32_t)i;
        uint32_t h = hash_slot(ids[i], c.multiplier, c.table_bits);
        for (;;) {
            uint32_t t = vt[h];
            if (t == kEmpty || t > cur) {
                uint32_t old = atomicMin(&tpos[h], cur);
                if (old == kEmpty) break;
                if (old > cur) cur = old;  // displaced the later insertion; carry it on
            }
            h = (h + 1) & tmask;
        }
    }
    __syncthreads();
    // phase 3
    for (int s = tid; s < (int)tsize; s += nt) {
        uint32_t p = tpos[s];
        tid_[s] = p == kEmpty ? kEmpty : ids[p];
        occ[s] = p != kEmpty;
    }
    __syncthreads();
    block_exclusive_scan(occ, (int)tsize, scratch);
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    for (int s = tid; s < (int)tsize; s += nt)
        if (tid_[s] != kEmpty) suid[occ[s]] = tid_[s];
    unsigned int csum = 0;
    int cmax = 0;
    for (int i = tid; i < n; i += nt) {
        uint32_t id = ids[i];
        uint32_t h0 = hash_slot(id, c.multiplier, c.table_bits), s = h0;
        while (tid_[s] != id) s = (s + 1) & tmask;
        int chain = (int)((s - h0) & tmask) + 1;
        csum += chain;
        cmax = max(cmax, chain);
        maps[i] = (uint16_t)occ[s];
    }
    atomicAdd(&s_chain_sum, (unsigned long long)csum);
    atomicMax(&s_chain_max, cmax);
    __syncthreads();
    if (c.out.d_assembly_map)
        for (int i = tid; i < n; i += nt) c.out.d_assembly_map[mo + i] = maps[i];
    if (tid == 0) {
        c.counts[b] = make_int2(1, nu);
        atomicAdd((unsigned long long*)&c.out.d_stats[VR_STAT_PROBES_FAST], s_chain_sum);
        atomicMax((long long*)&c.out.d_stats[VR_STAT_PROBE_MAX_CHAIN], (long long)s_chain_max);
        if (c.enforce_budget && nu > c.max_unique) report_error(c.out.d_stats, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K2: exclusive scan of per-batch (rounds, invocations); totals and statistics.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) count_scan_kernel(RunCtx c) {
    __shared__ int scratch[40];
    __shared__ int chunk_r[1024];
    __shared__ int chunk_u[1024];
    __shared__ long long carry_r, carry_u;
    const int tid = threadIdx.x;
    if (c.flags[0]) {
        if (tid == 0) {
            c.out.d_stats[VR_STAT_BATCHES] = c.n_batches;
        }
        return;
    }
    if (tid == 0) { carry_r = 0; carry_u = 0; }
    __syncthreads();
    for (int base = 0; base < c.n_batches; base += 1024) {
        int b = base + tid;
        int2 v = b < c.n_batches ? c.counts[b] : make_int2(0, 0);
        chunk_r[tid] = v.x;
        chunk_u[tid] = v.y;
        __syncthreads();
        int tr = block_exclusive_scan(chunk_r, 1024, scratch);
        int tu = block_exclusive_scan(chunk_u, 1024, scratch);
        long long br = carry_r, bu = carry_u;
        if (b < c.n_batches) {
            c.round_off[b] = (int32_t)(br + chunk_r[tid]);
            if (c.out.d_batch_round_off) c.out.d_batch_round_off[b] = (int32_t)(br + chunk_r[tid]);
            c.uid_off[b] = (int32_t)(bu + chunk_u[tid]);
        }
        __syncthreads();
        if (tid == 0) { carry_r = br + tr; carry_u = bu + tu; }
        __syncthreads();
    }
    if (tid == 0) {
        long long R = carry_r, U = carry_u;
        c.round_off[c.n_batches] = (int32_t)R;
        if (c.out.d_batch_round_off) c.out.d_batch_round_off[c.n_batches] = (int32_t)R;
        c.uid_off[c.n_batches] = (int32_t)U;
        int64_t* st = c.out.d_stats;
        st[VR_STAT_INDICES] = c.map_off[c.n_batches];
        st[VR_STAT_INVOCATIONS] = U;
        st[VR_STAT_BATCHES] = c.n_batches;
        st[VR_STAT_ROUNDS] = R;
        if (U > c.out.cap_unique || R > c.out.cap_rounds || U > 0x7fffffffLL) {
            report_error(st, 0, VR_ERR_CAPACITY);
            c.flags[0] = 1;
        } else if (c.out.d_round_uid_off) {
            c.out.d_round_uid_off[R] = (int32_t)U;
        }
    }
}

__global__ void finish_stats_kernel(RunCtx c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (c.out.d_stats[VR_STAT_ERROR] == 0x7fffffffffffffffLL) c.out.d_stats[VR_STAT_ERROR] = -1;
    }
}

// ---------------------------------------------------------------------------------
// K3: one warp per batch.  Round records and unique ids move to their final offsets; the
// vertex shader runs once per unique id (strategies.py:456-460) with 16-byte gathers and
// 16-byte coalesced stores; optional attribute pass-through and per-vertex tally.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void shade_one(const RunCtx& c, const ShaderParams& sp, int64_t dst, uint32_t uid) {
    if (c.out.d_unique_ids) c.out.d_unique_ids[dst] = uid;
    if (sp.kind == VR_SHADER_POSITION)
        reinterpret_cast<float4*>(c.out.d_shaded4)[dst] = shade_position(sp, uid);
    if (sp.attr_words && c.out.d_shaded_attr)
        for (int k = 0; k < sp.attr_words; k++)
            c.out.d_shaded_attr[dst * sp.attr_words + k] = __ldg(sp.attr + (int64_t)uid * sp.attr_words + k);
    if (c.out.d_shade_counts) atomicAdd(&c.out.d_shade_counts[uid], 1);
}

template <int STRATEGY>
__global__ void __launch_bounds__(256) finalize_kernel(RunCtx c, ShaderParams sp) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= c.n_batches || c.flags[0]) return;
    const int mo = c.map_off[b];
    const int span = c.map_off[b + 1] - mo;
    const int u0 = c.uid_off[b];
    const int nu = c.uid_off[b + 1] - u0;
    if (STRATEGY == VR_NAIVE) {
        const uint32_t* __restrict__ ids = c.idx + c.bbegin[b];
        const int ps = c.ps;
        for (int k = lane; k < span; k += 32) {
            shade_one(c, sp, (int64_t)u0 + k, ids[k]);
            if (c.out.d_assembly_map) c.out.d_assembly_map[mo + k] = (uint16_t)(k % ps);
        }
        const int r0 = mo / ps;
        for (int r = lane; r < span / ps; r += 32) {
            if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0 + r] = u0 + r * ps;
            if (c.out.d_round_prims) c.out.d_round_prims[r0 + r] = 1;
        }
        return;
    }
    const int r0 = c.round_off[b];
    if (STRATEGY == VR_WARP) {
        const int nr = c.round_off[b + 1] - r0;
        const int32_t* srn = c.stage_rn + stage_round_base(c, b, mo);
        const int32_t* srp = c.stage_rp + stage_round_base(c, b, mo);
        int run = u0;
        for (int base = 0; base < nr; base += 32) {
            int r = base + lane;
            int cnt = r < nr ? srn[r] : 0;
            int inc = warp_incl_scan(cnt, lane);
            if (r < nr) {
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0 + r] = run + inc - cnt;
                if (c.out.d_round_prims) c.out.d_round_prims[r0 + r] = srp[r];
            }
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
    } else {
        if (lane == 0) {
            if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0] = u0;
            if (c.out.d_round_prims) c.out.d_round_prims[r0] = span / c.ps;
        }
    }
    const uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    for (int k = lane; k < nu; k += 32) shade_one(c, sp, (int64_t)u0 + k, suid[k]);
}

// ---------------------------------------------------------------------------------
// strategies.py:456-463 expanded per-corner stream (the paper's stage output queue).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) expand_kernel(const int32_t* __restrict__ bro, const int32_t* __restrict__ ruo,
                                                      const int32_t* __restrict__ rprims, const uint16_t* __restrict__ amap,
                                                      const uint32_t* __restrict__ uids, const float4* __restrict__ shaded,
                                                      int n_batches, const int32_t* __restrict__ map_off, int ps,
                                                      float* __restrict__ out_pos3, uint32_t* __restrict__ out_ids) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= n_batches) return;
    int m = map_off[b];
    for (int r = bro[b]; r < bro[b + 1]; r++) {
        const int base = ruo[r];
        const int slots = rprims[r] * ps;
        for (int k = lane; k < slots; k += 32) {
            const int src = base + amap[m + k];
            if (out_ids) out_ids[m + k] = uids[src];
            if (out_pos3) {
                float4 v = shaded[src];
                out_pos3[3 * (int64_t)(m + k) + 0] = v.x;
                out_pos3[3 * (int64_t)(m + k) + 1] = v.y;
                out_pos3[3 * (int64_t)(m + k) + 2] = v.z;
            }
        }
        m += slots;
    }
}

__global__ void __launch_bounds__(1024) span_only_scan_kernel(const int32_t* __restrict__ bbegin, const int32_t* __restrict__ bend,
                                                               int n_batches, int32_t* __restrict__ map_off) {
    __shared__ int scratch[40];
    __shared__ int chunk[1024];
    __shared__ long long carry;
    const int tid = threadIdx.x;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n_batches; base += 1024) {
        int b = base + tid;
        chunk[tid] = b < n_batches ? bend[b] - bbegin[b] : 0;
        __syncthreads();
        int total = block_exclusive_scan(chunk, 1024, scratch);
        long long cb = carry;
        if (b < n_batches) map_off[b] = (int32_t)(cb + chunk[tid]);
        __syncthreads();
        if (tid == 0) carry = cb + total;
        __syncthreads();
    }
    if (tid == 0) map_off[n_batches] = (int32_t)carry;
}

__global__ void static_offsets_kernel(int64_t n, int bs, int64_t nb, int32_t* __restrict__ off) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nb) off[i] = (int32_t)(i * bs);
    if (i == nb) off[i] = (int32_t)n;
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct WsLayout {
    size_t map_off, counts, uid_off, round_off, stage_uid, stage_rn, stage_rp, flags, total;
    int stage_factor;
};

static WsLayout ws_layout(int strategy, int64_t span_total, int64_t nb, const vr_batch_config* cfg) {
    WsLayout L{};
    const int ps = cfg->primitive_size, w = cfg->warp_width;
    L.stage_factor = 1;
    if (strategy == VR_WARP) L.stage_factor = (int)ceil_div(w, w - ps + 1 > 0 ? w - ps + 1 : 1);
    size_t o = 0;
    L.map_off = o; o += align_up((size_t)(nb + 1) * 4);
    L.counts = o; o += align_up((size_t)(nb + 1) * 8);
    L.uid_off = o; o += align_up((size_t)(nb + 1) * 4);
    L.round_off = o; o += align_up((size_t)(nb + 1) * 4);
    L.flags = o; o += align_up(64);
    L.stage_uid = o;
    if (strategy != VR_NAIVE) o += align_up(((size_t)span_total * L.stage_factor + (size_t)nb * ps + 64) * 4);
    L.stage_rn = o;
    if (strategy == VR_WARP) o += align_up(((size_t)span_total / ps + nb + 64) * 4);
    L.stage_rp = o;
    if (strategy == VR_WARP) o += align_up(((size_t)span_total / ps + nb + 64) * 4);
    L.total = o;
    return L;
}

// Optional per-kernel timing of the last vr_run (a profiling aid for bench.py: CUDA events on
// the launching stream between the pipeline's kernels).  Process-wide state: while enabled,
// vr_run is not re-entrant.
static cudaEvent_t g_prof_ev[VR_PROFILE_STAGES + 1];
static int g_prof_on = 0, g_prof_marks = 0;
static inline void prof_mark(cudaStream_t s) {
    if (g_prof_on && g_prof_marks <= VR_PROFILE_STAGES) cudaEventRecord(g_prof_ev[g_prof_marks++], s);
}

}  // namespace vr

using namespace vr;

extern "C" {

int vr_profile_enable(int on) {
    if (on && !g_prof_on) {
        if (vr_device_count() == 0) return VR_ERR_CUDA;
        for (int i = 0; i <= VR_PROFILE_STAGES; i++) VR_CUDA_CHECK(cudaEventCreate(&g_prof_ev[i]));
    } else if (!on && g_prof_on) {
        for (int i = 0; i <= VR_PROFILE_STAGES; i++) cudaEventDestroy(g_prof_ev[i]);
    }
    g_prof_on = on ? 1 : 0;
    g_prof_marks = 0;
    return VR_OK;
}

int vr_profile_read(float* ms, int cap) {
    if (!g_prof_on || g_prof_marks < 2) return 0;
    if (cudaEventSynchronize(g_prof_ev[g_prof_marks - 1]) != cudaSuccess) return 0;
    int n = g_prof_marks - 1;
    for (int i = 0; i < n && i < cap; i++) cudaEventElapsedTime(&ms[i], g_prof_ev[i], g_prof_ev[i + 1]);
    return n < cap ? n : cap;
}

int vr_abi_version(void) { return VRGEOM_ABI_VERSION; }

const char* vr_status_string(int s) {
    switch (s) {
    case VR_OK: return "ok";
    case VR_ERR_UNKNOWN_STRATEGY: return "unknown strategy";
    case VR_ERR_BAD_BATCH: return "batch is not a primitive-aligned range of the buffer";
    case VR_ERR_TABLE_BELOW_BUDGET: return "hash table_size below max_unique";
    case VR_ERR_OVER_BUDGET: return "batch holds more unique ids than max_unique; dynamic strategies require splitter-honored batches";
    case VR_ERR_HASH_FULL: return "hash table full before all unique ids were inserted";
    case VR_ERR_WARP_NO_PROGRESS: return "warp voting made no progress; primitive exceeds warp capacity";
    case VR_ERR_WARP_WIDTH: return "warp width below primitive size cannot make progress";
    case VR_ERR_UNALIGNED: return "index count is not primitive-aligned";
    case VR_ERR_BAD_CONFIG: return "invalid configuration";
    case VR_ERR_UNSUPPORTED: return "configuration outside the device limits";
    case VR_ERR_CUDA: return "CUDA failure or no CUDA device";
    case VR_ERR_CAPACITY: return "output buffer too small";
    case VR_ERR_WORKSPACE: return "workspace too small";
    case VR_ERR_PRIM_OVER_BUDGET: return "primitive has more unique indices than max_unique";
    default: return "unknown status";
    }
}

int vr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
    return n;
}

int vr_check_batch_config(const vr_batch_config* c) {
    if (!c) return VR_ERR_BAD_CONFIG;
    const int ps = c->primitive_size;
    if (ps < 1) return VR_ERR_BAD_CONFIG;
    if (c->batch_size < ps || c->batch_size % ps != 0) return VR_ERR_BAD_CONFIG;
    if (c->max_unique < ps || c->max_indices < ps || c->block_size < 1) return VR_ERR_BAD_CONFIG;
    const int w = c->warp_width;
    if (!(w == 4 || w == 8 || w == 16 || w == 32 || w == 64)) return VR_ERR_BAD_CONFIG;
    return VR_OK;
}

int vr_check_hash_config(const vr_hash_config* h) {
    if (!h) return VR_ERR_BAD_CONFIG;
    if (h->table_size < 1 || (h->table_size & (h->table_size - 1))) return VR_ERR_BAD_CONFIG;
    if ((h->multiplier & 1u) == 0) return VR_ERR_BAD_CONFIG;
    if (h->max_fast_probes < 1) return VR_ERR_BAD_CONFIG;
    return VR_OK;
}

int64_t vr_static_batch_count(int64_t n, const vr_batch_config* cfg) {
    if (!cfg || cfg->batch_size < 1 || n <= 0) return 0;
    return ceil_div(n, cfg->batch_size);
}

int vr_static_offsets(int64_t n, const vr_batch_config* cfg, int32_t* d_offsets, void* stream) {
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    if (n % cfg->primitive_size != 0) return VR_ERR_UNALIGNED;  // batching.py:79-80
    if (n > 0x7fffffffLL) return VR_ERR_UNSUPPORTED;
    int64_t nb = vr_static_batch_count(n, cfg);
    if (nb == 0) return VR_OK;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    int blocks = (int)ceil_div(nb + 1, 256);
    static_offsets_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, cfg->batch_size, nb, d_offsets);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_output_bounds(int strategy, int64_t span_total, int64_t nb, const vr_batch_config* cfg,
                     const vr_hash_config* hcfg, int64_t* max_inv, int64_t* max_rounds) {
    (void)hcfg;
    if (strategy < VR_NAIVE || strategy > VR_PHASH) return VR_ERR_UNKNOWN_STRATEGY;
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    const int ps = cfg->primitive_size, w = cfg->warp_width;
    int64_t inv = span_total, rounds = nb;
    if (strategy == VR_NAIVE) rounds = span_total / ps;
    if (strategy == VR_WARP) {
        if (w < ps) return VR_ERR_WARP_WIDTH;
        inv = span_total * w / (w - ps + 1) + nb * ps + w;
        rounds = span_total / ps;
    }
    if (max_inv) *max_inv = inv + 1;
    if (max_rounds) *max_rounds = rounds + 1;
    return VR_OK;
}

size_t vr_run_workspace_bytes(int strategy, int64_t span_total, int64_t nb, const vr_batch_config* cfg,
                              const vr_hash_config* hcfg) {
    (void)hcfg;
    if (vr_check_batch_config(cfg)) return 0;
    if (strategy == VR_WARP && cfg->warp_width < cfg->primitive_size) return 0;
    return ws_layout(strategy, span_total, nb, cfg).total;
}

int vr_run(int strategy, const uint32_t* d_idx, int64_t n_idx, const int32_t* d_bbegin, const int32_t* d_bend,
           int64_t nb, int64_t span_total, int32_t max_span, const vr_batch_config* cfg, const vr_hash_config* hcfg,
           const vr_shader* shader, const vr_outputs* out, void* d_ws, size_t ws_bytes, void* stream_) {
    const bool no_budget = (strategy & VR_FLAG_NO_BUDGET) != 0;
    strategy &= 0xFF;
    if (strategy < VR_NAIVE || strategy > VR_PHASH) return VR_ERR_UNKNOWN_STRATEGY;  // strategies.py:422-423
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    if (!out || !out->d_stats) return VR_ERR_BAD_CONFIG;
    vr_hash_config hc{(uint32_t)cfg->block_size, 2654435769u, 8u};  // strategies.py:431 default
    if (strategy == VR_HASH || strategy == VR_PHASH) {
        if (hcfg) hc = *hcfg;
        st = vr_check_hash_config(&hc);
        if (st) return st;
        if (!no_budget && (int64_t)hc.table_size < cfg->max_unique) return VR_ERR_TABLE_BELOW_BUDGET;  // strategies.py:432-435
    }
    if (strategy == VR_PHASH) return VR_ERR_UNSUPPORTED;
    if (n_idx > 0x7fffffffLL || nb > 0x7fffffffLL || span_total > 0x7fffffffLL || n_idx < 0 || nb < 0 || span_total < 0)
        return VR_ERR_UNSUPPORTED;
    if (strategy == VR_WARP && nb > 0 && cfg->warp_width < cfg->primitive_size) return VR_ERR_WARP_WIDTH;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    cudaStream_t stream = (cudaStream_t)stream_;
    const int ps = cfg->primitive_size;
    if (max_span < ps) max_span = ps;
    WsLayout L = ws_layout(strategy, span_total, nb, cfg);
    if (ws_bytes < L.total || !d_ws) return VR_ERR_WORKSPACE;
    RunCtx c{};
    c.idx = d_idx; c.n_idx = n_idx; c.bbegin = d_bbegin; c.bend = d_bend;
    c.n_batches = (int)nb; c.max_span = max_span; c.ps = ps; c.max_unique = cfg->max_unique;
    c.warp_width = cfg->warp_width; c.table_size = hc.table_size; c.multiplier = hc.multiplier;
    c.table_bits = ilog2(hc.table_size);
    c.enforce_budget = strategy >= VR_SORT && !no_budget;
    c.stage_factor = L.stage_factor;
    unsigned char* ws = (unsigned char*)d_ws;
    c.map_off = (int32_t*)(ws + L.map_off);
    c.counts = (int2*)(ws + L.counts);
    c.uid_off = (int32_t*)(ws + L.uid_off);
    c.round_off = (int32_t*)(ws + L.round_off);
    c.span_cap = span_total;
    c.stage_uid = (uint32_t*)(ws + L.stage_uid);
    c.stage_rn = (int32_t*)(ws + L.stage_rn);
    c.stage_rp = (int32_t*)(ws + L.stage_rp);
    c.flags = (int32_t*)(ws + L.flags);
    c.out = *out;
    ShaderParams sp{};
    if (shader) {
        sp.kind = shader->kind; sp.has_matrix = shader->has_matrix;
        for (int i = 0; i < 16; i++) sp.m[i] = shader->matrix[i];
        sp.pos4 = (const float4*)shader->d_positions4; sp.attr = shader->d_attributes;
        sp.attr_words = shader->d_attributes ? shader->attr_words : 0; sp.vertex_count = shader->vertex_count;
        if (sp.kind == VR_SHADER_POSITION && (!sp.pos4 || !out->d_shaded4)) return VR_ERR_BAD_CONFIG;
    }

    g_prof_marks = 0;
    prof_mark(stream);
    span_scan_kernel<<<1, 1024, 0, stream>>>(c);
    prof_mark(stream);
    if (nb > 0) {
        const int nbi = (int)nb;
        if (strategy == VR_NAIVE) {
            naive_counts_kernel<<<(nbi + 255) / 256, 256, 0, stream>>>(c);
        } else if (strategy == VR_WARP) {
            warp_generic_kernel<<<(nbi + 127) / 128, 128, 0, stream>>>(c);
        } else if (strategy == VR_SORT) {
            if (max_span > 8192) return VR_ERR_UNSUPPORTED;
            int pmax = (int)next_pow2((uint32_t)(max_span < 2 ? 2 : max_span));
            size_t smem = (size_t)pmax * (8 + 4 + 2);
            VR_CUDA_CHECK(cudaFuncSetAttribute(sort_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            sort_batch_kernel<<<nbi, 256, smem, stream>>>(c, pmax);
        } else {
            int nmax = (max_span + 3) & ~3;
            int q = (int)next_pow2((uint32_t)(2 * nmax < 64 ? 64 : 2 * nmax));
            size_t smem = (size_t)nmax * 4 + (size_t)q * 8 + (size_t)hc.table_size * 12 + (size_t)nmax * 2 + (size_t)nmax + 16;
            if (smem > 200 * 1024 || max_span > 65535) return VR_ERR_UNSUPPORTED;
            VR_CUDA_CHECK(cudaFuncSetAttribute(hash_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            hash_batch_kernel<<<nbi, 256, smem, stream>>>(c, nmax, q);
        }
    }
    prof_mark(stream);
    count_scan_kernel<<<1, 1024, 0, stream>>>(c);
    prof_mark(stream);
    if (nb > 0) {
        const int blocks = (int)ceil_div(nb, 8);
        switch (strategy) {
        case VR_NAIVE: finalize_kernel<VR_NAIVE><<<blocks, 256, 0, stream>>>(c, sp); break;
        case VR_WARP: finalize_kernel<VR_WARP><<<blocks, 256, 0, stream>>>(c, sp); break;
        default: finalize_kernel<VR_SORT><<<blocks, 256, 0, stream>>>(c, sp); break;
        }
    }
    prof_mark(stream);
    finish_stats_kernel<<<1, 32, 0, stream>>>(c);
    prof_mark(stream);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_expand_stream(const int32_t* d_bro, const int32_t* d_ruo, const int32_t* d_rprims, const uint16_t* d_amap,
                     const uint32_t* d_uids, const float* d_shaded4, int64_t nb, const int32_t* d_bbegin,
                     const int32_t* d_bend, int32_t ps, float* d_pos3, uint32_t* d_ids, void* d_ws, size_t ws_bytes,
                     void* stream_) {
    if (nb <= 0) return VR_OK;
    if (ws_bytes < (size_t)(nb + 1) * 4 || !d_ws) return VR_ERR_WORKSPACE;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (d_pos3 && !d_shaded4) return VR_ERR_BAD_CONFIG;
    cudaStream_t stream = (cudaStream_t)stream_;
    int32_t* map_off = (int32_t*)d_ws;
    span_only_scan_kernel<<<1, 1024, 0, stream>>>(d_bbegin, d_bend, (int)nb, map_off);
    expand_kernel<<<(int)ceil_div(nb, 8), 256, 0, stream>>>(d_bro, d_ruo, d_rprims, d_amap, d_uids,
                                                             (const float4*)d_shaded4, (int)nb, map_off, ps, d_pos3, d_ids);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

}  // extern "C"
