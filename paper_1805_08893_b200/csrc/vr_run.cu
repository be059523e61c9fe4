// vr_run.cu -- per-batch dedup kernels, shading/assembly and the vr_run entry point.
//
// Pipeline of one vr_run call (all on the caller's stream, no host synchronisation):
//   K0 init          clears the accumulators; for NON-contiguous batch lists also the scan of
//                    batch spans that places every batch in the concatenated assembly map
//   K1 dedup_*       one thread / CTA per batch: validation (strategies.py:426-428) and the
//                    strategy's dedup (strategies.py:159-298) -> assembly map (final), unique
//                    ids and round records (staged), per-batch (rounds, invocations)
//   K2 scan          exclusive scan of (rounds, invocations) over SEGMENTS (a batch, or the 32
//                    batches of one warp of the warp-voting kernel) -> output offsets,
//                    totals, statistics (strategies.py:472-483)
//   K3 shade         one warp per segment: round tables and unique ids to their final
//                    offsets and the vertex shader once per unique id
//                    (strategies.py:456-463), 16-byte gathers / coalesced 16-byte stores,
//                    optional attribute pass-through and per-vertex tally (:485-489)
#include <type_traits>

#include "vr_common.cuh"

namespace vr {

enum { ACC_PROBES_FAST = 0, ACC_PROBES_SLOW, ACC_MAX_CHAIN, ACC_ERROR, ACC_ABORT, ACC_TICKET, ACC_DONE, ACC_WORDS = 8 };

// The output pointers the kernels use: vr_outputs without the queue (which only kernel C of vr_dyn3.cuh and the
// closing kernel write).  Kept apart from the ABI struct on purpose: the 80-register tile kernel's allocation is
// sensitive to the parameter layout (8 more bytes here cost it 16 bytes of spills and 1.5 % of the headline).
struct RunOut {
    int32_t* d_batch_round_off;
    int32_t* d_round_uid_off;
    int32_t* d_round_prims;
    uint32_t* d_unique_ids;
    uint16_t* d_assembly_map;
    float* d_shaded4;
    uint32_t* d_shaded_attr;
    int32_t* d_shade_counts;
    int64_t* d_stats;
    int64_t cap_unique;
    int64_t cap_rounds;
};

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
    int stage_factor;    // staged unique ids per batch <= span * stage_factor
    int contiguous;      // batches tile [bbegin[0], bend[n-1]) in order: map offset = begin - first
    int seg_batches;     // batches per segment: 32 for the warp-voting kernel, else 1
    int n_segs;
    int n_scan_tiles;    // 1024-segment tiles of the three-kernel scan (0: single-CTA scan)
    int64_t span_cap;    // caller's bound on the sum of batch spans
    // workspace
    int32_t* map_off;       // [n_batches+1] (non-contiguous lists only)
    int2* counts;           // [n_batches] (rounds, invocations)
    int2* seg_counts;       // [n_segs] (aliases counts when seg_batches == 1)
    int2* seg_off;          // [n_segs+1] exclusive prefix of seg_counts
    int2* tile_sums;        // [n_scan_tiles] / tile_off [n_scan_tiles+1]
    int2* tile_off;
    uint32_t* stage_uid;    // staged unique ids
    uint32_t* stage_round;  // staged round records: primitives << 8 | claims (warp)
    long long* acc;         // [ACC_WORDS]
    unsigned long long* tile_state;  // [n_fused_tiles] decoupled look-back: flag<<62 | rounds<<32 | ids
    int n_fused_tiles;
    int n_state_words;  // words of tile_state to clear: the tiles, and for the tile kernel its group tables behind them
    // outputs
    RunOut out;
};

// First failing batch wins, as in the reference's in-order loop (strategies.py:470):
// the accumulator starts at 0 and takes the max of ((2^47-1 - batch) << 8 | status).
__device__ inline void report_error(const RunCtx& c, int64_t batch, int status) {
    long long word = (long long)(((0x7FFFFFFFFFFFLL - batch) << 8) | (long long)status);
    atomicMax(&c.acc[ACC_ERROR], word);
}
// Errors found after the statistics block may already have been written (shading runs behind the offset
// scan): straight into the error word.  It is -1 when clean (init_kernel), i.e. the largest unsigned
// value, so the minimum of (batch << 8 | status) keeps the first failing batch.
__device__ inline void report_late_error(const RunCtx& c, int64_t batch, int status) {
    atomicMin(reinterpret_cast<unsigned long long*>(c.out.d_stats + VR_STAT_ERROR),
              ((unsigned long long)batch << 8) | (unsigned long long)status);
}
// strategies.py:62-65 positions[vid] raises for an id outside the vertex buffer; the device must neither
// gather nor tally out of bounds.  `v` = first vertex of the batch's draw + id.
__device__ __forceinline__ bool vertex_in_range(const ShaderParams& sp, uint32_t v) {
    return sp.vertex_count <= 0 || v < (uint32_t)sp.vertex_count;
}

__device__ __forceinline__ int batch_map_off(const RunCtx& c, int b, int begin) {
    return c.contiguous ? begin - __ldg(c.bbegin) : c.map_off[b];
}
__device__ __forceinline__ int64_t stage_uid_base(const RunCtx& c, int b, int mo) {
    return ((int64_t)mo * c.stage_factor + (int64_t)b * 8) & ~3LL;  // 16-byte aligned, >= 5 words of slack
}
__device__ __forceinline__ int64_t stage_round_base(const RunCtx& c, int b, int mo) {
    return (int64_t)mo / c.ps + b;
}

// strategies.py:427: 0 <= begin < end <= len(idx) and span % ps == 0 (+ device limits).
__device__ __forceinline__ bool validate_batch(const RunCtx& c, int b, int& begin, int& span) {
    const int bg = __ldg(c.bbegin + b), en = __ldg(c.bend + b);
    begin = bg;
    span = en - bg;
    bool ok = bg >= 0 && bg < en && (int64_t)en <= c.n_idx && (span % c.ps) == 0;
    if (ok && c.contiguous && b + 1 < c.n_batches) ok = __ldg(c.bbegin + b + 1) == en;
    if (!ok) { report_error(c, b, VR_ERR_BAD_BATCH); return false; }
    if (span > c.max_span) { report_error(c, b, VR_ERR_UNSUPPORTED); return false; }
    return true;
}

// ---------------------------------------------------------------------------------
// K0
// ---------------------------------------------------------------------------------
__global__ void init_kernel(RunCtx c) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the tile kernel may be scheduled; it waits below
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ACC_WORDS) c.acc[i] = 0;
    if (i == 0) c.out.d_stats[VR_STAT_ERROR] = -1;  // see report_late_error
    if (i < c.n_state_words) c.tile_state[i] = 0ull;
}

// Non-contiguous batch lists: single-CTA scan of the spans (general path, not the hot one).
__global__ void __launch_bounds__(1024) span_scan_kernel(RunCtx c) {
    __shared__ int scratch[40];
    __shared__ int chunk[1024];
    __shared__ long long carry;
    const int tid = threadIdx.x;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < c.n_batches; base += 1024) {
        int b = base + tid;
        int span = 0;
        if (b < c.n_batches) {
            int bg = c.bbegin[b], en = c.bend[b];
            if (bg >= 0 && bg < en && (int64_t)en <= c.n_idx) span = en - bg;  // K1 reports the bad ones
        }
        chunk[tid] = span;
        __syncthreads();
        int total = block_exclusive_scan(chunk, 1024, scratch);
        long long cbase = carry;
        if (b < c.n_batches) c.map_off[b] = (int32_t)min(cbase + chunk[tid], 0x7fffffffLL);
        __syncthreads();
        if (tid == 0) carry = cbase + total;
        __syncthreads();
    }
    if (tid == 0) {
        c.map_off[c.n_batches] = (int32_t)min((long long)carry, 0x7fffffffLL);
        if (carry > c.span_cap) { report_error(c, 0, VR_ERR_CAPACITY); c.acc[ACC_ABORT] = 1; }
    }
}

// ---------------------------------------------------------------------------------
// K1 (naive): strategies.py:159-170 -- one round per primitive, no reuse.  Closed form:
// nothing to stage, the finalize kernel reads the index buffer directly.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) naive_counts_kernel(RunCtx c) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= c.n_batches || c.acc[ACC_ABORT]) return;
    int begin, span;
    if (!validate_batch(c, b, begin, span)) { c.counts[b] = make_int2(0, 0); return; }
    c.counts[b] = make_int2(span / c.ps, span);
}

// ---------------------------------------------------------------------------------
// K1 (warp voting): strategies.py:173-232 in closed form, one THREAD per batch.
//
// Per round over the not yet consumed ids v[cursor..n):
//   claims   = distinct values in first-occurrence order (Algorithm 1 assigns each new id
//              to the lowest free lane, strategies.py:207-212), at most W of them;
//   the round stops at the first value that would be the (W+1)-th distinct one
//   (outgoing == 0, strategies.py:220), or at the end of the W-wide fetch in which the
//   W-th claim was made (loop condition fill < W, strategies.py:201), or at the batch end
//   (sentinel lanes, strategies.py:202,220);
//   primitives emitted = done // ps, cursor += emitted * ps (strategies.py:225-231);
//   every claim is shaded, including those only referenced by the discarded tail.
//
// The lock-step lanes of Algorithm 1 are the claim slots; on the B200 the 32 batches of a
// warp advance together instead.  Each thread streams its batch with 16-byte loads (one
// prefetched ahead), looks ids up in a private 2W-slot open-addressing table in shared
// memory ([slot][thread] layout: bank == lane, conflict-free; entries are tagged with the
// round number so nothing is cleared between rounds), stages claims and round records,
// and writes local indices 8 at a time as one 16-byte store from a 16-entry ring.
// ---------------------------------------------------------------------------------
constexpr int kTpbThreads = 128;

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) { uint16_t v; asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a)); return v; }
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) { uint32_t v; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) { asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory"); }
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

__device__ __forceinline__ uint4 lds_u128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// 16-byte asynchronous global->shared copy (LDGSTS); bytes past src_bytes are zero-filled.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int W>
__global__ void __launch_bounds__(kTpbThreads) warp_tpb_kernel(RunCtx c) {
    constexpr int S = 2 * W;  // table slots per thread
    constexpr int LOG2W = W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
    constexpr int LOG2S = LOG2W + 1;
    constexpr uint32_t kRankMask = W - 1;
    constexpr uint32_t kTagFree = (1u << (8 - LOG2W)) - 1;  // tag value of an unused entry (0xFF >> LOG2W)
    constexpr int T = kTpbThreads;
    // shared memory per thread: index quads uint4[4] (cp.async ring) | claims u32[W] |
    // table u8[S] (tag << LOG2W | rank) | ring u16[16]; every array is [entry][thread], so a
    // warp access with any per-lane entry is conflict-free for the 16-/4-byte arrays and at
    // most 4-/2-way for the byte / half arrays.
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));  // keep the thread id in a register (no S2R per use)
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_quads = sbase + 16 * t;                                  // + 16*T*(quad & 3)
    const uint32_t a_claims = sbase + 64 * T + 4 * t;                         // + 4*T*rank
    // byte / half arrays keep each thread's entries inside its own 32-bit column:
    //   table slot h  -> word (h >> 2) of the column, byte h & 3
    //   ring  pos  p  -> word ((p >> 1) & 7) of the column, half p & 1
    const uint32_t a_table = sbase + 64 * T + 4 * T * W + 4 * t;
    const uint32_t a_ring = sbase + 64 * T + 4 * T * W + T * S + 4 * t;
    auto tab = [&](uint32_t h) { return a_table + 4 * T * (h >> 2) + (h & 3); };
    auto rng = [&](int p) { return a_ring + 4 * T * ((p >> 1) & 7) + 2 * (p & 1); };
    const int b = blockIdx.x * T + t;
#pragma unroll
    for (int h = 0; h < S / 4; h++) sts_u32(a_table + 4 * T * h, 0xFFFFFFFFu);
    bool active = b < c.n_batches && !c.acc[ACC_ABORT];
    int begin = 0, n = 0;
    if (active && !validate_batch(c, b, begin, n)) { c.counts[b] = make_int2(0, 0); active = false; }
    const int mo = active ? batch_map_off(c, b, begin) : 0;
    const int ps = c.ps;
    uint16_t* __restrict__ amap = (active && c.out.d_assembly_map) ? c.out.d_assembly_map + mo : nullptr;
    const bool amap_vec = (mo & 7) == 0;
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    uint32_t* __restrict__ srd = c.stage_round + stage_round_base(c, b, mo);
    const int n_idx = (int)c.n_idx;

    // index stream: quad q of the buffer lives in ring slot q & 3; quads up to (current + 2)
    // are in flight, the previous quad is still resident for the <= 2-slot rewind of a round end
    auto issue_quad = [&](int gq) {
        const int rem = n_idx - 4 * gq;  // indices left from this quad on
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? 4 * rem : 0);
        cp_async16(a_quads + 16 * T * (gq & 3), c.idx + (bytes ? 4 * (int64_t)gq : 0), bytes);
        cp_async_commit();
    };
    auto flush_group = [&](int g, int count) {
        if (!amap) return;
        uint32_t r[8];
#pragma unroll
        for (int j = 0; j < 4; j++) {  // two ranks per 32-bit word of the ring
            const uint32_t w2 = lds_u32(a_ring + 4 * T * ((4 * g + j) & 7));
            r[2 * j] = w2 & 0xFFFFu;
            r[2 * j + 1] = w2 >> 16;
        }
        if (count == 8 && amap_vec) {
            uint4 v = make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), r[4] | (r[5] << 16), r[6] | (r[7] << 16));
            *reinterpret_cast<uint4*>(amap + 8 * g) = v;
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < count) amap[8 * g + j] = (uint16_t)r[j];
        }
    };

    int issued = (begin >> 2) - 1;  // highest quad handed to cp.async
    if (active) { issue_quad(++issued); issue_quad(++issued); }
    int cursor = 0, i = 0, fill = 0, stop = n, rounds = 0, inv = 0, flushed = 0, done = 0;
    uint32_t tagno = 0;
    bool run = false, round_end = false, finished = false;
    uint4 cl = make_uint4(0, 0, 0, 0);  // up to four staged claims not yet written

    // One index slot of this lane's batch (strategies.py:204-213 for one lane of the fetch).
    auto element = [&](const int e, const uint32_t x) {
        if (!run || ((begin + i) & 3) != e) return;
        if (i >= stop) { done = stop; round_end = true; run = false; return; }
        uint32_t h = (x * 0x9E3779B1u) >> (32 - LOG2S);
        int r = -1;
        for (;;) {
            const uint32_t ent = lds_u8(tab(h));
            if ((ent >> LOG2W) != tagno) break;  // free: never used or left over from an earlier round
            const uint32_t rr = ent & kRankMask;
            if (lds_u32(a_claims + 4 * T * rr) == x) { r = (int)rr; break; }
            h = (h + 1) & (S - 1);
        }
        if (r < 0) {
            if (fill >= W) { done = i; round_end = true; run = false; return; }  // first unassignable slot
            sts_u32(a_claims + 4 * T * fill, x);
            sts_u8(tab(h), (tagno << LOG2W) | (uint32_t)fill);
            {   // staged claims leave as 16-byte stores (the staging base is 16-byte aligned)
                const int k = inv + fill;
                const int k4 = k & 3;
                if (k4 == 0) cl.x = x; else if (k4 == 1) cl.y = x; else if (k4 == 2) cl.z = x; else cl.w = x;
                if (k4 == 3) *reinterpret_cast<uint4*>(suid + (k & ~3)) = cl;
            }
            r = fill++;
            if (fill == W) stop = min(n, cursor + ((i - cursor) / W + 1) * W);
        }
        sts_u16(rng(i), (uint32_t)r);
        i++;
    };

    // One loop for the whole warp, re-converged every iteration: each lane advances its own
    // batch by up to one 16-byte quad of indices; round ends and batch ends are handled in place.
    while (__any_sync(0xffffffffu, active)) {
        if (!active) continue;
        const int gq = (begin + i) >> 2;
        if (issued < gq + 2) issue_quad(++issued);  // one new quad per forward step
        else cp_async_commit();                     // keep one group per iteration
        cp_async_wait<2>();                         // everything but the two newest groups has landed
        const uint4 q = lds_u128(a_quads + 16 * T * (gq & 3));
        run = true;
        round_end = false;
        element(0, q.x);
        element(1, q.y);
        element(2, q.z);
        element(3, q.w);
        if (i >= 8 * flushed + 10) {  // positions <= i-3 are final
            flush_group(flushed, 8);
            flushed++;
        }
        if (round_end) {
            const int emitted = (done - cursor) / ps;
            if (emitted == 0) {  // strategies.py:226-227 (unreachable for W >= ps)
                report_error(c, b, VR_ERR_WARP_NO_PROGRESS);
                c.counts[b] = make_int2(0, 0);
                active = false;
                continue;
            }
            srd[rounds] = ((uint32_t)emitted << 8) | (uint32_t)fill;
            rounds++;
            inv += fill;
            cursor += emitted * ps;
            i = cursor;
            fill = 0;
            stop = n;
            if (++tagno == kTagFree) {  // tag space exhausted: wipe this thread's column
                for (int h = 0; h < S / 4; h++) sts_u32(a_table + 4 * T * h, 0xFFFFFFFFu);
                tagno = 0;
            }
            if (cursor >= n) {
                for (int g = flushed; 8 * g < n; g++) flush_group(g, min(8, n - 8 * g));
                if (inv & 3) *reinterpret_cast<uint4*>(suid + (inv & ~3)) = cl;  // partial last group
                c.counts[b] = make_int2(rounds, inv);
                finished = true;
                active = false;
            }
        }
    }
    cp_async_wait<0>();
    // the 32 batches of this warp form one segment of the offset scan
    int seg_r = finished ? rounds : 0, seg_u = finished ? inv : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        seg_r += __shfl_xor_sync(0xffffffffu, seg_r, d);
        seg_u += __shfl_xor_sync(0xffffffffu, seg_u, d);
    }
    const int seg = b >> 5;
    if ((t & 31) == 0 && seg < c.n_segs) c.seg_counts[seg] = make_int2(seg_r, seg_u);
}

// Totals, statistics and the closing table entries (strategies.py:472-502); one thread.
__device__ void finish_stats(const RunCtx& c, long long R, long long U) {
    int64_t* st = c.out.d_stats;
    for (int i = 0; i < VR_STATS_WORDS; i++)
        if (i != VR_STAT_ERROR) st[i] = 0;
    long long span_total = 0;
    if (c.n_batches > 0)
        span_total = c.contiguous ? (long long)c.bend[c.n_batches - 1] - c.bbegin[0] : c.map_off[c.n_batches];
    if (span_total > c.span_cap) report_error(c, 0, VR_ERR_CAPACITY);
    if (U > c.out.cap_unique || R > c.out.cap_rounds || U > 0x7fffffffLL) report_error(c, 0, VR_ERR_CAPACITY);
    st[VR_STAT_INDICES] = span_total;
    st[VR_STAT_INVOCATIONS] = U;
    st[VR_STAT_BATCHES] = c.n_batches;
    st[VR_STAT_ROUNDS] = R;
    // (read from L2: a fused kernel calls this from its last CTA, whose L1 may hold an older copy of the line)
    st[VR_STAT_PROBES_FAST] = __ldcg(c.acc + ACC_PROBES_FAST);
    st[VR_STAT_PROBES_SLOW] = __ldcg(c.acc + ACC_PROBES_SLOW);
    st[VR_STAT_PROBE_MAX_CHAIN] = __ldcg(c.acc + ACC_MAX_CHAIN);
    const long long e = __ldcg(c.acc + ACC_ERROR);
    if (e == 0) {
        if (c.out.d_batch_round_off) c.out.d_batch_round_off[c.n_batches] = (int32_t)R;
        if (c.out.d_round_uid_off) c.out.d_round_uid_off[R] = (int32_t)U;
    } else {
        report_late_error(c, 0x7FFFFFFFFFFFLL - (e >> 8), (int)(e & 0xFF));
        c.acc[ACC_ABORT] = 1;  // K3 must not touch the outputs
    }
}

// ---------------------------------------------------------------------------------
// K1 (warp voting), static-batch fast path: primitive_size 3, batch_size % 8 == 0 and
// begin[b] = begin[0] + b * batch_size (batching.py:76-84).  Same closed form as above,
// with everything position-aligned so that the whole warp stays converged:
//   * every lane streams its batch as 16-byte loads, one group of 8 slots ahead, into two
//     alternating register sets (no shared memory and no register moves on the index path);
//   * the <= 2 index slots of a round's discarded tail are re-claimed in place when the round
//     ends (they are the first slots of the next round), so the cursor never moves backwards;
//   * local indices accumulate in registers, 8 per 16-byte store; a round's claims leave the
//     shared claim array as 16-byte stores when the round ends.
// Shared memory per lane: claims u32[W] + table u8[2W] = 192 B at W = 32.
// ---------------------------------------------------------------------------------
constexpr int kFastThreads = 128;

// FUSED: the same CTA goes on to place and shade its own unique ids.  Output offsets come from a
// decoupled look-back over CTA tiles (tiles are handed out by an atomic ticket, so every
// predecessor of a tile is resident or finished): while some warps of an SM wait on gathers
// in the shading phase, others are busy with the (latency-bound) dedup phase.
constexpr unsigned long long kStateAggregate = 1ull << 62, kStateInclusive = 2ull << 62;

template <int W, bool FUSED>
__global__ void __launch_bounds__(kFastThreads) warp_fast_kernel(RunCtx c, int bs, ShaderParams sp) {
    constexpr int S = 2 * W;
    constexpr int LOG2W = W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
    constexpr int LOG2S = LOG2W + 1;
    constexpr uint32_t kRankMask = W - 1;
    constexpr uint32_t kTagFree = (1u << (8 - LOG2W)) - 1;
    constexpr int T = kFastThreads;
    // shared memory: index quads uint4 [4][T] (cp.async ring) | claims u32 [W][T] | table u8 [S]
    // per thread as words [S/4][T] (tag << LOG2W | rank): every access stays inside the lane's
    // own column
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    const int lane = t & 31;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_quads = sbase + 16 * t;
    const uint32_t a_claims = sbase + 64 * T + 4 * t;
    const uint32_t a_table = sbase + 64 * T + 4 * T * W + 4 * t;
    auto tab = [&](uint32_t h) { return a_table + 4 * T * (h >> 2) + (h & 3); };
    __shared__ int s_tile;
    __shared__ int2 s_warp_tot[T / 32];
    __shared__ int2 s_base;
    int tile = blockIdx.x;
    if (FUSED) {  // tiles in ticket order
        if (t == 0) s_tile = (int)atomicAdd((unsigned long long*)&c.acc[ACC_TICKET], 1ull);
        __syncthreads();
        tile = s_tile;
    }
    const int b = tile * T + t;
#pragma unroll
    for (int h = 0; h < S / 4; h++) sts_u32(a_table + 4 * T * h, 0xFFFFFFFFu);
    bool active = b < c.n_batches && !c.acc[ACC_ABORT];
    int begin = 0, n = 0;
    if (active && !validate_batch(c, b, begin, n)) { c.counts[b] = make_int2(0, 0); active = false; }
    if (active && (begin - __ldg(c.bbegin) != b * bs || (n != bs && b != c.n_batches - 1) || (begin & 3))) {
        report_error(c, b, VR_ERR_BAD_BATCH);  // not the static batching this path was promised
        c.counts[b] = make_int2(0, 0);
        active = false;
    }
    if (!active) n = 0;
    const int mo = b * bs;
    uint16_t* __restrict__ amap = (active && c.out.d_assembly_map) ? c.out.d_assembly_map + mo : nullptr;
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    uint32_t* __restrict__ srd = c.stage_round + stage_round_base(c, b, mo);
    const uint32_t* __restrict__ ids = c.idx + begin;

    // indices 4q..4q+3 of this lane's batch -> ring slot q & 3 (zero-filled past the batch end)
    auto issue_quad = [&](int q) {
        const int rem = n - 4 * q;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? 4 * rem : 0);
        cp_async16(a_quads + 16 * T * (q & 3), bytes ? ids + 4 * q : c.idx, bytes);
    };

    int fill = 0, cursor = 0, stop = n, rounds = 0, inv = 0;
    uint32_t tagno = 0;
    uint32_t h = 0;  // free slot found by the last failed lookup

    auto lookup = [&](uint32_t x) -> int {
        h = (x * 0x9E3779B1u) >> (32 - LOG2S);
        for (;;) {
            const uint32_t ent = lds_u8(tab(h));
            if ((ent >> LOG2W) != tagno) return -1;  // free: never used or from an earlier round
            const uint32_t rr = ent & kRankMask;
            if (lds_u32(a_claims + 4 * T * rr) == x) return (int)rr;
            h = (h + 1) & (S - 1);
        }
    };
    auto claim = [&](uint32_t x, int p) -> int {  // strategies.py:207-212
        sts_u32(a_claims + 4 * T * fill, x);
        sts_u8(tab(h), (tagno << LOG2W) | (uint32_t)fill);
        const int r = fill++;
        if (fill == W) stop = min(n, cursor + ((p - cursor) / W + 1) * W);  // end of this fetch
        return r;
    };
    auto flush_claims = [&]() {  // the round's claims, 16 bytes at a time (inv % 4 == 0)
        for (int j = 0; j < fill; j += 4) {
            uint4 v;
            v.x = lds_u32(a_claims + 4 * T * (j + 0));
            v.y = lds_u32(a_claims + 4 * T * ((j + 1) & (W - 1)));
            v.z = lds_u32(a_claims + 4 * T * ((j + 2) & (W - 1)));
            v.w = lds_u32(a_claims + 4 * T * ((j + 3) & (W - 1)));
            *reinterpret_cast<uint4*>(suid + inv + j) = v;
        }
    };

    uint32_t r[8];                       // local indices of the current group of 8 slots
    uint4 gp = make_uint4(0, 0, 0, 0);   // previous group, packed, not yet stored
    uint32_t px6 = 0, px7 = 0;           // last two ids of the previous group
    auto store_group = [&](int kg, const uint4& g) {  // 8 local indices = one 16-byte store
        if (!amap || 8 * kg >= n) return;
        if (8 * kg + 8 <= n) {
            *reinterpret_cast<uint4*>(amap + 8 * kg) = g;
        } else {
            const uint32_t w4[4] = {g.x, g.y, g.z, g.w};
            for (int e = 0; e < 8 && 8 * kg + e < n; e++)
                amap[8 * kg + e] = (uint16_t)(w4[e >> 1] >> (16 * (e & 1)));
        }
    };

    // one group of 8 index slots; a round end inside the group is handled once, then the
    // group resumes at the slot that closed the round
    auto process_group = [&](const int k, const uint4& qa, const uint4& qb) {
        const uint32_t xs[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        int e0 = 0;
        for (;;) {
            int pe = -1;  // slot of this group before which the current round ends
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const int p = 8 * k + e;
                if (e >= e0 && pe < 0 && p < n) {
                    int rr = -1;
                    if (p < stop) {  // else: the fetch that filled the warp is exhausted
                        rr = lookup(xs[e]);
                        if (rr < 0 && fill < W) rr = claim(xs[e], p);
                    }
                    if (rr < 0) pe = e;  // p >= stop, or first unassignable slot
                    else r[e] = (uint32_t)rr;
                }
                if (e == 1 && k > 0 && pe < 0 && e0 <= 1) store_group(k - 1, gp);  // slots < 8k are final now
            }
            if (pe < 0) break;
            // strategies.py:220-231: the round ends before slot p; emit whole primitives, re-open
            // at the first unconsumed slot and give the discarded tail its claims of the new round
            const int p = 8 * k + pe;
            const int emitted = (p - cursor) / 3;
            const int consumed = cursor + 3 * emitted;
            flush_claims();
            srd[rounds++] = ((uint32_t)emitted << 8) | (uint32_t)fill;
            inv += fill;
            fill = 0;
            cursor = consumed;
            stop = n;
            if (++tagno == kTagFree) {
                for (int hh = 0; hh < S / 4; hh++) sts_u32(a_table + 4 * T * hh, 0xFFFFFFFFu);
                tagno = 0;
            }
            for (int tp = consumed; tp < p; tp++) {
                uint32_t id = (tp & 7) == 6 ? px6 : px7;
                if ((tp >> 3) == k) {
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((tp & 7) == e) id = xs[e];
                }
                int rr = lookup(id);
                if (rr < 0) rr = claim(id, tp);
                if ((tp >> 3) == k) {
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if ((tp & 7) == e) r[e] = (uint32_t)rr;
                } else if ((tp & 7) == 6) {
                    gp.w = (gp.w & 0xFFFF0000u) | (uint32_t)rr;
                } else {
                    gp.w = (gp.w & 0x0000FFFFu) | ((uint32_t)rr << 16);
                }
            }
            if (pe <= 1 && k > 0) store_group(k - 1, gp);  // tail fixed: the previous group is final
            e0 = pe;
        }
        gp = make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), r[4] | (r[5] << 16), r[6] | (r[7] << 16));
        px6 = xs[6];
        px7 = xs[7];
    };

    const int groups = (bs + 7) >> 3;
#pragma unroll
    for (int e = 0; e < 8; e++) r[e] = 0;
    issue_quad(0);
    issue_quad(1);
    cp_async_commit();
    for (int k = 0; k < groups; k++) {
        issue_quad(2 * k + 2);  // one group ahead
        issue_quad(2 * k + 3);
        cp_async_commit();
        cp_async_wait<1>();
        const uint4 qa = lds_u128(a_quads + 16 * T * ((2 * k) & 3)), qb = lds_u128(a_quads + 16 * T * ((2 * k + 1) & 3));
        process_group(k, qa, qb);
    }
    cp_async_wait<0>();
    int seg_r = 0, seg_u = 0;
    if (active) {
        // last group, then the final round (the batch end closes it; nothing is discarded)
        store_group(groups - 1, gp);
        flush_claims();
        srd[rounds++] = ((uint32_t)((n - cursor) / 3) << 8) | (uint32_t)fill;
        inv += fill;
        c.counts[b] = make_int2(rounds, inv);
        seg_r = rounds;
        seg_u = inv;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        seg_r += __shfl_xor_sync(0xffffffffu, seg_r, d);
        seg_u += __shfl_xor_sync(0xffffffffu, seg_u, d);
    }
    if (!FUSED) {
        const int seg = b >> 5;
        if (lane == 0 && seg < c.n_segs) c.seg_counts[seg] = make_int2(seg_r, seg_u);
        return;
    }
    // ---- output offsets: CTA aggregate, then decoupled look-back by warp 0
    const int wid = t >> 5;
    if (lane == 0) s_warp_tot[wid] = make_int2(seg_r, seg_u);
    __syncthreads();
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
        for (int p = tile - 1; p >= 0; p -= 32) {
            const int idx = p - lane;
            unsigned long long word = kStateInclusive;  // tiles before the first one: inclusive zero
            int spins = 0;
            for (;;) {
                if (idx >= 0) word = state[idx];
                if (!__any_sync(0xffffffffu, (word >> 62) == 0)) break;
                if (++spins > (1 << 20)) { lost = true; break; }
                __nanosleep(40);
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
    __syncthreads();
    int2 off = s_base;
    if (off.x < 0) return;  // offsets unknown or outputs too small: leave them untouched
    for (int w = 0; w < wid; w++) { off.x += s_warp_tot[w].x; off.y += s_warp_tot[w].y; }

    // ---- this warp's segment: round tables, then unique ids + shading (as in shade_kernel)
    {
        const int my_r = active ? rounds : 0, my_u = active ? inv : 0;
        const int inc_r = warp_incl_scan(my_r, lane), inc_u = warp_incl_scan(my_u, lane);
        const int u0 = off.y + inc_u - my_u;
        if (active) {
            const int r0 = off.x + inc_r - my_r;
            int run = u0;
            if (c.out.d_batch_round_off) c.out.d_batch_round_off[b] = r0;
            for (int q = 0; q < my_r; q++) {
                const uint32_t wv = srd[q];
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0 + q] = run;
                if (c.out.d_round_prims) c.out.d_round_prims[r0 + q] = (int)(wv >> 8);
                run += (int)(wv & 0xFFu);
            }
        }
        const unsigned long long my_src = (unsigned long long)suid;
        const int ex = inc_u - my_u;
        const int tot = __shfl_sync(0xffffffffu, inc_u, 31);
        const bool want_uid = c.out.d_unique_ids != nullptr;
        const bool want_pos = sp.kind == VR_SHADER_POSITION;
        const bool want_attr = sp.attr_words && c.out.d_shaded_attr;
        const bool want_cnt = c.out.d_shade_counts != nullptr;
        uint32_t* __restrict__ out_uid = c.out.d_unique_ids + off.y;
        float4* __restrict__ shaded = reinterpret_cast<float4*>(c.out.d_shaded4) + off.y;
        const uint32_t lt = (1u << lane) - 1;
        int first_owner = 0;
        constexpr int U4 = 4;
        for (int j0 = 0; j0 < tot; j0 += 32 * U4) {
            uint32_t uid[U4];
            bool live[U4];
            float4 pv[U4];
#pragma unroll
            for (int u = 0; u < U4; u++) {
                const int jb = j0 + 32 * u;
                const int d = inc_u - jb - 1;
                const uint32_t ends = __reduce_or_sync(0xffffffffu, (my_u > 0 && d >= 0 && d < 32) ? (1u << d) : 0u);
                const int owner = (first_owner + __popc(ends & lt)) & 31;
                first_owner += __popc(ends);
                const int oex = __shfl_sync(0xffffffffu, ex, owner);
                const uint32_t* osrc = (const uint32_t*)__shfl_sync(0xffffffffu, my_src, owner);
                const int j = jb + lane;
                uid[u] = j < tot ? osrc[j - oex] : 0u;
                live[u] = j < tot && vertex_in_range(sp, uid[u]);
                if (j < tot && !live[u]) report_late_error(c, (int64_t)tile * T + 32 * wid + owner, VR_ERR_VERTEX_RANGE);
            }
            if (want_pos) {
#pragma unroll
                for (int u = 0; u < U4; u++)
                    if (live[u]) pv[u] = __ldg(sp.pos4 + uid[u]);
            }
#pragma unroll
            for (int u = 0; u < U4; u++) {
                const int j = j0 + 32 * u + lane;
                if (j >= tot) continue;
                if (want_uid) out_uid[j] = uid[u];
                if (!live[u]) continue;
                if (want_pos) shaded[j] = transform_position(sp, pv[u]);
                if (want_attr)
                    for (int q = 0; q < sp.attr_words; q++)
                        c.out.d_shaded_attr[((int64_t)off.y + j) * sp.attr_words + q] = __ldg(sp.attr + (int64_t)uid[u] * sp.attr_words + q);
                if (want_cnt) atomicAdd(&c.out.d_shade_counts[uid[u]], 1);
            }
        }
    }
}

#include "vr_warp_rows.cuh"

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
    if (c.acc[ACC_ABORT]) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    int begin, n;
    if (!validate_batch(c, b, begin, n)) {  // uniform: every thread evaluates the same values
        if (tid == 0) c.counts[b] = make_int2(0, 0);
        return;
    }
    const int mo = batch_map_off(c, b, begin);
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
        if (c.enforce_budget && nu > c.max_unique) report_error(c, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K1 (sort), one WARP per batch: the result of strategies.py:235-260 is "unique ids ascending,
// local index = rank of the id", which does not need the batch sorted -- only its DISTINCT ids
// (at most max_unique of them under the budget of strategies.py:451-455).  So: (1) distinct ids
// by insertion into a private open-addressing set (CAS), remembering every element's set slot;
// (2) the distinct ids are compacted out of the set and sorted (bitonic, in shared memory, padded
// to the next power of two of their number); (3) every sorted id looks its set slot up again and
// leaves its rank there; (4) local index of element i = rank at its set slot.
// ---------------------------------------------------------------------------------
// Bitonic sort of 32 * R keys held R per lane (key index = r * 32 + lane): partners at distance >= 32 are
// registers of the same lane, nearer ones come by shuffle; no shared memory, no barriers.
template <int R>
__device__ __forceinline__ void warp_bitonic_regs(uint32_t (&v)[R], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    if ((r & jr) == 0) {
                        const bool asc = ((r * 32) & k) == 0;  // k >= 64 here: the direction depends on r alone
                        const uint32_t a = v[r], d = v[r | jr];
                        const uint32_t lo = min(a, d), hi = max(a, d);
                        v[r] = asc ? lo : hi;
                        v[r | jr] = asc ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool asc = (((r * 32) | lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    v[r] = (lower == asc) ? min(v[r], o) : max(v[r], o);
                }
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void warp_sort_shared(uint32_t* sorted, int lane) {
    uint32_t v[R];
#pragma unroll
    for (int r = 0; r < R; r++) v[r] = sorted[r * 32 + lane];
    warp_bitonic_regs<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; r++) sorted[r * 32 + lane] = v[r];
}

__global__ void __launch_bounds__(256) sort_warp_kernel(RunCtx c, int n_max, int q, int u_bound, int p_max, int per_warp_bytes) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5;
    const int b = blockIdx.x * warps + wid;
    if (b >= c.n_batches || c.acc[ACC_ABORT]) return;
    unsigned char* base = smem_raw + (size_t)wid * per_warp_bytes;
    uint32_t* kkey = reinterpret_cast<uint32_t*>(base);                // [q] the set (the batch is read in place)
    uint32_t* sorted = kkey + q;                                       // [p_max]
    uint16_t* kslot = reinterpret_cast<uint16_t*>(sorted + p_max);     // [n_max] set slot of every element
    uint16_t* rank_at = kslot + n_max;                                 // [q] rank of the id in a set slot
    int begin, n;
    if (!validate_batch(c, b, begin, n)) {
        if (lane == 0) c.counts[b] = make_int2(0, 0);
        return;
    }
    const int mo = batch_map_off(c, b, begin);
    const uint32_t qmask = (uint32_t)q - 1;
    const int qbits = ilog2((uint32_t)q);
    const uint32_t* __restrict__ ids = c.idx + begin;
    for (int i = lane; i < q; i += 32) kkey[i] = kEmpty;
    __syncwarp();
    int fresh = 0;
    bool overflow = false;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        if (i < n) {
            const uint32_t id = __ldg(ids + i);
            uint32_t h = (id * 0x9E3779B1u) >> (32 - qbits);
            for (;;) {
                const uint32_t prev = atomicCAS(&kkey[h], kEmpty, id);
                if (prev == kEmpty) fresh++;
                if (prev == kEmpty || prev == id) break;
                h = (h + 1) & qmask;
            }
            kslot[i] = (uint16_t)h;
        }
        const int tot = __reduce_add_sync(0xffffffffu, fresh);  // one REDUX instead of five shuffles
        if (tot > u_bound) { overflow = true; break; }  // uniform: stop before the set can fill up
    }
    if (overflow) {  // only under the unique budget: more distinct ids than max_unique (strategies.py:451-455)
        if (lane == 0) {
            report_error(c, b, VR_ERR_OVER_BUDGET);
            c.counts[b] = make_int2(0, 0);
        }
        return;
    }
    __syncwarp();
    // distinct ids out of the set
    int nu = 0;
    for (int s0 = 0; s0 < q; s0 += 32) {
        const uint32_t k = kkey[s0 + lane];
        const uint32_t m = __ballot_sync(0xffffffffu, k != kEmpty);
        if (k != kEmpty) sorted[nu + __popc(m & ((1u << lane) - 1))] = k;
        nu += __popc(m);
    }
    const int P = (int)next_pow2((uint32_t)max(nu, 32));
    for (int i = nu + lane; i < P; i += 32) sorted[i] = kEmpty;  // pads sort last
    __syncwarp();
    // up to 256 distinct ids (the default budget): sorted in registers; more: in shared memory
    if (P == 32) warp_sort_shared<1>(sorted, lane);
    else if (P == 64) warp_sort_shared<2>(sorted, lane);
    else if (P == 128) warp_sort_shared<4>(sorted, lane);
    else if (P == 256) warp_sort_shared<8>(sorted, lane);
    __syncwarp();
    for (int k = 2; k <= P && P > 256; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = lane; t < (P >> 1); t += 32) {
                const int lo = 2 * t - (t & (j - 1));
                const int hi = lo + j;
                const bool asc = (lo & k) == 0;
                const uint32_t a = sorted[lo], d = sorted[hi];
                if ((a > d) == asc) { sorted[lo] = d; sorted[hi] = a; }
            }
            __syncwarp();
        }
    }
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    for (int r = lane; r < nu; r += 32) {
        const uint32_t id = sorted[r];
        uint32_t h = (id * 0x9E3779B1u) >> (32 - qbits);
        while (kkey[h] != id) h = (h + 1) & qmask;
        rank_at[h] = (uint16_t)r;
        suid[r] = id;
    }
    __syncwarp();
    if (c.out.d_assembly_map) {
        uint16_t* __restrict__ amap = c.out.d_assembly_map + mo;
        for (int i = lane; i < n; i += 32) amap[i] = rank_at[kslot[i]];
    }
    if (lane == 0) {
        c.counts[b] = make_int2(1, nu);
        if (c.enforce_budget && nu > c.max_unique) report_error(c, b, VR_ERR_OVER_BUDGET);
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
    if (c.acc[ACC_ABORT]) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    int begin, n;
    if (!validate_batch(c, b, begin, n)) {
        if (tid == 0) c.counts[b] = make_int2(0, 0);
        return;
    }
    const int mo = batch_map_off(c, b, begin);
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
            report_error(c, b, VR_ERR_HASH_FULL);
            c.counts[b] = make_int2(0, 0);
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
    // phase 3: no walking -- the final slot of every first occurrence is read off the table
    // (slot_of[position] = slot), duplicates take the slot of their first occurrence, and the
    // probe chain of the reference's loop is the circular distance from the home slot + 1.
    for (int s = tid; s < (int)tsize; s += nt) {
        uint32_t p = tpos[s];
        tid_[s] = p == kEmpty ? kEmpty : ids[p];
        occ[s] = p != kEmpty;
        if (p != kEmpty) kpos[maps[p]] = (uint32_t)s;  // private-set slot of this id -> table slot
    }
    __syncthreads();
    block_exclusive_scan(occ, (int)tsize, scratch);
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    for (int s = tid; s < (int)tsize; s += nt)
        if (tid_[s] != kEmpty) suid[occ[s]] = tid_[s];
    unsigned int csum = 0;
    int cmax = 0;
    for (int i = tid; i < n; i += nt) {
        const uint32_t s = kpos[maps[i]];
        const uint32_t h0 = hash_slot(ids[i], c.multiplier, c.table_bits);
        const int chain = (int)((s - h0) & tmask) + 1;
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
        atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_FAST], s_chain_sum);
        atomicMax(&c.acc[ACC_MAX_CHAIN], (long long)s_chain_max);
        if (c.enforce_budget && nu > c.max_unique) report_error(c, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K1 (hash), one WARP per batch: same three phases as hash_batch_kernel, sized for the dynamic
// batches of the paper (<= 1023 indices, <= 256 unique ids): 8 batches per 256-thread CTA, no
// CTA barriers, lanes stride the batch.  The private first-occurrence set is sized by the
// unique budget (2x, power of two), not by the batch length.
// ---------------------------------------------------------------------------------
struct HashWarpSmem { int n_max, q, per_warp_bytes; };

__global__ void __launch_bounds__(256) hash_warp_kernel(RunCtx c, int n_max, int q, int u_bound, int per_warp_bytes) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5;
    const int b = blockIdx.x * warps + wid;
    if (b >= c.n_batches || c.acc[ACC_ABORT]) return;
    unsigned char* base = smem_raw + (size_t)wid * per_warp_bytes;
    // (the batch itself is not copied: its indices are read where they lie, through L1 -- the 4 KB per warp
    // decide how many warps an SM holds, and this kernel lives on occupancy)
    uint32_t* kkey = reinterpret_cast<uint32_t*>(base);
    uint32_t* kpos = kkey + q;
    uint32_t* tpos = kpos + q;
    uint16_t* rank_of = reinterpret_cast<uint16_t*>(tpos + c.table_size);
    uint16_t* kslot = rank_of + c.table_size;
    int begin, n;
    if (!validate_batch(c, b, begin, n)) {
        if (lane == 0) c.counts[b] = make_int2(0, 0);
        return;
    }
    const int mo = batch_map_off(c, b, begin);
    const uint32_t tsize = c.table_size, tmask = tsize - 1;
    const uint32_t qmask = (uint32_t)q - 1;
    const int qbits = ilog2((uint32_t)q);
    const uint32_t* __restrict__ ids = c.idx + begin;
    for (int i = lane; i < q; i += 32) { kkey[i] = kEmpty; kpos[i] = kEmpty; }
    for (int i = lane; i < (int)tsize; i += 32) tpos[i] = kEmpty;
    __syncwarp();
    // phase 1: first occurrences.  The set holds at most u_bound + 32 distinct ids.
    int fresh = 0;
    bool overflow = false;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        if (i < n && !overflow) {
            const uint32_t id = __ldg(ids + i);
            uint32_t h = (id * 0x9E3779B1u) >> (32 - qbits);
            for (;;) {
                const uint32_t prev = atomicCAS(&kkey[h], kEmpty, id);
                if (prev == kEmpty) fresh++;
                if (prev == kEmpty || prev == id) break;
                h = (h + 1) & qmask;
            }
            atomicMin(&kpos[h], (uint32_t)i);
            kslot[i] = (uint16_t)h;
        }
        const int tot = __reduce_add_sync(0xffffffffu, fresh);  // one REDUX instead of five shuffles
        overflow = tot > u_bound;  // uniform: stop before the set can fill up
        if (overflow) break;
    }
    const int nu = __reduce_add_sync(0xffffffffu, fresh);
    if (overflow || nu > (int)tsize) {
        // more unique ids than table slots: the reference's chain would exceed table_size (strategies.py:283-284)
        if (lane == 0) {
            report_error(c, b, VR_ERR_HASH_FULL);
            c.counts[b] = make_int2(0, 0);
        }
        return;
    }
    __syncwarp();
    // phase 2: first occurrences enter the reference table in WAVES of 32, in position order.
    // When a wave starts every earlier first occurrence sits in its final slot, so the wave's
    // elements jump over those slots with a find-next-zero on an occupancy bitmap (that is what
    // the reference's probe loop does one slot at a time) and only compete among themselves:
    // atomicMin with displacement, the earlier position wins the slot (strategies.py:277-294).
    uint32_t* bitmap = reinterpret_cast<uint32_t*>(kslot + n_max);  // [max(1, tsize/32)] occupied slots
    const int n_words = tsize >= 32 ? (int)(tsize >> 5) : 1;
    for (int w = lane; w < n_words; w += 32) bitmap[w] = (tsize >= 32) ? 0u : ~((1u << tsize) - 1u);
    // list of first-occurrence positions, ascending (kept in rank_of until phase 3 rewrites it)
    {
        int run = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            const bool f = i < n && kpos[kslot[i]] == (uint32_t)i;
            const uint32_t m = __ballot_sync(0xffffffffu, f);
            if (f) rank_of[run + __popc(m & ((1u << lane) - 1))] = (uint16_t)i;
            run += __popc(m);
        }
    }
    __syncwarp();
    for (int w0 = 0; w0 < nu; w0 += 32) {
        uint32_t cur = (w0 + lane < nu) ? (uint32_t)rank_of[w0 + lane] : kEmpty;
        uint32_t h = cur != kEmpty ? hash_slot(__ldg(ids + cur), c.multiplier, c.table_bits) : 0u;
        uint32_t taken = kEmpty;  // slot this lane turned from empty to occupied
        while (__any_sync(0xffffffffu, cur != kEmpty)) {
            if (cur != kEmpty) {
                // next slot at or after h that no earlier wave occupies
                uint32_t wi = h >> 5;
                uint32_t bits = ~bitmap[wi] & (0xFFFFFFFFu << (h & 31));
                while (bits == 0) { wi = (wi + 1) & (uint32_t)(n_words - 1); bits = ~bitmap[wi]; }
                const uint32_t sl = (wi << 5) + (uint32_t)__ffs((int)bits) - 1;
                const uint32_t old = atomicMin(&tpos[sl], cur);
                if (old == kEmpty) {
                    taken = sl;  // a lane takes at most one empty slot per wave
                    cur = kEmpty;
                } else {
                    if (old > cur) cur = old;  // displaced a later insertion of this wave: carry it on
                    h = (sl + 1) & tmask;
                }
            }
        }
        __syncwarp();
        if (taken != kEmpty) atomicOr(&bitmap[taken >> 5], 1u << (taken & 31));
        __syncwarp();
    }
    // phase 3: ranks in table order, unique ids, slot of every id
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    int run = 0;
    for (int s0 = 0; s0 < (int)tsize; s0 += 32) {
        const int s = s0 + lane;
        const uint32_t p = s < (int)tsize ? tpos[s] : kEmpty;
        const uint32_t occ = __ballot_sync(0xffffffffu, p != kEmpty);
        if (p != kEmpty) {
            const int rk = run + __popc(occ & ((1u << lane) - 1));
            rank_of[s] = (uint16_t)rk;
            suid[rk] = __ldg(ids + p);
            kpos[kslot[p]] = (uint32_t)s;
        }
        run += __popc(occ);
    }
    __syncwarp();
    unsigned int csum = 0;
    int cmax = 0;
    uint16_t* __restrict__ amap = c.out.d_assembly_map ? c.out.d_assembly_map + mo : nullptr;
    for (int i = lane; i < n; i += 32) {
        const uint32_t s = kpos[kslot[i]];
        const uint32_t h0 = hash_slot(__ldg(ids + i), c.multiplier, c.table_bits);
        const int chain = (int)((s - h0) & tmask) + 1;
        csum += chain;
        cmax = max(cmax, chain);
        if (amap) amap[i] = rank_of[s];
    }
    csum = __reduce_add_sync(0xffffffffu, csum);
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    if (lane == 0) {
        c.counts[b] = make_int2(1, nu);
        atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_FAST], (unsigned long long)csum);
        atomicMax(&c.acc[ACC_MAX_CHAIN], (long long)cmax);
        if (c.enforce_budget && nu > c.max_unique) report_error(c, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K1 (phash): strategies.py:301-367 -- two-tier hashing.  The reference is a sequential emulation
// whose table layout and probe statistics depend on the exact order of events: per group of
// warp_width slots every element probes at most max_fast_probes slots of a table that already
// holds the group's earlier insertions, then the deferred elements are inserted one at a time by
// scanning warp_width-slot windows.  One WARP per batch: the batch, the table and the slot map
// live in shared memory; the elements are replayed in the reference's order, one at a time, and the
// probes of one element are examined by the lanes in parallel (see below); all lanes stage the batch and
// produce the outputs (occupied slots ranked in table order, strategies.py:370-380).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) phash_warp_kernel(RunCtx c, int n_max, int w, int mfp, int per_warp_bytes) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5;
    const int b = blockIdx.x * warps + wid;
    if (b >= c.n_batches || c.acc[ACC_ABORT]) return;
    const uint32_t tsize = c.table_size, tmask = tsize - 1;  // a power of two (HashConfig, strategies.py:78-80)
    unsigned char* base = smem_raw + (size_t)wid * per_warp_bytes;
    uint32_t* tab = reinterpret_cast<uint32_t*>(base);                  // [tsize] ids (the batch is read in place)
    int32_t* d_i = reinterpret_cast<int32_t*>(tab + tsize);             // deferred elements of a group: index,
    int32_t* d_p = d_i + 64;                                            //   slot where fast probing stopped,
    int32_t* d_chain = d_p + 64;                                        //   probes so far
    uint16_t* slot_map = reinterpret_cast<uint16_t*>(d_chain + 64);     // [n_max]
    uint16_t* rank_of = slot_map + n_max;                               // [tsize]
    uint8_t* occ = reinterpret_cast<uint8_t*>(rank_of + tsize);         // [tsize]
    int begin, n;
    if (!validate_batch(c, b, begin, n)) {
        if (lane == 0) c.counts[b] = make_int2(0, 0);
        return;
    }
    const int mo = batch_map_off(c, b, begin);
    const uint32_t* __restrict__ ids = c.idx + begin;
    for (int s = lane; s < (int)tsize; s += 32) occ[s] = 0;
    __syncwarp();
    int status = VR_OK;
    long long fast = 0, slow = 0;
    int max_chain = 0;
    // The reference's order of events is kept element by element (every element sees the table exactly as
    // the sequential emulation leaves it), but the PROBES of one element -- up to max_fast_probes slots, then
    // warp_width-slot windows -- are looked at by the lanes side by side: the table does not change while one
    // element probes, so "first slot that is free or holds the id" is a ballot + ffs instead of a chain of
    // dependent shared-memory loads.  All variables below are warp-uniform.
    for (int gb = 0; gb < n && status == VR_OK; gb += w) {  // strategies.py:321
        int nd = 0;
        const int top = min(gb + w, n);
        for (int i = gb; i < top; i++) {
            const uint32_t vid = __ldg(ids + i);
            const uint32_t p0 = hash_slot(vid, c.multiplier, c.table_bits);
            int chain = mfp, resolved = -1;
            for (int k0 = 0; k0 < mfp; k0 += 32) {  // :328, 32 probes at a time
                const int k = k0 + lane;
                const uint32_t sl = (p0 + (uint32_t)k) & tmask;
                const bool in = k < mfp;
                const bool fr = in && !occ[sl];
                const bool hit = in && !fr && tab[sl] == vid;
                const uint32_t stop = __ballot_sync(0xffffffffu, fr || hit);
                if (stop) {
                    const int first = __ffs((int)stop) - 1;
                    chain = k0 + first + 1;
                    resolved = (int)((p0 + (uint32_t)(k0 + first)) & tmask);
                    if (lane == first && fr) { occ[sl] = 1; tab[sl] = vid; }
                    break;
                }
            }
            __syncwarp();
            fast += chain;
            if (resolved >= 0) {
                if (lane == 0) slot_map[i] = (uint16_t)resolved;
                max_chain = max(max_chain, chain);
            } else {
                if (lane == 0) { d_i[nd] = i; d_p[nd] = (int)((p0 + (uint32_t)mfp) & tmask); d_chain[nd] = mfp; }
                nd++;
            }
        }
        __syncwarp();
        for (int d = 0; d < nd && status == VR_OK; d++) {  // :345
            const int i = d_i[d];
            uint32_t p = (uint32_t)d_p[d];
            int chain = d_chain[d];
            const uint32_t vid = __ldg(ids + i);
            long long scanned = 0;
            for (;;) {
                if (scanned > (long long)tsize + w) { status = VR_ERR_HASH_FULL; break; }  // :348-349
                slow += w;  // :351
                int pos = 0;
                uint32_t psl = 0;
                for (int l0 = 0; l0 < w && !pos; l0 += 32) {  // ballot + ffs over the window
                    const int l = l0 + lane;
                    const uint32_t sl = (p + (uint32_t)l) & tmask;
                    const bool in = l < w;
                    const bool fr = in && !occ[sl];
                    const bool hit = in && !fr && tab[sl] == vid;
                    const uint32_t stop = __ballot_sync(0xffffffffu, fr || hit);
                    if (stop) {
                        const int first = __ffs((int)stop) - 1;
                        pos = l0 + first + 1;
                        psl = (p + (uint32_t)(pos - 1)) & tmask;
                        if (lane == first && fr) { occ[sl] = 1; tab[sl] = vid; }
                    }
                }
                __syncwarp();
                if (pos) {
                    if (lane == 0) slot_map[i] = (uint16_t)psl;
                    max_chain = max(max_chain, chain + pos);
                    break;
                }
                p = (p + (uint32_t)w) & tmask;
                chain += w;
                scanned += w;
            }
        }
        __syncwarp();
    }
    status = __shfl_sync(0xffffffffu, status, 0);
    __syncwarp();
    if (status != VR_OK) {
        if (lane == 0) { report_error(c, b, status); c.counts[b] = make_int2(0, 0); }
        return;
    }
    // occupied slots ranked in table order, unique ids, local indices
    uint32_t* __restrict__ suid = c.stage_uid + stage_uid_base(c, b, mo);
    int run = 0;
    for (int s0 = 0; s0 < (int)tsize; s0 += 32) {
        const int s = s0 + lane;
        const bool o = s < (int)tsize && occ[s];
        const uint32_t m = __ballot_sync(0xffffffffu, o);
        if (o) {
            const int rk = run + __popc(m & ((1u << lane) - 1));
            rank_of[s] = (uint16_t)rk;
            suid[rk] = tab[s];
        }
        run += __popc(m);
    }
    __syncwarp();
    if (c.out.d_assembly_map)
        for (int i = lane; i < n; i += 32) c.out.d_assembly_map[mo + i] = rank_of[slot_map[i]];
    if (lane == 0) {
        c.counts[b] = make_int2(1, run);
        atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_FAST], (unsigned long long)fast);
        atomicAdd((unsigned long long*)&c.acc[ACC_PROBES_SLOW], (unsigned long long)slow);
        atomicMax(&c.acc[ACC_MAX_CHAIN], (long long)max_chain);
        if (c.enforce_budget && run > c.max_unique) report_error(c, b, VR_ERR_OVER_BUDGET);
    }
}

// ---------------------------------------------------------------------------------
// K2: exclusive scan of per-segment (rounds, invocations).  Up to 32768 segments one CTA
// does it all; beyond that, 1024-segment tiles are reduced, the tile sums scanned by the
// same single-CTA kernel, and a down-sweep writes the per-segment offsets.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) scan_block_kernel(RunCtx c, const int2* __restrict__ in, int2* __restrict__ out, int n) {
    __shared__ long long wr[32], wu[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + 1023) >> 10;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    long long r = 0, u = 0;
    for (int k = lo; k < hi; k++) { const int2 v = in[k]; r += v.x; u += v.y; }
    long long ir = r, iu = u;  // inclusive scan over the CTA's 1024 partial sums
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long tr = __shfl_up_sync(0xffffffffu, ir, d), tu = __shfl_up_sync(0xffffffffu, iu, d);
        if (lane >= d) { ir += tr; iu += tu; }
    }
    if (lane == 31) { wr[wid] = ir; wu[wid] = iu; }
    __syncthreads();
    if (wid == 0) {
        long long xr = wr[lane], xu = wu[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long tr = __shfl_up_sync(0xffffffffu, xr, d), tu = __shfl_up_sync(0xffffffffu, xu, d);
            if (lane >= d) { xr += tr; xu += tu; }
        }
        wr[lane] = xr;
        wu[lane] = xu;
    }
    __syncthreads();
    long long br = (wid ? wr[wid - 1] : 0) + ir - r, bu = (wid ? wu[wid - 1] : 0) + iu - u;
    for (int k = lo; k < hi; k++) {
        const int2 v = in[k];
        out[k] = make_int2((int)min(br, 0x7fffffffLL), (int)min(bu, 0x7fffffffLL));
        br += v.x;
        bu += v.y;
    }
    if (tid == 1023) {
        const long long R = wr[31], U = wu[31];
        out[n] = make_int2((int)min(R, 0x7fffffffLL), (int)min(U, 0x7fffffffLL));
        finish_stats(c, R, U);
    }
}

__global__ void __launch_bounds__(256) scan_reduce_kernel(RunCtx c) {
    __shared__ int sr[8], su[8];
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int k0 = tile * 1024, k1 = min(c.n_segs, k0 + 1024);
    int r = 0, u = 0;
    for (int k = k0 + tid; k < k1; k += 256) { int2 v = c.seg_counts[k]; r += v.x; u += v.y; }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        r += __shfl_xor_sync(0xffffffffu, r, d);
        u += __shfl_xor_sync(0xffffffffu, u, d);
    }
    if ((tid & 31) == 0) { sr[tid >> 5] = r; su[tid >> 5] = u; }
    __syncthreads();
    if (tid == 0) {
        int tr = 0, tu = 0;
        for (int w = 0; w < 8; w++) { tr += sr[w]; tu += su[w]; }
        c.tile_sums[tile] = make_int2(tr, tu);
    }
}

__global__ void __launch_bounds__(1024) scan_down_kernel(RunCtx c) {
    __shared__ int scratch[40];
    __shared__ int chunk_r[1024];
    __shared__ int chunk_u[1024];
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int k = tile * 1024 + tid;
    int2 v = k < c.n_segs ? c.seg_counts[k] : make_int2(0, 0);
    chunk_r[tid] = v.x;
    chunk_u[tid] = v.y;
    __syncthreads();
    block_exclusive_scan(chunk_r, 1024, scratch);
    block_exclusive_scan(chunk_u, 1024, scratch);
    const int2 base = c.tile_off[tile];
    if (k < c.n_segs) c.seg_off[k] = make_int2(base.x + chunk_r[tid], base.y + chunk_u[tid]);
    if (k == c.n_segs - 1) c.seg_off[c.n_segs] = c.tile_off[c.n_scan_tiles];
}

// ---------------------------------------------------------------------------------
// K3: one warp per segment.
// ---------------------------------------------------------------------------------
constexpr int kShadeThreads = 256;
#ifndef VR_SHADE_UNROLL
#define VR_SHADE_UNROLL 4
#endif
constexpr int kShadeUnroll = VR_SHADE_UNROLL;

// Streams `cnt` staged unique ids src[0..cnt) to outputs dst0.. with `width` cooperating lanes
// (l = lane within the group): coalesced id load, 16-byte gather, transform, coalesced stores.
template <int STRATEGY>
__device__ __forceinline__ void shade_stream(const RunCtx& c, const ShaderParams& sp, const uint32_t* __restrict__ src,
                                             int cnt, int64_t dst0, int l, int width, int naive_mo, int vbase, int batch,
                                             float4* keep = nullptr) {
    const bool want_uid = c.out.d_unique_ids != nullptr;
    const bool want_pos = sp.kind == VR_SHADER_POSITION;
    const bool want_attr = sp.attr_words && c.out.d_shaded_attr;
    const bool want_cnt = c.out.d_shade_counts != nullptr;
    const L2Policies pol = make_l2_policies();
    uint32_t* __restrict__ out_uid = c.out.d_unique_ids + dst0;
    float4* __restrict__ shaded = reinterpret_cast<float4*>(c.out.d_shaded4) + dst0;
    for (int j0 = 0; j0 < cnt; j0 += width * kShadeUnroll) {
        uint32_t uid[kShadeUnroll];
        float4 p[kShadeUnroll];
        bool live[kShadeUnroll];
#pragma unroll
        for (int u = 0; u < kShadeUnroll; u++) {
            const int j = j0 + u * width + l;
            uid[u] = j < cnt ? src[j] : 0u;
            live[u] = j < cnt && vertex_in_range(sp, (uint32_t)vbase + uid[u]);
            if (j < cnt && !live[u]) report_late_error(c, batch, VR_ERR_VERTEX_RANGE);
        }
        if (want_pos) {
#pragma unroll
            for (int u = 0; u < kShadeUnroll; u++)
                if (live[u]) p[u] = ldg_keep_f4(sp.pos4 + vbase + uid[u], pol.keep);
        }
#pragma unroll
        for (int u = 0; u < kShadeUnroll; u++) {
            const int j = j0 + u * width + l;
            if (j >= cnt) continue;
            if (want_uid) st_stream_u32(out_uid + j, uid[u], pol.stream);
            if (!live[u]) continue;
            if (want_pos) {
                const float4 rec = transform_position<true>(sp, p[u]);
                st_stream_f4(shaded + j, rec, pol.stream);
                if (keep) keep[j] = rec;  // (shared memory: the caller expands the batch's corners from it)
            }
            if (STRATEGY == VR_NAIVE && c.out.d_assembly_map) c.out.d_assembly_map[naive_mo + j] = (uint16_t)(j % c.ps);
            if (want_attr)
                for (int k = 0; k < sp.attr_words; k++)
                    c.out.d_shaded_attr[(dst0 + j) * sp.attr_words + k] = __ldg(sp.attr + ((int64_t)vbase + uid[u]) * sp.attr_words + k);
            if (want_cnt) atomicAdd(&c.out.d_shade_counts[vbase + uid[u]], 1);
        }
    }
}

template <int STRATEGY>
__global__ void __launch_bounds__(kShadeThreads) shade_kernel(RunCtx c, ShaderParams sp) {
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (kShadeThreads / 32) + (threadIdx.x >> 5);
    if (s >= c.n_segs || c.acc[ACC_ABORT]) return;
    const int2 off = c.seg_off[s];
    const int ps = c.ps;
    if (STRATEGY == VR_WARP) {
        // lanes <-> the 32 batches of the segment: round tables
        const int b = 32 * s + lane;
        const bool valid = b < c.n_batches;
        const int2 cnt = valid ? c.counts[b] : make_int2(0, 0);
        const int inc_r = warp_incl_scan(cnt.x, lane), inc_u = warp_incl_scan(cnt.y, lane);
        const int begin = valid ? __ldg(c.bbegin + b) : 0;
        const int mo = valid ? batch_map_off(c, b, begin) : 0;
        const int u0 = off.y + inc_u - cnt.y;
        if (valid) {
            const int r0 = off.x + inc_r - cnt.x;
            int run = u0;
            if (c.out.d_batch_round_off) c.out.d_batch_round_off[b] = r0;
            const uint32_t* srd = c.stage_round + stage_round_base(c, b, mo);
            for (int r = 0; r < cnt.x; r++) {
                const uint32_t w = srd[r];
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[r0 + r] = run;
                if (c.out.d_round_prims) c.out.d_round_prims[r0 + r] = (int)(w >> 8);
                run += (int)(w & 0xFFu);
            }
        }
        // unique ids: flat over the segment's outputs, 32 per step.  The owner batch of an output
        // comes from one warp-wide OR: lane L sets the bit of the last output of its batch, and an
        // output's owner is the first owner of the step plus the number of batch ends before it.
        const unsigned long long my_src = (unsigned long long)(c.stage_uid + stage_uid_base(c, b, mo));
        const int my_vbase = valid && sp.batch_base ? __ldg(sp.batch_base + b) : 0;
        const int ex = inc_u - cnt.y;
        const int tot = __shfl_sync(0xffffffffu, inc_u, 31);
        const bool want_uid = c.out.d_unique_ids != nullptr;
        const bool want_pos = sp.kind == VR_SHADER_POSITION;
        const bool want_attr = sp.attr_words && c.out.d_shaded_attr;
        const bool want_cnt = c.out.d_shade_counts != nullptr;
        uint32_t* __restrict__ out_uid = c.out.d_unique_ids + off.y;
        float4* __restrict__ shaded = reinterpret_cast<float4*>(c.out.d_shaded4) + off.y;
        const uint32_t lt = (1u << lane) - 1;
        int first_owner = 0;
        for (int j0 = 0; j0 < tot; j0 += 32 * kShadeUnroll) {
            uint32_t uid[kShadeUnroll];
            int vb[kShadeUnroll];
            bool live[kShadeUnroll];
            float4 p[kShadeUnroll];
#pragma unroll
            for (int u = 0; u < kShadeUnroll; u++) {
                const int jb = j0 + 32 * u;
                const int d = inc_u - jb - 1;
                const uint32_t ends = __reduce_or_sync(0xffffffffu, (cnt.y > 0 && d >= 0 && d < 32) ? (1u << d) : 0u);
                const int owner = (first_owner + __popc(ends & lt)) & 31;
                first_owner += __popc(ends);
                const int oex = __shfl_sync(0xffffffffu, ex, owner);
                const uint32_t* osrc = (const uint32_t*)__shfl_sync(0xffffffffu, my_src, owner);
                vb[u] = __shfl_sync(0xffffffffu, my_vbase, owner);
                const int j = jb + lane;
                uid[u] = j < tot ? osrc[j - oex] : 0u;
                live[u] = j < tot && vertex_in_range(sp, (uint32_t)vb[u] + uid[u]);
                if (j < tot && !live[u]) report_late_error(c, 32 * s + owner, VR_ERR_VERTEX_RANGE);
            }
            if (want_pos) {
#pragma unroll
                for (int u = 0; u < kShadeUnroll; u++)
                    if (live[u]) p[u] = __ldg(sp.pos4 + vb[u] + uid[u]);
            }
#pragma unroll
            for (int u = 0; u < kShadeUnroll; u++) {
                const int j = j0 + 32 * u + lane;
                if (j >= tot) continue;
                if (want_uid) out_uid[j] = uid[u];
                if (!live[u]) continue;
                if (want_pos) shaded[j] = transform_position<true>(sp, p[u]);
                if (want_attr)
                    for (int k = 0; k < sp.attr_words; k++)
                        c.out.d_shaded_attr[((int64_t)off.y + j) * sp.attr_words + k] = __ldg(sp.attr + ((int64_t)vb[u] + uid[u]) * sp.attr_words + k);
                if (want_cnt) atomicAdd(&c.out.d_shade_counts[vb[u] + uid[u]], 1);
            }
        }
    } else {
        const int b = s;
        const int2 cnt = c.counts[b];
        const int begin = __ldg(c.bbegin + b);
        const int mo = batch_map_off(c, b, begin);
        if (lane == 0 && c.out.d_batch_round_off) c.out.d_batch_round_off[b] = off.x;
        const uint32_t* src;
        if (STRATEGY == VR_NAIVE) {  // one round per primitive, closed form
            for (int r = lane; r < cnt.x; r += 32) {
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[off.x + r] = off.y + r * ps;
                if (c.out.d_round_prims) c.out.d_round_prims[off.x + r] = 1;
            }
            src = c.idx + begin;
        } else {
            if (lane == 0 && cnt.x > 0) {
                if (c.out.d_round_uid_off) c.out.d_round_uid_off[off.x] = off.y;
                if (c.out.d_round_prims) c.out.d_round_prims[off.x] = (__ldg(c.bend + b) - begin) / ps;
            }
            src = c.stage_uid + stage_uid_base(c, b, mo);
        }
        shade_stream<STRATEGY>(c, sp, src, cnt.y, off.y, lane, 32, mo, sp.batch_base ? __ldg(sp.batch_base + b) : 0, b);
    }
}

#include "vr_dyn3.cuh"

// ---------------------------------------------------------------------------------
// strategies.py:456-463 expanded per-corner stream (the paper's stage output queue).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) expand_kernel(const int32_t* __restrict__ bro, const int32_t* __restrict__ ruo,
                                                      const int32_t* __restrict__ rprims, const uint16_t* __restrict__ amap,
                                                      const uint32_t* __restrict__ uids, const float4* __restrict__ shaded,
                                                      int n_batches, const int32_t* __restrict__ map_off, int ps,
                                                      float* __restrict__ out_pos3, uint32_t* __restrict__ out_ids,
                                                      int32_t* __restrict__ out_src, const int32_t* __restrict__ contiguous_begin = nullptr) {
    __shared__ float s_row[8][96];  // 32 records of a warp on their way out: see below
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int b = blockIdx.x * (blockDim.x >> 5) + wid;
    if (b >= n_batches) return;
    // (batches that tile one range of the buffer sit in the map where they sit in the buffer: no span scan)
    int m = contiguous_begin ? contiguous_begin[b] - contiguous_begin[0] : map_off[b];
    float* row = s_row[wid];
    for (int r = bro[b]; r < bro[b + 1]; r++) {
        const int base = ruo[r];
        const int slots = rprims[r] * ps;
        for (int k0 = 0; k0 < slots; k0 += 32) {
            const int k = k0 + lane;
            if (k < slots) {
                const int src = base + amap[m + k];
                if (out_src) out_src[m + k] = src;
                if (out_ids) out_ids[m + k] = uids[src];
                if (out_pos3) {
                    const float4 v = shaded[src];
                    row[3 * lane] = v.x; row[3 * lane + 1] = v.y; row[3 * lane + 2] = v.z;
                }
            }
            if (out_pos3) {
                // the 32 records are 96 consecutive floats: three coalesced 4-byte stores per lane instead of a
                // 12-byte record per lane (12 sectors per store instruction)
                __syncwarp();
                const int words = 3 * min(32, slots - k0);
                float* q = out_pos3 + 3 * (int64_t)(m + k0);
#pragma unroll
                for (int w = 0; w < 3; w++)
                    if (lane + 32 * w < words) q[lane + 32 * w] = row[lane + 32 * w];
                __syncwarp();
            }
        }
        m += slots;
    }
}

// Exclusive scan of the batch spans -> position of every batch in the concatenated assembly map.  One CTA; every
// thread owns a run of consecutive batches (two passes over its run, one CTA-wide scan of the 1024 partial sums) --
// not a loop of CTA barriers per 1024 batches (0.4 ms for the 225 000 batches of configs[2]).
__global__ void __launch_bounds__(1024) span_only_scan_kernel(const int32_t* __restrict__ bbegin, const int32_t* __restrict__ bend,
                                                               int n_batches, int32_t* __restrict__ map_off) {
    __shared__ long long wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n_batches + 1023) >> 10;
    const int lo = min(n_batches, tid * per), hi = min(n_batches, lo + per);
    long long mine = 0;
    for (int b = lo; b < hi; b++) mine += bend[b] - bbegin[b];
    long long inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        long long x = wsum[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += t;
        }
        wsum[lane] = x;
    }
    __syncthreads();
    long long run = (wid ? wsum[wid - 1] : 0) + inc - mine;
    for (int b = lo; b < hi; b++) {
        map_off[b] = (int32_t)run;
        run += bend[b] - bbegin[b];
    }
    if (tid == 1023) map_off[n_batches] = (int32_t)wsum[31];
}

// multi-draw: first vertex of the draw that holds each batch (include/vrgeom.h vr_batch_vertex_base)
__global__ void __launch_bounds__(256) batch_vertex_base_kernel(const int32_t* __restrict__ bbegin, int64_t nb,
                                                                const int32_t* __restrict__ draw_start,
                                                                const int32_t* __restrict__ draw_vbase, int n_draws,
                                                                int32_t* __restrict__ out) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int pos = bbegin[b];
    int lo = 0, hi = n_draws;  // last draw with draw_start[d] <= pos (empty draws share a start: the last one wins)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (draw_start[mid] <= pos) lo = mid; else hi = mid;
    }
    out[b] = draw_vbase[lo];
}

// float4 (x/w, y/w, z/w, w) -> the reference's float32[3] record: 4 records in, 3 x 16 bytes out per thread
__global__ void __launch_bounds__(256) pack_xyz_kernel(const float4* __restrict__ in, int64_t n, float* __restrict__ out) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // group of 4 records
    const int64_t i = 4 * q;
    if (i + 4 <= n) {
        const float4 a = in[i], b = in[i + 1], c4 = in[i + 2], d = in[i + 3];
        float4* o = reinterpret_cast<float4*>(out + 3 * i);
        o[0] = make_float4(a.x, a.y, a.z, b.x);
        o[1] = make_float4(b.y, b.z, c4.x, c4.y);
        o[2] = make_float4(c4.z, d.x, d.y, d.z);
    } else {
        for (int64_t k = i; k < n; k++) {
            const float4 v = in[k];
            out[3 * k] = v.x; out[3 * k + 1] = v.y; out[3 * k + 2] = v.z;
        }
    }
}

// uint16 local indices -> bytes, 16 per thread (the map is padded to a multiple of 8 entries by every caller of vr_run)
__global__ void __launch_bounds__(256) pack_u8_kernel(const uint16_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out, int32_t* flag) {
    const int64_t i = 16 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    uint32_t big = 0;
    if (i + 16 <= n && (((uintptr_t)(in + i)) & 15) == 0 && (((uintptr_t)(out + i)) & 15) == 0) {
        const uint4 a = *reinterpret_cast<const uint4*>(in + i), b = *reinterpret_cast<const uint4*>(in + i + 8);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            big |= (w[2 * k] | w[2 * k + 1]) & 0xFF00FF00u;
            o[k] = __byte_perm(w[2 * k], w[2 * k + 1], 0x6420);
        }
        *reinterpret_cast<uint4*>(out + i) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
        for (int64_t k = i; k < n && k < i + 16; k++) { big |= in[k] & 0xFF00u; out[k] = (uint8_t)in[k]; }
    }
    if (big && flag) *flag = 1;
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
    size_t map_off, counts, seg_counts, seg_off, tile_sums, tile_off, acc, tile_state, stage_uid, stage_round, aux, total;
    int stage_factor, seg_batches, n_segs, n_scan_tiles;
};

static WsLayout ws_layout(int strategy, int64_t span_total, int64_t nb, const vr_batch_config* cfg) {
    WsLayout L{};
    const int ps = cfg->primitive_size, w = cfg->warp_width;
    L.stage_factor = 1;
    if (strategy == VR_WARP) L.stage_factor = (int)ceil_div(w, w - ps + 1 > 0 ? w - ps + 1 : 1);
    L.seg_batches = strategy == VR_WARP ? 32 : 1;
    L.n_segs = (int)ceil_div(nb, L.seg_batches);
    L.n_scan_tiles = L.n_segs > 32768 ? (int)ceil_div(L.n_segs, 1024) : 0;
    size_t o = 0;
    L.map_off = o; o += align_up((size_t)(nb + 1) * 4);
    L.counts = o; o += align_up((size_t)(nb + 1) * 8);
    L.seg_counts = L.counts;
    if (L.seg_batches > 1) { L.seg_counts = o; o += align_up((size_t)(L.n_segs + 1) * 8); }
    L.seg_off = o; o += align_up((size_t)(L.n_segs + 2) * 8);
    L.tile_sums = o; o += align_up((size_t)(L.n_scan_tiles + 1) * 8);
    L.tile_off = o; o += align_up((size_t)(L.n_scan_tiles + 2) * 8);
    L.acc = o; o += align_up(ACC_WORDS * 8);
    // kRowThreads tiles (>= kFastThreads tiles) + the tile kernel's two group tables (one group = 32 tiles)
    // (and the kDyn3Warps-batch tiles of the three-kernel sort/hash path)
    L.tile_state = o; o += align_up((size_t)(ceil_div(nb, 8) + ceil_div(nb, 128) + 16 + 2 * (ceil_div(ceil_div(nb, 64), 32) + 1)) * 8);  // (>= dyn3_state_words(nb / 8))
    L.stage_uid = o;
    if (strategy != VR_NAIVE) {
        size_t words = (size_t)span_total * L.stage_factor + (size_t)nb * 8 + 64;
        if (strategy == VR_WARP) {  // the tile kernel keeps its claim lists here (vr_warp_rows.cuh)
            const size_t tw = rows_scratch_words(w, cfg->batch_size, nb);
            if (tw > words) words = tw;
        } else {  // the three-kernel path: a fixed-stride slot per batch (vr_dyn3.cuh)
            const size_t dw = dyn3_dist_words(nb, cfg);
            if (dw > words) words = dw;
        }
        o += align_up(words * 4);
    }
    L.stage_round = o;
    if (strategy == VR_WARP) o += align_up(((size_t)span_total / ps + nb + 64) * 4);
    L.aux = o;  // vr_dyn3.cuh: home slot / table slot / group of every distinct id
    if (strategy == VR_HASH || strategy == VR_PHASH) o += align_up(dyn3_aux_bytes(nb, cfg));
    L.total = o;
    return L;
}

// Optional per-kernel timing of the last vr_run (a profiling aid for bench.py: CUDA events on
// the launching stream between the pipeline's kernels).  Per host thread, like the two "last run" values
// below: vr_run itself keeps no state, so concurrent callers on different threads / streams do not disturb
// each other's diagnostics.
static thread_local cudaEvent_t g_prof_ev[VR_PROFILE_STAGES + 1];
static thread_local int g_prof_on = 0, g_prof_marks = 0;
static thread_local int g_last_launches = 0;  // kernels launched by this thread's last vr_run
static thread_local int g_last_path = 0;      // see vr_last_kernel_path()
static inline void prof_mark(cudaStream_t s) {
    if (g_prof_on && g_prof_marks <= VR_PROFILE_STAGES) cudaEventRecord(g_prof_ev[g_prof_marks++], s);
}

template <int W>
static int launch_warp_tpb(const RunCtx& c, cudaStream_t stream) {
    const size_t smem = (size_t)kTpbThreads * (64 + 4 * W + 2 * W + 2 * 16);
    if (smem > 48 * 1024)
        VR_CUDA_CHECK(cudaFuncSetAttribute(warp_tpb_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    warp_tpb_kernel<W><<<(int)ceil_div(c.n_batches, kTpbThreads), kTpbThreads, smem, stream>>>(c);
    return VR_OK;
}

template <int W>
static int launch_warp_fast(const RunCtx& c, int bs, bool fused, const ShaderParams& sp, cudaStream_t stream) {
    const size_t smem = (size_t)kFastThreads * (64 + 4 * W + 2 * W);
    const int blocks = (int)ceil_div(c.n_batches, kFastThreads);
    if (fused) {
        if (smem > 48 * 1024)
            VR_CUDA_CHECK(cudaFuncSetAttribute(warp_fast_kernel<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        warp_fast_kernel<W, true><<<blocks, kFastThreads, smem, stream>>>(c, bs, sp);
    } else {
        if (smem > 48 * 1024)
            VR_CUDA_CHECK(cudaFuncSetAttribute(warp_fast_kernel<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        warp_fast_kernel<W, false><<<blocks, kFastThreads, smem, stream>>>(c, bs, sp);
    }
    return VR_OK;
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
    case VR_ERR_VERTEX_RANGE: return "index outside the vertex buffer";
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
    strategy &= 0xFF;
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
    strategy &= 0xFF;
    if (vr_check_batch_config(cfg)) return 0;
    if (strategy == VR_WARP && cfg->warp_width < cfg->primitive_size) return 0;
    return ws_layout(strategy, span_total, nb, cfg).total;
}

static int run_impl(int strategy, const uint32_t* d_idx, int64_t n_idx, const int32_t* d_bbegin, const int32_t* d_bend,
                    int64_t nb, int64_t span_total, int32_t max_span, const vr_batch_config* cfg, const vr_hash_config* hcfg,
                    const vr_shader* shader, const vr_outputs* out, void* d_ws, size_t ws_bytes, void* stream_,
                    const int64_t* d_n_batches) {
    const bool no_budget = (strategy & VR_FLAG_NO_BUDGET) != 0;
    const bool static_batches = (strategy & VR_FLAG_STATIC) != 0;
    const bool allow_fuse = (strategy & VR_FLAG_NO_FUSE) == 0;
    const bool contiguous = (strategy & VR_FLAG_CONTIGUOUS) != 0 || static_batches;
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
    if (n_idx > 0x7fffffffLL || nb > 0x7fffffffLL || span_total > 0x7fffffffLL || n_idx < 0 || nb < 0 || span_total < 0)
        return VR_ERR_UNSUPPORTED;
    if (strategy == VR_WARP && nb > 0 && cfg->warp_width < cfg->primitive_size) return VR_ERR_WARP_WIDTH;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (((uintptr_t)d_idx & 15) != 0) return VR_ERR_UNSUPPORTED;  // 16-byte index loads
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
    c.contiguous = contiguous ? 1 : 0;
    c.seg_batches = L.seg_batches;
    c.n_segs = L.n_segs;
    c.n_scan_tiles = L.n_scan_tiles;
    c.span_cap = span_total;
    unsigned char* ws = (unsigned char*)d_ws;
    c.map_off = (int32_t*)(ws + L.map_off);
    c.counts = (int2*)(ws + L.counts);
    c.seg_counts = (int2*)(ws + L.seg_counts);
    c.seg_off = (int2*)(ws + L.seg_off);
    c.tile_sums = (int2*)(ws + L.tile_sums);
    c.tile_off = (int2*)(ws + L.tile_off);
    c.acc = (long long*)(ws + L.acc);
    c.tile_state = (unsigned long long*)(ws + L.tile_state);
    c.stage_uid = (uint32_t*)(ws + L.stage_uid);
    c.stage_round = (uint32_t*)(ws + L.stage_round);
    c.out = RunOut{out->d_batch_round_off, out->d_round_uid_off, out->d_round_prims, out->d_unique_ids, out->d_assembly_map,
                   out->d_shaded4, out->d_shaded_attr, out->d_shade_counts, out->d_stats, out->cap_unique, out->cap_rounds};
    ShaderParams sp{};
    if (shader) {
        sp.kind = shader->kind; sp.has_matrix = shader->has_matrix;
        for (int i = 0; i < 16; i++) sp.m[i] = shader->matrix[i];
        sp.pos4 = (const float4*)shader->d_positions4; sp.attr = shader->d_attributes;
        sp.attr_words = shader->d_attributes ? shader->attr_words : 0; sp.vertex_count = shader->vertex_count;
        sp.batch_base = shader->d_batch_vertex_base;
        sp.extra_cycles = shader->extra_cycles > 0 ? shader->extra_cycles : 0;
        sp.load_a = 1.0f; sp.load_b = 0.0f;
        if (sp.kind == VR_SHADER_POSITION && (!sp.pos4 || !out->d_shaded4)) return VR_ERR_BAD_CONFIG;
    }
    const bool want_queue = out->d_stream_xyz != nullptr && sp.kind == VR_SHADER_POSITION && nb > 0;
    if (want_queue && (!out->d_assembly_map || !out->d_batch_round_off || !out->d_round_uid_off || !out->d_round_prims))
        return VR_ERR_BAD_CONFIG;
    const int nbi = (int)nb;
    // limits of the CTA-per-batch kernels
    int pmax = 0, nmax = 0, q = 0;
    size_t smem = 0;
    if (strategy == VR_SORT && nb > 0) {
        if (max_span > 8192) return VR_ERR_UNSUPPORTED;
        pmax = (int)next_pow2((uint32_t)(max_span < 2 ? 2 : max_span));
        smem = (size_t)pmax * (8 + 4 + 2);
        VR_CUDA_CHECK(cudaFuncSetAttribute(sort_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    } else if (strategy == VR_PHASH && nb > 0) {
        if (max_span > 65535 || hc.table_size > 65536) return VR_ERR_UNSUPPORTED;  // 16-bit slot map / ranks
    } else if (strategy == VR_HASH && nb > 0) {
        nmax = (max_span + 3) & ~3;
        q = (int)next_pow2((uint32_t)(2 * nmax < 64 ? 64 : 2 * nmax));
        smem = (size_t)nmax * 4 + (size_t)q * 8 + (size_t)hc.table_size * 12 + (size_t)nmax * 2 + (size_t)nmax + 16;
        if (smem > 200 * 1024 || max_span > 65535) return VR_ERR_UNSUPPORTED;
        VR_CUDA_CHECK(cudaFuncSetAttribute(hash_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }

    // (the position-aligned kernels read one vertex buffer: multi-draw runs take the general path)
    const bool fast_warp = strategy == VR_WARP && static_batches && ps == 3 && cfg->batch_size % 8 == 0 && nb > 0 && !sp.batch_base;
    const bool fused = fast_warp && allow_fuse && sp.extra_cycles == 0;  // (the fused kernels shade without the synthetic load)
    // tile kernel (vr_warp_rows.cuh) when a batch row fits shared memory comfortably
    RowsGeom rg{};
    // (its packed table entries hold 24-bit ids: the caller must state a vertex count that fits)
    const bool rows = fused && rows_geometry(cfg->warp_width, cfg->batch_size, rg) &&
                      (((uintptr_t)out->d_assembly_map) & 15) == 0 && shader && shader->vertex_count > 0 &&
                      shader->vertex_count <= (1 << 24);
    // budgeted sort / hash / phash batches: the three-kernel path of vr_dyn3.cuh
    Dyn3Plan d3 = dyn3_plan(strategy, cfg, hc, max_span, c.enforce_budget != 0, shader, out);
    if (!allow_fuse || nb == 0 || nb >= (1 << 30)) d3.ok = false;
    d3.g.aux = ws + L.aux;
    d3.g.queue = out->d_stream_xyz;
    d3.g.nb_dev = d_n_batches;
    if (d_n_batches && !d3.ok) return VR_ERR_UNSUPPORTED;  // (the device-side batch count is implemented by the three-kernel path)
    d3.g.prefetch = debug_knobs().dyn3_prefetch;
    // (short runs: fewer batches per CTA of the set dedup, so that the grid still covers the GPU)
    d3.g.tile_shift = nb >= 16384 ? 5 : nb >= 4096 ? 4 : 3;
    if (debug_knobs().dyn3_tile_shift >= 3 && debug_knobs().dyn3_tile_shift <= 5) d3.g.tile_shift = debug_knobs().dyn3_tile_shift;
    c.n_fused_tiles = rows ? (int)ceil_div(nb, kRowThreads) : fused ? (int)ceil_div(nb, kFastThreads) : d3.ok ? (int)ceil_div(nb, (int64_t)1 << d3.g.tile_shift) : 0;
    g_prof_marks = 0;
    g_last_path = rows ? 3 : fused ? 2 : fast_warp ? 1 : d3.ok ? 4 : 0;
    prof_mark(stream);
    c.n_state_words = rows ? c.n_fused_tiles + 1 + 2 * ((int)ceil_div(c.n_fused_tiles, kRowGroup) + 1)
                      : d3.ok ? dyn3_state_words(c.n_fused_tiles) : c.n_fused_tiles;
    init_kernel<<<(int)ceil_div(c.n_state_words + ACC_WORDS, 256), 256, 0, stream>>>(c);
    if (!contiguous && nb > 0) span_scan_kernel<<<1, 1024, 0, stream>>>(c);
    prof_mark(stream);
    if (nb > 0) {
        if (strategy == VR_NAIVE) {
            naive_counts_kernel<<<(nbi + 255) / 256, 256, 0, stream>>>(c);
        } else if (d3.ok) {
            const int tiles = c.n_fused_tiles, ftiles = (int)ceil_div(nb, kDyn3Warps);
            // long batches (strip-ordered meshes), sort: two elements per lane and step; see dyn3_dedup_kernel.  (With the
            // ordered numbering of hash / phash the wide variant measured slower on both kinds of mesh: 58 registers.)
            const bool wide = strategy == VR_SORT && span_total / nb >= 384;
            auto launch_a = [&](auto kernel) -> int {
                if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d3.smem_a) != cudaSuccess) return VR_ERR_CUDA;
                kernel<<<tiles, kDyn3Warps * 32, d3.smem_a, stream>>>(c, d3.g);
                return VR_OK;
            };
            if (strategy == VR_SORT) st = wide ? launch_a(dyn3_dedup_kernel<false, false, true>) : launch_a(dyn3_dedup_kernel<false, false, false>);
            else if (strategy == VR_HASH) st = launch_a(dyn3_dedup_kernel<true, false, false>);
            else st = launch_a(dyn3_dedup_kernel<true, true, false>);
            if (st) return st;
            if (strategy == VR_HASH) dyn3_insert_kernel<false><<<(int)ceil_div(nb, kDyn3InsertThreads), kDyn3InsertThreads, 0, stream>>>(c, d3.g);
            if (strategy == VR_PHASH)
                dyn3_insert_kernel<true><<<(int)ceil_div(nb, kDyn3InsertThreads / 2), kDyn3InsertThreads / 2, (size_t)2 * cfg->warp_width * (kDyn3InsertThreads / 2), stream>>>(c, d3.g);
            prof_mark(stream);
            prof_mark(stream);
            const size_t csmem = want_queue ? (size_t)kDyn3Warps * (256 * sizeof(float4) + 96 * sizeof(float)) : 0;  // the batch's shaded records + a row of the queue
            if (want_queue) {  // (static + dynamic shared memory is within 512 bytes of the 48 KB default: opt in explicitly)
                VR_CUDA_CHECK(cudaFuncSetAttribute(dyn3_finish_kernel<VR_SORT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
                VR_CUDA_CHECK(cudaFuncSetAttribute(dyn3_finish_kernel<VR_HASH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
                VR_CUDA_CHECK(cudaFuncSetAttribute(dyn3_finish_kernel<VR_PHASH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
            }
            auto launch_c = [&](auto kernel) { kernel<<<ftiles, kDyn3Warps * 32, csmem, stream>>>(c, sp, d3.g); };
            switch (strategy * 2 + (want_queue ? 1 : 0)) {
            case VR_SORT * 2: launch_c(dyn3_finish_kernel<VR_SORT, false>); break;
            case VR_SORT * 2 + 1: launch_c(dyn3_finish_kernel<VR_SORT, true>); break;
            case VR_HASH * 2: launch_c(dyn3_finish_kernel<VR_HASH, false>); break;
            case VR_HASH * 2 + 1: launch_c(dyn3_finish_kernel<VR_HASH, true>); break;
            case VR_PHASH * 2: launch_c(dyn3_finish_kernel<VR_PHASH, false>); break;
            default: launch_c(dyn3_finish_kernel<VR_PHASH, true>); break;
            }
            prof_mark(stream);
            g_last_launches = strategy == VR_SORT ? 3 : 4;
            VR_CUDA_CHECK(cudaGetLastError());
            return VR_OK;  // (kernel C wrote the queue)
        } else if (rows) {
            const int bs = cfg->batch_size;
            switch (cfg->warp_width) {
            case 4: st = launch_warp_rows<4>(c, bs, rg, sp, stream); break;
            case 8: st = launch_warp_rows<8>(c, bs, rg, sp, stream); break;
            case 16: st = launch_warp_rows<16>(c, bs, rg, sp, stream); break;
            case 32: st = launch_warp_rows<32>(c, bs, rg, sp, stream); break;
            default: st = launch_warp_rows<64>(c, bs, rg, sp, stream); break;
            }
            if (st) return st;
        } else if (fast_warp) {
            const int bs = cfg->batch_size;
            switch (cfg->warp_width) {
            case 4: st = launch_warp_fast<4>(c, bs, fused, sp, stream); break;
            case 8: st = launch_warp_fast<8>(c, bs, fused, sp, stream); break;
            case 16: st = launch_warp_fast<16>(c, bs, fused, sp, stream); break;
            case 32: st = launch_warp_fast<32>(c, bs, fused, sp, stream); break;
            default: st = launch_warp_fast<64>(c, bs, fused, sp, stream); break;
            }
            if (st) return st;
        } else if (strategy == VR_WARP) {
            switch (cfg->warp_width) {
            case 4: st = launch_warp_tpb<4>(c, stream); break;
            case 8: st = launch_warp_tpb<8>(c, stream); break;
            case 16: st = launch_warp_tpb<16>(c, stream); break;
            case 32: st = launch_warp_tpb<32>(c, stream); break;
            default: st = launch_warp_tpb<64>(c, stream); break;
            }
            if (st) return st;
        } else if (strategy == VR_PHASH) {
            const int wn = (max_span + 3) & ~3;
            const int per_warp = ((int)hc.table_size * 4 + 3 * 64 * 4 + wn * 2 + (int)hc.table_size * 2 + (int)hc.table_size + 15) & ~15;
            if (per_warp > 200 * 1024) return VR_ERR_UNSUPPORTED;
            int warps = 8;
            while (warps > 1 && warps * per_warp > 64 * 1024) warps >>= 1;
            const size_t wsmem = (size_t)warps * per_warp;
            VR_CUDA_CHECK(cudaFuncSetAttribute(phash_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
            phash_warp_kernel<<<(int)ceil_div(nb, warps), warps * 32, wsmem, stream>>>(c, wn, cfg->warp_width, (int)hc.max_fast_probes, per_warp);
        } else if (strategy == VR_SORT) {
            // one warp per batch (distinct ids, then a sort of those only) when its tables fit; else the CTA sort
            const int u_bound = c.enforce_budget && cfg->max_unique < max_span ? cfg->max_unique : max_span;
            const int wn = (max_span + 31) & ~31;
            const int wq = (int)next_pow2((uint32_t)((u_bound + 32) * 3 / 2 + 2));  // the set holds <= u_bound + 32 ids
            const int wp = (int)next_pow2((uint32_t)(u_bound + 32));
            const int per_warp = (wq * 4 + wp * 4 + wn * 2 + wq * 2 + 15) & ~15;
            // (a few long batches -- configs[0]: 509 batches of 768 -- do not fill the GPU with one warp each:
            // the CTA sort is faster there)
            const bool few_long = nb < 2048 && wp > 512;
            if (per_warp <= 24 * 1024 && wq <= 65536 && !few_long && !debug_knobs().sort_cta) {
                int warps = 8;
                while (warps > 1 && warps * per_warp > 64 * 1024) warps >>= 1;
                const size_t wsmem = (size_t)warps * per_warp;
                VR_CUDA_CHECK(cudaFuncSetAttribute(sort_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
                sort_warp_kernel<<<(int)ceil_div(nb, warps), warps * 32, wsmem, stream>>>(c, wn, wq, u_bound, wp, per_warp);
            } else {
                sort_batch_kernel<<<nbi, 256, smem, stream>>>(c, pmax);
            }
        } else {
            // one warp per batch when a warp's tables fit comfortably; else one CTA per batch
            const int u_bound = (uint32_t)max_span < hc.table_size ? max_span : (int)hc.table_size;
            const int wn = (max_span + 31) & ~31;
            const int wq = (int)next_pow2((uint32_t)((u_bound + 32) * 3 / 2 + 2));  // the set holds <= u_bound + 32 ids: load <= 2/3
            const int per_warp = (wq * 8 + (int)hc.table_size * 6 + wn * 2 + ((int)hc.table_size >> 3) + 4 + 15) & ~15;
            if (per_warp <= 24 * 1024 && hc.table_size <= 4096) {
                int warps = 8;
                while (warps > 1 && warps * per_warp > 64 * 1024) warps >>= 1;
                const size_t wsmem = (size_t)warps * per_warp;
                VR_CUDA_CHECK(cudaFuncSetAttribute(hash_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
                hash_warp_kernel<<<(int)ceil_div(nb, warps), warps * 32, wsmem, stream>>>(c, wn, wq, u_bound, per_warp);
            } else {
                hash_batch_kernel<<<nbi, 256, smem, stream>>>(c, nmax, q);
            }
        }
    }
    prof_mark(stream);
    // the output queue on the paths that do not write it inside the stage: a closing kernel (strategies.py:456-463)
    auto closing_queue = [&]() {
        if (!want_queue) return 0;
        if (!contiguous) span_only_scan_kernel<<<1, 1024, 0, stream>>>(d_bbegin, d_bend, nbi, c.map_off);
        expand_kernel<<<(int)ceil_div(nb, 8), 256, 0, stream>>>(out->d_batch_round_off, out->d_round_uid_off, out->d_round_prims,
                                                                 out->d_assembly_map, nullptr, (const float4*)out->d_shaded4, nbi, c.map_off, ps,
                                                                 out->d_stream_xyz, nullptr, nullptr, contiguous ? d_bbegin : nullptr);
        return contiguous ? 1 : 2;
    };
    if (fused) {
        prof_mark(stream);
        prof_mark(stream);
        g_last_launches = 2 + closing_queue();  // init + one kernel that dedups, places and shades
        VR_CUDA_CHECK(cudaGetLastError());
        return VR_OK;
    }
    if (L.n_scan_tiles == 0) {
        scan_block_kernel<<<1, 1024, 0, stream>>>(c, c.seg_counts, c.seg_off, c.n_segs);
    } else {
        scan_reduce_kernel<<<L.n_scan_tiles, 256, 0, stream>>>(c);
        scan_block_kernel<<<1, 1024, 0, stream>>>(c, c.tile_sums, c.tile_off, L.n_scan_tiles);
        scan_down_kernel<<<L.n_scan_tiles, 1024, 0, stream>>>(c);
    }
    prof_mark(stream);
    if (nb > 0) {
        const int blocks = (int)ceil_div(L.n_segs, kShadeThreads / 32);
        switch (strategy) {
        case VR_NAIVE: shade_kernel<VR_NAIVE><<<blocks, kShadeThreads, 0, stream>>>(c, sp); break;
        case VR_WARP: shade_kernel<VR_WARP><<<blocks, kShadeThreads, 0, stream>>>(c, sp); break;
        default: shade_kernel<VR_SORT><<<blocks, kShadeThreads, 0, stream>>>(c, sp); break;
        }
    }
    prof_mark(stream);
    g_last_launches = (nb > 0 ? 3 : 1) + ((!contiguous && nb > 0) ? 1 : 0) + (L.n_scan_tiles ? 3 : 1) + closing_queue();
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_run(int strategy, const uint32_t* d_idx, int64_t n_idx, const int32_t* d_bbegin, const int32_t* d_bend,
           int64_t nb, int64_t span_total, int32_t max_span, const vr_batch_config* cfg, const vr_hash_config* hcfg,
           const vr_shader* shader, const vr_outputs* out, void* d_ws, size_t ws_bytes, void* stream_) {
    return run_impl(strategy, d_idx, n_idx, d_bbegin, d_bend, nb, span_total, max_span, cfg, hcfg, shader, out, d_ws, ws_bytes, stream_, nullptr);
}

int64_t vr_dynamic_batch_bound(int64_t n, const vr_batch_config* cfg, int32_t n_draws) {
    if (vr_check_batch_config(cfg) || n <= 0) return 0;
    // batching.py:106-118: a batch closes because the next primitive would not fit, i.e. it holds more than
    // max_unique - ps distinct ids (so at least that many indices) or max_primitives primitives; only the last batch of
    // a draw may be shorter
    const int64_t ps = cfg->primitive_size;
    int64_t by_unique = (int64_t)cfg->max_unique - ps + 1;
    if (by_unique < ps) by_unique = ps;
    const int64_t by_cap = (cfg->max_indices / ps) * ps;
    const int64_t shortest = by_unique < by_cap ? by_unique : by_cap;
    return n / (shortest > 0 ? shortest : 1) + (n_draws > 0 ? n_draws : 1) + 1;
}

int vr_run_counted(int strategy, const uint32_t* d_idx, int64_t n_idx, const int32_t* d_offsets, int64_t nb_max,
                   const int64_t* d_n_batches, int32_t max_span, const vr_batch_config* cfg, const vr_hash_config* hcfg,
                   const vr_shader* shader, const vr_outputs* out, void* d_ws, size_t ws_bytes, void* stream_) {
    if (!d_n_batches || !d_offsets || nb_max <= 0) return VR_ERR_BAD_CONFIG;
    return run_impl((strategy & ~0xF00) | VR_FLAG_CONTIGUOUS | (strategy & VR_FLAG_NO_BUDGET), d_idx, n_idx, d_offsets, d_offsets + 1, nb_max,
                    n_idx, max_span, cfg, hcfg, shader, out, d_ws, ws_bytes, stream_, d_n_batches);
}

int vr_last_launch_count(void) { return g_last_launches; }
int vr_debug_reload_knobs(void) {
    debug_knobs_storage() = parse_debug_knobs();
    return VR_OK;
}
int vr_last_kernel_path(void) { return g_last_path; }

int vr_batch_vertex_base(const int32_t* d_batch_begin, int64_t n_batches, const int32_t* d_draw_index_start,
                         const int32_t* d_draw_vertex_base, int32_t n_draws, int32_t* d_out, void* stream) {
    if (n_batches < 0 || n_draws <= 0 || !d_draw_index_start || !d_draw_vertex_base) return VR_ERR_BAD_BATCH;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (n_batches == 0) return VR_OK;
    if (!d_batch_begin || !d_out) return VR_ERR_BAD_BATCH;
    batch_vertex_base_kernel<<<(int)ceil_div(n_batches, 256), 256, 0, (cudaStream_t)stream>>>(
        d_batch_begin, n_batches, d_draw_index_start, d_draw_vertex_base, n_draws, d_out);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

#ifdef VR_TIMELINE
// debugging aid (not part of the ABI): copies the phase time stamps of the last tile-kernel launch
int vr_debug_timeline(unsigned long long* host, int cap) {
    const int n = kTimelineMarks * 2 * kTimelineTiles;
    if (cap < n) return -n;
    if (cudaMemcpyFromSymbol(host, g_timeline, sizeof(unsigned long long) * n) != cudaSuccess) return 0;
    return n;
}
#endif

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
                                                             (const float4*)d_shaded4, (int)nb, map_off, ps, d_pos3, d_ids, nullptr);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_pack_xyz(const float* d_shaded4, int64_t n, float* d_xyz, void* stream) {
    if (n < 0) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (n == 0) return VR_OK;
    if (!d_shaded4 || !d_xyz || ((uintptr_t)d_xyz & 15) || ((uintptr_t)d_shaded4 & 15)) return VR_ERR_BAD_CONFIG;
    pack_xyz_kernel<<<(int)ceil_div(ceil_div(n, 4), 256), 256, 0, (cudaStream_t)stream>>>((const float4*)d_shaded4, n, d_xyz);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_pack_bytes(const uint16_t* d_map, int64_t n, uint8_t* d_out, int32_t* d_flag, void* stream) {
    if (n < 0) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (n == 0) return VR_OK;
    if (!d_map || !d_out) return VR_ERR_BAD_CONFIG;
    pack_u8_kernel<<<(int)ceil_div(ceil_div(n, 16), 256), 256, 0, (cudaStream_t)stream>>>(d_map, n, d_out, d_flag);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_expand_sources(const int32_t* d_bro, const int32_t* d_ruo, const int32_t* d_rprims, const uint16_t* d_amap, int64_t nb,
                      const int32_t* d_bbegin, const int32_t* d_bend, int32_t ps, int32_t* d_src, void* d_ws, size_t ws_bytes,
                      void* stream_) {
    if (nb <= 0) return VR_OK;
    if (ws_bytes < (size_t)(nb + 1) * 4 || !d_ws) return VR_ERR_WORKSPACE;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (!d_src) return VR_ERR_BAD_CONFIG;
    cudaStream_t stream = (cudaStream_t)stream_;
    int32_t* map_off = (int32_t*)d_ws;
    span_only_scan_kernel<<<1, 1024, 0, stream>>>(d_bbegin, d_bend, (int)nb, map_off);
    expand_kernel<<<(int)ceil_div(nb, 8), 256, 0, stream>>>(d_bro, d_ruo, d_rprims, d_amap, nullptr, nullptr, (int)nb, map_off, ps,
                                                             nullptr, nullptr, d_src);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

}  // extern "C"
