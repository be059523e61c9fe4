// vr_dynamic.cu -- exact parallel restatement of the greedy dynamic batch splitter
// (/root/reference/pkg/src/vrlab/batching.py:87-125).
//
// The reference walks the index buffer front to back with a Python set: a primitive joins the
// open batch iff |uniques U prim| <= max_unique and the primitive cap is not exceeded, except
// that the first primitive of a batch is always accepted (batching.py:106-118).  Every batch
// boundary depends on the previous one, so the scan is restated as two exact stages:
//
//  Stage A  next[s] = end of the greedy batch that would START at primitive s.  It depends on
//           s alone:  next[s] = max e <= min(T, s+cap) with
//                     #{ i in [ps*s, ps*e) : prev_occurrence(i) < ps*s } <= max_unique, e > s.
//           A1 (occurrence_links): nearest earlier / later position holding the same id,
//              exact within one batch window, from a per-warp shared-memory table walked in
//              32-wide steps (__match_any_sync orders duplicates inside a step).
//           A2 (greedy_next): every thread slides a two-pointer window over its own run of
//              start primitives; appending index i adds a unique iff prev[i] < window start,
//              retiring index i removes one iff nxt[i] >= window end.  No set, no hashing.
//  Stage B  the boundaries are the chain b0 = 0, b(k+1) = next[b(k)].  A chunk of the stream
//           is a function "entry offset -> (exit offset, batches emitted)"; these functions
//           compose associatively, so the chain is resolved by a reduce-then-scan over chunk
//           tables (B1 chunk tables, B2 group tables, B3 group scan, B4 chunk entries) and
//           B5 writes the offsets array (batching.py:128-137).
//
// Kernel choice (vr_dynamic_batches_draws below): batch windows up to ~4000 indices take the tile link
// kernel (A1), the shared-memory window walk (A2) and the shared-memory chain walks (B3/B4); longer
// windows fall back to the warp-synchronous link kernel and the global-memory walks.  Ablation knobs
// (environment, read per call): VR_LINKS_WARP=1, VR_GREEDY_GLOBAL=1, VR_WALK_GLOBAL=1 force the fallbacks;
// VR_LINK_TILE=<positions>, VR_GREEDY_RUN=<primitives> resize the tile / the per-thread run of the fallback.
#include "vr_common.cuh"

namespace vr {

constexpr int kNoLink = 0x7fffffff;  // "no later occurrence"
constexpr int kGroup = 64;           // chunks per group in the two-level scan

struct DynCtx {
    const uint32_t* __restrict__ ids;
    int n;        // indices
    int T;        // primitives
    int ps;
    int max_unique;
    int cap;      // max primitives per batch (batching.py:58-61)
    int window;   // ps * cap positions
    int tile;     // positions per A1 tile (multiple of 32)
    int slots;    // A1 table slots (any multiple of 32)
    int chunk;    // primitives per chunk, >= cap
    int n_chunks;
    int n_groups;
    int32_t* prev;
    int32_t* nxt;
    int32_t* next;     // [T]
    int32_t* c_exit;   // [n_chunks * cap]
    int32_t* c_cnt;    // [n_chunks * cap]
    int32_t* g_exit;   // [n_groups * cap]
    int32_t* g_cnt;    // [n_groups * cap]
    int32_t* g_entry;  // [n_groups + 1]
    int32_t* g_base;   // [n_groups + 1]
    int32_t* c_entry;  // [n_chunks]
    int32_t* c_base;   // [n_chunks]
    int32_t* offsets;  // out
    int64_t* n_batches;  // out: [0] count, [1] status
    // multi-draw streams: draw d owns positions [draw_start[d], draw_start[d+1]); a batch never
    // crosses a draw (the reference runs dynamic_batches once per draw).  NULL = one draw.
    const int32_t* __restrict__ draw_start;
    int n_draws;
    // a RANGE of the stream (multi-GPU, SURVEY.md 8e option (ii)): whole groups [g_lo, g_hi) = chunks [k_lo, k_hi) =
    // start primitives [s_lo, s_hi).  The whole stream: 0 .. n_groups / n_chunks / T.
    int g_lo, g_hi, k_lo, k_hi, s_lo, s_hi;
    int tile_lo;            // first tile of the link kernel
    int ranged;             // 1: offsets are written relative to the range's first batch, see vr_dynamic_range_*
    int32_t* r_table;       // [2 * cap] out: entry offset -> (exit offset, batches) of the whole range
    const int32_t* entry;   // [2] in (ranged): entry offset into the range, global number of its first batch
    int link_end;           // positions [.., link_end) have their prev[] link (n, or the range's end + one batch window)
    int want_nxt;           // 1: the link kernels also write nxt[] (the global-memory window walk reads it; the shared-memory one derives it from prev[])
    int entries_in_tables;  // 1: c_exit / c_cnt hold, per entry offset of the chunk's GROUP, the chunk's entry offset and the batches before it
};

// (the buffer starts 256-byte aligned and is padded: whole 16-byte stores)
__global__ void fill_kernel(int32_t* p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i < n) reinterpret_cast<int4*>(p)[i] = make_int4(v, v, v, v);
}

// ---- A1 -----------------------------------------------------------------------------------
// One warp per tile of positions, preceded by a halo of one batch window.  The table (open addressing,
// no deletions) holds every distinct id of tile + halo: `slots` is NOT a power of two (multiply-high
// hash), sized for a load of 0.8, and the last position of an id is kept relative to the halo start
// in 16 bits -- 6 bytes per slot instead of 16, which is what decides how many warps an SM can hold.
template <typename LastT>
__global__ void __launch_bounds__(128) occurrence_links_kernel(DynCtx c, int n_tiles, int per_warp_bytes) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tile_id = blockIdx.x * (blockDim.x >> 5) + wid;
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw + (size_t)wid * per_warp_bytes);
    LastT* last = reinterpret_cast<LastT*>(keys + c.slots);
    if (tile_id >= n_tiles) return;
    const uint32_t nslots = (uint32_t)c.slots;
    for (int i = lane; i < c.slots; i += 32) keys[i] = kEmpty;
    __syncwarp();
    const int t0 = tile_id * c.tile;
    const int t1 = min(c.n, t0 + c.tile);
    int hs = t0 - c.window;
    hs = hs < 0 ? 0 : (hs & ~31);
    const uint32_t lt = (1u << lane) - 1;
    for (int base = hs; base < t1; base += 32) {
        const int i = base + lane;
        const bool valid = i < t1;
        const uint32_t id = valid ? c.ids[i] : kEmpty;
        const uint32_t peers = __match_any_sync(0xffffffffu, id);
        const uint32_t lower = peers & lt;
        const bool leader = valid && lower == 0;
        const int hipeer = 31 - __clz(peers);
        uint32_t h = __umulhi(id * 0x9E3779B1u, nslots);
        bool active = leader, existed = false;
        while (__any_sync(0xffffffffu, active)) {
            uint32_t k = active ? keys[h] : 0u;
            bool claim = active && k == kEmpty;
            if (active && k == id) { existed = true; active = false; }
            if (claim) keys[h] = id;
            __syncwarp();
            if (claim) {
                if (keys[h] == id) active = false; else h = h + 1 == nslots ? 0u : h + 1;
            } else if (active) {
                h = h + 1 == nslots ? 0u : h + 1;
            }
            __syncwarp();
        }
        int pv = -1;
        if (leader) {
            if (existed) pv = hs + (int)last[h];
            last[h] = (LastT)(base + hipeer - hs);
        } else if (valid) {
            pv = base + (31 - __clz(lower));
        }
        __syncwarp();
        if (valid && i >= t0) {
            c.prev[i] = pv;
            if (pv >= 0 && c.want_nxt) c.nxt[pv] = i;
        }
    }
}

// ---- A1, tile version ------------------------------------------------------------------------
// One CTA per tile of 2048 positions (+ a halo of one batch window), one THREAD per position, no
// warp-synchronous probing: the positions are bucketed by id with a counting sort over the slots of
// a shared open-addressing table (insert + count, scan, scatter), then every tile position takes the
// largest earlier position in its bucket.  Buckets are unordered (the scatter uses atomics), so a
// position reads its whole bucket: a few entries for any mesh-like stream; ids with very many
// occurrences inside the window fall back to walking the index buffer backwards (their previous
// occurrence is then near on average).  Used when tile + halo fit 16-bit relative positions.
constexpr int kLinkThreads = 256;
constexpr int kBigBucket = 48;

__global__ void __launch_bounds__(kLinkThreads) occurrence_links_tile_kernel(DynCtx c, int tile, int halo, int nslots) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw);          // [nslots]
    uint32_t* cnt = keys + nslots;                                    // [nslots + 1] count, then bucket end
    uint16_t* slot_of = reinterpret_cast<uint16_t*>(cnt + nslots + 1);  // [tile + halo]
    uint16_t* bucket = slot_of + tile + halo;                         // [tile + halo] relative positions
    __shared__ uint32_t s_part[kLinkThreads];
    const int t = threadIdx.x;
    const int t0 = (c.tile_lo + blockIdx.x) * tile;
    const int t1 = min(c.n, t0 + tile);
    int hs = t0 - halo;
    if (hs < 0) hs = 0;
    const int np = t1 - hs;  // positions of halo + tile
    const uint32_t mask = (uint32_t)nslots - 1, shift = (uint32_t)__clz(nslots) + 1;  // nslots is a power of two: 32 - log2
    for (int i = t; i <= nslots; i += kLinkThreads) {
        if (i < nslots) keys[i] = kEmpty;
        cnt[i] = 0;
    }
    __syncthreads();
    // insert + count.  Every thread owns the positions t, t + 256, ... and inserts them as a per-lane STATE
    // MACHINE: one probe per trip; a lane whose probe resolves moves straight on to its next position
    // instead of waiting for the longest chain among the 32 lanes.  The loop then runs max-over-lanes of
    // the lane's TOTAL probes (~2 per position) rather than the sum of per-position maxima (~8 each;
    // ncu: 15 of 32 lanes active in the probe loop before).  The next position's id is loaded one ahead.
    {
        // the thread's positions t, t + 256, ...: pointers that move on when a probe resolves, a count of what is left
        const uint32_t* __restrict__ idp = c.ids + hs + t;
        uint16_t* slp = slot_of + t;
        int left = t < np ? (np - t + kLinkThreads - 1) / kLinkThreads : 0;
        uint32_t id = left > 0 ? idp[0] : 0u;
        uint32_t id_next = left > 1 ? idp[kLinkThreads] : 0u;
        // double hashing over a power-of-two table (odd step)
        uint32_t h = (id * 0x9E3779B1u) >> shift;
        uint32_t step = ((id * 0x85EBCA6Bu) >> shift) | 1u;
        // branch-free trips: every lane issues the two atomics (a lane whose probe collided, or that is done, on a word
        // of its own -- s_part is free until the scan), the next state is chosen by selects
        const uint32_t a_keys = (uint32_t)__cvta_generic_to_shared(keys), a_cnt = (uint32_t)__cvta_generic_to_shared(cnt);
        const uint32_t a_spare = (uint32_t)__cvta_generic_to_shared(&s_part[t]);
        while (__any_sync(0xffffffffu, left > 0)) {
            const bool active = left > 0;
            uint32_t k;
            asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(k) : "r"(active ? a_keys + 4u * h : a_spare), "r"(kEmpty), "r"(id) : "memory");
            const bool res = active && (k == kEmpty || k == id);
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(res ? a_cnt + 4u * h : a_spare) : "memory");
            if (res) *slp = (uint16_t)h;
            slp += res ? kLinkThreads : 0;
            idp += res ? kLinkThreads : 0;
            left -= res ? 1 : 0;
            const uint32_t idn = res ? id_next : id;
            if (res && left > 1) id_next = idp[kLinkThreads];
            h = res ? (idn * 0x9E3779B1u) >> shift : (h + step) & mask;
            step = res ? ((idn * 0x85EBCA6Bu) >> shift) | 1u : step;
            id = idn;
        }
    }
    __syncthreads();
    // exclusive scan of the counts -> bucket starts (cnt[h] becomes the start; the scatter turns it into the end)
    {
        const int per = ((nslots + kLinkThreads - 1) / kLinkThreads) | 1;  // odd: the threads' chunks start on different banks
        const int lo = t * per, hi = min(nslots, lo + per);
        uint32_t sum = 0;
        for (int i = lo; i < hi; i++) sum += cnt[i];
        s_part[t] = sum;
        __syncthreads();
        if (t < 32) {  // 256 partials: 8 per lane
            uint32_t v[8], tot = 0;
            for (int k = 0; k < 8; k++) { v[k] = s_part[t * 8 + k]; tot += v[k]; }
            uint32_t inc = tot;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (t >= d) inc += o;
            }
            uint32_t run = inc - tot;
            for (int k = 0; k < 8; k++) { s_part[t * 8 + k] = run; run += v[k]; }
        }
        __syncthreads();
        uint32_t run = s_part[t];
        for (int i = lo; i < hi; i++) { const uint32_t v = cnt[i]; cnt[i] = run; run += v; }
    }
    __syncthreads();
    // scatter
    for (int r = t; r < np; r += kLinkThreads) bucket[atomicAdd(&cnt[slot_of[r]], 1u)] = (uint16_t)r;
    __syncthreads();
    // nearest earlier occurrence of every tile position
    for (int r = t0 - hs + t; r < np; r += kLinkThreads) {
        const uint32_t h = slot_of[r];
        const uint32_t end = cnt[h], begin = h ? cnt[h - 1] : 0u;  // starts are the previous slot's end
        int pv = -1;
        if (end - begin <= (uint32_t)kBigBucket) {
            for (uint32_t e = begin; e < end; e++) {
                const int q = bucket[e];
                if (q < r && q > pv) pv = q;
            }
        } else {
            const uint32_t id = c.ids[hs + r];
            for (int q = r - 1; q >= 0; q--)
                if (c.ids[hs + q] == id) { pv = q; break; }
        }
        const int i = hs + r;
        const int pva = pv >= 0 ? hs + pv : -1;
        c.prev[i] = pva;
        if (pva >= 0 && c.want_nxt) c.nxt[pva] = i;
    }
}

// ---- A2 -----------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) greedy_next_kernel(DynCtx c, int run) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int s0 = t * run;
    if (s0 >= c.T) return;
    const int s1 = min(c.T, s0 + run);
    const int ps = c.ps;
    int e = s0, cnt = 0;
    // multi-draw: the window never grows past the end of the draw that holds its first primitive.
    // Occurrence links that cross a draw boundary are harmless: a link to an earlier draw lies
    // before every window start of this draw, a link to a later one past every window end.
    int d = 0, dend = c.T;
    if (c.draw_start) {
        int lo = 0, hi = c.n_draws;  // last d with draw_start[d] <= ps * s0
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (c.draw_start[mid] <= ps * s0) lo = mid; else hi = mid;
        }
        d = lo;
        dend = c.draw_start[d + 1] / ps;
    }
    for (int s = s0; s < s1; s++) {
        const int S = ps * s;
        while (s >= dend) dend = c.draw_start[++d + 1] / ps;  // (only with draws: dend == T otherwise)
        const int lim = min(dend, s + c.cap);
        if (e < s) { e = s; cnt = 0; }
        while (e < lim) {
            int fresh = 0;
            for (int k = 0; k < ps; k++) fresh += c.prev[ps * e + k] < S;
            if (e != s && cnt + fresh > c.max_unique) break;  // first primitive always accepted
            cnt += fresh;
            e++;
        }
        c.next[s] = e;
        const int E = ps * e;
        int lost = 0;
        for (int k = 0; k < ps; k++) lost += c.nxt[S + k] >= E;
        cnt -= lost;
    }
}

// A2 with the links of a CTA's stretch of the stream staged in shared memory.  In the kernel above every
// thread walks its own part of prev / nxt in global memory: a warp's 32 streams are 768 bytes apart, each
// step waits for the slowest lane's cache miss, and a trip takes ~1 us (ncu: 12 % issue utilisation, 70 % of
// the samples on the prev load).  Here the CTA first copies the links of its run of start primitives plus
// one batch window, coalesced, as 16-bit DISTANCES (position - prev, next - position; 65535 = none, which
// compares like "outside any window" because a window is shorter than that), then runs the same two-pointer
// walk out of shared memory.
template <int PS>
__global__ void __launch_bounds__(128) greedy_next_smem_kernel(DynCtx c, int run, int npos_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t* dp = reinterpret_cast<uint16_t*>(smem_raw);  // [npos_max] position - prev
    uint16_t* dn = dp + npos_max;                          // [npos_max] next - position
    const int ps = c.ps;
    const int p0 = c.s_lo + blockIdx.x * blockDim.x * run;  // first start primitive of the CTA
    const int base = ps * p0;
    const int npos = min(c.link_end - base, npos_max);  // (no position past link_end is needed by a start of the range)
    // Only prev[] is read: a position's NEXT occurrence inside the staged stretch is the position whose previous
    // occurrence it is, so the distances to the next occurrence are scattered in shared memory (every position has at
    // most one next occurrence: one writer per word).  A next occurrence past the staged stretch lies past every window
    // that can hold the position, like "none".  (No nxt[] array: 86 MB less written by the link kernel -- scattered
    // 4-byte stores --, 86 MB less read here, and no kernel to fill it with "none".)
    for (int q = threadIdx.x; q < (npos_max + 7) / 8; q += blockDim.x)  // "none" everywhere first (16-byte stores)
        reinterpret_cast<uint4*>(dn)[q] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    __syncthreads();
    auto put = [&](int r, int pv) {
        const int i = base + r;
        const int dd = pv < 0 || pv >= i ? 65535 : min(i - pv, 65535);
        dp[r] = (uint16_t)dd;
        if (dd <= r) dn[r - dd] = (uint16_t)dd;  // (dd = 65535 > r: the stretch is shorter than that)
    };
    if ((base & 3) == 0) {  // 16-byte loads, several in flight per thread: the copy is the bulk of this kernel's traffic
        const int4* __restrict__ pv4 = reinterpret_cast<const int4*>(c.prev + base);
        const int nq = npos >> 2;
#pragma unroll 4
        for (int qd = threadIdx.x; qd < nq; qd += blockDim.x) {
            const int4 a = __ldg(pv4 + qd);
            put(4 * qd, a.x); put(4 * qd + 1, a.y); put(4 * qd + 2, a.z); put(4 * qd + 3, a.w);
        }
        for (int r = 4 * nq + threadIdx.x; r < npos; r += blockDim.x) put(r, c.prev[base + r]);
    } else {
        for (int r = threadIdx.x; r < npos; r += blockDim.x) put(r, c.prev[base + r]);
    }
    __syncthreads();
    const int s0 = p0 + threadIdx.x * run;
    const int s1 = s0 < c.s_hi ? min(c.s_hi, s0 + run) : s0;  // (a thread past the end stays in the warp's votes, with no starts)
    int e = s0, cnt = 0;
    int d = 0, dend = c.T;
    if (c.draw_start && s0 < s1) {
        int lo = 0, hi = c.n_draws;  // last d with draw_start[d] <= ps * s0
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (c.draw_start[mid] <= ps * s0) lo = mid; else hi = mid;
        }
        d = lo;
        dend = c.draw_start[d + 1] / ps;
    }
    // The walk as a per-lane STATE MACHINE: a trip either appends primitive e to the window of start s, or closes s
    // (next[s] = e, its indices retire) and moves to s + 1 -- both sides are computed, selects pick.  A lane makes
    // (starts + appended primitives) trips whatever their order, so the warp makes about as many; with a loop per
    // start the warp ran the longest inner loop among its lanes for every start (ncu: 85 M warp instructions).
    int s = s0;
    if (PS == 3) {
        // triangles: the three distances of primitive e (to the previous occurrence) and of start s (to the next one)
        // stay in registers; a trip reloads only the triple that moved
        int dpv[3], dnv[3];
#pragma unroll
        for (int k = 0; k < 3; k++) { dpv[k] = dp[3 * s0 + k - base]; dnv[k] = dn[3 * s0 + k - base]; }
        // (e >= s throughout: a start's first primitive is always appended -- lim > s -- before the start can close, so
        // the restatement's "if (e < s) restart the window" never fires and is not compiled in here)
        auto trip = [&]() {
            const bool live = s < s1;
            if (c.draw_start) {
                while (live && s >= dend) dend = c.draw_start[++d + 1] / 3;
            }
            const int lim = min(dend, s + c.cap);
            const bool room = live && e < lim;
            const int gap = 3 * (e - s);  // E - S
            int fresh = 0, lost = 0;
#pragma unroll
            for (int k = 0; k < 3; k++) {
                fresh += room && dpv[k] > gap + k;   // prev < S
                lost += live && dnv[k] >= gap - k;   // next >= E
            }
            const bool adv = room && (e == s || cnt + fresh <= c.max_unique);  // first primitive always accepted
            if (live && !adv) c.next[s] = e;
            cnt += adv ? fresh : -lost;
            e += adv ? 1 : 0;
            s += live && !adv ? 1 : 0;
            const uint16_t* __restrict__ src = adv ? dp + (3 * e - base) : dn + (3 * s - base);
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const int v = src[k];
                dpv[k] = adv ? v : dpv[k];
                dnv[k] = adv ? dnv[k] : v;
            }
        };
        while (__any_sync(0xffffffffu, s < s1)) {  // two trips per vote (a finished lane's trip changes nothing)
            trip();
            trip();
        }
    } else {
    while (__any_sync(0xffffffffu, s < s1)) {
        const bool live = s < s1;
        const int S = ps * s;
        if (c.draw_start) {
            while (live && s >= dend) dend = c.draw_start[++d + 1] / ps;
        }
        const int lim = min(dend, s + c.cap);
        if (e < s) { e = s; cnt = 0; }
        const bool room = live && e < lim;
        int fresh = 0, lost = 0;
        const int E = ps * e;
        for (int k = 0; k < ps; k++) {
            const int i = E + k;
            fresh += room && (int)dp[room ? i - base : 0] > i - S;            // prev < S
            lost += live && (int)dn[live ? S + k - base : 0] >= E - (S + k);  // next >= E
        }
        const bool adv = room && (e == s || cnt + fresh <= c.max_unique);  // first primitive always accepted
        if (live && !adv) c.next[s] = e;
        cnt += adv ? fresh : -lost;
        e += adv ? 1 : 0;
        s += live && !adv ? 1 : 0;
    }
    }
}

// draw table sanity (multi-draw): starts at 0, ends at n, non-decreasing, primitive-aligned
__global__ void draws_check_kernel(DynCtx c) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d > c.n_draws) return;
    const int v = c.draw_start[d];
    bool bad = v % c.ps != 0 || v < 0 || v > c.n;
    if (d == 0) bad |= v != 0;
    if (d == c.n_draws) bad |= v != c.n;
    if (d < c.n_draws) bad |= c.draw_start[d + 1] < v;
    if (bad) c.n_batches[1] = VR_ERR_BAD_BATCH;
}

// ---- B1: chunk tables ---------------------------------------------------------------------
__global__ void __launch_bounds__(256) chunk_table_kernel(DynCtx c) {
    const int k = c.k_lo + blockIdx.x;
    const int lo = k * c.chunk, hi = min(c.T, lo + c.chunk);
    for (int o = threadIdx.x; o < c.cap; o += blockDim.x) {
        int s = lo + o, cnt = 0;
        while (s < hi) { s = c.next[s]; cnt++; }
        // entries at or past the end of the stream emit nothing and exit at offset 0
        c.c_exit[(size_t)k * c.cap + o] = s >= hi ? s - hi : 0;
        c.c_cnt[(size_t)k * c.cap + o] = cnt;
    }
}

// ---- B2: group tables (compose kGroup chunk tables for every entry offset) -----------------
__global__ void __launch_bounds__(256) group_table_kernel(DynCtx c) {
    const int g = c.g_lo + blockIdx.x;
    const int k0 = g * kGroup, k1 = min(c.n_chunks, k0 + kGroup);
    for (int o = threadIdx.x; o < c.cap; o += blockDim.x) {
        int e = o, cnt = 0;
        for (int k = k0; k < k1; k++) {
            size_t at = (size_t)k * c.cap + e;
            cnt += c.c_cnt[at];
            e = c.c_exit[at];
        }
        c.g_exit[(size_t)g * c.cap + o] = e;
        c.g_cnt[(size_t)g * c.cap + o] = cnt;
    }
}

// B1 / B2 out of shared memory.  In the two kernels above every thread follows a chain of dependent global loads
// (~12 batches per chunk, 64 chunk tables per group: ncu shows 48-60 warps waiting on the load per issued
// instruction, 34 + 36 us for the 7 M-triangle stream).  Here the CTA first copies what its chains walk through --
// the chunk's stretch of next[], the group's chunk tables -- coalesced, with all loads in flight, and the chains
// run out of shared memory.
__global__ void __launch_bounds__(256) chunk_table_smem_kernel(DynCtx c) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int* s_next = reinterpret_cast<int*>(smem_raw);  // [chunk] next start, relative to the chunk
    const int k = c.k_lo + blockIdx.x;
    const int lo = k * c.chunk, hi = min(c.T, lo + c.chunk), len = hi - lo;
#pragma unroll 4
    for (int i = threadIdx.x; i < len; i += blockDim.x) s_next[i] = __ldg(c.next + lo + i) - lo;
    __syncthreads();
    for (int o = threadIdx.x; o < c.cap; o += blockDim.x) {
        int s = o, cnt = 0;
        while (s < len) { s = s_next[s]; cnt++; }
        c.c_exit[(size_t)k * c.cap + o] = s >= len ? s - len : 0;
        c.c_cnt[(size_t)k * c.cap + o] = cnt;
    }
}
__global__ void __launch_bounds__(1024) group_table_smem_kernel(DynCtx c) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int g = c.g_lo + blockIdx.x;
    const int k0 = g * kGroup, k1 = min(c.n_chunks, k0 + kGroup), nr = k1 - k0;
    int* s_exit = reinterpret_cast<int*>(smem_raw);  // [nr][cap]
    int* s_cnt = s_exit + kGroup * c.cap;
    const int* __restrict__ ge = c.c_exit + (size_t)k0 * c.cap;
    const int* __restrict__ gc = c.c_cnt + (size_t)k0 * c.cap;
#pragma unroll 8
    for (int i = threadIdx.x; i < nr * c.cap; i += blockDim.x) {
        s_exit[i] = __ldg(ge + i);
        s_cnt[i] = __ldg(gc + i);
    }
    __syncthreads();
    // ... and, on the way, where a chain that enters the GROUP at offset o enters every chunk, and how many batches it
    // has emitted by then: written over the chunk tables (nothing reads them after this kernel), so that once the
    // group's true entry offset is known (B3) a chunk's entry is one look-up instead of a walk (B4)
    for (int o = threadIdx.x; o < c.cap; o += blockDim.x) {
        int e = o, cnt = 0;
        for (int r = 0; r < nr; r++) {
            const int at = r * c.cap + e;
            c.c_exit[(size_t)(k0 + r) * c.cap + o] = e;
            c.c_cnt[(size_t)(k0 + r) * c.cap + o] = cnt;
            cnt += s_cnt[at];
            e = s_exit[at];
        }
        c.g_exit[(size_t)g * c.cap + o] = e;
        c.g_cnt[(size_t)g * c.cap + o] = cnt;
    }
}

// ---- ranges (multi-GPU): the range's own table = its group tables composed, for every entry offset ----
__global__ void __launch_bounds__(256) range_table_kernel(DynCtx c) {
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < c.cap; o += gridDim.x * blockDim.x) {
        int e = o, cnt = 0;
        for (int g = c.g_lo; g < c.g_hi; g++) {
            const size_t at = (size_t)g * c.cap + e;
            cnt += c.g_cnt[at];
            e = c.g_exit[at];
        }
        c.r_table[o] = e;
        c.r_table[c.cap + o] = cnt;
    }
}
// ... and the entry of range `rank` from the tables of all ranges (gathered): the chain enters range 0 at offset
// 0; out[0] = entry offset into range `rank`, out[1] = number of its first batch, out[2] = batches of the stream
__global__ void range_entry_kernel(const int32_t* __restrict__ tables, int world, int rank, int cap, int32_t* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int e = 0, base = 0;
    for (int q = 0; q < world; q++) {
        if (q == rank) { out[0] = e; out[1] = base; }
        const int32_t* t = tables + (size_t)q * 2 * cap;
        base += t[cap + e];
        e = t[e];
    }
    out[2] = base;
}

// ---- B3: scan over groups (one thread; n_groups is T / (chunk * kGroup)) --------------------
__global__ void group_scan_kernel(DynCtx c) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int e = 0, base = 0;
    for (int g = 0; g < c.n_groups; g++) {
        c.g_entry[g] = e;
        c.g_base[g] = base;
        size_t at = (size_t)g * c.cap + e;
        base += c.g_cnt[at];
        e = c.g_exit[at];
    }
    c.g_entry[c.n_groups] = e;
    c.g_base[c.n_groups] = base;
    c.n_batches[0] = base;
    c.n_batches[1] = 0;
    c.offsets[base] = c.n;  // batching.py:124,136: last entry = end of the final batch
}

// B3 / B4 with the table rows staged in shared memory.  Walking a chain of tables is one dependent
// global load per step (~0.5 us each: 110 steps for the groups, 64 for the chunks of a group); here the
// CTA copies the (exit, count) rows of `rows` consecutive tables at once -- one latency -- and thread 0
// walks them in shared memory.
__global__ void __launch_bounds__(1024) table_walk_kernel(DynCtx c, int level, int rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int* s_exit = reinterpret_cast<int*>(smem_raw);  // [rows][cap]
    int* s_cnt = s_exit + rows * c.cap;
    __shared__ int s_e, s_base;
    // level 0: the groups (one CTA); level 1: the chunks of group blockIdx.x
    const int* __restrict__ t_exit = level == 0 ? c.g_exit : c.c_exit;
    const int* __restrict__ t_cnt = level == 0 ? c.g_cnt : c.c_cnt;
    int k0, k1;
    const int grp = c.g_lo + blockIdx.x;  // level 1
    if (level == 0) { k0 = c.g_lo; k1 = c.g_hi; }
    else { k0 = grp * kGroup; k1 = min(c.n_chunks, k0 + kGroup); }
    if (threadIdx.x == 0) {
        s_e = level == 0 ? (c.ranged ? c.entry[0] : 0) : c.g_entry[grp];
        s_base = level == 0 ? (c.ranged ? c.entry[1] : 0) : c.g_base[grp];
    }
    for (int kb = k0; kb < k1; kb += rows) {
        const int nr = min(rows, k1 - kb);
        const int* __restrict__ ge = t_exit + (size_t)kb * c.cap;
        const int* __restrict__ gc = t_cnt + (size_t)kb * c.cap;
#pragma unroll 4
        for (int i = threadIdx.x; i < nr * c.cap; i += blockDim.x) {  // all loads of a batch of rows in flight together
            s_exit[i] = __ldg(ge + i);
            s_cnt[i] = __ldg(gc + i);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int e = s_e, base = s_base;
            for (int r = 0; r < nr; r++) {
                if (level == 0) { c.g_entry[kb + r] = e; c.g_base[kb + r] = base; }
                else { c.c_entry[kb + r] = e; c.c_base[kb + r] = base; }
                base += s_cnt[r * c.cap + e];
                e = s_exit[r * c.cap + e];
            }
            s_e = e;
            s_base = base;
        }
        __syncthreads();
    }
    if (level == 0 && threadIdx.x == 0) {
        c.g_entry[c.g_hi] = s_e;
        c.g_base[c.g_hi] = s_base;
        if (!c.ranged) {
            c.n_batches[0] = s_base;
            c.n_batches[1] = 0;
            c.offsets[s_base] = c.n;  // batching.py:124,136: last entry = end of the final batch
        } else {  // the range's own batches, numbered from 0; the closing entry is where the chain leaves the range
            const int local = s_base - c.entry[1];
            c.n_batches[0] = local;
            c.n_batches[1] = 0;
            c.n_batches[2] = c.entry[1];
            c.n_batches[3] = c.entry[2];
            c.offsets[local] = (int32_t)min((long long)c.n, (long long)(c.s_hi + s_e) * c.ps);
        }
    }
}

// ---- B4: true entry offset / first batch number of every chunk -----------------------------
__global__ void __launch_bounds__(128) chunk_entry_kernel(DynCtx c) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= c.n_groups) return;
    const int k0 = g * kGroup, k1 = min(c.n_chunks, k0 + kGroup);
    int e = c.g_entry[g], base = c.g_base[g];
    for (int k = k0; k < k1; k++) {
        c.c_entry[k] = e;
        c.c_base[k] = base;
        size_t at = (size_t)k * c.cap + e;
        base += c.c_cnt[at];
        e = c.c_exit[at];
    }
}

// ---- B5: offsets ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) emit_offsets_kernel(DynCtx c) {
    const int k = c.k_lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= c.k_hi) return;
    const int lo = k * c.chunk, hi = min(c.T, lo + c.chunk);
    int entry, base;
    if (c.entries_in_tables) {  // (group_table_smem_kernel left every chunk's entry per group entry offset)
        const int g = k / kGroup, eg = c.g_entry[g];
        entry = c.c_exit[(size_t)k * c.cap + eg];
        base = c.g_base[g] + c.c_cnt[(size_t)k * c.cap + eg];
    } else {
        entry = c.c_entry[k];
        base = c.c_base[k];
    }
    int s = lo + entry, j = base - (c.ranged ? c.entry[1] : 0);
    while (s < hi) {
        c.offsets[j++] = s * c.ps;
        s = c.next[s];
    }
}

static inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct DynLayout {
    size_t prev, nxt, next, c_exit, c_cnt, g_exit, g_cnt, g_entry, g_base, c_entry, c_base, r_entry, total;
    int T, cap, chunk, n_chunks, n_groups, tile, slots, window;
};

static DynLayout dyn_layout(int64_t n, const vr_batch_config* cfg) {
    DynLayout L{};
    const int ps = cfg->primitive_size;
    L.T = (int)(n / ps);
    int64_t cap = cfg->max_indices / ps;
    if (cap > L.T) cap = L.T > 0 ? L.T : 1;
    L.cap = (int)cap;
    L.window = L.cap * ps;
    L.chunk = L.cap > 1024 ? L.cap : 1024;
    L.n_chunks = (int)ceil_div(L.T > 0 ? L.T : 1, L.chunk);
    L.n_groups = (int)ceil_div(L.n_chunks, kGroup);
    int tile = (L.window + 31) & ~31;
    if (tile < 1024) tile = 1024;  // (2048 halves the halo overhead but also the warps per SM: measured slower)
    L.tile = tile;
    {   // distinct ids seen by one warp <= tile + halo
        const int cnt = tile + ((L.window + 31) & ~31) + 32;
        L.slots = ((cnt + cnt / 4) + 31) & ~31;  // load <= 0.8
    }
    size_t o = 0;
    L.prev = o; o += al((size_t)n * 4 + 64);
    L.nxt = o; o += al((size_t)n * 4 + 64);
    L.next = o; o += al((size_t)L.T * 4 + 64);
    L.c_exit = o; o += al((size_t)L.n_chunks * L.cap * 4);
    L.c_cnt = o; o += al((size_t)L.n_chunks * L.cap * 4);
    L.g_exit = o; o += al((size_t)L.n_groups * L.cap * 4);
    L.g_cnt = o; o += al((size_t)L.n_groups * L.cap * 4);
    L.g_entry = o; o += al((size_t)(L.n_groups + 1) * 4);
    L.g_base = o; o += al((size_t)(L.n_groups + 1) * 4);
    L.c_entry = o; o += al((size_t)L.n_chunks * 4);
    L.c_base = o; o += al((size_t)L.n_chunks * 4);
    L.r_entry = o; o += al(16);
    L.total = o;
    return L;
}

}  // namespace vr

using namespace vr;

extern "C" {

size_t vr_dynamic_workspace_bytes(int64_t n, const vr_batch_config* cfg) {
    if (vr_check_batch_config(cfg) || n <= 0 || n > 0x7fffffffLL) return 0;
    return dyn_layout(n, cfg).total;
}

int vr_dynamic_batches(const uint32_t* d_idx, int64_t n, const vr_batch_config* cfg, int32_t* d_offsets,
                       int64_t* d_n_batches, void* d_ws, size_t ws_bytes, void* stream_) {
    return vr_dynamic_batches_draws(d_idx, n, cfg, nullptr, 0, d_offsets, d_n_batches, d_ws, ws_bytes, stream_);
}

// mode 0: the whole stream in one call; mode 1: tables of the range [g_lo, g_hi) (stage A, B1, B2 and the range's
// own table); mode 2: offsets of the range, given the tables of all ranges (range entry, B3 .. B5 on the range)
static int dyn_launch(int mode, const uint32_t* d_idx, int64_t n, const vr_batch_config* cfg, const int32_t* d_draw_index_start,
                      int32_t n_draws, int g_lo, int g_hi, int32_t* d_table, const int32_t* d_tables, int world, int rank,
                      int32_t* d_offsets, int64_t* d_n_batches, void* d_ws, size_t ws_bytes, cudaStream_t stream) {
    DynLayout L = dyn_layout(n, cfg);
    if (!d_ws || ws_bytes < L.total) return VR_ERR_WORKSPACE;
    if (mode != 0 && (g_lo < 0 || g_hi < g_lo || g_hi > L.n_groups)) return VR_ERR_BAD_CONFIG;
    // link table: 4-byte key + last position of the id relative to the halo start (16 bits when the
    // tile and its halo span fewer than 65 536 positions)
    const bool small_last = (int64_t)L.tile + L.window + 64 < 65536;
    const int per_warp = (L.slots * (small_last ? 6 : 8) + 15) & ~15;
    int wpc = 4;
    while ((size_t)wpc * per_warp > 200 * 1024 && wpc > 1) wpc >>= 1;
    const size_t smem = (size_t)wpc * per_warp;
    if (smem > 200 * 1024) return VR_ERR_UNSUPPORTED;  // batch window too long for the link table
    unsigned char* ws = (unsigned char*)d_ws;
    DynCtx c{};
    c.ids = d_idx; c.n = (int)n; c.T = L.T; c.ps = cfg->primitive_size; c.max_unique = cfg->max_unique;
    c.cap = L.cap; c.window = L.window; c.tile = L.tile; c.slots = L.slots; c.chunk = L.chunk;
    c.n_chunks = L.n_chunks; c.n_groups = L.n_groups;
    c.prev = (int32_t*)(ws + L.prev); c.nxt = (int32_t*)(ws + L.nxt); c.next = (int32_t*)(ws + L.next);
    c.c_exit = (int32_t*)(ws + L.c_exit); c.c_cnt = (int32_t*)(ws + L.c_cnt);
    c.g_exit = (int32_t*)(ws + L.g_exit); c.g_cnt = (int32_t*)(ws + L.g_cnt);
    c.g_entry = (int32_t*)(ws + L.g_entry); c.g_base = (int32_t*)(ws + L.g_base);
    c.c_entry = (int32_t*)(ws + L.c_entry); c.c_base = (int32_t*)(ws + L.c_base);
    c.offsets = d_offsets; c.n_batches = d_n_batches;
    c.draw_start = d_draw_index_start; c.n_draws = d_draw_index_start ? n_draws : 0;
    c.ranged = mode != 0;
    c.g_lo = mode ? g_lo : 0; c.g_hi = mode ? g_hi : L.n_groups;
    c.k_lo = c.g_lo * kGroup; c.k_hi = (int)(c.g_hi * (int64_t)kGroup < L.n_chunks ? c.g_hi * kGroup : L.n_chunks);
    c.s_lo = (int)((int64_t)c.k_lo * L.chunk < L.T ? (int64_t)c.k_lo * L.chunk : L.T);
    c.s_hi = (int)((int64_t)c.k_hi * L.chunk < L.T ? (int64_t)c.k_hi * L.chunk : L.T);
    c.r_table = d_table;
    c.entry = (const int32_t*)(ws + L.r_entry);
    const DebugKnobs& knobs = debug_knobs();
    const int halo2 = (L.window + 31) & ~31;
    const int tile2 = knobs.link_tile;  // (4096 / 6144: fewer CTAs per SM, measured slower)
    const int np2 = tile2 + halo2;
    const int nslots2 = (int)next_pow2((uint32_t)(np2 + np2 / 3));  // load <= 0.75
    const size_t smem2 = (size_t)nslots2 * 4 + (size_t)(nslots2 + 1) * 4 + (size_t)np2 * 4 + 16;
    const bool links_tile = np2 <= 65535 && nslots2 <= 65535 && smem2 <= 100 * 1024 && !knobs.links_warp;
    int run_s = knobs.greedy_run_s > 0 ? knobs.greedy_run_s : 30;
    for (int k = 0; k < 3 && (run_s * c.ps) % 4 != 2; k++) run_s++;
    const int64_t npos_s = ((int64_t)128 * run_s * c.ps + L.window + c.ps + 7) & ~(int64_t)7;  // (whole 16-byte rows of halfwords)
    const bool greedy_smem = npos_s * 4 <= 56 * 1024 && L.window < 60000 && !knobs.greedy_global;
    c.want_nxt = greedy_smem ? 0 : 1;
    int walk_rows = 8;
    while (walk_rows > 1 && (size_t)walk_rows * L.cap * 8 > 48 * 1024) walk_rows >>= 1;
    const bool walk_smem = (size_t)walk_rows * L.cap * 8 <= 48 * 1024 && walk_rows >= 2 && !knobs.walk_global;
    // the walk over the groups is one CTA: as many rows at once as shared memory holds
    int walk_rows0 = walk_rows;
    while ((size_t)2 * walk_rows0 * L.cap * 8 <= 200 * 1024 && walk_rows0 < L.n_groups) walk_rows0 *= 2;
    const size_t ct_smem = (size_t)L.chunk * 4, gt_smem = (size_t)kGroup * L.cap * 8;
    const bool tables_smem = walk_smem && gt_smem <= 200 * 1024;
    c.entries_in_tables = tables_smem ? 1 : 0;
    // (ranges are implemented by the default kernels only)
    if (mode != 0 && (!links_tile || !greedy_smem || !walk_smem || c.draw_start)) return VR_ERR_UNSUPPORTED;
    const int n_prims_r = c.s_hi - c.s_lo, n_chunks_r = c.k_hi - c.k_lo, n_groups_r = c.g_hi - c.g_lo;

    if (mode != 2) {
        // positions whose links are needed: the range and one batch window behind it
        const int64_t p_lo = (int64_t)c.s_lo * c.ps;
        const int64_t p_end = mode ? ((int64_t)c.s_hi * c.ps + L.window < n ? (int64_t)c.s_hi * c.ps + L.window : n) : n;
        c.link_end = (int)p_end;
        if (p_end > p_lo && c.want_nxt) fill_kernel<<<(int)ceil_div(ceil_div(p_end - p_lo, 4), 256), 256, 0, stream>>>(c.nxt + p_lo, (int)(p_end - p_lo), kNoLink);
        const int n_tiles = (int)ceil_div(n, L.tile);
        if (links_tile) {
            // tile version: thread per position, counting sort by table slot (16-bit relative positions)
            c.tile_lo = (int)(p_lo / tile2);
            const int tiles = (int)(ceil_div(p_end, tile2) - c.tile_lo);
            VR_CUDA_CHECK(cudaFuncSetAttribute(occurrence_links_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
            if (tiles > 0) occurrence_links_tile_kernel<<<tiles, kLinkThreads, smem2, stream>>>(c, tile2, halo2, nslots2);
        } else if (small_last) {
            VR_CUDA_CHECK(cudaFuncSetAttribute(occurrence_links_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            occurrence_links_kernel<uint16_t><<<(int)ceil_div(n_tiles, wpc), wpc * 32, smem, stream>>>(c, n_tiles, per_warp);
        } else {
            VR_CUDA_CHECK(cudaFuncSetAttribute(occurrence_links_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            occurrence_links_kernel<int32_t><<<(int)ceil_div(n_tiles, wpc), wpc * 32, smem, stream>>>(c, n_tiles, per_warp);
        }
        // shared-memory version when a CTA's stretch (128 runs + one batch window) fits as 16-bit distances
        // (run * ps halfwords between the lanes' streams: an odd number of 32-bit words keeps their reads on
        // different banks)
        if (greedy_smem) {
            auto kernel = c.ps == 3 ? greedy_next_smem_kernel<3> : greedy_next_smem_kernel<0>;
            VR_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(npos_s * 4)));
            if (n_prims_r > 0) kernel<<<(int)ceil_div(n_prims_r, 128 * run_s), 128, (size_t)npos_s * 4, stream>>>(c, run_s, (int)npos_s);
        } else {
            const int run = knobs.greedy_run;
            greedy_next_kernel<<<(int)ceil_div(ceil_div(L.T, run), 128), 128, 0, stream>>>(c, run);
        }
        if (n_chunks_r > 0) {
            if (ct_smem <= 48 * 1024 && !knobs.walk_global) chunk_table_smem_kernel<<<n_chunks_r, 256, ct_smem, stream>>>(c);
            else chunk_table_kernel<<<n_chunks_r, 256, 0, stream>>>(c);
        }
        if (n_groups_r > 0) {
            if (tables_smem) {
                VR_CUDA_CHECK(cudaFuncSetAttribute(group_table_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gt_smem));
                group_table_smem_kernel<<<n_groups_r, 1024, gt_smem, stream>>>(c);
            } else {
                group_table_kernel<<<n_groups_r, 256, 0, stream>>>(c);
            }
        }
        if (mode == 1) range_table_kernel<<<(int)ceil_div(L.cap, 256), 256, 0, stream>>>(c);
    }
    if (mode != 1) {
        if (mode == 2) range_entry_kernel<<<1, 32, 0, stream>>>(d_tables, world, rank, L.cap, (int32_t*)(ws + L.r_entry));
        // B3 / B4: rows of 8 tables at a time through shared memory when they fit
        if (walk_smem) {
            VR_CUDA_CHECK(cudaFuncSetAttribute(table_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((size_t)walk_rows0 * L.cap * 8)));
            table_walk_kernel<<<1, 1024, (size_t)walk_rows0 * L.cap * 8, stream>>>(c, 0, walk_rows0);
        } else {
            group_scan_kernel<<<1, 32, 0, stream>>>(c);
        }
        if (c.draw_start) draws_check_kernel<<<(n_draws + 256) / 256, 256, 0, stream>>>(c);
        if (tables_smem) { /* B4 is a look-up in emit_offsets_kernel */ }
        else if (walk_smem) { if (n_groups_r > 0) table_walk_kernel<<<n_groups_r, 1024, (size_t)walk_rows * L.cap * 8, stream>>>(c, 1, walk_rows); }
        else chunk_entry_kernel<<<(int)ceil_div(L.n_groups, 128), 128, 0, stream>>>(c);
        if (n_chunks_r > 0) emit_offsets_kernel<<<(int)ceil_div(n_chunks_r, 128), 128, 0, stream>>>(c);
    }
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_dynamic_batches_draws(const uint32_t* d_idx, int64_t n, const vr_batch_config* cfg,
                             const int32_t* d_draw_index_start, int32_t n_draws, int32_t* d_offsets,
                             int64_t* d_n_batches, void* d_ws, size_t ws_bytes, void* stream_) {
    if (d_draw_index_start && n_draws <= 0) return VR_ERR_BAD_BATCH;
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    if (n % cfg->primitive_size != 0) return VR_ERR_UNALIGNED;  // batching.py:96-97
    if (n < 0 || n > 0x7fffffffLL) return VR_ERR_UNSUPPORTED;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    cudaStream_t stream = (cudaStream_t)stream_;
    if (n == 0) {  // batching.py:99-100
        VR_CUDA_CHECK(cudaMemsetAsync(d_n_batches, 0, 16, stream));
        return VR_OK;
    }
    return dyn_launch(0, d_idx, n, cfg, d_draw_index_start, n_draws, 0, 0, nullptr, nullptr, 1, 0, d_offsets, d_n_batches,
                      d_ws, ws_bytes, stream);
}

// ---- multi-GPU batch formation: ranges of whole groups, one exchange of small tables (SURVEY.md 8e option (ii)) ----
int64_t vr_dynamic_group_count(int64_t n, const vr_batch_config* cfg) {
    if (vr_check_batch_config(cfg) || n <= 0 || n > 0x7fffffffLL || n % cfg->primitive_size) return 0;
    return dyn_layout(n, cfg).n_groups;
}
int64_t vr_dynamic_group_indices(const vr_batch_config* cfg) {
    if (vr_check_batch_config(cfg)) return 0;
    const int64_t cap = cfg->max_indices / cfg->primitive_size;
    return (cap > 1024 ? cap : 1024) * (int64_t)kGroup * cfg->primitive_size;
}
int64_t vr_dynamic_table_words(int64_t n, const vr_batch_config* cfg) {
    if (vr_check_batch_config(cfg) || n <= 0 || n > 0x7fffffffLL || n % cfg->primitive_size) return 0;
    return 2 * (int64_t)dyn_layout(n, cfg).cap;
}
int vr_dynamic_range_tables(const uint32_t* d_idx, int64_t n, const vr_batch_config* cfg, int64_t group_lo, int64_t group_hi,
                            int32_t* d_table, void* d_ws, size_t ws_bytes, void* stream_) {
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    if (n <= 0 || n % cfg->primitive_size != 0) return VR_ERR_UNALIGNED;
    if (n > 0x7fffffffLL) return VR_ERR_UNSUPPORTED;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (!d_table) return VR_ERR_BAD_CONFIG;
    return dyn_launch(1, d_idx, n, cfg, nullptr, 0, (int)group_lo, (int)group_hi, d_table, nullptr, 1, 0, nullptr, nullptr, d_ws, ws_bytes,
                      (cudaStream_t)stream_);
}
int vr_dynamic_range_offsets(const uint32_t* d_idx, int64_t n, const vr_batch_config* cfg, int64_t group_lo, int64_t group_hi,
                             const int32_t* d_tables, int32_t world, int32_t rank, int32_t* d_offsets, int64_t* d_counts,
                             void* d_ws, size_t ws_bytes, void* stream_) {
    int st = vr_check_batch_config(cfg);
    if (st) return st;
    if (n <= 0 || n % cfg->primitive_size != 0) return VR_ERR_UNALIGNED;
    if (n > 0x7fffffffLL) return VR_ERR_UNSUPPORTED;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (!d_tables || !d_offsets || !d_counts || world < 1 || rank < 0 || rank >= world) return VR_ERR_BAD_CONFIG;
    return dyn_launch(2, d_idx, n, cfg, nullptr, 0, (int)group_lo, (int)group_hi, nullptr, d_tables, world, rank, d_offsets, d_counts, d_ws,
                      ws_bytes, (cudaStream_t)stream_);
}

}  // extern "C"
