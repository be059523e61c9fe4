// vr_clients.cu -- what sits either side of the geometry stage in the reference:
//   * ideal_report (analytics.py:105-119): one invocation per referenced vertex;
//   * simulate_parallel_cache (cache.py:66-130): the per-multiprocessor LRU post-transform cache the paper
//     compares the reuse strategies with;
//   * the random-walk client (walk.py): likelihood "shader" per occupied cell, counter-based uniforms,
//     move selection.
#include "vr_common.cuh"

namespace vr {

// ---------------------------------------------------------------------------------
// ideal_report
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ideal_mark_kernel(const uint32_t* __restrict__ idx, int64_t n, int32_t vertex_count,
                                                         int32_t* __restrict__ counts, long long* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t v = __ldg(idx + i);
        if (v < (uint32_t)vertex_count) counts[v] = 1;  // every writer stores the same value
        else atomicMax(out + 1, (long long)VR_ERR_VERTEX_RANGE);
    }
}
__global__ void __launch_bounds__(256) ideal_count_kernel(const int32_t* __restrict__ counts, int32_t vertex_count,
                                                          long long* __restrict__ out) {
    long long mine = 0;
    const int stride = gridDim.x * blockDim.x;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < vertex_count; v += stride) mine += counts[v];
    mine = __reduce_add_sync(0xffffffffu, (int)mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd((unsigned long long*)out, (unsigned long long)mine);
}

// ---------------------------------------------------------------------------------
// simulate_parallel_cache: one CTA per processor chunk.  Recency is a time stamp: a hit at offset o of the wave
// that starts at stamp t0 gets t0 + o (the last hit wins: atomicMax), the wave's distinct missed ids get
// t0 + W + (offset of their first miss), the next wave starts at t0 + 2 W -- the order of the stamps is the
// order of the reference's OrderedDict (cache.py:113-129), and "pop the oldest while over capacity" keeps the
// `capacity` largest stamps.
// ---------------------------------------------------------------------------------
struct CacheTables {
    uint32_t* key[2];           // [T] open addressing, kEmpty = free
    unsigned long long* ts[2];  // [T]
    uint32_t* mkey;             // [M] ids missed in the current wave
    uint32_t* mpos;             // [M] offset of their first miss
};
constexpr int kCacheThreads = 1024;

__device__ __forceinline__ uint32_t cache_hash(uint32_t id, int bits) { return bits ? (id * 0x9E3779B1u) >> (32 - bits) : 0u; }

__global__ void __launch_bounds__(kCacheThreads) cache_sim_kernel(const uint32_t* __restrict__ idx, int64_t n, int64_t per_proc,
                                                                  int wave, int capacity, int T, int M, unsigned char* ws,
                                                                  size_t per_proc_bytes, int32_t vertex_count,
                                                                  int32_t* __restrict__ miss_counts, long long* __restrict__ out) {
    __shared__ long long s_hits, s_misses;
    __shared__ int s_count, s_size, s_new;
    __shared__ unsigned long long s_lo, s_hi;
    const int tid = threadIdx.x;
    const int64_t start = (int64_t)blockIdx.x * per_proc;
    if (start >= n) return;
    const int64_t len = min(per_proc, n - start);
    unsigned char* base = ws + (size_t)blockIdx.x * per_proc_bytes;
    CacheTables tb;
    tb.ts[0] = reinterpret_cast<unsigned long long*>(base);
    tb.ts[1] = tb.ts[0] + T;
    tb.key[0] = reinterpret_cast<uint32_t*>(tb.ts[1] + T);
    tb.key[1] = tb.key[0] + T;
    tb.mkey = tb.key[1] + T;
    tb.mpos = tb.mkey + M;
    const int tbits = ilog2((uint32_t)T), mbits = ilog2((uint32_t)M);
    const uint32_t tmask = (uint32_t)T - 1, mmask = (uint32_t)M - 1;
    for (int i = tid; i < T; i += kCacheThreads) { tb.key[0][i] = kEmpty; tb.key[1][i] = kEmpty; }
    if (tid == 0) { s_hits = 0; s_misses = 0; s_size = 0; }
    __syncthreads();
    int cur = 0;
    unsigned long long t0 = 1;
    for (int64_t wb = 0; wb < len; wb += wave, t0 += 2ull * (unsigned long long)wave) {
        const int wn = (int)min((int64_t)wave, len - wb);
        uint32_t* __restrict__ key = tb.key[cur];
        unsigned long long* __restrict__ ts = tb.ts[cur];
        for (int i = tid; i < M; i += kCacheThreads) { tb.mkey[i] = kEmpty; tb.mpos[i] = kEmpty; }
        if (tid == 0) s_new = 0;
        __syncthreads();
        // lookups against the cache as it stood before the wave (cache.py:113-121)
        int hits = 0, misses = 0;
        for (int o = tid; o < wn; o += kCacheThreads) {
            const uint32_t id = __ldg(idx + start + wb + o);
            if (vertex_count > 0 && id >= (uint32_t)vertex_count) { atomicMax(out + 2, (long long)VR_ERR_VERTEX_RANGE); continue; }
            uint32_t h = cache_hash(id, tbits);
            bool hit = false;
            for (;;) {
                const uint32_t k = key[h];
                if (k == id) { hit = true; break; }
                if (k == kEmpty) break;
                h = (h + 1) & tmask;
            }
            if (hit) {
                hits++;
                atomicMax(&ts[h], t0 + (unsigned long long)o);
            } else {
                misses++;
                if (miss_counts) atomicAdd(&miss_counts[id], 1);
                uint32_t m = cache_hash(id, mbits);
                for (;;) {
                    const uint32_t prev = atomicCAS(&tb.mkey[m], kEmpty, id);
                    if (prev == kEmpty) atomicAdd(&s_new, 1);
                    if (prev == kEmpty || prev == id) break;
                    m = (m + 1) & mmask;
                }
                atomicMin(&tb.mpos[m], (uint32_t)o);
            }
        }
        if (hits) atomicAdd((unsigned long long*)&s_hits, (unsigned long long)hits);
        if (misses) atomicAdd((unsigned long long*)&s_misses, (unsigned long long)misses);
        __syncthreads();
        const int total = s_size + s_new;
        // the stamp below which entries leave: the (total - capacity)-th smallest (stamps are distinct)
        unsigned long long cut = 0;
        if (total > capacity) {
            const int drop = total - capacity;
            if (tid == 0) { s_lo = 0; s_hi = t0 + 2ull * (unsigned long long)wave; }
            __syncthreads();
            for (;;) {  // smallest x with |{stamp < x}| >= drop  ->  survivors are the stamps >= x - 1 ... found by bisection
                const unsigned long long lo = s_lo, hi = s_hi;
                if (hi - lo <= 1) break;
                const unsigned long long mid = lo + (hi - lo) / 2;
                if (tid == 0) s_count = 0;
                __syncthreads();
                int c = 0;
                for (int i = tid; i < T; i += kCacheThreads) c += key[i] != kEmpty && ts[i] < mid;
                for (int i = tid; i < M; i += kCacheThreads)
                    c += tb.mkey[i] != kEmpty && t0 + (unsigned long long)wave + tb.mpos[i] < mid;
                if (c) atomicAdd(&s_count, c);
                __syncthreads();
                if (tid == 0) { if (s_count >= drop) s_hi = mid; else s_lo = mid; }
                __syncthreads();
            }
            cut = s_hi;  // exactly `drop` stamps lie below it
        }
        // rebuild: survivors of the old table and of the wave's new ids into the other table
        const int nxt = cur ^ 1;
        uint32_t* __restrict__ nkey = tb.key[nxt];
        unsigned long long* __restrict__ nts = tb.ts[nxt];
        for (int i = tid; i < T; i += kCacheThreads) nkey[i] = kEmpty;
        __syncthreads();
        auto insert = [&](uint32_t id, unsigned long long stamp) {
            uint32_t h = cache_hash(id, tbits);
            for (;;) {
                if (atomicCAS(&nkey[h], kEmpty, id) == kEmpty) break;
                h = (h + 1) & tmask;
            }
            nts[h] = stamp;
        };
        for (int i = tid; i < T; i += kCacheThreads)
            if (key[i] != kEmpty && ts[i] >= cut) insert(key[i], ts[i]);
        for (int i = tid; i < M; i += kCacheThreads) {
            const unsigned long long stamp = t0 + (unsigned long long)wave + tb.mpos[i];
            if (tb.mkey[i] != kEmpty && stamp >= cut) insert(tb.mkey[i], stamp);
        }
        if (tid == 0) s_size = min(total, capacity);
        cur = nxt;
        __syncthreads();
    }
    if (tid == 0) {
        atomicAdd((unsigned long long*)out, (unsigned long long)s_hits);
        atomicAdd((unsigned long long*)(out + 1), (unsigned long long)s_misses);
    }
}

// ---------------------------------------------------------------------------------
// random-walk client
// ---------------------------------------------------------------------------------
constexpr int kWalkMaxCandidates = 1024;  // moves within max_move_distance (797 at the default 16)
constexpr int kWalkWarps = 4;

constexpr int kWalkMaxDistance = 18;  // 1009 candidate moves; 19 would be 1129
struct WalkParams {
    int grid_w, grid_h, d, kept, n_g, n_cand;
    double cx[VR_WALK_MAX_GAUSSIANS], cy[VR_WALK_MAX_GAUSSIANS], inv2s2[VR_WALK_MAX_GAUSSIANS], amp[VR_WALK_MAX_GAUSSIANS];
    // walk.py:85-99: the candidate moves in row-major scan order are the rows dy = -d .. d of a disk; row r holds
    // dx = -half[r] .. half[r] and starts at candidate number row_start[r].  (Kernel parameters, not a __constant__
    // table: concurrent calls with different radii must not share state.)
    short row_start[2 * kWalkMaxDistance + 2];
    signed char half[2 * kWalkMaxDistance + 1];
};
// candidate number -> (dx, dy)
__device__ __forceinline__ void walk_candidate(const WalkParams& p, int k, int& dx, int& dy) {
    int r = 0;
    while (p.row_start[r + 1] <= k) r++;
    dy = r - p.d;
    dx = k - p.row_start[r] - p.half[r];
}

// walk.py:110-137 for one cell per warp.  Candidates in row-major scan order (walk.py:85-99); activity =
// 1e-12 + sum of the Gaussians at the destination, in the order of cfg.gaussians (walk.py:102-109);
// likelihood = activity / sum over the legal candidates; the kept_moves largest, ties by scan position.
__global__ void __launch_bounds__(kWalkWarps * 32) walk_likelihood_kernel(const uint32_t* __restrict__ cells, int64_t n, WalkParams p,
                                                                         double* __restrict__ moves, long long* __restrict__ status) {
    __shared__ double s_act[kWalkWarps][kWalkMaxCandidates];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t cell_i = (int64_t)blockIdx.x * kWalkWarps + wid;
    if (cell_i >= n) return;
    const uint32_t cell = __ldg(cells + cell_i);
    const int x = (int)(cell & 0xFFFFu), y = (int)(cell >> 16);
    double* act = s_act[wid];
    double sum = 0.0;
    int legal = 0;
    int row = 0;  // row of the lane's current candidate (candidates ascend, so the row only moves forward)
    for (int k = lane; k < p.n_cand; k += 32) {
        while (p.row_start[row + 1] <= k) row++;
        const int dx = k - p.row_start[row] - p.half[row], dy = row - p.d;
        const int tx = x + dx, ty = y + dy;
        double a = -1.0;  // not on the grid
        if (tx >= 0 && tx < p.grid_w && ty >= 0 && ty < p.grid_h) {
            a = 1.0;
            if (p.n_g > 0) {
                a = 1e-12;
                for (int g = 0; g < p.n_g; g++) {
                    const double ex = (double)tx - p.cx[g], ey = (double)ty - p.cy[g];
                    const double d2 = ex * ex + ey * ey;
                    a += p.amp[g] * exp(-d2 / p.inv2s2[g]);  // inv2s2 holds 2 sigma^2 (the reference divides)
                }
            }
            sum += a;
            legal++;
        }
        act[k] = a;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, d);
        legal += __shfl_xor_sync(0xffffffffu, legal, d);
    }
    __syncwarp();
    if (legal < p.kept) {  // walk.py:123-126
        if (lane == 0) atomicMax(status, (long long)((cell_i << 8) | VR_ERR_BAD_CONFIG));
        return;
    }
    for (int k = lane; k < p.n_cand; k += 32)
        if (act[k] >= 0.0) act[k] = act[k] / sum;
    __syncwarp();
    double* out = moves + cell_i * p.kept * 3;
    for (int j = 0; j < p.kept; j++) {
        double best = -1.0;
        int best_k = 0x7fffffff;
        for (int k = lane; k < p.n_cand; k += 32) {  // ascending k: the first maximum is the earliest in scan order
            const double a = act[k];
            if (a > best) { best = a; best_k = k; }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, d);
            const int ok = __shfl_xor_sync(0xffffffffu, best_k, d);
            if (ob > best || (ob == best && ok < best_k)) { best = ob; best_k = ok; }
        }
        if (lane == 0) {
            int bdx, bdy;
            walk_candidate(p, best_k, bdx, bdy);
            out[3 * j + 0] = (double)bdx;
            out[3 * j + 1] = (double)bdy;
            out[3 * j + 2] = best;
            act[best_k] = -1.0;
        }
        __syncwarp();
    }
}

// splitmix64 finalizer (walk.py:140-149)
__host__ __device__ inline unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void __launch_bounds__(256) walk_advance_kernel(const int32_t* __restrict__ pin, int64_t n, const int32_t* __restrict__ src,
                                                           const double* __restrict__ moves, int kept, unsigned long long base,
                                                           int32_t* __restrict__ pout) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    // walk.py:152-158 agent_uniforms: 53 random bits -> [0, 1)
    const unsigned long long z = mix64((unsigned long long)a + base);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    const double* m = moves + (src ? (int64_t)src[a] : a) * kept * 3;
    // walk.py:161-165 choose_move: cumulative likelihoods, first j with cum[j] > u * cum[-1]
    double total = 0.0;
    for (int j = 0; j < kept; j++) total += m[3 * j + 2];
    const double r = u * total;
    double cum = 0.0;
    int pick = kept - 1;
    for (int j = 0; j < kept; j++) {
        cum += m[3 * j + 2];
        if (cum > r) { pick = j; break; }
    }
    pout[2 * a + 0] = pin[2 * a + 0] + (int)m[3 * pick + 0];
    pout[2 * a + 1] = pin[2 * a + 1] + (int)m[3 * pick + 1];
}

__global__ void __launch_bounds__(256) walk_pack_kernel(const int32_t* __restrict__ pos, int64_t n, uint32_t* __restrict__ cells) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a < n) cells[a] = ((uint32_t)pos[2 * a + 1] << 16) | (uint32_t)pos[2 * a + 0];
}

}  // namespace vr

using namespace vr;

extern "C" {

int vr_ideal_counts(const uint32_t* d_idx, int64_t n, int32_t vertex_count, int32_t* d_counts, int64_t* d_out, void* stream_) {
    if (n < 0 || vertex_count < 0 || !d_out) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    cudaStream_t stream = (cudaStream_t)stream_;
    VR_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 2 * sizeof(int64_t), stream));
    if (vertex_count == 0 && n == 0) return VR_OK;
    if (!d_counts || (n > 0 && !d_idx)) return VR_ERR_BAD_CONFIG;
    VR_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, (size_t)vertex_count * sizeof(int32_t), stream));
    if (n > 0) ideal_mark_kernel<<<(int)(ceil_div(n, 256) < 148 * 16 ? ceil_div(n, 256) : 148 * 16), 256, 0, stream>>>(d_idx, n, vertex_count, d_counts, (long long*)d_out);
    if (vertex_count > 0)
        ideal_count_kernel<<<(int)(ceil_div(vertex_count, 256) < 148 * 8 ? ceil_div(vertex_count, 256) : 148 * 8), 256, 0, stream>>>(d_counts, vertex_count, (long long*)d_out);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

static int cache_geometry(int64_t n, const vr_cache_config* cfg, int64_t* per_proc, int* T, int* M, size_t* per_bytes) {
    if (!cfg || cfg->num_processors < 1 || cfg->wave_width < 1 || cfg->capacity < 1 || cfg->primitive_size < 1) return VR_ERR_BAD_CONFIG;
    if (n % cfg->primitive_size != 0) return VR_ERR_UNALIGNED;  // cache.py:85-86
    if (cfg->capacity > (1 << 24) || cfg->wave_width > (1 << 24)) return VR_ERR_UNSUPPORTED;
    const int64_t prims = n / cfg->primitive_size;
    *per_proc = ceil_div(prims, cfg->num_processors) * cfg->primitive_size;  // cache.py:88-89
    *T = (int)next_pow2((uint32_t)(2 * cfg->capacity < 64 ? 64 : 2 * cfg->capacity));
    *M = (int)next_pow2((uint32_t)(2 * cfg->wave_width < 64 ? 64 : 2 * cfg->wave_width));
    *per_bytes = ((size_t)*T * (8 + 4) * 2 + (size_t)*M * 8 + 255) & ~(size_t)255;
    return VR_OK;
}

size_t vr_cache_workspace_bytes(int64_t n, const vr_cache_config* cfg) {
    int64_t per_proc; int T, M; size_t pb;
    if (cache_geometry(n, cfg, &per_proc, &T, &M, &pb)) return 0;
    return pb * (size_t)cfg->num_processors;
}

int vr_simulate_cache(const uint32_t* d_idx, int64_t n, const vr_cache_config* cfg, int32_t vertex_count, int32_t* d_miss_counts,
                      int64_t* d_out, void* d_ws, size_t ws_bytes, void* stream_) {
    int64_t per_proc; int T, M; size_t pb;
    const int st = cache_geometry(n, cfg, &per_proc, &T, &M, &pb);
    if (st) return st;
    if (!d_out || n < 0) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    cudaStream_t stream = (cudaStream_t)stream_;
    VR_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 4 * sizeof(int64_t), stream));
    if (n == 0) return VR_OK;
    if (!d_ws || ws_bytes < pb * (size_t)cfg->num_processors) return VR_ERR_WORKSPACE;
    if (d_miss_counts && vertex_count <= 0) return VR_ERR_BAD_CONFIG;
    const int blocks = (int)ceil_div(n, per_proc);
    cache_sim_kernel<<<blocks, kCacheThreads, 0, stream>>>(d_idx, n, per_proc, cfg->wave_width, cfg->capacity, T, M, (unsigned char*)d_ws, pb,
                                                          vertex_count, d_miss_counts, (long long*)d_out);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_walk_likelihoods(const uint32_t* d_cells, int64_t n, const vr_walk_config* cfg, double* d_moves, int64_t* d_status, void* stream_) {
    if (!cfg || !d_status) return VR_ERR_BAD_CONFIG;
    if (cfg->grid_w < 2 || cfg->grid_h < 2 || cfg->grid_w > 65536 || cfg->grid_h > 65536) return VR_ERR_BAD_CONFIG;  // walk.py:62-64
    if (cfg->max_move_distance < 1 || cfg->kept_moves < 1 || cfg->n_gaussians < 0 || cfg->n_gaussians > VR_WALK_MAX_GAUSSIANS) return VR_ERR_BAD_CONFIG;
    if (cfg->max_move_distance > kWalkMaxDistance) return VR_ERR_UNSUPPORTED;  // more than 1024 candidate moves
    WalkParams p{};
    const int d = cfg->max_move_distance;
    int nc = 0;
    for (int dy = -d; dy <= d; dy++) {  // walk.py:85-99 candidate moves, row-major scan order
        int h = 0;
        while ((h + 1) * (h + 1) + dy * dy <= d * d) h++;
        p.row_start[dy + d] = (short)nc;
        p.half[dy + d] = (signed char)h;
        nc += 2 * h + 1;
    }
    p.row_start[2 * d + 1] = (short)nc;
    if (nc > kWalkMaxCandidates) return VR_ERR_UNSUPPORTED;
    if (cfg->kept_moves > nc) return VR_ERR_BAD_CONFIG;  // walk.py:69-70
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    cudaStream_t stream = (cudaStream_t)stream_;
    VR_CUDA_CHECK(cudaMemsetAsync(d_status, 0, sizeof(int64_t), stream));
    if (n <= 0) return VR_OK;
    if (!d_cells || !d_moves) return VR_ERR_BAD_CONFIG;
    p.grid_w = cfg->grid_w; p.grid_h = cfg->grid_h; p.d = d; p.kept = cfg->kept_moves; p.n_g = cfg->n_gaussians; p.n_cand = nc;
    for (int g = 0; g < cfg->n_gaussians; g++) {
        p.cx[g] = cfg->gaussians[g][0]; p.cy[g] = cfg->gaussians[g][1];
        p.inv2s2[g] = 2.0 * cfg->gaussians[g][2] * cfg->gaussians[g][2];  // walk.py:108
        p.amp[g] = cfg->gaussians[g][3];
    }
    walk_likelihood_kernel<<<(int)ceil_div(n, kWalkWarps), kWalkWarps * 32, 0, stream>>>(d_cells, n, p, d_moves, (long long*)d_status);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_walk_advance(const int32_t* d_pin, int64_t n, const int32_t* d_src, const double* d_moves, int32_t kept, uint64_t seed, int64_t step,
                    int32_t* d_pout, void* stream) {
    if (n < 0 || kept < 1) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (n == 0) return VR_OK;
    if (!d_pin || !d_moves || !d_pout) return VR_ERR_BAD_CONFIG;
    // walk.py:154-155: key = seed + golden * (step + 1) (mod 2^64), base = mix64(key)
    const unsigned long long key = (unsigned long long)seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(step + 1);
    walk_advance_kernel<<<(int)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(d_pin, n, d_src, d_moves, kept, mix64(key), d_pout);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

int vr_walk_pack(const int32_t* d_pos, int64_t n, uint32_t* d_cells, void* stream) {
    if (n < 0) return VR_ERR_BAD_CONFIG;
    if (vr_device_count() == 0) return VR_ERR_CUDA;
    if (n == 0) return VR_OK;
    if (!d_pos || !d_cells) return VR_ERR_BAD_CONFIG;
    walk_pack_kernel<<<(int)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(d_pos, n, d_cells);
    VR_CUDA_CHECK(cudaGetLastError());
    return VR_OK;
}

}  // extern "C"
