// vr_common.cuh -- shared device helpers for libvrgeom (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/vrgeom.h"

namespace vr {

constexpr int kWarp = 32;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;  // mesh.py:11-13: reserved, never a vertex id

#define VR_CUDA_CHECK(expr)                         \
    do {                                            \
        cudaError_t _e = (expr);                    \
        if (_e != cudaSuccess) return VR_ERR_CUDA;  \
    } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint32_t next_pow2(uint32_t x) {
#ifdef __CUDA_ARCH__
    return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));  // (the kernels call this once per batch)
#else
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
#endif
}
__host__ __device__ inline int ilog2(uint32_t pow2) {
#ifdef __CUDA_ARCH__
    return pow2 <= 1 ? 0 : 32 - __clz(pow2 - 1);
#else
    int b = 0;
    while ((1u << b) < pow2) b++;
    return b;
#endif
}

// Ablation / debugging knobs.  Read from the environment ONCE per process (the first library call that
// asks); the launch paths never call getenv.  Defaults are the product behaviour.
struct DebugKnobs {
    int link_tile = 2048;     // VR_LINK_TILE     batch formation: positions per tile of the link kernel
    int links_warp = 0;       // VR_LINKS_WARP    batch formation: per-warp link kernel instead of the tile kernel
    int greedy_run = 64;      // VR_GREEDY_RUN
    int greedy_run_s = 30;    // VR_GREEDY_RUN_S   start primitives per thread of the shared-memory window walk
    int greedy_global = 0;    // VR_GREEDY_GLOBAL batch formation: windows walked in global memory
    int walk_global = 0;      // VR_WALK_GLOBAL   batch formation: chain walks in global memory
    int sort_cta = 0;         // VR_SORT_CTA      general sort path: one CTA per batch
    int rows_prefetch = 0;    // VR_PREFETCH      tile kernel: L2 prefetch of a tile's vertices
    int rows_lag = 0;         // VR_LAG           tile kernel: shade lag in tiles (0 = 1.5 x resident CTAs)
    int no_pdl = 0;           // VR_NO_PDL        no programmatic dependent launch
    int dyn3_prefetch = 0;    // VR_DYN3_PREFETCH three-kernel path: L2 prefetch of the distinct vertices before the sort
    int dyn3_tile_shift = 0;  // VR_DYN3_TILE_SHIFT three-kernel path: log2 of the batches per CTA of the set dedup (3..5; 0 = by run length)
};
inline DebugKnobs parse_debug_knobs() {
    DebugKnobs d;
    auto geti = [](const char* name, int& v) { if (const char* e = getenv(name)) v = atoi(e); };
    auto flag = [](const char* name, int& v) { if (getenv(name)) v = 1; };
    geti("VR_LINK_TILE", d.link_tile); flag("VR_LINKS_WARP", d.links_warp); geti("VR_GREEDY_RUN", d.greedy_run); geti("VR_GREEDY_RUN_S", d.greedy_run_s);
    flag("VR_GREEDY_GLOBAL", d.greedy_global); flag("VR_WALK_GLOBAL", d.walk_global); flag("VR_SORT_CTA", d.sort_cta);
    geti("VR_PREFETCH", d.rows_prefetch); geti("VR_LAG", d.rows_lag); flag("VR_NO_PDL", d.no_pdl);
    geti("VR_DYN3_PREFETCH", d.dyn3_prefetch); geti("VR_DYN3_TILE_SHIFT", d.dyn3_tile_shift);
    return d;
}
inline DebugKnobs& debug_knobs_storage() {
    static DebugKnobs k = parse_debug_knobs();
    return k;
}
inline const DebugKnobs& debug_knobs() { return debug_knobs_storage(); }

// strategies.py:88-91 HashConfig.slot; bits == 0 (table_size 1) -> slot 0.
__device__ __forceinline__ uint32_t hash_slot(uint32_t vid, uint32_t mult, int bits) {
    uint32_t prod = vid * mult;
    return bits == 0 ? 0u : (prod >> (32 - bits));
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// Exclusive scan of data[0..n) in shared memory by the whole CTA (any blockDim that is a
// multiple of 32, <= 1024).  Returns the total.  `scratch` holds >= 33 ints.
__device__ inline int block_exclusive_scan(int* data, int n, int* scratch) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + nt - 1) / nt;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    int sum = 0;
    for (int i = lo; i < hi; i++) sum += data[i];
    int inc = warp_incl_scan(sum, lane);
    if (lane == 31) scratch[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int nw = nt >> 5;
        int w = lane < nw ? scratch[lane] : 0;
        int winc = warp_incl_scan(w, lane);
        scratch[lane] = winc - w;  // exclusive warp offsets
        if (lane == 31) scratch[32] = winc;
    }
    __syncthreads();
    int run = scratch[wid] + inc - sum;
    const int total = scratch[32];
    for (int i = lo; i < hi; i++) {
        int v = data[i];
        data[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

// strategies.py:53-67 position_shader in FP32: record = (m @ [x,y,z,1])[:3] / w.
struct ShaderParams {
    int kind;
    int has_matrix;
    float m[16];
    const float4* __restrict__ pos4;
    const uint32_t* __restrict__ attr;
    int attr_words;
    int vertex_count;
    const int32_t* __restrict__ batch_base;  // multi-draw: first vertex of each batch's draw, or NULL
    int extra_cycles;   // synthetic shader load: dependent FMAs per invocation (vr_shader.extra_cycles)
    float load_a, load_b;  // 1, 0 at run time (kernel parameters, so the chain is not folded away)
};

// L2 eviction policies (createpolicy + .L2::cache_hint): a random 16-byte gather pulls a 32-byte sector, so a
// vertex buffer that has to come from DRAM costs twice its algorithmic bytes per invocation; kept in L2 (it is
// 58 MB at 3.6 M vertices) it costs them once per run.  The outputs are written once and never read here.
struct L2Policies { unsigned long long keep, stream; };
__device__ __forceinline__ L2Policies make_l2_policies() {
    L2Policies p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.stream));
    return p;
}
__device__ __forceinline__ float4 ldg_keep_f4(const float4* p, unsigned long long pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream_f4(float4* p, float4 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream_u32(uint32_t* p, uint32_t v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// The w-divide uses one hardware reciprocal (MUFU.RCP, <= 1 ulp) and three multiplies: a few ulp
// of FP32 from the reference's float64 result, far inside the 1e-5 relative bound.
// LOAD: honour sp.extra_cycles (the general shading kernels); the fused warp-voting kernels are compiled without it
// and vr_run does not select them for a loaded shader.
template <bool LOAD = false>
__device__ __forceinline__ float4 transform_position(const ShaderParams& sp, float4 p) {
    if (!sp.has_matrix) {
        float w = 1.0f;
        if (LOAD)
            for (int k = 0; k < sp.extra_cycles; k++) w = fmaf(w, sp.load_a, sp.load_b);
        return make_float4(p.x, p.y, p.z, w);
    }
    const float ox = fmaf(sp.m[0], p.x, fmaf(sp.m[1], p.y, fmaf(sp.m[2], p.z, sp.m[3])));
    const float oy = fmaf(sp.m[4], p.x, fmaf(sp.m[5], p.y, fmaf(sp.m[6], p.z, sp.m[7])));
    const float oz = fmaf(sp.m[8], p.x, fmaf(sp.m[9], p.y, fmaf(sp.m[10], p.z, sp.m[11])));
    const float ow = fmaf(sp.m[12], p.x, fmaf(sp.m[13], p.y, fmaf(sp.m[14], p.z, sp.m[15])));
    float iw;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(iw) : "f"(ow));
    float w = ow;
    // the paper's synthetic shader loads: a dependent chain w = w * 1 + 0, exact, one FMA per "cycle"
    if (LOAD)
        for (int k = 0; k < sp.extra_cycles; k++) w = fmaf(w, sp.load_a, sp.load_b);
    return make_float4(ox * iw, oy * iw, oz * iw, w);
}

}  // namespace vr
