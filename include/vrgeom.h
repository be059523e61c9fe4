/*
 * vrgeom.h -- C ABI of the B200-native geometry stage (libvrgeom.so).
 *
 * Drop-in boundary for the hot path of the reference package `vrlab`
 * (paths below are relative to /root/reference/pkg/src/vrlab/):
 *
 *   index buffer + vertex buffer -> batch formation -> per-batch dedup
 *   (naive / warp voting / sort / hash) -> vertex shader once per unique
 *   vertex per batch -> primitive assembly with local-index remap ->
 *   reuse statistics.
 *
 * Conventions
 *   - every pointer named d_* is DEVICE memory owned by the caller; the library
 *     never frees caller memory and keeps no state between calls;
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*);
 *     results are valid after the caller synchronises that stream;
 *   - calls are re-entrant across streams and host threads as long as outputs/workspaces differ (the only
 *     library state is the per-thread diagnostics of vr_profile_* / vr_last_*, and debugging knobs read from
 *     the environment once per process);
 *   - functions return a vr_status; host-detectable misuse is reported
 *     immediately, data-dependent violations (found by the kernels) are reported
 *     through vr_stats.error_code / error_batch, read back by the caller;
 *   - no function falls back to the CPU.  Without a CUDA device every compute
 *     entry point returns VR_ERR_CUDA.
 */
#ifndef VRGEOM_H
#define VRGEOM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VRGEOM_ABI_VERSION 4

/* strategies.py:387  STRATEGY_NAMES = ("naive", "warp", "sort", "hash", "phash") */
enum vr_strategy {
    VR_NAIVE = 0, /* strategies.py:159-170 naive_batch          */
    VR_WARP = 1,  /* strategies.py:173-232 warp_vote_batch      */
    VR_SORT = 2,  /* strategies.py:235-260 sort_batch           */
    VR_HASH = 3,  /* strategies.py:263-298 hash_batch           */
    VR_PHASH = 4  /* strategies.py:301-367 parallel_hash_batch  */
};

/* OR into the `strategy` argument of vr_run to call a per-batch kernel on its own
 * (strategies.py:235-298 have no unique budget; the guards of strategies.py:432-435 and
 * :451-455 belong to run_on_indices). */
#define VR_FLAG_NO_BUDGET 0x100
/* OR into `strategy` when the batches tile one range of the buffer in order
 * (batch_end[b] == batch_begin[b+1], e.g. any offsets array of batching.py:128-137):
 * the span scan is skipped.  The kernels verify the claim and report VR_ERR_BAD_BATCH. */
#define VR_FLAG_CONTIGUOUS 0x200
/* OR into `strategy` when the batches are static_batches(n, cfg) (batching.py:76-84):
 * batch_begin[b] = batch_begin[0] + b * cfg->batch_size, last batch possibly shorter.  Implies
 * VR_FLAG_CONTIGUOUS and selects the position-aligned kernels; verified on the device. */
#define VR_FLAG_STATIC 0x400
/* OR into `strategy` to keep dedup, offset scan and shading in separate kernels even where
 * a fused kernel exists (ablation / debugging; results are identical). */
#define VR_FLAG_NO_FUSE 0x800

enum vr_status {
    VR_OK = 0,
    VR_ERR_UNKNOWN_STRATEGY = 1,   /* strategies.py:422-423 ConfigError                    */
    VR_ERR_BAD_BATCH = 2,          /* strategies.py:426-428 ConfigError (range/alignment)  */
    VR_ERR_TABLE_BELOW_BUDGET = 3, /* strategies.py:432-435 ConfigError                    */
    VR_ERR_OVER_BUDGET = 4,        /* strategies.py:451-455 ConfigError (> max_unique)     */
    VR_ERR_HASH_FULL = 5,          /* strategies.py:283-284, :348-349 RuntimeError         */
    VR_ERR_WARP_NO_PROGRESS = 6,   /* strategies.py:226-227 RuntimeError                   */
    VR_ERR_WARP_WIDTH = 7,         /* strategies.py:187-188 ConfigError (w < prim size)    */
    VR_ERR_UNALIGNED = 8,          /* batching.py:79-80, :96-97 ConfigError                */
    VR_ERR_BAD_CONFIG = 9,         /* batching.py:44-56, strategies.py:78-86, warp.py:32-35 */
    VR_ERR_UNSUPPORTED = 10,       /* legal in the reference, outside the device limits    */
    VR_ERR_CUDA = 11,              /* CUDA runtime failure / no device                     */
    VR_ERR_CAPACITY = 12,          /* an output buffer is smaller than the result          */
    VR_ERR_WORKSPACE = 13,         /* workspace smaller than vr_*_workspace_bytes()        */
    VR_ERR_PRIM_OVER_BUDGET = 14,  /* batching.py:119-123 ConfigError                      */
    VR_ERR_VERTEX_RANGE = 15       /* strategies.py:62-65 positions[vid]: IndexError (an id
                                      outside [0, vertex_count); nothing is gathered or tallied) */
};

/* batching.py:23-61 BatchConfig (same fields, same defaults: 96/256/1023/32/256/3) */
typedef struct vr_batch_config {
    int32_t batch_size;
    int32_t max_unique;
    int32_t max_indices;
    int32_t warp_width;
    int32_t block_size;
    int32_t primitive_size;
} vr_batch_config;

/* strategies.py:70-91 HashConfig (defaults 256 / 2654435769 / 8) */
typedef struct vr_hash_config {
    uint32_t table_size;
    uint32_t multiplier;
    uint32_t max_fast_probes;
} vr_hash_config;

/* strategies.py:36-67 ShaderFn: the device shaders are a closed set. */
enum vr_shader_kind {
    VR_SHADER_NONE = 0,     /* dedup + assembly only                                        */
    VR_SHADER_IDENTITY = 1, /* strategies.py:48-50: record = vertex id (== unique_ids)      */
    VR_SHADER_POSITION = 2  /* strategies.py:53-67: [m @ (x,y,z,1)] / w, FP32               */
};

typedef struct vr_shader {
    int32_t kind;              /* vr_shader_kind                                             */
    int32_t has_matrix;        /* 0: record = position as is (strategies.py:56-58)           */
    float matrix[16];          /* row-major 4x4 (strategies.py:60-65)                        */
    const float *d_positions4; /* float4[vertex_count] = (x, y, z, 1); 16-byte aligned       */
    const uint32_t *d_attributes; /* optional opaque per-vertex payload (mesh.py:40-41), or NULL */
    int32_t attr_words;        /* 32-bit words of payload per vertex                         */
    int32_t vertex_count;      /* 0 if unknown; needed for d_shade_counts                    */
    const int32_t *d_batch_vertex_base; /* multi-draw: ids of batch b are relative to vertex
                                  d_batch_vertex_base[b] of the (concatenated) vertex buffers: the
                                  shader reads positions/attributes at base + id and tallies
                                  d_shade_counts[base + id]; unique ids stay draw-local, as the
                                  reference's per-draw runs report them.  NULL = one vertex buffer */
    int32_t extra_cycles;      /* synthetic shader load ("256/512/1024 cycles"; ShaderFn.cycles,
                                  strategies.py:40-44): a dependent chain of this many FP32 FMAs per
                                  invocation that leaves the record unchanged.  0 = the plain transform */
} vr_shader;

/* Statistics block: int64[VR_STATS_WORDS] in device memory, written by vr_run.
 * analytics.py:20-50 ReuseReport + strategies.py:94-111 ProbeStats. */
enum vr_stats_word {
    VR_STAT_INDICES = 0,     /* indices consumed                         */
    VR_STAT_INVOCATIONS = 1, /* shader invocations                       */
    VR_STAT_BATCHES = 2,
    VR_STAT_ROUNDS = 3,
    VR_STAT_PROBES_FAST = 4,
    VR_STAT_PROBES_SLOW = 5,
    VR_STAT_PROBE_MAX_CHAIN = 6,
    VR_STAT_ERROR = 7, /* (first failing batch << 8) | vr_status, or -1 when clean */
    VR_STATS_WORDS = 16
};

/* Flattened list of DedupResult (strategies.py:114-129), batch order.
 * Any pointer except d_stats may be NULL when that output is not wanted
 * (d_shaded is required for VR_SHADER_POSITION). */
typedef struct vr_outputs {
    int32_t *d_batch_round_off; /* [n_batches+1] first round of each batch                  */
    int32_t *d_round_uid_off;   /* [rounds+1]    first unique id of each round              */
    int32_t *d_round_prims;     /* [rounds]      Round.primitives_emitted                   */
    uint32_t *d_unique_ids;     /* [invocations] Round.unique_ids, concatenated             */
    uint16_t *d_assembly_map;   /* [sum of batch spans] Round.assembly_map, concatenated    */
    float *d_shaded4;           /* float4[invocations] = (x/w, y/w, z/w, w)                 */
    uint32_t *d_shaded_attr;    /* [invocations * attr_words] pass-through payload          */
    int32_t *d_shade_counts;    /* [vertex_count] per-vertex tally (strategies.py:485-489);
                                   must be zeroed by the caller                              */
    int64_t *d_stats;           /* [VR_STATS_WORDS]                                          */
    int64_t cap_unique;         /* capacity of d_unique_ids / d_shaded4 (elements)           */
    int64_t cap_rounds;         /* capacity of d_round_prims (elements)                      */
    float *d_stream_xyz;        /* optional, VR_SHADER_POSITION: the stage's output QUEUE (strategies.py:456-463,
                                   PAPER.md:656), float[3 * sum of batch spans]: the record of every corner,
                                   out[slot] = shaded[round base + assembly_map[slot]].xyz.  Written inside the
                                   stage by the three-kernel sort/hash path (from the shaded records in shared
                                   memory), by a closing kernel of vr_run on the other paths.  Needs the round
                                   tables and d_assembly_map.  NULL = no queue (vr_expand_stream builds it later) */
} vr_outputs;

int vr_abi_version(void);
const char *vr_status_string(int status);

/* Number of CUDA devices visible, or 0 (never fails). */
int vr_device_count(void);

/* Validation of the two parameter blocks (batching.py:44-56; strategies.py:78-86). */
int vr_check_batch_config(const vr_batch_config *cfg);
int vr_check_hash_config(const vr_hash_config *hcfg);

/* batching.py:76-84 static_batches.  Writes ceil(n/batch_size)+1 offsets
 * (the "auxiliary buffer" of batching.py:128-137) to d_offsets. */
int64_t vr_static_batch_count(int64_t n_indices, const vr_batch_config *cfg);
int vr_static_offsets(int64_t n_indices, const vr_batch_config *cfg, int32_t *d_offsets, void *stream);

/* batching.py:87-125 dynamic_batches: exact parallel restatement of the greedy scan.
 * d_offsets must hold n_indices/primitive_size + 1 entries; d_n_batches is device int64[2]:
 * [0] receives the batch count (0 for an empty buffer), [1] a vr_status found on the device. */
size_t vr_dynamic_workspace_bytes(int64_t n_indices, const vr_batch_config *cfg);
int vr_dynamic_batches(const uint32_t *d_indices, int64_t n_indices, const vr_batch_config *cfg,
                       int32_t *d_offsets, int64_t *d_n_batches, void *d_workspace,
                       size_t workspace_bytes, void *stream);

/* Multi-draw streams (BASELINE.json configs[4]; the reference calls dynamic_batches and
 * run_on_indices once per mesh, strategies.py:404-415): the index buffers of n_draws draws are
 * concatenated, draw d owning positions [d_draw_index_start[d], d_draw_index_start[d+1]) with
 * [0] = 0 and [n_draws] = n_indices (device int32[n_draws+1], primitive-aligned, verified on the
 * device).  Every draw restarts the greedy scan, so no batch crosses a draw; the offsets are
 * positions in the concatenated buffer.  NULL / 0 draws = vr_dynamic_batches. */
int vr_dynamic_batches_draws(const uint32_t *d_indices, int64_t n_indices, const vr_batch_config *cfg,
                             const int32_t *d_draw_index_start, int32_t n_draws, int32_t *d_offsets,
                             int64_t *d_n_batches, void *d_workspace, size_t workspace_bytes,
                             void *stream);
/* Batch formation over a stream that is SHARDED across GPUs (SURVEY.md 8e option (ii)).  A greedy boundary depends on
 * all boundaries before it, so a rank cannot cut its own range of the stream on its own -- but what a range does to
 * the chain of boundaries is a small table "offset at which the chain enters the range -> (offset at which it enters
 * the next range, batches started inside)", cap = max_indices / primitive_size entries, and tables compose.  So:
 *   1. every rank calls vr_dynamic_range_tables on ITS range (whole groups [group_lo, group_hi) of
 *      vr_dynamic_group_indices() indices each; the index buffer is replicated): stage A and the chunk / group
 *      tables for that range only, and the range's table -> d_table[vr_dynamic_table_words()];
 *   2. ONE all-gather of the tables (2 * cap int32 per rank: 2.7 KB at the defaults) -- the path's only exchange;
 *   3. every rank calls vr_dynamic_range_offsets with the gathered tables [world][table_words] (same workspace as
 *      in step 1, untouched in between): its true entry offset, then the offsets of the batches that START in
 *      its range, d_offsets[0 .. count] (positions in the whole buffer; the closing entry is the start of the next
 *      rank's first batch, or n_indices), d_counts (device int64[4]) = {count, vr_status, global number of the
 *      range's first batch, batches of the whole stream}.
 * The concatenation of the ranks' offsets is exactly vr_dynamic_batches' array.  Workspace: vr_dynamic_workspace_bytes.
 * VR_ERR_UNSUPPORTED for batch windows the default kernels do not take (fall back to a redundant whole-stream scan). */
int64_t vr_dynamic_group_count(int64_t n_indices, const vr_batch_config *cfg);
int64_t vr_dynamic_group_indices(const vr_batch_config *cfg);
int64_t vr_dynamic_table_words(int64_t n_indices, const vr_batch_config *cfg);
int vr_dynamic_range_tables(const uint32_t *d_indices, int64_t n_indices, const vr_batch_config *cfg,
                            int64_t group_lo, int64_t group_hi, int32_t *d_table, void *d_workspace,
                            size_t workspace_bytes, void *stream);
int vr_dynamic_range_offsets(const uint32_t *d_indices, int64_t n_indices, const vr_batch_config *cfg,
                             int64_t group_lo, int64_t group_hi, const int32_t *d_tables, int32_t world,
                             int32_t rank, int32_t *d_offsets, int64_t *d_counts, void *d_workspace,
                             size_t workspace_bytes, void *stream);

/* Per-batch first vertex for vr_shader.d_batch_vertex_base: batch b lies in the draw that holds
 * d_batch_begin[b]; d_out[b] = d_draw_vertex_base[that draw] (device int32 arrays). */
int vr_batch_vertex_base(const int32_t *d_batch_begin, int64_t n_batches, const int32_t *d_draw_index_start,
                         const int32_t *d_draw_vertex_base, int32_t n_draws, int32_t *d_out, void *stream);

/* Upper bounds for the data-dependent output sizes of vr_run. */
int vr_output_bounds(int strategy, int64_t span_total, int64_t n_batches, const vr_batch_config *cfg,
                     const vr_hash_config *hcfg, int64_t *max_invocations, int64_t *max_rounds);

size_t vr_run_workspace_bytes(int strategy, int64_t span_total, int64_t n_batches,
                              const vr_batch_config *cfg, const vr_hash_config *hcfg);

/* strategies.py:404-502 run_on_indices on device.
 * d_batch_begin / d_batch_end: int32[n_batches] half-open ranges (batching.py:64-73); for a
 * contiguous offsets array pass (offsets, offsets + 1).  span_total >= the sum of the batch
 * spans (n_indices when the batches tile the buffer; it sizes d_assembly_map and the
 * workspace), max_span >= the longest batch. */
int vr_run(int strategy, const uint32_t *d_indices, int64_t n_indices, const int32_t *d_batch_begin,
           const int32_t *d_batch_end, int64_t n_batches, int64_t span_total, int32_t max_span,
           const vr_batch_config *cfg, const vr_hash_config *hcfg, const vr_shader *shader,
           const vr_outputs *out, void *d_workspace, size_t workspace_bytes, void *stream);

/* Batch formation -> stage with NO host round trip: the batch count stays on the device.
 *   d_offsets, d_n_batches   as written by vr_dynamic_batches / vr_dynamic_batches_draws on the same stream
 *                            (d_n_batches: int64[2] = {count, vr_status}; a non-zero status is reported through the
 *                            statistics block, as is a count above n_batches_max);
 *   n_batches_max            upper bound the launch, the outputs and the workspace are sized for:
 *                            vr_dynamic_batch_bound(n_indices, cfg, n_draws) -- every batch but the last of a draw holds
 *                            at least min(max_unique - ps + 1, max_primitives * ps) indices (batching.py:106-118).
 * Outputs as vr_run with contiguous batches; VR_STAT_BATCHES and the closing table entries use the device count.
 * Implemented by the three-kernel sort / hash / phash path (budgeted batches): VR_ERR_UNSUPPORTED otherwise. */
int64_t vr_dynamic_batch_bound(int64_t n_indices, const vr_batch_config *cfg, int32_t n_draws);
int vr_run_counted(int strategy, const uint32_t *d_indices, int64_t n_indices, const int32_t *d_offsets,
                   int64_t n_batches_max, const int64_t *d_n_batches, int32_t max_span,
                   const vr_batch_config *cfg, const vr_hash_config *hcfg, const vr_shader *shader,
                   const vr_outputs *out, void *d_workspace, size_t workspace_bytes, void *stream);

/* strategies.py:456-463 + :132-152: expanded per-corner record stream,
 * out[slot] = shaded[round base + assembly_map[slot]].  d_stream_pos3 is float[3*n_slots]
 * (TriangleStream.as_array() for the position shader), d_stream_ids uint32[n_slots]
 * (identity shader); either may be NULL. */
int vr_expand_stream(const int32_t *d_batch_round_off, const int32_t *d_round_uid_off,
                     const int32_t *d_round_prims, const uint16_t *d_assembly_map,
                     const uint32_t *d_unique_ids, const float *d_shaded4, int64_t n_batches,
                     const int32_t *d_batch_begin, const int32_t *d_batch_end, int32_t primitive_size,
                     float *d_stream_pos3, uint32_t *d_stream_ids, void *d_workspace,
                     size_t workspace_bytes, void *stream);

/* strategies.py:53-67 records are float32[3] (x/w, y/w, z/w); the stage keeps float4 (+ w) for 16-byte stores.
 * Packs d_shaded4[n] to float[3*n] -- what a caller copies to the host when it wants the reference's record. */
int vr_pack_xyz(const float *d_shaded4, int64_t n, float *d_xyz, void *stream);
/* Local indices are < warp_width (warp voting) or < max_unique (sort / hash), i.e. bytes for every configuration of
 * the paper: packs d_assembly_map[n] (uint16) to uint8[n] for the trip to the host.  d_flag (device int32[1], may be
 * NULL) is set to 1 if a value did not fit. */
int vr_pack_bytes(const uint16_t *d_assembly_map, int64_t n, uint8_t *d_out, int32_t *d_flag, void *stream);

/* Same walk as vr_expand_stream, but out[slot] = round base + assembly_map[slot]: the position of the
 * slot's record in the unique-id / shaded arrays (int32[n_slots]).  Clients that attach their own
 * per-unique payload (the random-walk client below) expand it with this. */
int vr_expand_sources(const int32_t *d_batch_round_off, const int32_t *d_round_uid_off,
                      const int32_t *d_round_prims, const uint16_t *d_assembly_map, int64_t n_batches,
                      const int32_t *d_batch_begin, const int32_t *d_batch_end, int32_t primitive_size,
                      int32_t *d_stream_src, void *d_workspace, size_t workspace_bytes, void *stream);

/* analytics.py:105-119 ideal_report: one invocation per REFERENCED vertex.  d_counts is int32[vertex_count]
 * (1 for a referenced vertex, else 0); d_out is device int64[2]: [0] the number of referenced vertices,
 * [1] a vr_status found on the device (VR_ERR_VERTEX_RANGE for an index outside the buffer). */
int vr_ideal_counts(const uint32_t *d_indices, int64_t n_indices, int32_t vertex_count, int32_t *d_counts,
                    int64_t *d_out, void *stream);

/* cache.py:66-130 simulate_parallel_cache: per-multiprocessor LRU post-transform cache with the concurrency
 * penalty of wide hardware (duplicates arriving in one wave all miss).  The buffer is cut into
 * num_processors primitive-aligned chunks (cache.py:88-90), one CTA each; a wave of wave_width indices is
 * looked up against the cache as it stood before the wave, hits refresh recency in wave order, the wave's
 * missed ids are inserted in first-miss order afterwards and the least recently used entries leave while the
 * cache is over capacity (cache.py:106-129).  d_out is device int64[4]: hits, misses, vr_status, 0.
 * d_miss_counts (int32[vertex_count], zeroed by the caller) receives one count per miss, or NULL. */
typedef struct vr_cache_config {
    int32_t num_processors; /* cache.py:29 default 28   */
    int32_t wave_width;     /* cache.py:30 default 1024 */
    int32_t capacity;       /* cache.py:43-47 entries   */
    int32_t primitive_size;
} vr_cache_config;
size_t vr_cache_workspace_bytes(int64_t n_indices, const vr_cache_config *cfg);
int vr_simulate_cache(const uint32_t *d_indices, int64_t n_indices, const vr_cache_config *cfg,
                      int32_t vertex_count, int32_t *d_miss_counts, int64_t *d_out, void *d_workspace,
                      size_t workspace_bytes, void *stream);

/* ---- random-walk client (walk.py) ------------------------------------------------------
 * Agents on a grid, positions packed as virtual indices (y << 16 | x, walk.py:75-82) and run through vr_run
 * with primitive_size 1, so that agents sharing a cell share one likelihood evaluation per batch. */
#define VR_WALK_MAX_GAUSSIANS 8
typedef struct vr_walk_config {   /* walk.py:51-72 WalkConfig */
    int32_t grid_w, grid_h;
    int32_t max_move_distance;
    int32_t kept_moves;
    int32_t n_gaussians;
    int32_t reserved;
    double gaussians[VR_WALK_MAX_GAUSSIANS][4]; /* walk.py:32-36: center x, center y, sigma, amplitude */
} vr_walk_config;
/* walk.py:110-137 cell_likelihoods for n cells: d_moves is double[n][kept_moves][3] = (dx, dy, likelihood),
 * descending likelihood, ties in row-major scan order; FP64.  d_status is device int64[1] (0 or
 * (cell index << 8) | VR_ERR_BAD_CONFIG when a cell has fewer legal moves than kept_moves, walk.py:123-126). */
int vr_walk_likelihoods(const uint32_t *d_cells, int64_t n_cells, const vr_walk_config *cfg, double *d_moves,
                        int64_t *d_status, void *stream);
/* walk.py:140-165 + :202-207: agent a draws u = agent_uniforms(seed, step, a) (splitmix64), picks move
 * choose_move(moves[src[a]], u) and advances.  Positions are int32 (x, y) pairs; d_src is the output of
 * vr_expand_sources (NULL: agent a uses record a -- the per-agent path of walk.py:210-219). */
int vr_walk_advance(const int32_t *d_positions_in, int64_t n_agents, const int32_t *d_src, const double *d_moves,
                    int32_t kept_moves, uint64_t seed, int64_t step, int32_t *d_positions_out, void *stream);
/* walk.py:167-170 pack_positions on the device: cells[a] = y << 16 | x. */
int vr_walk_pack(const int32_t *d_positions, int64_t n_agents, uint32_t *d_cells, void *stream);

/* Profiling aid (bench.py): per-kernel device time of the last vr_run, measured with CUDA
 * events on the launching stream.  Stages, in order: init (+ span scan), dedup, offset scan
 * (+ statistics), shade/finalize (the three-kernel sort/hash path reports its kernels A (+ B) as "dedup" and C as
 * "shade/finalize").  State is per host THREAD: a thread reads what its own last vr_run recorded.
 * vr_profile_read synchronises the last event and returns the number of stages written. */
#define VR_PROFILE_STAGES 4
int vr_profile_enable(int on);
/* Number of kernels the calling thread's last vr_run launched (bench.py's gpu_launches). */
int vr_last_launch_count(void);
int vr_profile_read(float *ms, int cap);
/* Which dedup path the calling thread's last vr_run took (tests and bench.py report it):
 * 0 = generic kernels (K1 -> K2 -> K3), 1 = static-batch warp kernel (unfused), 2 = static-batch warp
 * kernel with fused look-back + shading, 3 = persistent tile kernel (csrc/vr_warp_rows.cuh), 4 = three-kernel
 * sort / hash / phash path for budgeted batches (csrc/vr_dyn3.cuh). */
int vr_last_kernel_path(void);
/* Debugging / ablation knobs (VR_LAG, VR_PREFETCH, VR_LINK_TILE, ...: `DebugKnobs` in csrc/vr_common.cuh) are read
 * from the environment once per process; this re-reads them.  For tests and sweeps that change a knob between
 * runs; not for use while another thread is inside the library. */
int vr_debug_reload_knobs(void);

#ifdef __cplusplus
}
#endif
#endif /* VRGEOM_H */
