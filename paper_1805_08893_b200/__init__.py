"""B200-native software geometry stage with on-the-fly vertex reuse (arXiv 1805.08893).

Drop-in for the hot path of the reference package `vrlab` (same names as
/root/reference/pkg/src/vrlab/__init__.py:9-65 for that path): batch formation, the
naive / warp-voting / sorting / hashing strategies, shading, primitive assembly and reuse
statistics, executed by hand-written sm_100a CUDA kernels behind include/vrgeom.h.
"""
from .analytics import CostEstimate, ReuseReport, build_report, estimate_cost, ideal_report
from .cache import CacheConfig, CacheReport, ideal_reuse, simulate_parallel_cache
from .batching import (Batch, BatchConfig, ConfigError, UnsupportedOnDevice, batches_to_offsets,
                       dynamic_batches, offsets_to_batches, static_batches)
from .mesh import (IndexedMesh, MeshError, VertexShadingCounts, gen_grid, gen_icosphere,
                   shuffle_triangles)
from .strategies import (DedupResult, HashConfig, ProbeStats, Round, ShaderFn, TriangleStream,
                         hash_batch, identity_shader, naive_batch, parallel_hash_batch,
                         position_shader, run_hashing, run_naive, run_on_indices,
                         run_parallel_hashing, run_sorting, run_warp_voting, sort_batch,
                         warp_vote_batch)
from .walk import (Gaussian, WalkConfig, WalkRun, agent_uniforms, cell_likelihoods, choose_move,
                   default_gaussians, initial_positions, likelihood_shader, naive_step, naive_walk,
                   pack_cell, pack_positions, run_walk, step_with_reuse, unpack_cell)
from .warp import WarpState, ballot, ffs, shfl

__version__ = "0.1.0"
