"""Parallel random walk whose per-cell move evaluation runs through the dedup engine, on the device.

Host mirror of `vrlab/walk.py` (/root/reference/pkg/src/vrlab/walk.py): same names,
signatures, defaults and exception types for

  Gaussian / default_gaussians / WalkConfig        :31-72
  pack_cell / unpack_cell / pack_positions         :75-82, :167-170
  cell_likelihoods / likelihood_shader             :110-137, :173-174
  agent_uniforms / choose_move                     :140-165
  step_with_reuse / naive_step                     :177-219
  initial_positions / run_walk / naive_walk        :222-276

Agent positions are packed into 32-bit virtual indices (y << 16 | x) and fed to the vertex-reuse
strategies with primitive size 1 (`vr_run`), so agents sharing a grid cell share one likelihood
evaluation per batch; the likelihood "shader" (`vr_walk_likelihoods`, FP64, one warp per unique cell),
the counter-based uniforms and the move selection (`vr_walk_advance`) run on the GPU.  `agent_uniforms`,
`choose_move` and the packing helpers are kept as small host functions for API parity (exact integer /
IEEE arithmetic, the same results as the device code).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as N
from .analytics import ReuseReport, build_report
from .batching import BatchConfig, ConfigError
from .strategies import HashConfig, ProbeStats, ShaderFn

PackedCell = int  # 32-bit word: y in the high 16 bits, x in the low 16

_GRID_LIMIT = 65536  # walk.py:24
_MAX_CANDIDATES = 1024  # device limit (kWalkMaxCandidates): moves within max_move_distance


@dataclass(frozen=True)
class Gaussian:  # walk.py:31-35
    center: tuple[float, float]
    sigma: float
    amplitude: float = 1.0


def default_gaussians(grid: tuple[int, int]) -> tuple[Gaussian, ...]:
    """Three activity peaks spread over the grid (walk.py:38-47)."""
    w, h = grid
    s = max(w, h) / 6.0
    return (
        Gaussian(center=(0.25 * w, 0.25 * h), sigma=s),
        Gaussian(center=(0.70 * w, 0.60 * h), sigma=s),
        Gaussian(center=(0.40 * w, 0.80 * h), sigma=s * 0.5, amplitude=0.5),
    )


@lru_cache(maxsize=8)
def _candidate_count(max_distance: int) -> int:
    d = max_distance
    return sum(1 for dy in range(-d, d + 1) for dx in range(-d, d + 1) if dx * dx + dy * dy <= d * d)


@dataclass(frozen=True)
class WalkConfig:  # walk.py:50-72
    grid: tuple[int, int] = (256, 256)
    agents: int = 300_000
    max_move_distance: int = 16
    kept_moves: int = 8
    gaussians: tuple[Gaussian, ...] | None = None
    steps: int = 10
    rng_seed: int = 0

    def __post_init__(self):
        w, h = self.grid
        if not (2 <= w <= _GRID_LIMIT and 2 <= h <= _GRID_LIMIT):
            raise ConfigError(f"grid sides must be in [2, {_GRID_LIMIT}]")
        if self.agents < 1:
            raise ConfigError("need at least one agent")
        if self.max_move_distance < 1:
            raise ConfigError("max_move_distance must be >= 1")
        if self.kept_moves < 1 or self.kept_moves > _candidate_count(self.max_move_distance):
            raise ConfigError("kept_moves must be within the candidate move count")
        if self.steps < 0:
            raise ConfigError("steps must be >= 0")
        if self.gaussians is None:
            object.__setattr__(self, "gaussians", default_gaussians(self.grid))


def pack_cell(x: int, y: int) -> PackedCell:
    return (y << 16) | x


def unpack_cell(packed: PackedCell) -> tuple[int, int]:
    return packed & 0xFFFF, packed >> 16


def pack_positions(positions: np.ndarray) -> np.ndarray:
    xs = positions[:, 0].astype(np.uint32)
    ys = positions[:, 1].astype(np.uint32)
    return (ys << np.uint32(16)) | xs


def _walk_c(cfg: WalkConfig) -> N.WalkConfigC:
    if len(cfg.gaussians) > N.VR_WALK_MAX_GAUSSIANS or _candidate_count(cfg.max_move_distance) > _MAX_CANDIDATES:
        from .batching import UnsupportedOnDevice
        raise UnsupportedOnDevice("walk configuration outside the device limits (8 Gaussians, 1024 candidate moves)")
    c = N.WalkConfigC()
    c.grid_w, c.grid_h = cfg.grid
    c.max_move_distance, c.kept_moves, c.n_gaussians = cfg.max_move_distance, cfg.kept_moves, len(cfg.gaussians)
    for i, g in enumerate(cfg.gaussians):
        c.gaussians[i][0], c.gaussians[i][1] = float(g.center[0]), float(g.center[1])
        c.gaussians[i][2], c.gaussians[i][3] = float(g.sigma), float(g.amplitude)
    return c


def _likelihoods_device(d_cells, cfg: WalkConfig):
    """(n, kept_moves, 3) float64 device tensor of (dx, dy, likelihood) rows for n packed cells."""
    from . import engine
    import torch

    lib = N.require_cuda()
    n = int(d_cells.numel())
    dev = d_cells.device
    moves = torch.empty((n, cfg.kept_moves, 3), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int64, device=dev)
    c = _walk_c(cfg)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_walk_likelihoods(engine._ptr(d_cells), n, C.byref(c), engine._ptr(moves),
                                                    engine._ptr(status), engine._stream_ptr()))
    return moves, status


def _check_cells(status, d_cells, cfg: WalkConfig):
    st = int(status.item())
    if st:  # walk.py:123-126
        x, y = unpack_cell(int(d_cells[st >> 8].item()) & 0xFFFFFFFF)
        raise ConfigError(f"cell ({x},{y}) has fewer legal moves than kept_moves {cfg.kept_moves}")


def cell_likelihoods(cell: PackedCell, cfg: WalkConfig) -> np.ndarray:
    """Top kept_moves (dx, dy, likelihood) rows for one grid cell (walk.py:110-137), evaluated on the device."""
    import torch

    d_cells = torch.tensor([int(cell) & 0xFFFFFFFF], dtype=torch.int64, device="cuda").to(torch.int32)
    moves, status = _likelihoods_device(d_cells, cfg)
    _check_cells(status, d_cells, cfg)
    out = moves[0].cpu().numpy()
    out.flags.writeable = False
    return out


def likelihood_shader(cfg: WalkConfig) -> ShaderFn:  # walk.py:173-174
    return ShaderFn(fn=lambda cell: cell_likelihoods(int(cell), cfg), cycles=1, name="likelihood",
                    device=("likelihood", cfg))


_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX_A = np.uint64(0xBF58476D1CE4E5B9)
_MIX_B = np.uint64(0x94D049BB133111EB)


def _mix64(z):  # walk.py:140-149
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = z ^ (z >> np.uint64(30))
        z = z * _MIX_A
        z = z ^ (z >> np.uint64(27))
        z = z * _MIX_B
        z = z ^ (z >> np.uint64(31))
    return z


def agent_uniforms(seed: int, step: int, agent_ids: np.ndarray) -> np.ndarray:
    """Counter-based uniforms in [0, 1), keyed by (seed, step, agent id) (walk.py:152-158); host copy of the
    generator inside vr_walk_advance."""
    key = (seed + 0x9E3779B97F4A7C15 * (step + 1)) & 0xFFFFFFFFFFFFFFFF
    base = _mix64(np.uint64(key))
    with np.errstate(over="ignore"):
        z = _mix64(np.asarray(agent_ids).astype(np.uint64) + base)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0**-53


def choose_move(moves: np.ndarray, u: float) -> int:  # walk.py:161-165
    cum = np.cumsum(moves[:, 2])
    r = u * cum[-1]
    return min(int(np.searchsorted(cum, r, side="right")), len(cum) - 1)


def _to_device_positions(positions):
    import torch

    if isinstance(positions, torch.Tensor):
        return positions.to("cuda", torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(positions, dtype=np.int32)).cuda()


def _advance(d_pos, d_src, moves, cfg: WalkConfig, step_index: int):
    from . import engine
    import torch

    lib = N.require_cuda()
    out = torch.empty_like(d_pos)
    with torch.cuda.device(d_pos.device):
        engine.raise_status(lib.vr_walk_advance(engine._ptr(d_pos), d_pos.shape[0],
                                                engine._ptr(d_src) if d_src is not None else None, engine._ptr(moves),
                                                cfg.kept_moves, cfg.rng_seed & 0xFFFFFFFFFFFFFFFF, step_index,
                                                engine._ptr(out), engine._stream_ptr()))
    return out


def _pack_device(d_pos):
    from . import engine
    import torch

    lib = N.require_cuda()
    cells = torch.empty(d_pos.shape[0], dtype=torch.int32, device=d_pos.device)
    with torch.cuda.device(d_pos.device):
        engine.raise_status(lib.vr_walk_pack(engine._ptr(d_pos), d_pos.shape[0], engine._ptr(cells), engine._stream_ptr()))
    return cells


def _step_device(d_pos, cfg: WalkConfig, step_index: int, strategy: str, bcfg: BatchConfig,
                 hash_cfg: HashConfig | None, scene: str):
    """One step with every stage on the device; returns (new positions, report)."""
    from . import engine
    import torch

    lib = N.require_cuda()
    if bcfg.primitive_size != 1:
        raise ConfigError("walk batching uses primitive_size 1")
    n = int(d_pos.shape[0])
    d_cells = _pack_device(d_pos)
    if strategy in ("sort", "hash", "phash"):
        offs = engine.dynamic_offsets_device(d_cells, bcfg)
        static = False
        if strategy != "sort":
            hash_cfg = hash_cfg or HashConfig(table_size=bcfg.block_size)  # strategies.py:431
            if hash_cfg.table_size < bcfg.max_unique:
                raise ConfigError(f"hash table_size {hash_cfg.table_size} below max_unique {bcfg.max_unique}")
    else:
        offs = engine.static_offsets_device(n, bcfg)
        static = True
    nb = int(offs.numel()) - 1
    run = engine.run_device(strategy, d_cells, offs[:-1], offs[1:], nb, n, max(bcfg.batch_size, bcfg.max_indices),
                            bcfg, hash_cfg, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY), contiguous=True,
                            static=static and strategy == "warp")
    run.check()
    u = run.invocations
    moves, status = _likelihoods_device(run.unique_ids[:u], cfg)
    src = torch.empty(n, dtype=torch.int32, device=d_pos.device)
    ws = torch.empty((nb + 1) * 4 + 256, dtype=torch.uint8, device=d_pos.device)
    with torch.cuda.device(d_pos.device):
        engine.raise_status(lib.vr_expand_sources(engine._ptr(run.batch_round_off), engine._ptr(run.round_uid_off),
                                                  engine._ptr(run.round_prims), engine._ptr(run.assembly_map), nb,
                                                  engine._ptr(run.batch_begin), engine._ptr(run.batch_end), 1,
                                                  engine._ptr(src), engine._ptr(ws), ws.numel(), engine._stream_ptr()))
    _check_cells(status, run.unique_ids[:u], cfg)
    new_pos = _advance(d_pos, src, moves, cfg, step_index)
    probe = None
    if strategy in ("hash", "phash"):
        fast, slow, mx = run.probes
        probe = ProbeStats(fast=fast, slow=slow, max_chain=mx)
    report = build_report(scene=f"{scene}/step{step_index}", strategy=strategy, indices=run.indices,
                          invocations=u, batches=nb, probe_stats=probe)
    return new_pos, report


def step_with_reuse(positions: np.ndarray, cfg: WalkConfig, step_index: int, strategy: str = "sort",
                    batch_cfg: BatchConfig | None = None, hash_cfg: HashConfig | None = None, *,
                    scene: str = "walk", workers: int = 1) -> tuple[np.ndarray, ReuseReport]:
    """Advance every agent one step, deduplicating likelihood evaluations (walk.py:177-207).  Returns the new
    (N, 2) positions and the step's ReuseReport; invocation counts equal the per-batch unique occupied cells."""
    bcfg = batch_cfg or BatchConfig(primitive_size=1)
    d_new, report = _step_device(_to_device_positions(positions), cfg, step_index, strategy, bcfg, hash_cfg, scene)
    return d_new.cpu().numpy().astype(np.asarray(positions).dtype), report


def naive_step(positions: np.ndarray, cfg: WalkConfig, step_index: int) -> np.ndarray:
    """Per-agent evaluation: no batching, no dedup (walk.py:210-219)."""
    d_pos = _to_device_positions(positions)
    d_cells = _pack_device(d_pos)
    moves, status = _likelihoods_device(d_cells, cfg)
    _check_cells(status, d_cells, cfg)
    return _advance(d_pos, None, moves, cfg, step_index).cpu().numpy().astype(np.asarray(positions).dtype)


def initial_positions(cfg: WalkConfig) -> np.ndarray:
    """Seeded uniform scatter over the grid, (N, 2) int64 (walk.py:222-230)."""
    rng = np.random.default_rng(cfg.rng_seed)
    w, h = cfg.grid
    out = np.empty((cfg.agents, 2), dtype=np.int64)
    out[:, 0] = rng.integers(0, w, cfg.agents)
    out[:, 1] = rng.integers(0, h, cfg.agents)
    return out


@dataclass(frozen=True)
class WalkRun:
    trajectory: np.ndarray  # (steps + 1, N, 2)
    reports: list


def run_walk(cfg: WalkConfig, strategy: str = "sort", batch_cfg: BatchConfig | None = None,
             hash_cfg: HashConfig | None = None, *, initial: np.ndarray | None = None, scene: str = "walk",
             workers: int = 1) -> WalkRun:
    """walk.py:239-258; the positions stay on the device between steps."""
    positions = initial.copy() if initial is not None else initial_positions(cfg)
    bcfg = batch_cfg or BatchConfig(primitive_size=1)
    trajectory = np.empty((cfg.steps + 1, len(positions), 2), dtype=np.int64)
    trajectory[0] = positions
    d_pos = _to_device_positions(positions)
    reports = []
    for t in range(cfg.steps):
        d_pos, report = _step_device(d_pos, cfg, t, strategy, bcfg, hash_cfg, scene)
        trajectory[t + 1] = d_pos.cpu().numpy()
        reports.append(report)
    return WalkRun(trajectory=trajectory, reports=reports)


def naive_walk(cfg: WalkConfig, *, initial: np.ndarray | None = None) -> np.ndarray:
    """Trajectory by the per-agent path (the dedup-transparency check, walk.py:261-276)."""
    positions = initial.copy() if initial is not None else initial_positions(cfg)
    trajectory = np.empty((cfg.steps + 1, len(positions), 2), dtype=np.int64)
    trajectory[0] = positions
    for t in range(cfg.steps):
        positions = naive_step(positions, cfg, t)
        trajectory[t + 1] = positions
    return trajectory
