"""The vertex-processing strategies behind the reference's Python API, executed on the GPU.

Host mirror of `vrlab/strategies.py` (/root/reference/pkg/src/vrlab/strategies.py): same names,
signatures, defaults, return shapes and exception types for

  ShaderFn / identity_shader / position_shader   :36-67
  HashConfig (+ .slot)                           :70-91
  ProbeStats, Round, DedupResult                 :94-129
  TriangleStream                                 :132-152
  naive_batch / warp_vote_batch / sort_batch / hash_batch       :159-298
  run_on_indices and the run_* wrappers          :404-533

All work happens in libvrgeom.so (csrc/*.cu) through include/vrgeom.h; there is no CPU fallback.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from . import analytics
from .batching import Batch, BatchConfig, ConfigError, UnsupportedOnDevice
from .mesh import IndexedMesh
from .warp import check_width

SENTINEL = -1  # strategies.py:27
WORKER_ENV = "VRLAB_THREADS"  # strategies.py:29
FIBONACCI_MULTIPLIER = 2654435769  # strategies.py:33
STRATEGY_NAMES = ("naive", "warp", "sort", "hash", "phash")  # strategies.py:387
_DYNAMIC = {"sort", "hash", "phash"}


@dataclass(frozen=True)
class ShaderFn:
    """Vertex shader descriptor (strategies.py:36-45).

    `fn` keeps the reference's per-id callable for API compatibility, but the runners never
    call it: they execute the device shader named by `device` (identity / position).  A
    ShaderFn built around an arbitrary Python callable has no device form and is rejected
    with ConfigError -- there is no CPU fallback."""

    fn: Callable[[int], object]
    cycles: int = 1
    name: str = "shader"
    device: tuple | None = field(default=None, compare=False, repr=False)


def identity_shader() -> ShaderFn:
    """Record = vertex id (strategies.py:48-50)."""
    return ShaderFn(fn=lambda vid: np.uint32(vid), cycles=1, name="identity", device=("identity",))


def position_shader(mesh: IndexedMesh, matrix: np.ndarray | None = None, cycles: int = 1) -> ShaderFn:
    """Record = (matrix-transformed, w-divided) position as float32[3] (strategies.py:53-67).
    On the device the transform runs in FP32 (1e-5 relative to the reference's float64)."""
    positions = mesh.positions
    m = None if matrix is None else np.asarray(matrix, dtype=np.float64)

    def fn(vid: int):
        if m is None:
            return positions[vid].astype(np.float32)
        out = m @ np.append(positions[vid], 1.0)
        return (out[:3] / out[3]).astype(np.float32)

    return ShaderFn(fn=fn, cycles=cycles, name="position", device=("position", mesh, m))


@dataclass(frozen=True)
class HashConfig:
    """Open-addressing table parameters (strategies.py:70-91)."""

    table_size: int = 256
    multiplier: int = FIBONACCI_MULTIPLIER
    max_fast_probes: int = 8

    def __post_init__(self):
        if self.table_size < 1 or self.table_size & (self.table_size - 1):
            raise ConfigError("table_size must be a power of two")
        if self.multiplier % 2 == 0:
            raise ConfigError("multiplier must be odd")
        if not 0 < self.multiplier < 2**32:
            raise ConfigError("multiplier must be a 32-bit constant")
        if self.max_fast_probes < 1:
            raise ConfigError("max_fast_probes must be >= 1")

    def slot(self, vid: int) -> int:
        """Multiplicative hash into [0, table_size) (strategies.py:88-91)."""
        shift = 32 - (self.table_size.bit_length() - 1)
        return ((vid * self.multiplier) & 0xFFFFFFFF) >> shift


@dataclass(frozen=True)
class ProbeStats:
    """Slot inspections of the hashing kernels (strategies.py:94-111)."""

    fast: int = 0
    slow: int = 0
    max_chain: int = 0

    @property
    def total(self) -> int:
        return self.fast + self.slow

    def merge(self, other: "ProbeStats") -> "ProbeStats":
        return ProbeStats(self.fast + other.fast, self.slow + other.slow,
                          max(self.max_chain, other.max_chain))


@dataclass(frozen=True)
class Round:
    """One shading round (strategies.py:114-120)."""

    unique_ids: tuple
    assembly_map: tuple
    primitives_emitted: int


@dataclass(frozen=True)
class DedupResult:
    """Per-batch output contract of all strategies (strategies.py:123-129)."""

    rounds: tuple
    invocations: int
    indices_consumed: int


class TriangleStream:
    """Queue of shaded-vertex records, primitive_size per primitive (strategies.py:132-152).

    Backed by the device result: the per-corner expansion `shaded[assembly_map]` is produced
    by vr_expand_stream on first access and cached as a NumPy array."""

    def __init__(self, primitive_size: int = 3, records: list | None = None, *, _run=None,
                 _positions: bool = False):
        self.primitive_size = primitive_size
        self._run = _run
        self._positions = _positions
        self._array = None
        self._records = records if records is not None else ([] if _run is None else None)

    def as_array(self) -> np.ndarray:
        """(n,3) float32 for the position shader, (n,) uint32 for identity (strategies.py:147-148)."""
        if self._run is None:
            return np.asarray(self._records)
        if self._array is None:
            dev = self._run.expand_stream(self._positions)
            arr = dev.cpu().numpy()
            self._array = arr if self._positions else arr.view(np.uint32)
        return self._array

    @property
    def records(self) -> list:
        if self._records is None:
            self._records = list(self.as_array())
        return self._records

    def __len__(self) -> int:
        if self._run is not None:
            return self._run.indices // self.primitive_size
        return len(self._records) // self.primitive_size

    def primitives(self):
        ps = self.primitive_size
        rec = self.records
        for i in range(0, len(rec), ps):
            yield tuple(rec[i:i + ps])

    def write_binary(self, path: str | Path) -> None:
        """Flat dump, native byte order (strategies.py:150-152)."""
        self.as_array().tofile(path)


# ---------------------------------------------------------------------------
# per-batch kernels: one-batch launches of the device path
# ---------------------------------------------------------------------------
def _single_batch(strategy: str, ids, cfg: BatchConfig, hcfg: HashConfig | None):
    from . import engine
    import torch

    arr = np.ascontiguousarray(np.asarray(ids), dtype=np.uint32)
    n = len(arr)
    d_idx = engine.to_device_indices(arr)
    offs = torch.tensor([0, n], dtype=torch.int32, device=d_idx.device)
    run = engine.run_device(strategy, d_idx, offs[:1], offs[1:], 1, n, max(n, 1), cfg, hcfg,
                            engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY), enforce_budget=False)
    return run, run.flat()


def _result_from_flat(flat: dict, ps: int, batch: int = 0) -> DedupResult:
    r0, r1 = int(flat["batch_round_off"][batch]), int(flat["batch_round_off"][batch + 1])
    rounds = []
    m = int(flat["round_prims"][:r0].sum()) * ps
    inv = 0
    for r in range(r0, r1):
        a, b = int(flat["round_uid_off"][r]), int(flat["round_uid_off"][r + 1])
        k = int(flat["round_prims"][r]) * ps
        rounds.append(Round(tuple(int(v) for v in flat["unique_ids"][a:b]),
                            tuple(int(v) for v in flat["assembly_map"][m:m + k]),
                            int(flat["round_prims"][r])))
        m += k
        inv += b - a
    consumed = sum(rd.primitives_emitted for rd in rounds) * ps
    return DedupResult(tuple(rounds), invocations=inv, indices_consumed=consumed)


def _batch_cfg(n: int, ps: int, warp_width: int = 32) -> BatchConfig:
    size = max(ps, n)
    return BatchConfig(batch_size=size, max_unique=max(size, ps), max_indices=max(size, ps),
                       warp_width=warp_width, primitive_size=ps)


def naive_batch(ids, primitive_size: int = 3) -> DedupResult:
    """No reuse: one invocation per index slot (strategies.py:159-170)."""
    if len(ids) == 0:
        return DedupResult((), 0, 0)
    _, flat = _single_batch("naive", ids, _batch_cfg(len(ids), primitive_size), None)
    return _result_from_flat(flat, primitive_size)


def warp_vote_batch(ids, warp_width: int, primitive_size: int = 3) -> DedupResult:
    """Warp-voting dedup of one static batch (strategies.py:173-232)."""
    w = check_width(warp_width)
    if w < primitive_size:
        raise ConfigError("warp width below primitive size cannot make progress")
    if len(ids) == 0:
        return DedupResult((), 0, 0)
    _, flat = _single_batch("warp", ids, _batch_cfg(len(ids), primitive_size, w), None)
    return _result_from_flat(flat, primitive_size)


def sort_batch(ids, primitive_size: int = 3) -> DedupResult:
    """Sorting dedup: unique ids ascending, map = rank (strategies.py:235-260)."""
    if len(ids) == 0:
        return DedupResult((), 0, 0)
    cfg = _batch_cfg(len(ids), primitive_size)
    run, flat = _single_batch("sort", ids, cfg, None)
    return _result_from_flat(flat, primitive_size)


def hash_batch(ids, hash_cfg: HashConfig, primitive_size: int = 3):
    """Hashing dedup with the reference's table layout and probe statistics (strategies.py:263-298)."""
    if len(ids) == 0:
        return DedupResult((Round((), (), 0),), 0, 0), ProbeStats()
    n = len(ids)
    size = max(primitive_size, n)
    # the per-batch kernel has no unique budget (strategies.py:451 belongs to the runner)
    cfg = BatchConfig(batch_size=size, max_unique=size, max_indices=size, primitive_size=primitive_size)
    run, flat = _single_batch("hash", ids, cfg, hash_cfg)
    fast, slow, mx = run.probes
    return _result_from_flat(flat, primitive_size), ProbeStats(fast=fast, slow=slow, max_chain=mx)


def parallel_hash_batch(ids, hash_cfg: HashConfig, warp_width: int, primitive_size: int = 3):
    """Two-tier hashing (strategies.py:301-367): same stream and invocation count as hash_batch, its own
    table layout and probe statistics (fast / slow)."""
    w = check_width(warp_width)
    if len(ids) == 0:
        return DedupResult((Round((), (), 0),), 0, 0), ProbeStats()
    n = len(ids)
    size = max(primitive_size, n)
    cfg = BatchConfig(batch_size=size, max_unique=size, max_indices=size, warp_width=w, primitive_size=primitive_size)
    run, flat = _single_batch("phash", ids, cfg, hash_cfg)
    fast, slow, mx = run.probes
    return _result_from_flat(flat, primitive_size), ProbeStats(fast=fast, slow=slow, max_chain=mx)


# ---------------------------------------------------------------------------
# runners
# ---------------------------------------------------------------------------
def effective_workers(requested: int) -> int:
    """strategies.py:392-401.  Accepted for compatibility: the device path ignores it."""
    cap = os.environ.get(WORKER_ENV)
    workers = max(1, int(requested))
    if cap is not None:
        try:
            workers = min(workers, max(1, int(cap)))
        except ValueError:
            raise ConfigError(f"{WORKER_ENV} must be an integer, got {cap!r}") from None
    return workers


def _shader_spec(shader: ShaderFn, device, vertex_count):
    from . import engine

    dev = getattr(shader, "device", None)
    if dev is None:
        raise ConfigError(
            f"shader {shader.name!r} is an arbitrary Python callable; the device path runs "
            "identity_shader() or position_shader() only (no CPU fallback)")
    if dev[0] == "identity":
        return engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=vertex_count or 0), False
    _, mesh, matrix = dev
    cache = mesh.__dict__.get("_vr_pos4")
    if cache is None or cache.device != device:
        cache = engine.to_device_positions4(mesh.positions, device)
        object.__setattr__(mesh, "_vr_pos4", cache)
    # ShaderFn.cycles (strategies.py:40-44) is the abstract per-invocation load of the cost model; on the device
    # cycles > 1 runs that many extra dependent FMAs per invocation (PAPER.md:661's synthetic shader loads)
    return engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=cache, matrix=matrix,
                             vertex_count=vertex_count or mesh.vertex_count,
                             extra_cycles=max(int(shader.cycles) - 1, 0)), True


def run_on_indices(strategy: str, indices, batches, cfg: BatchConfig, shader: ShaderFn,
                   hash_cfg: HashConfig | None = None, *, vertex_count: int | None = None,
                   scene: str = "", workers: int = 1):
    """Run one strategy over raw indices on the GPU (strategies.py:404-502).

    `batches` is a sequence of Batch as in the reference, or a device-resident int32 offsets
    tensor from engine.static_offsets_device / dynamic_offsets_device.  Returns (stream, report)
    and additionally ProbeStats for the hashing strategies."""
    from . import engine
    import torch

    if strategy not in STRATEGY_NAMES:
        raise ConfigError(f"unknown strategy {strategy!r}; expected one of {STRATEGY_NAMES}")
    effective_workers(workers)
    ps = cfg.primitive_size
    n_idx = int(indices.numel()) if isinstance(indices, torch.Tensor) else len(indices)

    offsets_on_device = isinstance(batches, torch.Tensor)
    if offsets_on_device:
        nb = max(int(batches.numel()) - 1, 0)
        max_span = max(cfg.batch_size, cfg.max_indices)
        span_total = n_idx
        contiguous = True
        static = getattr(batches, "vr_static_batch_size", None) == cfg.batch_size
    else:
        nb = len(batches)
        if nb:
            bb = np.fromiter((b.begin for b in batches), dtype=np.int64, count=nb)
            be = np.fromiter((b.end for b in batches), dtype=np.int64, count=nb)
            bad = ~((0 <= bb) & (bb < be) & (be <= n_idx) & ((be - bb) % ps == 0))
            if bad.any():  # strategies.py:426-428
                k = int(np.argmax(bad))
                raise ConfigError(f"batch {batches[k]} is not a primitive-aligned range of the buffer")
            max_span = int((be - bb).max())
            span_total = int((be - bb).sum())
            contiguous = bool((bb[1:] == be[:-1]).all())
            # static_batches(n, cfg) shifted to a 16-byte aligned start (the position-aligned kernels load
            # index quads); any other equally spaced list takes the general kernels
            static = bool(contiguous and bb[0] % 4 == 0 and (np.diff(bb) == cfg.batch_size).all()
                          and (be[-1] - bb[-1]) <= cfg.batch_size)

    if strategy in ("hash", "phash"):
        hash_cfg = hash_cfg or HashConfig(table_size=cfg.block_size)  # strategies.py:431
        if hash_cfg.table_size < cfg.max_unique:
            raise ConfigError(
                f"hash table_size {hash_cfg.table_size} below max_unique {cfg.max_unique}")
    if strategy == "warp" and nb and cfg.warp_width < ps:
        raise ConfigError("warp width below primitive size cannot make progress")

    probe_total = ProbeStats() if strategy in ("hash", "phash") else None
    if nb == 0:  # strategies.py:472-502 with an empty result list
        stream = TriangleStream(primitive_size=ps)
        counts = np.zeros(vertex_count, dtype=np.int64) if vertex_count is not None else None
        report = analytics.build_report(scene=scene, strategy=strategy, indices=0, invocations=0,
                                        batches=0, shade_counts=counts, probe_stats=probe_total)
        return (stream, report, probe_total) if probe_total is not None else (stream, report)

    d_idx = engine.to_device_indices(indices)
    dev = d_idx.device
    if offsets_on_device:
        offs = batches.to(dev, torch.int32)
        d_begin, d_end = offs[:-1], offs[1:]
    else:
        both = torch.from_numpy(np.stack([bb, be]).astype(np.int32)).to(dev)
        d_begin, d_end = both[0], both[1]
    spec, positions = _shader_spec(shader, dev, vertex_count)
    run = engine.run_device(strategy, d_idx, d_begin, d_end, nb, span_total, max_span, cfg, hash_cfg,
                            spec, want_counts=vertex_count is not None, contiguous=contiguous, static=static)
    run.check()

    shade_counts = None
    if vertex_count is not None:
        shade_counts = run.shade_counts[:vertex_count].cpu().numpy().astype(np.int64)
    if probe_total is not None:
        fast, slow, mx = run.probes
        probe_total = ProbeStats(fast=fast, slow=slow, max_chain=mx)
    report = analytics.build_report(scene=scene, strategy=strategy, indices=run.indices,
                                    invocations=run.invocations, batches=nb,
                                    shade_counts=shade_counts, probe_stats=probe_total)
    stream = TriangleStream(primitive_size=ps, _run=run, _positions=positions)
    stream.device_run = run
    if probe_total is not None:
        return stream, report, probe_total
    return stream, report


def run_naive(mesh: IndexedMesh, batches, shader: ShaderFn, *, cfg: BatchConfig | None = None,
              scene: str = "", workers: int = 1):
    """strategies.py:505-509."""
    cfg = cfg or BatchConfig()
    return run_on_indices("naive", mesh.indices, batches, cfg, shader,
                          vertex_count=mesh.vertex_count, scene=scene, workers=workers)


def run_warp_voting(mesh: IndexedMesh, batches, cfg: BatchConfig, shader: ShaderFn, *,
                    scene: str = "", workers: int = 1):
    """strategies.py:512-515."""
    return run_on_indices("warp", mesh.indices, batches, cfg, shader,
                          vertex_count=mesh.vertex_count, scene=scene, workers=workers)


def run_sorting(mesh: IndexedMesh, batches, cfg: BatchConfig, shader: ShaderFn, *,
                scene: str = "", workers: int = 1):
    """strategies.py:518-521."""
    return run_on_indices("sort", mesh.indices, batches, cfg, shader,
                          vertex_count=mesh.vertex_count, scene=scene, workers=workers)


def run_hashing(mesh: IndexedMesh, batches, cfg: BatchConfig, hash_cfg: HashConfig,
                shader: ShaderFn, *, scene: str = "", workers: int = 1):
    """strategies.py:524-527."""
    return run_on_indices("hash", mesh.indices, batches, cfg, shader, hash_cfg,
                          vertex_count=mesh.vertex_count, scene=scene, workers=workers)


def run_parallel_hashing(mesh: IndexedMesh, batches, cfg: BatchConfig, hash_cfg: HashConfig,
                         shader: ShaderFn, *, scene: str = "", workers: int = 1):
    """strategies.py:530-533."""
    return run_on_indices("phash", mesh.indices, batches, cfg, shader, hash_cfg,
                          vertex_count=mesh.vertex_count, scene=scene, workers=workers)
