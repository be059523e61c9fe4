"""Multi-draw workloads (BASELINE.json configs[4]: ~1000 meshes, ~20 M triangles, dynamic batching).

The reference has no multi-draw entry point: a scene of many meshes is a loop of
`dynamic_batches(mesh.indices, cfg)` + `run_on_indices(...)` per mesh (strategies.py:404-415),
each with its own vertex buffer and its own greedy scan starting at index 0.  On the device a
loop of a thousand small launches would be launch-bound, so the draws are packed once into ONE
index stream + ONE vertex buffer and processed by one sequence of kernels:

  * batch formation takes the draw boundaries and never lets a batch cross one
    (vr_dynamic_batches_draws), which is exactly "every draw restarts the scan";
  * the dedup kernels see the draw-local ids unchanged, so unique ids, hash tables, local
    indices and statistics are bit-identical to the per-draw runs;
  * the shader reads vertex `base[draw of the batch] + id` (vr_shader.d_batch_vertex_base).

The results are the concatenation, in draw order, of what the reference's per-draw runs return.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import engine
from .analytics import ReuseReport, build_report
from .batching import BatchConfig, ConfigError
from .mesh import IndexedMesh, gen_grid, gen_icosphere, shuffle_triangles


def scene_corpus(count: int, seed: int = 2018, lo: int = 64, hi: int = 176, ico=(4, 6)) -> list:
    """a mixed corpus in the style of the reference's tests/helpers.py:20-40
    (grids, icospheres and shuffled variants, kind = k % 4), at game-scene sizes.  With the
    defaults and count=1000: 20 397 942 triangles, 10 319 577 vertices."""
    rng = np.random.default_rng(seed)
    meshes = []
    spheres = {}  # the few distinct icospheres are built once
    for k in range(count):
        kind = k % 4
        if kind in (0, 2):
            r = int(rng.integers(lo, hi))
            c = int(rng.integers(lo, hi))
            m = gen_grid(r, c)
        else:
            sub = int(rng.integers(ico[0], ico[1]))
            m = spheres.get(sub) or spheres.setdefault(sub, gen_icosphere(sub))
        if kind >= 2:
            m = shuffle_triangles(m, int(rng.integers(0, 2 ** 31)))
        meshes.append(m)
    return meshes


@dataclass
class DrawSet:
    """Packed multi-draw input, resident on the device."""

    indices: torch.Tensor            # int32[sum of index counts], draw-local ids
    positions4: torch.Tensor         # float32[sum of vertex counts, 4]
    index_start: np.ndarray          # int64[n_draws + 1]
    vertex_base: np.ndarray          # int64[n_draws + 1]
    d_index_start: torch.Tensor      # int32 copies on the device
    d_vertex_base: torch.Tensor
    names: tuple = ()

    @property
    def n_draws(self) -> int:
        return len(self.index_start) - 1

    @property
    def triangles(self) -> int:
        return int(self.index_start[-1]) // 3


def pack_draws(meshes, device=None) -> DrawSet:
    """Concatenate the index and vertex buffers of `meshes` (IndexedMesh or (indices, positions))."""
    dev = engine._device(device)
    idx, pos, names = [], [], []
    for m in meshes:
        if isinstance(m, IndexedMesh):
            i, p, nm = m.indices, m.positions, getattr(m, "name", "")
        else:
            i, p = m
            nm = ""
        i = np.ascontiguousarray(i, dtype=np.uint32)
        if len(i) and int(i.max()) >= len(p):
            raise ConfigError("index outside the draw's vertex buffer")
        idx.append(i)
        pos.append(np.asarray(p, dtype=np.float32).reshape(-1, 3))
        names.append(nm)
    istart = np.concatenate([[0], np.cumsum([len(i) for i in idx])]).astype(np.int64)
    vbase = np.concatenate([[0], np.cumsum([len(p) for p in pos])]).astype(np.int64)
    if istart[-1] > 0x7FFFFFFF or vbase[-1] > 0x7FFFFFFF:
        raise ConfigError("multi-draw stream too long for 32-bit positions")
    all_idx = np.concatenate(idx) if idx else np.zeros(0, dtype=np.uint32)
    p4 = np.ones((int(vbase[-1]), 4), dtype=np.float32)
    if pos:
        p4[:, :3] = np.concatenate(pos)
    return DrawSet(indices=engine.to_device_indices(all_idx, dev),
                   positions4=torch.from_numpy(p4).to(dev),
                   index_start=istart, vertex_base=vbase,
                   d_index_start=torch.from_numpy(istart.astype(np.int32)).to(dev),
                   d_vertex_base=torch.from_numpy(vbase.astype(np.int32)).to(dev),
                   names=tuple(names))


def dynamic_offsets_draws(ds: DrawSet, cfg: BatchConfig, workspace=None) -> torch.Tensor:
    """batching.py:87-125 once per draw, in one pass over the packed stream -> int32 offsets
    (positions in the packed stream; length n_batches + 1, or 0 for an empty scene)."""
    lib = N.require_cuda()
    n = ds.indices.numel()
    dev = ds.indices.device
    ps = cfg.primitive_size
    if any(int(v) % ps for v in ds.index_start):
        raise ConfigError("a draw's index count is not primitive-aligned")
    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev)
    c = engine._cfg_c(cfg)
    ws_bytes = lib.vr_dynamic_workspace_bytes(n, C.byref(c))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    offs = torch.empty(n // ps + 1, dtype=torch.int32, device=dev)
    nb = torch.zeros(2, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_dynamic_batches_draws(
            engine._ptr(ds.indices), n, C.byref(c), engine._ptr(ds.d_index_start), ds.n_draws,
            engine._ptr(offs), engine._ptr(nb), engine._ptr(workspace), ws_bytes, engine._stream_ptr()))
    nbh = nb.cpu()
    if int(nbh[1]) != 0:
        engine.raise_status(int(nbh[1]))
    return offs[: int(nbh[0]) + 1]


def static_offsets_draws(ds: DrawSet, cfg: BatchConfig) -> torch.Tensor:
    """batching.py:76-84 once per draw (host arithmetic: the boundaries are closed-form)."""
    parts = []
    for d in range(ds.n_draws):
        a, b = int(ds.index_start[d]), int(ds.index_start[d + 1])
        if (b - a) % cfg.primitive_size:
            raise ConfigError("a draw's index count is not primitive-aligned")
        parts.append(np.arange(a, b, cfg.batch_size, dtype=np.int64))
    parts.append(np.array([int(ds.index_start[-1])], dtype=np.int64))
    offs = np.concatenate(parts)
    if len(offs) == 1:
        return torch.zeros(0, dtype=torch.int32, device=ds.indices.device)
    return torch.from_numpy(offs.astype(np.int32)).to(ds.indices.device)


def batch_vertex_base(ds: DrawSet, offsets: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """First vertex of each batch's draw (vr_batch_vertex_base)."""
    lib = N.require_cuda()
    nb = max(offsets.numel() - 1, 0)
    dev = ds.indices.device
    if out is None or out.numel() < max(nb, 1):
        out = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_batch_vertex_base(engine._ptr(offsets), nb, engine._ptr(ds.d_index_start),
                                                     engine._ptr(ds.d_vertex_base), ds.n_draws, engine._ptr(out),
                                                     engine._stream_ptr()))
    return out


def run_draws(strategy: str, ds: DrawSet, offsets: torch.Tensor, cfg: BatchConfig, hcfg=None, *,
              matrix=None, shade: bool = True, want_counts: bool = False, buffers=None,
              vbase: torch.Tensor | None = None) -> engine.DeviceRun:
    """One vr_run over every batch of every draw.  `max_span` is the longest batch the batching
    rule allows, so no host round trip is needed between batch formation and the run."""
    nb = max(offsets.numel() - 1, 0)
    n = ds.indices.numel()
    if vbase is None:
        vbase = batch_vertex_base(ds, offsets)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION if shade else N.VR_SHADER_IDENTITY,
                             positions4=ds.positions4 if shade else None, matrix=matrix,
                             vertex_count=int(ds.vertex_base[-1]), batch_vertex_base=vbase)
    max_span = min(max(cfg.batch_size, cfg.max_indices - cfg.max_indices % cfg.primitive_size), max(n, 1))
    run = engine.run_device(strategy, ds.indices, offsets[:-1] if nb else offsets, offsets[1:] if nb else offsets,
                            nb, n, max_span, cfg, hcfg, spec, want_counts=want_counts, buffers=buffers)
    return run


def per_draw_reports(run: engine.DeviceRun, ds: DrawSet, offsets: torch.Tensor, strategy: str) -> list:
    """One ReuseReport per draw (analytics.py:20-50), as the reference's per-mesh runs would print."""
    flat_bro = run.batch_round_off[: run.n_batches + 1].cpu().numpy().astype(np.int64)
    ruo = run.round_uid_off[: run.rounds + 1].cpu().numpy().astype(np.int64)
    offs = offsets.cpu().numpy().astype(np.int64)
    first = np.searchsorted(offs[:-1], ds.index_start[:-1], side="left") if len(offs) else np.zeros(ds.n_draws, int)
    last = np.searchsorted(offs[:-1], ds.index_start[1:], side="left") if len(offs) else np.zeros(ds.n_draws, int)
    out = []
    for d in range(ds.n_draws):
        b0, b1 = int(first[d]), int(last[d])
        inv = int(ruo[flat_bro[b1]] - ruo[flat_bro[b0]]) if b1 > b0 else 0
        out.append(build_report(scene=ds.names[d] if d < len(ds.names) else "", strategy=strategy,
                                indices=int(ds.index_start[d + 1] - ds.index_start[d]), invocations=inv,
                                batches=b1 - b0))
    return out
