"""Per-multiprocessor LRU post-transform cache simulation and the ideal rate, on the device.

Host mirror of `vrlab/cache.py` (/root/reference/pkg/src/vrlab/cache.py): `CacheConfig` :18-47,
`CacheReport` :50-58, `ideal_reuse` :61-66, `simulate_parallel_cache` :69-100 (the simulation itself,
`_simulate_one` :103-130, is `cache_sim_kernel` in csrc/vr_clients.cu: one CTA per processor chunk).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class CacheConfig:
    """Parallel cache model parameters (cache.py:18-47)."""

    num_processors: int = 28
    wave_width: int = 1024
    cache_bytes: int = 16384
    entry_bytes: int = 64
    entries: int | None = None

    def __post_init__(self):
        if self.num_processors < 1 or self.wave_width < 1:
            raise ValueError("num_processors and wave_width must be >= 1")
        if self.capacity < 1:
            raise ValueError("cache must hold at least one entry")

    @property
    def capacity(self) -> int:
        if self.entries is not None:
            return self.entries
        return self.cache_bytes // self.entry_bytes


@dataclass(frozen=True)
class CacheReport:
    hits: int
    misses: int
    hit_rate: float

    @property
    def total(self) -> int:
        return self.hits + self.misses


def ideal_reuse(indices) -> float:
    """1 - unique/total: the reuse ceiling any mechanism can attain (cache.py:61-66), counted on the device."""
    from . import engine
    import torch

    n = int(indices.numel()) if isinstance(indices, torch.Tensor) else len(indices)
    if n == 0:
        raise ValueError("empty index buffer")
    d_idx = engine.to_device_indices(indices)
    referenced, _ = engine.ideal_counts(d_idx, int(d_idx.max().item()) + 1)
    return 1.0 - referenced / n


def simulate_parallel_cache(indices, cfg: CacheConfig, primitive_size: int = 3,
                            miss_counts: np.ndarray | None = None) -> CacheReport:
    """LRU simulation across num_processors independent caches (cache.py:69-100).  `miss_counts`, when given,
    accumulates one shader invocation per miss per vertex id."""
    from . import engine
    import torch

    lib = N.require_cuda()
    n = int(indices.numel()) if isinstance(indices, torch.Tensor) else len(indices)
    if n % primitive_size != 0:
        raise ValueError(f"index count {n} is not primitive-aligned")
    if n == 0:
        return CacheReport(hits=0, misses=0, hit_rate=0.0)
    d_idx = engine.to_device_indices(indices)
    dev = d_idx.device
    c = N.CacheConfigC(cfg.num_processors, cfg.wave_width, cfg.capacity, primitive_size)
    ws = torch.empty(lib.vr_cache_workspace_bytes(n, C.byref(c)) + 256, dtype=torch.uint8, device=dev)
    out = torch.zeros(4, dtype=torch.int64, device=dev)
    d_miss = None
    vcount = 0
    if miss_counts is not None:
        vcount = len(miss_counts)
        d_miss = torch.zeros(vcount, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_simulate_cache(engine._ptr(d_idx), n, C.byref(c), vcount,
                                                  engine._ptr(d_miss) if d_miss is not None else None,
                                                  engine._ptr(out), engine._ptr(ws), ws.numel(), engine._stream_ptr()))
    hits, misses, status, _ = (int(v) for v in out.cpu().numpy())
    if status:
        engine.raise_status(status)
    if miss_counts is not None:
        miss_counts += d_miss.cpu().numpy().astype(miss_counts.dtype)
    total = hits + misses
    return CacheReport(hits=hits, misses=misses, hit_rate=1.0 - misses / total if total else 0.0)
