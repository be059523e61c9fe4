"""CPU restatement of the reference's random-walk client and LRU cache model (TEST INFRASTRUCTURE ONLY).

Plain Python / NumPy, small cases only.  Follows /root/reference/pkg/src/vrlab/walk.py and cache.py (lines cited
per function); pinned against fixtures generated from the unmodified reference (tests/golden/walk.npz,
cache.json, written by tests/golden/make_golden.py) in tests/test_oracle_golden.py.  Nothing in the product
imports this module.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1


# ---- walk.py -------------------------------------------------------------------------------------
def candidate_moves(max_distance: int) -> list:
    """walk.py:85-99: every (dx, dy) within the Euclidean radius, dy outer / dx inner (row-major scan)."""
    d = max_distance
    return [(dx, dy) for dy in range(-d, d + 1) for dx in range(-d, d + 1) if dx * dx + dy * dy <= d * d]


def activity(xs: np.ndarray, ys: np.ndarray, gaussians) -> np.ndarray:
    """walk.py:102-109: 1e-12 + sum of the Gaussians, accumulated in their order; all ones without Gaussians."""
    if not gaussians:
        return np.ones(len(xs))
    acc = np.full(len(xs), 1e-12)
    for (cx, cy, sigma, amp) in gaussians:
        dist2 = (xs - cx) ** 2 + (ys - cy) ** 2
        acc += amp * np.exp(-dist2 / (2.0 * sigma * sigma))
    return acc


def cell_moves(cell: int, grid, max_distance: int, kept: int, gaussians):
    """walk.py:110-137: the `kept` most likely moves of one cell as rows (dx, dy, likelihood); likelihood =
    activity at the destination / sum over the on-grid candidates (numpy's pairwise sum, as the reference);
    descending likelihood, ties in scan order.  None when fewer than `kept` moves stay on the grid (:123-126)."""
    x, y = cell & 0xFFFF, cell >> 16
    w, h = grid
    cand = np.array(candidate_moves(max_distance), dtype=np.int64)
    tx, ty = cand[:, 0] + x, cand[:, 1] + y
    ok = (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h)
    if int(ok.sum()) < kept:
        return None
    on_grid = cand[ok]
    act = activity(tx[ok].astype(np.float64), ty[ok].astype(np.float64), gaussians)
    lik = act / act.sum()
    order = sorted(range(len(lik)), key=lambda k: (-lik[k], k))[:kept]
    return np.array([[on_grid[k, 0], on_grid[k, 1], lik[k]] for k in order], dtype=np.float64)


def mix64(z: int) -> int:
    """walk.py:140-149 splitmix64 finalizer on Python integers."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def uniform(seed: int, step: int, agent: int) -> float:
    """walk.py:152-158: 53 bits of mix64(agent + mix64(seed + golden * (step + 1))) as a double in [0, 1)."""
    base = mix64((seed + 0x9E3779B97F4A7C15 * (step + 1)) & MASK64)
    return float(mix64((agent + base) & MASK64) >> 11) * 2.0 ** -53


def pick_move(moves: np.ndarray, u: float) -> int:
    """walk.py:161-165: first row whose running likelihood sum exceeds u * total (the last row otherwise)."""
    cum = 0.0
    sums = []
    for row in moves:
        cum += row[2]
        sums.append(cum)
    r = u * sums[-1]
    for j, s in enumerate(sums):
        if s > r:
            return j
    return len(sums) - 1


def walk_step(positions: np.ndarray, grid, max_distance, kept, gaussians, seed: int, step: int) -> np.ndarray:
    """walk.py:210-219 (= :202-207: dedup is transparent): every agent moves by its own cell's table."""
    out = np.empty_like(positions)
    tables = {}
    for a, (x, y) in enumerate(positions):
        cell = (int(y) << 16) | int(x)
        if cell not in tables:
            tables[cell] = cell_moves(cell, grid, max_distance, kept, gaussians)
        m = tables[cell]
        j = pick_move(m, uniform(seed, step, a))
        out[a, 0], out[a, 1] = x + int(m[j, 0]), y + int(m[j, 1])
    return out


# ---- cache.py ------------------------------------------------------------------------------------
def lru_chunk(chunk, wave_width: int, capacity: int, miss_counts=None):
    """cache.py:103-130: one processor.  Per wave: hit iff cached before the wave (refreshes recency, in wave
    order); the wave's distinct missed ids enter afterwards in first-miss order, the least recently used entry
    leaving whenever the cache is over capacity."""
    order = {}  # insertion-ordered: oldest first
    hits = misses = 0
    for base in range(0, len(chunk), wave_width):
        new_ids = []
        seen = set()
        for v in chunk[base:base + wave_width]:
            v = int(v)
            if v in order:
                hits += 1
                del order[v]
                order[v] = None
            else:
                misses += 1
                if miss_counts is not None:
                    miss_counts[v] += 1
                if v not in seen:
                    seen.add(v)
                    new_ids.append(v)
        for v in new_ids:
            order[v] = None
            if len(order) > capacity:
                del order[next(iter(order))]
    return hits, misses


def simulate_cache(indices, num_processors: int, wave_width: int, capacity: int, primitive_size: int = 3,
                   miss_counts=None):
    """cache.py:69-100: equal primitive-aligned chunks, one independent cache each; (hits, misses, hit rate)."""
    idx = np.asarray(indices)
    n = len(idx)
    per = math.ceil((n // primitive_size) / num_processors) * primitive_size
    hits = misses = 0
    for s in range(0, n, per):
        h, m = lru_chunk(idx[s:s + per], wave_width, capacity, miss_counts)
        hits += h
        misses += m
    total = hits + misses
    return hits, misses, (1.0 - misses / total if total else 0.0)


def ideal_counts(indices, vertex_count: int):
    """analytics.py:105-119: 1 per referenced vertex."""
    counts = np.zeros(vertex_count, dtype=np.int64)
    counts[np.unique(np.asarray(indices))] = 1
    return int(counts.sum()), counts
