#!/usr/bin/env python
"""Randomised stress of the three-kernel sort / hash / phash path, the LRU cache model and the walk client against the
oracle (run on the GPU box):  python scripts/stress_dyn3.py [cases] [seed]
Random budgets, table sizes, group widths, fast-probe counts; id streams from meshes, uniform ids, few hot ids,
long runs of one id; batch lists from the greedy splitter and hand-cut short batches."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import oracle as O
from oracle import clients as OC
import paper_1805_08893_b200 as P
from helpers import assert_flat_equal, oracle_flat
from paper_1805_08893_b200 import _native as N, engine
from paper_1805_08893_b200.batching import BatchConfig
from paper_1805_08893_b200.strategies import HashConfig

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)


def stream(kind, n_tris):
    if kind == 0:
        m = P.gen_grid(int(rng.integers(5, 90)), int(rng.integers(5, 90)))
        return m.indices if rng.random() < 0.5 else P.shuffle_triangles(m, int(rng.integers(1 << 30))).indices
    if kind == 1:  # uniform ids over a small / large range
        return rng.integers(0, int(rng.choice([7, 300, 70000, 1 << 24])), size=3 * n_tris).astype(np.uint32)
    if kind == 2:  # a few hot ids among cold ones
        hot = rng.integers(0, 1 << 20, size=5)
        ids = rng.integers(0, 1 << 20, size=3 * n_tris)
        mask = rng.random(3 * n_tris) < 0.6
        ids[mask] = hot[rng.integers(0, 5, size=int(mask.sum()))]
        return ids.astype(np.uint32)
    ids = np.repeat(rng.integers(0, 1 << 22, size=n_tris // 4 + 1), 12)[:3 * n_tris]  # long runs of one id
    return ids.astype(np.uint32)


for k in range(cases):
    mu = int(rng.choice([3, 4, 9, 16, 33, 64, 100, 255, 256]))
    mi = int(rng.integers(mu, 4 * mu + 2)) // 3 * 3
    mi = max(mi, 3)
    ts = 1 << int(np.ceil(np.log2(mu)))
    if rng.random() < 0.3 and ts < 256:
        ts *= 2
    w = int(rng.choice([4, 8, 16, 32, 64]))
    mfp = int(rng.choice([1, 2, 3, 8, 17, 300]))
    idx = stream(int(rng.integers(4)), int(rng.integers(1, 4000)))
    cfg = BatchConfig(max_unique=mu, max_indices=mi, warp_width=w)
    hc = HashConfig(table_size=ts, max_fast_probes=mfp)
    offs = O.dynamic_batches(idx, max_unique=mu, max_indices=mi)
    if rng.random() < 0.3 and len(offs) > 3:  # cut some batches short (still within the budget)
        cuts = sorted(set(offs.tolist()) | set((rng.integers(0, len(idx) // 3, size=5) * 3).tolist()))
        offs = np.array([c for c in cuts if c <= len(idx)], dtype=np.int64)
    d_idx = engine.to_device_indices(idx)
    o = torch.from_numpy(offs.astype(np.int32)).cuda()
    vcount = int(idx.max()) + 1
    for strat in ("sort", "hash", "phash"):
        fr = O.run(strat, idx, offs[:-1], offs[1:], max_unique=mu, warp_width=w, table_size=ts, max_fast_probes=mfp)
        run = engine.run_device(strat, d_idx, o[:-1], o[1:], len(offs) - 1, len(idx), int(np.diff(offs).max()), cfg, hc,
                                engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=min(vcount, 1 << 24) if vcount <= (1 << 24) else 0))
        ctx = f"case {k} {strat} mu={mu} mi={mi} ts={ts} w={w} mfp={mfp} n={len(idx)}"
        assert_flat_equal(run.flat(), oracle_flat(fr), ctx)
        assert run.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain), ctx
        if vcount <= (1 << 24):
            assert run.kernel_path == 4, ctx
    # LRU cache model
    procs, wave, cap = int(rng.integers(1, 9)), int(rng.choice([1, 3, 32, 100, 1024])), int(rng.choice([1, 2, 16, 64, 300]))
    got = P.simulate_parallel_cache(idx, P.CacheConfig(num_processors=procs, wave_width=wave, entries=cap))
    want = OC.simulate_cache(idx, procs, wave, cap)
    assert (got.hits, got.misses, got.hit_rate) == want, f"case {k} cache {procs} {wave} {cap}"
    if k % 10 == 0:
        print(f"{k} cases ok", flush=True)

# walk client: random small configurations, every strategy, against the oracle's per-agent step
for k in range(max(cases // 10, 3)):
    gw, gh = int(rng.integers(8, 50)), int(rng.integers(8, 50))
    dist = int(rng.integers(1, 7))
    ncand = sum(1 for dy in range(-dist, dist + 1) for dx in range(-dist, dist + 1) if dx * dx + dy * dy <= dist * dist)
    kept = int(rng.integers(1, min(8, ncand // 3) + 1))
    gs = tuple(P.Gaussian(center=(float(rng.uniform(0, gw)), float(rng.uniform(0, gh))), sigma=float(rng.uniform(1, 10)),
                          amplitude=float(rng.uniform(0.2, 2))) for _ in range(int(rng.integers(0, 4))))
    cfg = P.WalkConfig(grid=(gw, gh), agents=int(rng.integers(1, 900)), max_move_distance=dist, kept_moves=kept, gaussians=gs,
                       steps=2, rng_seed=int(rng.integers(1 << 30)))
    pos = P.initial_positions(cfg)
    g = [(x.center[0], x.center[1], x.sigma, x.amplitude) for x in gs]
    try:
        want = pos
        for t in range(cfg.steps):
            want = OC.walk_step(want, cfg.grid, dist, kept, g, cfg.rng_seed, t)
    except TypeError:  # a corner cell with fewer legal moves than kept_moves: the reference raises ConfigError
        continue
    for strat in ("sort", "hash", "phash", "warp", "naive"):
        run = P.run_walk(cfg, strat, BatchConfig(primitive_size=1, batch_size=96 if strat in ("warp", "naive") else 576))
        assert np.array_equal(run.trajectory[-1], want), f"walk case {k} {strat}"
print(f"{cases} random cases bit-exact (sort / hash / phash, cache model), walk cases ok")
