#!/usr/bin/env python
"""Generate the golden fixtures from the UNMODIFIED reference (`vrlab`).

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Writes, next to this file:
  kernels.npz   per-batch kernel results on random id arrays (all five kernels)
  runs.npz      run_on_indices results on a small mesh corpus (all strategies,
                identity + position shader, per-vertex tallies, streams)
  dynamic.npz   dynamic_batches offsets on meshes / random buffers
  grid256.json  the config-1/2 table of BASELINE.md (gen_grid(256,256))
  walk.npz      random-walk client: likelihood tables, uniforms, trajectories and reports (walk.py)
  cache.json    simulate_parallel_cache / ideal_report results on small meshes (cache.py, analytics.py)
The files are committed; the GPU box never sees /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import vrlab  # noqa: E402
from helpers import mesh_corpus, random_batches  # noqa: E402
from vrlab.batching import (BatchConfig, batches_to_offsets, dynamic_batches,  # noqa: E402
                            static_batches)
from vrlab.strategies import (HashConfig, hash_batch, identity_shader, naive_batch,  # noqa: E402
                              parallel_hash_batch, position_shader, run_on_indices, sort_batch,
                              warp_vote_batch)

HERE = os.path.dirname(os.path.abspath(__file__))
MATRIX = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]], dtype=np.float64)


def flatten(results):
    """list[DedupResult] -> flat arrays (the layout the CUDA path emits)."""
    bro, ruo, rp, uid, amap = [0], [0], [], [], []
    for res in results:
        for rnd in res.rounds:
            uid.extend(rnd.unique_ids)
            amap.extend(rnd.assembly_map)
            rp.append(rnd.primitives_emitted)
            ruo.append(len(uid))
        bro.append(len(rp))
    return dict(batch_round_off=np.array(bro, np.int64), round_uid_off=np.array(ruo, np.int64),
                round_prims=np.array(rp, np.int32), unique_ids=np.array(uid, np.uint32),
                assembly_map=np.array(amap, np.int32))


def kernel_results(strategy, ids_list, cfg, hcfg):
    out, fast, slow, mx = [], 0, 0, 0
    for ids in ids_list:
        if strategy == "naive":
            r = naive_batch(ids, cfg.primitive_size)
        elif strategy == "warp":
            r = warp_vote_batch(ids, cfg.warp_width, cfg.primitive_size)
        elif strategy == "sort":
            r = sort_batch(ids, cfg.primitive_size)
        elif strategy == "hash":
            r, s = hash_batch(ids, hcfg, cfg.primitive_size)
            fast, slow, mx = fast + s.fast, slow + s.slow, max(mx, s.max_chain)
        else:
            r, s = parallel_hash_batch(ids, hcfg, cfg.warp_width, cfg.primitive_size)
            fast, slow, mx = fast + s.fast, slow + s.slow, max(mx, s.max_chain)
        out.append(r)
    return out, (fast, slow, mx)


def make_kernels():
    store = {}
    cases = []
    k = 0
    for seed, max_unique, max_tris, tsize in ((21, 256, 341, 256), (3, 64, 100, 64), (5, 16, 40, 32)):
        for ids in random_batches(8, seed=seed, max_unique=max_unique, max_tris=max_tris):
            for w in (4, 8, 16, 32, 64):
                cfg = BatchConfig(warp_width=w)
                hcfg = HashConfig(table_size=tsize, max_fast_probes=2 + (k % 3))
                case = {"id": k, "warp_width": w, "table_size": tsize,
                        "max_fast_probes": hcfg.max_fast_probes}
                store[f"k{k}_ids"] = ids
                for strat in ("naive", "warp", "sort", "hash", "phash"):
                    res, probes = kernel_results(strat, [ids], cfg, hcfg)
                    for name, arr in flatten(res).items():
                        store[f"k{k}_{strat}_{name}"] = arr
                    case[strat] = {"invocations": res[0].invocations, "probes": list(probes)}
                cases.append(case)
                k += 1
                if w == 32:
                    pass
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **store)
    with open(os.path.join(HERE, "kernels.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    print("kernels:", k, "cases")


def make_runs():
    store = {}
    meta = []
    widths = (4, 8, 16, 32)
    for i, mesh in enumerate(mesh_corpus(20, seed=100)):  # test_strategies.py:214-218 corpus
        w = widths[i % 4]
        cfg = BatchConfig(batch_size=(96, 12, 30, 768)[i % 4], max_unique=(256, 8, 16, 256)[i % 4],
                          max_indices=(1023, 30, 99, 1023)[i % 4], warp_width=w,
                          block_size=(256, 8, 16, 256)[i % 4])
        hcfg = HashConfig(table_size=cfg.block_size, max_fast_probes=(8, 2, 3, 8)[i % 4])
        stat = static_batches(len(mesh.indices), cfg)
        dyn = dynamic_batches(mesh.indices, cfg)
        store[f"m{i}_positions"] = mesh.positions
        store[f"m{i}_indices"] = mesh.indices
        store[f"m{i}_static"] = batches_to_offsets(stat)
        store[f"m{i}_dynamic"] = batches_to_offsets(dyn)
        entry = {"id": i, "cfg": cfg.__dict__, "hash": hcfg.__dict__, "runs": {}}
        for strat, batches in (("naive", stat), ("warp", stat), ("sort", dyn), ("hash", dyn),
                               ("phash", dyn)):
            res, _ = kernel_results(strat, [mesh.indices[b.begin:b.end] for b in batches], cfg, hcfg)
            for name, arr in flatten(res).items():
                store[f"m{i}_{strat}_{name}"] = arr
            out = run_on_indices(strat, mesh.indices, batches, cfg, position_shader(mesh, MATRIX),
                                 hcfg, vertex_count=mesh.vertex_count, scene=f"m{i}")
            stream, rep = out[0], out[1]
            store[f"m{i}_{strat}_stream"] = stream.as_array().astype(np.float32)
            store[f"m{i}_{strat}_counts"] = rep.per_vertex.counts
            out_id = run_on_indices(strat, mesh.indices, batches, cfg, identity_shader(), hcfg)
            assert np.array_equal(out_id[0].as_array().astype(np.uint32), mesh.indices)
            entry["runs"][strat] = rep.to_dict()
        meta.append(entry)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **store)
    with open(os.path.join(HERE, "runs.json"), "w") as fh:
        json.dump({"matrix": MATRIX.tolist(), "meshes": meta}, fh, indent=1)
    print("runs:", len(meta), "meshes")


def make_dynamic():
    store = {}
    meta = []
    k = 0
    rng = np.random.default_rng(1234)  # test_batching.py:100-113
    bufs = [rng.integers(0, 4000, size=3 * 10_000).astype(np.uint32)]
    rng = np.random.default_rng(7)
    bufs.append(rng.integers(0, 500, size=3 * 2000).astype(np.uint32))
    bufs += [vrlab.gen_grid(40, 33).indices, vrlab.shuffle_triangles(vrlab.gen_grid(40, 33), 9).indices,
             vrlab.gen_icosphere(3).indices, vrlab.shuffle_triangles(vrlab.gen_icosphere(3), 2).indices,
             np.array([7, 7, 7] * 50 + [1, 2, 3] * 10, dtype=np.uint32),
             np.arange(30, dtype=np.uint32)]
    for buf in bufs:
        for mu, mi in ((256, 1023), (64, 255), (4, 9), (3, 3), (6, 1023), (256, 9), (32, 127)):
            cfg = BatchConfig(max_unique=mu, max_indices=mi)
            store[f"d{k}_ids"] = buf
            store[f"d{k}_offsets"] = batches_to_offsets(dynamic_batches(buf, cfg))
            meta.append({"id": k, "max_unique": mu, "max_indices": mi})
            k += 1
    # primitive_size = 1 (walk client, batching.py:33-35)
    buf = np.random.default_rng(5).integers(0, 300, size=5000).astype(np.uint32)
    for mu, mi in ((64, 576), (16, 100), (1, 1023)):
        cfg = BatchConfig(batch_size=96, max_unique=mu, max_indices=mi, primitive_size=1)
        store[f"d{k}_ids"] = buf
        store[f"d{k}_offsets"] = batches_to_offsets(dynamic_batches(buf, cfg))
        meta.append({"id": k, "max_unique": mu, "max_indices": mi, "primitive_size": 1})
        k += 1
    np.savez_compressed(os.path.join(HERE, "dynamic.npz"), **store)
    with open(os.path.join(HERE, "dynamic.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("dynamic:", k, "cases")


def make_walk():
    from vrlab import walk as W
    out = {}
    cfgs = {
        "default_small": W.WalkConfig(grid=(48, 40), agents=700, max_move_distance=5, kept_moves=4, steps=4, rng_seed=3),
        "radius16": W.WalkConfig(grid=(64, 64), agents=300, steps=2, rng_seed=11),
        "uniform_field": W.WalkConfig(grid=(30, 30), agents=200, max_move_distance=3, kept_moves=6, gaussians=(), steps=3,
                                      rng_seed=5),
        "one_peak": W.WalkConfig(grid=(40, 56), agents=500, max_move_distance=7, kept_moves=8, steps=3, rng_seed=9,
                                 gaussians=(W.Gaussian(center=(10.5, 30.25), sigma=4.0, amplitude=2.0),)),
    }
    for name, cfg in cfgs.items():
        out[f"{name}/cfg"] = np.array([cfg.grid[0], cfg.grid[1], cfg.agents, cfg.max_move_distance, cfg.kept_moves,
                                       cfg.steps, cfg.rng_seed], dtype=np.int64)
        out[f"{name}/gaussians"] = np.array([[g.center[0], g.center[1], g.sigma, g.amplitude] for g in cfg.gaussians],
                                            dtype=np.float64).reshape(-1, 4)
        rng = np.random.default_rng(1)
        cells = np.array([W.pack_cell(int(rng.integers(0, cfg.grid[0])), int(rng.integers(0, cfg.grid[1])))
                          for _ in range(40)] + [W.pack_cell(0, 0), W.pack_cell(cfg.grid[0] - 1, cfg.grid[1] - 1),
                                                 W.pack_cell(0, cfg.grid[1] - 1)], dtype=np.uint32)
        out[f"{name}/cells"] = cells
        out[f"{name}/tables"] = np.stack([W.cell_likelihoods(int(c), cfg) for c in cells])
        out[f"{name}/uniforms"] = np.stack([W.agent_uniforms(cfg.rng_seed, t, np.arange(cfg.agents)) for t in range(3)])
        traj = W.naive_walk(cfg)
        out[f"{name}/trajectory"] = traj
        for strategy in ("sort", "hash", "warp", "naive", "phash"):
            bcfg = BatchConfig(primitive_size=1, batch_size=96 if strategy in ("warp", "naive") else 576)
            run = W.run_walk(cfg, strategy, bcfg)
            assert np.array_equal(run.trajectory, traj), (name, strategy)
            out[f"{name}/{strategy}/reports"] = np.array(
                [[r.indices, r.invocations, r.batches,
                  r.probe_stats.fast if r.probe_stats else -1, r.probe_stats.slow if r.probe_stats else -1,
                  r.probe_stats.max_chain if r.probe_stats else -1] for r in run.reports], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "walk.npz"), **out)
    print("walk.npz:", len(out), "arrays")


def make_cache():
    from vrlab.analytics import ideal_report
    from vrlab.cache import CacheConfig, ideal_reuse, simulate_parallel_cache
    from vrlab.mesh import gen_grid, gen_icosphere, shuffle_triangles
    meshes = {"grid40x31": gen_grid(40, 31), "grid40x31s": shuffle_triangles(gen_grid(40, 31), 4),
              "sphere3": gen_icosphere(3), "grid9x9": gen_grid(9, 9)}
    cases = []
    for mname, mesh in meshes.items():
        ir = ideal_report(mesh)
        for (procs, wave, entries) in [(28, 1024, 256), (4, 32, 16), (1, 1, 10 ** 6), (3, 96, 64), (7, 8, 5),
                                       (2, 3, 1), (1, 64, 48), (5, 1024, 8)]:
            miss = np.zeros(mesh.vertex_count, dtype=np.int64)
            rep = simulate_parallel_cache(mesh.indices, CacheConfig(num_processors=procs, wave_width=wave, entries=entries),
                                          miss_counts=miss)
            cases.append(dict(mesh=mname, procs=procs, wave=wave, entries=entries, hits=rep.hits, misses=rep.misses,
                              hit_rate=rep.hit_rate, miss_counts_sum=int(miss.sum()),
                              miss_counts_crc=int((miss * (np.arange(len(miss)) % 9973 + 1)).sum())))
        cases.append(dict(mesh=mname, ideal_invocations=ir.invocations, ideal_reuse=ideal_reuse(mesh.indices),
                          ideal_rate=ir.reuse_rate))
    with open(os.path.join(HERE, "cache.json"), "w") as fh:
        json.dump(cases, fh, indent=1)
    print("cache.json:", len(cases), "cases")


def next_pow2(x):
    p = 1
    while p < x:
        p *= 2
    return p


def make_grid256():
    """BASELINE.md section 2 table (SURVEY.md 8d parameter mapping)."""
    mesh = vrlab.gen_grid(256, 256)
    rows = []
    for B in (32, 64, 128, 256, 512, 1024):
        scfg = BatchConfig(batch_size=3 * B, max_unique=3 * B, warp_width=32)
        shc = HashConfig(table_size=next_pow2(3 * B))
        stat = static_batches(len(mesh.indices), scfg)
        dcfg = BatchConfig(max_unique=B, max_indices=4 * B - 1, block_size=B)
        dhc = HashConfig(table_size=B)
        dyn = dynamic_batches(mesh.indices, dcfg)
        for batching, strat, cfg, hc, batches in (
                ("static", "warp", scfg, shc, stat), ("static", "sort", scfg, shc, stat),
                ("static", "hash", scfg, shc, stat), ("dynamic", "sort", dcfg, dhc, dyn),
                ("dynamic", "hash", dcfg, dhc, dyn)):
            res, probes = kernel_results(strat, [mesh.indices[b.begin:b.end] for b in batches], cfg, hc)
            rows.append({"B": B, "batching": batching, "strategy": strat, "batches": len(batches),
                         "rounds": sum(len(r.rounds) for r in res),
                         "invocations": sum(r.invocations for r in res),
                         "probes_fast": probes[0], "probe_max_chain": probes[2],
                         "table_size": hc.table_size})
            print(rows[-1], flush=True)
    with open(os.path.join(HERE, "grid256.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    only = sys.argv[1:]
    for name, fn in (("kernels", make_kernels), ("dynamic", make_dynamic), ("runs", make_runs),
                     ("grid256", make_grid256), ("walk", make_walk), ("cache", make_cache)):
        if not only or name in only:
            fn()
