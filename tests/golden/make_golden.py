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
    make_kernels()
    make_dynamic()
    make_runs()
    make_grid256()
