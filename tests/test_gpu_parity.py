"""Parity of the CUDA path (through the C ABI) with the CPU oracle and the golden fixtures.
Integer outputs are compared bit-exactly; FP32 positions within rtol 1e-5 (BASELINE.json)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1805_08893_b200 as P
from helpers import (FLAT_KEYS, MATRIX, assert_flat_equal, load_json, load_npz, next_pow2, oracle_flat,
                     random_batches)
from paper_1805_08893_b200 import _native as N
from paper_1805_08893_b200 import engine
from paper_1805_08893_b200.batching import Batch, BatchConfig, ConfigError
from paper_1805_08893_b200.strategies import HashConfig

pytestmark = pytest.mark.gpu
RTOL = 1e-5  # north_star: shaded positions within 1e-5 relative FP32 tolerance


def device_run(strategy, idx, offs, cfg, hcfg=None, shader=None, counts=False):
    import torch
    d_idx = engine.to_device_indices(idx)
    o = torch.from_numpy(np.asarray(offs, dtype=np.int32)).to(d_idx.device)
    spans = np.diff(offs)
    return engine.run_device(strategy, d_idx, o[:-1], o[1:], len(offs) - 1, int(spans.sum()),
                             int(spans.max()), cfg, hcfg, shader, want_counts=counts)


def oracle_run(strategy, idx, offs, cfg, hcfg=None):
    hc = hcfg or HashConfig(table_size=cfg.block_size)
    return O.run(strategy, idx, offs[:-1], offs[1:], primitive_size=cfg.primitive_size,
                 max_unique=cfg.max_unique, warp_width=cfg.warp_width, table_size=hc.table_size,
                 multiplier=hc.multiplier, max_fast_probes=hc.max_fast_probes)


def check_against_oracle(strategy, idx, offs, cfg, hcfg=None, ctx=""):
    run = device_run(strategy, idx, offs, cfg, hcfg, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY))
    fr = oracle_run(strategy, idx, offs, cfg, hcfg)
    assert_flat_equal(run.flat(), oracle_flat(fr), f"{ctx} {strategy}")
    assert (run.invocations, run.rounds, run.indices) == (fr.invocations, fr.rounds, fr.indices)
    if strategy in ("hash", "phash"):
        assert run.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain), ctx
    return run, fr


# ---- reference KATs straight through the public per-batch API -----------------------------
def test_reference_kats(cuda_lib):
    r = P.warp_vote_batch(np.array([0, 1, 2, 0, 2, 3], dtype=np.uint32), 4)  # test_strategies.py:49-58
    assert r.invocations == 4 and len(r.rounds) == 1
    assert r.rounds[0].unique_ids == (0, 1, 2, 3) and r.rounds[0].assembly_map == (0, 1, 2, 0, 2, 3)
    assert r.rounds[0].primitives_emitted == 2
    r = P.warp_vote_batch(np.array([0, 1, 2, 3, 4, 5], dtype=np.uint32), 4)  # :60-67
    assert r.invocations == 7 and [x.unique_ids for x in r.rounds] == [(0, 1, 2, 3), (3, 4, 5)]
    assert [x.primitives_emitted for x in r.rounds] == [1, 1] and r.indices_consumed == 6
    assert P.warp_vote_batch(np.array([10, 20, 30], dtype=np.uint32), 32).invocations == 3
    assert P.warp_vote_batch(np.array([9] * 6, dtype=np.uint32), 4).invocations == 1
    with pytest.raises(ConfigError):  # :79-81
        P.warp_vote_batch(np.array([0, 1, 2, 3], dtype=np.uint32), 4, primitive_size=5)
    r = P.sort_batch(np.array([5, 5, 7, 3, 7, 3], dtype=np.uint32))  # :92-97
    assert r.rounds[0].unique_ids == (3, 5, 7) and r.rounds[0].assembly_map == (1, 1, 2, 0, 2, 0)
    assert P.sort_batch(np.array([0, 1, 2], dtype=np.uint32)).rounds[0].assembly_map == (0, 1, 2)
    r, st = P.hash_batch(np.array([5, 5, 7, 3, 7, 3], dtype=np.uint32), HashConfig(table_size=8))  # :112-124
    assert r.rounds[0].unique_ids == (5, 7, 3) and r.rounds[0].assembly_map == (0, 0, 1, 2, 1, 2)
    assert (st.fast, st.slow, st.max_chain) == (6, 0, 1) and r.invocations == 3
    r, _ = P.hash_batch(np.array([9, 9, 9], dtype=np.uint32), HashConfig(table_size=8))  # :126-129
    assert r.invocations == 1 and len(set(r.rounds[0].assembly_map)) == 1
    with pytest.raises(RuntimeError):  # :146-149 table full
        P.hash_batch(np.arange(9, dtype=np.uint32).repeat(3)[:27], HashConfig(table_size=8))
    r = P.naive_batch(np.array([0, 1, 2, 0, 2, 3], dtype=np.uint32))  # :27-31
    assert r.invocations == 6 and len(r.rounds) == 2 and r.rounds[1].unique_ids == (0, 2, 3)


def test_phash_engineered_collisions(cuda_lib):
    """Reference tests/test_strategies.py:170-181: ids that all collide in a table of 8 force the
    warp-cooperative slow path; same corner stream as hash_batch, slow probes recorded."""
    ids = np.repeat(np.array([0, 5, 13, 18, 26, 34], dtype=np.uint32), 3)
    hc = HashConfig(table_size=8, max_fast_probes=2)
    rp, sp = P.parallel_hash_batch(ids, hc, 4)
    rh, _ = P.hash_batch(ids, hc)
    want_rounds, inv, _, probes = O.parallel_hash_batch(ids, 4, table_size=8, max_fast_probes=2)
    assert (sp.fast, sp.slow, sp.max_chain) == tuple(probes) and sp.slow > 0 and rp.invocations == inv == 6
    assert [tuple(r.unique_ids) for r in rp.rounds] == [tuple(int(v) for v in r[0]) for r in want_rounds]
    corners = lambda res: [r.unique_ids[s] for r in res.rounds for s in r.assembly_map]
    assert corners(rp) == corners(rh) == ids.tolist()
    with pytest.raises(RuntimeError):  # more unique ids than slots (strategies.py:348-349)
        P.parallel_hash_batch(np.arange(9, dtype=np.uint32).repeat(3)[:27], HashConfig(table_size=8), 4)


def test_kernels_golden(cuda_lib):
    data, meta = load_npz("kernels.npz"), load_json("kernels.json")
    for case in meta:
        k = case["id"]
        ids = data[f"k{k}_ids"]
        n = len(ids)
        cfg = BatchConfig(batch_size=n, max_unique=max(n, 3), max_indices=n, warp_width=case["warp_width"])
        hc = HashConfig(table_size=case["table_size"], max_fast_probes=case["max_fast_probes"])
        for strat in ("naive", "warp", "sort", "hash", "phash"):
            run = engine.run_device(strat, engine.to_device_indices(ids), *_one(ids), 1, n, n, cfg, hc,
                                    engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY), enforce_budget=False)
            want = {name: data[f"k{k}_{strat}_{name}"] for name in FLAT_KEYS}
            assert_flat_equal(run.flat(), want, f"case {k} w={case['warp_width']} {strat}")
            if strat in ("hash", "phash"):
                assert list(run.probes) == case[strat]["probes"], f"case {k} {strat} probes"


def _one(ids):
    import torch
    o = torch.tensor([0, len(ids)], dtype=torch.int32, device="cuda")
    return o[:1], o[1:]


def test_runs_golden(cuda_lib):
    """run_on_indices on the reference's 20-mesh corpus: flat results, stream, tallies, report."""
    data, meta = load_npz("runs.npz"), load_json("runs.json")
    for m in meta["meshes"]:
        i = m["id"]
        cfg = BatchConfig(**m["cfg"])
        hc = HashConfig(**m["hash"])
        mesh = P.IndexedMesh(positions=data[f"m{i}_positions"], indices=data[f"m{i}_indices"])
        stat = P.static_batches(len(mesh.indices), cfg)
        dyn = P.dynamic_batches(mesh.indices, cfg)
        assert np.array_equal(P.batches_to_offsets(dyn), data[f"m{i}_dynamic"]), f"mesh {i} dynamic"
        for strat, batches in (("naive", stat), ("warp", stat), ("sort", dyn), ("hash", dyn), ("phash", dyn)):
            out = P.run_on_indices(strat, mesh.indices, batches, cfg, P.position_shader(mesh, MATRIX), hc,
                                   vertex_count=mesh.vertex_count, scene=f"m{i}")
            stream, rep = out[0], out[1]
            want = {name: data[f"m{i}_{strat}_{name}"] for name in FLAT_KEYS}
            assert_flat_equal(stream.device_run.flat(), want, f"mesh {i} {strat}")
            assert rep.to_dict() == m["runs"][strat], f"mesh {i} {strat} report"
            assert np.array_equal(rep.per_vertex.counts, data[f"m{i}_{strat}_counts"])
            ref_stream = data[f"m{i}_{strat}_stream"]
            np.testing.assert_allclose(stream.as_array(), ref_stream, rtol=RTOL,
                                       atol=RTOL * max(1.0, float(np.abs(ref_stream).max())))
            assert len(stream) == mesh.triangle_count
            ident = P.run_on_indices(strat, mesh.indices, batches, cfg, P.identity_shader(), hc)[0]
            assert np.array_equal(ident.as_array(), mesh.indices), f"mesh {i} {strat} stream != input"


def test_dynamic_golden(cuda_lib):
    data, meta = load_npz("dynamic.npz"), load_json("dynamic.json")
    for case in meta:
        k = case["id"]
        cfg = BatchConfig(max_unique=case["max_unique"], max_indices=case["max_indices"],
                          primitive_size=case.get("primitive_size", 3))
        got = engine.dynamic_offsets_device(data[f"d{k}_ids"], cfg).cpu().numpy()
        assert np.array_equal(got, data[f"d{k}_offsets"]), f"dynamic case {k} {case}"


def test_dynamic_examples(cuda_lib):  # reference tests/test_batching.py:71-97
    d = lambda ids, **k: P.dynamic_batches(np.array(ids, dtype=np.uint32), BatchConfig(**k))
    assert d([0, 1, 2, 0, 2, 3, 4, 5, 6], max_unique=4) == [Batch(0, 6), Batch(6, 9)]
    assert d([0, 1, 2, 3, 4, 5], max_unique=6) == [Batch(0, 6)]
    assert d([0, 1, 2, 1, 2, 3], max_unique=4) == [Batch(0, 6)]
    b = d(list(range(30)), max_unique=256, max_indices=9)
    assert b[0] == Batch(0, 9) and all(x.span <= 9 for x in b)
    assert d([]) == []
    with pytest.raises(ConfigError):
        d([0, 1])


def test_random_batches_vs_oracle(cuda_lib):
    """test_acceptance.py criterion 2 shape: many ragged batches in one launch."""
    for seed, mu, mt in ((2000, 256, 341), (7, 32, 50), (8, 5, 9)):
        ids_list = random_batches(150, seed=seed, max_unique=mu, max_tris=mt)
        idx = np.concatenate(ids_list)
        offs = np.concatenate([[0], np.cumsum([len(x) for x in ids_list])]).astype(np.int64)
        span = int(np.diff(offs).max())
        for strat, w in (("naive", 32), ("warp", 32), ("warp", 4), ("warp", 8), ("warp", 16), ("warp", 64),
                         ("sort", 32), ("hash", 32), ("phash", 32), ("phash", 8)):
            cfg = BatchConfig(batch_size=span, max_unique=mu, max_indices=span, warp_width=w,
                              block_size=next_pow2(mu))
            run, fr = check_against_oracle(strat, idx, offs, cfg, HashConfig(table_size=next_pow2(mu)),
                                           ctx=f"seed {seed} w={w}")
            if strat in ("sort", "hash", "phash"):
                assert fr.invocations == sum(len(set(x.tolist())) for x in ids_list)


def test_grid256_table(cuda_lib):
    """BASELINE.md section 2 (configs 1 and 2): every strategy at batch sizes 32..1024."""
    mesh = P.gen_grid(256, 256)
    idx = mesh.indices
    d_idx = engine.to_device_indices(idx)
    for row in load_json("grid256.json"):
        B = row["B"]
        if row["batching"] == "static":
            cfg = BatchConfig(batch_size=3 * B, max_unique=3 * B, warp_width=32)
            offs = engine.static_offsets_device(len(idx), cfg)
        else:
            cfg = BatchConfig(max_unique=B, max_indices=4 * B - 1, block_size=B)
            offs = engine.dynamic_offsets_device(d_idx, cfg)
        hc = HashConfig(table_size=row["table_size"])
        nb = offs.numel() - 1
        assert nb == row["batches"], row
        run = engine.run_device(row["strategy"], d_idx, offs[:-1], offs[1:], nb, len(idx),
                                max(cfg.batch_size, cfg.max_indices), cfg, hc,
                                engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY)).check()
        assert (run.rounds, run.invocations) == (row["rounds"], row["invocations"]), row
        if row["strategy"] == "hash":
            assert run.probes == (row["probes_fast"], 0, row["probe_max_chain"]), row
        assert np.array_equal(run.expand_stream(False).cpu().numpy().view(np.uint32), idx), row
        # every array of every row against the oracle (all batch sizes, all strategies)
        h_offs = offs.cpu().numpy().astype(np.int64)
        fr = oracle_run(row["strategy"], idx, h_offs, cfg, hc)
        assert_flat_equal(run.flat(), oracle_flat(fr), str(row))
        if row["strategy"] in ("hash", "phash"):
            assert run.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain), row


def test_config1_headline_numbers(cuda_lib):
    """configs[0]: 256x256 grid, static 256-triangle batches, sort dedup."""
    mesh = P.gen_grid(256, 256)
    cfg = BatchConfig(batch_size=768, max_unique=768, block_size=1024)
    stream, rep = P.run_sorting(mesh, P.static_batches(len(mesh.indices), cfg), cfg,
                                P.position_shader(mesh, MATRIX), scene="grid256")
    assert (rep.batches, rep.invocations, rep.indices) == (509, 131574, 390150)
    assert abs(rep.reuse_rate - 0.6628) < 5e-5 and abs(rep.shading_rate - 2.008) < 5e-4
    pos = np.hstack([mesh.positions, np.ones((mesh.vertex_count, 1))]) @ MATRIX.T
    want = (pos[:, :3] / pos[:, 3:4]).astype(np.float32)[mesh.indices]
    np.testing.assert_allclose(stream.as_array(), want, rtol=RTOL, atol=RTOL * 256)
    # with the default max_unique=256 the reference raises ConfigError on this config
    with pytest.raises(ConfigError):
        bad = BatchConfig(batch_size=768)
        P.run_sorting(mesh, P.static_batches(len(mesh.indices), bad), bad, P.identity_shader())


def test_error_semantics(cuda_lib):
    ids = np.array([0, 1, 2, 3, 4, 5], dtype=np.uint32)
    with pytest.raises(ConfigError):  # test_strategies.py:311-316 over budget is a hard error
        P.run_on_indices("sort", ids, [Batch(0, 6)], BatchConfig(max_unique=3, block_size=256), P.identity_shader())
    with pytest.raises(ConfigError):
        P.run_on_indices("hash", ids, [Batch(0, 6)], BatchConfig(max_unique=3, block_size=256), P.identity_shader())
    # static hash with more uniques than slots: RuntimeError from the kernel (strategies.py:283-284)
    many = np.arange(30, dtype=np.uint32)
    with pytest.raises(RuntimeError):
        P.run_on_indices("hash", many, [Batch(0, 30)], BatchConfig(batch_size=30, max_unique=8, block_size=8),
                         P.identity_shader(), HashConfig(table_size=8))
    # arbitrary python shaders have no device form
    with pytest.raises(ConfigError):
        P.run_on_indices("naive", ids, [Batch(0, 6)], BatchConfig(), P.ShaderFn(fn=lambda v: v))
    # first failing batch decides the exception, as in the in-order reference loop
    idx = np.concatenate([np.arange(6), np.arange(30), np.arange(6)]).astype(np.uint32)
    batches = [Batch(0, 6), Batch(6, 36), Batch(36, 42)]
    with pytest.raises(RuntimeError):
        P.run_on_indices("hash", idx, batches, BatchConfig(batch_size=30, max_unique=8, block_size=8),
                         P.identity_shader(), HashConfig(table_size=8))


def test_arbitrary_batch_lists(cuda_lib):
    """Any strategy accepts any list of primitive-aligned ranges: gaps, overlaps, ragged."""
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 60, size=3 * 400).astype(np.uint32)
    begins = (rng.integers(0, 380, size=40) * 3).astype(np.int64)
    ends = np.minimum(begins + 3 * rng.integers(1, 20, size=40), len(idx)).astype(np.int64)
    batches = [Batch(int(b), int(e)) for b, e in zip(begins, ends)]
    cfg = BatchConfig(batch_size=60, max_unique=60, max_indices=60, block_size=64, warp_width=8)
    for strat in ("naive", "warp", "sort", "hash"):
        out = P.run_on_indices(strat, idx, batches, cfg, P.identity_shader(), HashConfig(table_size=64))
        fr = O.run(strat, idx, begins, ends, max_unique=60, warp_width=8, table_size=64)
        assert_flat_equal(out[0].device_run.flat(), oracle_flat(fr), strat)
        want_stream = np.concatenate([idx[b:e] for b, e in zip(begins, ends)])
        assert np.array_equal(out[0].as_array(), want_stream)


def test_primitive_size_one(cuda_lib):
    """batching.py:33-35: the random-walk client feeds single-index primitives."""
    rng = np.random.default_rng(11)
    idx = rng.integers(0, 300, size=5000).astype(np.uint32)
    cfg = BatchConfig(batch_size=96, max_unique=64, max_indices=576, primitive_size=1, block_size=64)
    offs = engine.dynamic_offsets_device(idx, cfg).cpu().numpy().astype(np.int64)
    assert np.array_equal(offs, O.dynamic_batches(idx, primitive_size=1, max_unique=64, max_indices=576))
    for strat in ("sort", "hash"):
        check_against_oracle(strat, idx, offs, cfg, HashConfig(table_size=64), ctx="ps=1")
    soffs = O.static_batches(len(idx), primitive_size=1, batch_size=96)
    for strat in ("naive", "warp"):
        check_against_oracle(strat, idx, soffs, cfg, ctx="ps=1 static")


def test_shader_matches_oracle_and_attributes(cuda_lib):
    import torch
    mesh = P.shuffle_triangles(P.gen_icosphere(3), 17)
    cfg = BatchConfig()
    offs = O.dynamic_batches(mesh.indices)
    attrs = (np.arange(mesh.vertex_count, dtype=np.uint32)[:, None] * np.array([3, 5, 7], dtype=np.uint32)
             + np.array([1, 2, 3], dtype=np.uint32)).astype(np.uint32)
    for matrix in (None, MATRIX):
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                 matrix=matrix, vertex_count=mesh.vertex_count,
                                 attributes=torch.from_numpy(attrs.view(np.int32)).cuda())
        run = device_run("sort", mesh.indices, offs, cfg, None, spec, counts=True)
        flat = run.flat()
        fr = oracle_run("sort", mesh.indices, offs, cfg)
        want = O.shade_positions(mesh.positions, fr.unique_ids, matrix)
        np.testing.assert_allclose(flat["shaded"][:, :3], want, rtol=RTOL, atol=1e-6)
        assert np.array_equal(flat["shaded_attr"].view(np.uint32), attrs[fr.unique_ids])  # bit-exact pass-through
        assert np.array_equal(flat["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count))
        if matrix is None:
            assert np.array_equal(flat["shaded"][:, :3], want)  # plain cast is exact


def test_determinism_across_launches(cuda_lib):
    """test_strategies.py:268-280: results do not depend on scheduling."""
    mesh = P.shuffle_triangles(P.gen_icosphere(3), 11)
    cfg = BatchConfig()
    offs = O.dynamic_batches(mesh.indices)
    blobs = []
    for _ in range(3):
        run = device_run("hash", mesh.indices, offs, cfg, HashConfig(), engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY))
        f = run.flat()
        blobs.append(b"".join(np.ascontiguousarray(f[k]).tobytes() for k in FLAT_KEYS) + bytes(str(run.probes), "ascii"))
    assert blobs[0] == blobs[1] == blobs[2]


def test_dynamic_adversarial_streams(cuda_lib):
    """Batch formation against the oracle on streams that stress the occurrence links: one id, a
    handful of ids (buckets far beyond the in-bucket scan limit), long runs, a pool around the
    budget, long windows (both link kernels), primitive size 1."""
    rng = np.random.default_rng(99)
    n = 3 * 40_000
    runs = np.repeat(rng.integers(0, 1 << 20, size=n // 50 + 1), 50)[:n]
    streams = {
        "one-id": np.full(n, 5, dtype=np.uint32),
        "two-ids": (np.arange(n) % 2).astype(np.uint32),
        "five-ids": rng.integers(0, 5, size=n).astype(np.uint32),
        "pool-300": rng.integers(0, 300, size=n).astype(np.uint32),
        "pool-60": rng.integers(0, 60, size=n).astype(np.uint32),
        "runs": runs.astype(np.uint32),
        "all-new": np.arange(n, dtype=np.uint32),
        "far-repeat": np.concatenate([np.arange(2000), np.arange(2000)] * 30).astype(np.uint32)[:n],
    }
    cfgs = [dict(), dict(max_unique=8), dict(max_unique=3, max_indices=30), dict(max_unique=256, max_indices=4095),
            dict(max_unique=1000, max_indices=8191), dict(max_unique=16, max_indices=64, primitive_size=1),
            dict(max_unique=50, max_indices=1023)]
    for name, ids in streams.items():
        for kw in cfgs:
            ps = kw.get("primitive_size", 3)
            cfg = BatchConfig(batch_size=96 if ps == 3 else 32, **kw)
            want = O.dynamic_batches(ids, primitive_size=ps, max_unique=cfg.max_unique, max_indices=cfg.max_indices)
            got = engine.dynamic_offsets_device(ids, cfg).cpu().numpy().astype(np.int64)
            assert np.array_equal(got, want), f"{name} {kw}: first difference at batch {int(np.argmax(got[:len(want)] != want[:len(got)]))}"


def test_fallback_kernels_agree(cuda_lib, monkeypatch):
    """The kernels kept for long batch windows / few long batches (warp-synchronous links, global-memory
    walks, CTA sort) are forced through their ablation knobs and must give the same bytes."""
    mesh = P.shuffle_triangles(P.gen_grid(150, 130), 4)
    cfg = BatchConfig()

    def once():
        offs = engine.dynamic_offsets_device(mesh.indices, cfg)
        run = engine.run_device("sort", engine.to_device_indices(mesh.indices), offs[:-1], offs[1:], offs.numel() - 1,
                                len(mesh.indices), 1023, cfg, None, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY))
        return offs.cpu().numpy(), run.flat()

    def once_general():  # VR_SORT_CTA acts on the general sort path (the three-kernel path does not take it)
        offs = engine.dynamic_offsets_device(mesh.indices, cfg)
        run = engine.run_device("sort", engine.to_device_indices(mesh.indices), offs[:-1], offs[1:], offs.numel() - 1,
                                len(mesh.indices), 1023, cfg, None, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY), fuse=False)
        assert run.kernel_path == 0
        return run.flat()

    offs_a, flat_a = once()
    gen_a = once_general()
    for k in ("VR_LINKS_WARP", "VR_GREEDY_GLOBAL", "VR_WALK_GLOBAL", "VR_SORT_CTA"):
        monkeypatch.setenv(k, "1")
    N.lib().vr_debug_reload_knobs()  # the knobs are read once per process
    try:
        offs_b, flat_b = once()
        gen_b = once_general()
    finally:
        for k in ("VR_LINKS_WARP", "VR_GREEDY_GLOBAL", "VR_WALK_GLOBAL", "VR_SORT_CTA"):
            monkeypatch.delenv(k)
        N.lib().vr_debug_reload_knobs()
    assert np.array_equal(offs_a, offs_b) and np.array_equal(offs_a.astype(np.int64), O.dynamic_batches(mesh.indices))
    assert_flat_equal(flat_a, flat_b, "fallback kernels")
    assert_flat_equal(gen_a, gen_b, "CTA sort")
    assert_flat_equal(gen_a, flat_a, "general vs three-kernel sort")
