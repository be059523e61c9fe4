"""Device versions of the stage's clients: random-walk client, LRU cache model, ideal counts, synthetic
shader load -- against the fixtures generated from the unmodified reference and against oracle/clients.py."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1805_08893_b200 as P
from helpers import MATRIX, load_json, load_npz
from oracle import clients as OC
from paper_1805_08893_b200.batching import BatchConfig
from paper_1805_08893_b200.strategies import HashConfig
from test_clients_oracle import WALK_CASES, walk_case

pytestmark = pytest.mark.gpu


def _walk_cfg(c, steps=None):
    return P.WalkConfig(grid=c["grid"], agents=c["agents"], max_move_distance=c["dist"], kept_moves=c["kept"],
                        gaussians=tuple(P.Gaussian(center=(g[0], g[1]), sigma=g[2], amplitude=g[3]) for g in c["gaussians"]),
                        steps=c["steps"] if steps is None else steps, rng_seed=c["seed"])


@pytest.mark.parametrize("name", WALK_CASES)
def test_walk_likelihood_tables(cuda_lib, name):
    """walk.py:110-137 in FP64 on the device: moves exact, likelihoods within 1e-12 relative of the reference's
    (device exp / warp-ordered sum instead of libm / numpy's pairwise sum)."""
    g = load_npz("walk.npz")
    c = walk_case(g, name)
    cfg = _walk_cfg(c)
    for cell, want in zip(g[f"{name}/cells"], g[f"{name}/tables"]):
        got = P.cell_likelihoods(int(cell), cfg)
        assert np.array_equal(got[:, :2], want[:, :2]), (name, int(cell))
        np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=1e-12, atol=0)
    with pytest.raises(P.ConfigError):
        P.cell_likelihoods(0, P.WalkConfig(grid=(2, 2), max_move_distance=1, kept_moves=4))  # tests/test_walk.py:94-98


@pytest.mark.parametrize("name", WALK_CASES)
@pytest.mark.parametrize("strategy", ["sort", "hash", "phash", "warp", "naive"])
def test_walk_trajectories_and_reports(cuda_lib, name, strategy):
    """tests/test_walk.py:150-154: trajectories equal the per-agent path for every strategy; reuse reports equal the
    reference's (invocations = per-batch unique occupied cells)."""
    g = load_npz("walk.npz")
    c = walk_case(g, name)
    cfg = _walk_cfg(c)
    bcfg = BatchConfig(primitive_size=1, batch_size=96 if strategy in ("warp", "naive") else 576)
    run = P.run_walk(cfg, strategy, bcfg)
    assert np.array_equal(run.trajectory, g[f"{name}/trajectory"])
    want = g[f"{name}/{strategy}/reports"]
    for t, r in enumerate(run.reports):
        ps = r.probe_stats
        got = [r.indices, r.invocations, r.batches, ps.fast if ps else -1, ps.slow if ps else -1, ps.max_chain if ps else -1]
        assert got == want[t].tolist(), (name, strategy, t)
        assert r.scene == f"walk/step{t}" and r.strategy == strategy


def test_walk_per_agent_path_and_helpers(cuda_lib):
    g = load_npz("walk.npz")
    c = walk_case(g, "default_small")
    cfg = _walk_cfg(c)
    assert np.array_equal(P.naive_walk(cfg), g["default_small/trajectory"])
    assert np.array_equal(P.initial_positions(cfg), g["default_small/trajectory"][0])
    uni = P.agent_uniforms(cfg.rng_seed, 1, np.arange(cfg.agents))
    assert np.array_equal(uni, g["default_small/uniforms"][1])
    # one step through the public step function, against the oracle's step
    pos = g["default_small/trajectory"][2]
    new, rep = P.step_with_reuse(pos, cfg, 2, "hash", BatchConfig(primitive_size=1, batch_size=576), HashConfig())
    want = OC.walk_step(pos, c["grid"], c["dist"], c["kept"], c["gaussians"], c["seed"], 2)
    assert np.array_equal(new, want) and new.dtype == pos.dtype
    with pytest.raises(P.ConfigError):  # tests/test_walk.py:135-139
        P.step_with_reuse(pos, cfg, 0, "sort", BatchConfig())
    # tests/test_walk.py:122-127: all agents in one cell -> one evaluation per batch
    same = np.tile(np.array([[7, 9]], dtype=np.int64), (500, 1))
    _, rep = P.step_with_reuse(same, cfg, 0, "sort", BatchConfig(primitive_size=1))
    assert rep.invocations == rep.batches


def test_cache_model_and_ideal_counts(cuda_lib):
    meshes = {"grid40x31": P.gen_grid(40, 31), "grid40x31s": P.shuffle_triangles(P.gen_grid(40, 31), 4),
              "sphere3": P.gen_icosphere(3), "grid9x9": P.gen_grid(9, 9)}
    for case in load_json("cache.json"):
        mesh = meshes[case["mesh"]]
        if "ideal_invocations" in case:
            rep = P.ideal_report(mesh, scene="s")
            assert rep.invocations == case["ideal_invocations"] and rep.reuse_rate == case["ideal_rate"]
            assert rep.strategy == "ideal" and rep.batches == 1
            assert np.array_equal(rep.per_vertex.counts, OC.ideal_counts(mesh.indices, mesh.vertex_count)[1])
            assert P.ideal_reuse(mesh.indices) == case["ideal_reuse"]
            continue
        miss = np.zeros(mesh.vertex_count, dtype=np.int64)
        rep = P.simulate_parallel_cache(mesh.indices, P.CacheConfig(num_processors=case["procs"], wave_width=case["wave"],
                                                                    entries=case["entries"]), miss_counts=miss)
        assert (rep.hits, rep.misses, rep.hit_rate) == (case["hits"], case["misses"], case["hit_rate"]), case
        assert int(miss.sum()) == case["miss_counts_sum"]
        assert int((miss * (np.arange(len(miss)) % 9973 + 1)).sum()) == case["miss_counts_crc"]
    # tests/test_cache.py:52-55 serial + unbounded == ideal exactly; :57-64 hand trace; :79-83 alignment
    mesh = P.gen_icosphere(2)
    rep = P.simulate_parallel_cache(mesh.indices, P.CacheConfig(num_processors=1, wave_width=1, entries=10 ** 6))
    assert rep.hit_rate == P.ideal_reuse(mesh.indices)
    rep = P.simulate_parallel_cache(np.array([0, 1, 0, 2, 1]), P.CacheConfig(num_processors=1, wave_width=1, entries=2),
                                    primitive_size=1)
    assert (rep.hits, rep.misses, rep.hit_rate) == (1, 4, 1 - 4 / 5)
    with pytest.raises(ValueError):
        P.simulate_parallel_cache(np.arange(7), P.CacheConfig())
    # a bigger randomised case against the oracle (capacity and wave of the paper's comparison column)
    big = P.shuffle_triangles(P.gen_grid(120, 100), 1)
    for procs, wave, entries in ((28, 1024, 256), (28, 1024, 1024), (8, 256, 100)):
        got = P.simulate_parallel_cache(big.indices, P.CacheConfig(num_processors=procs, wave_width=wave, entries=entries))
        want = OC.simulate_cache(big.indices, procs, wave, entries)
        assert (got.hits, got.misses, got.hit_rate) == want, (procs, wave, entries)


@pytest.mark.parametrize("strategy", ["naive", "warp", "sort", "hash"])
def test_synthetic_shader_load_leaves_results_unchanged(cuda_lib, strategy):
    """ShaderFn.cycles (strategies.py:40-44) as PAPER.md:661's synthetic load: the records must not change."""
    mesh = P.gen_grid(70, 50)
    cfg = BatchConfig()
    batches = P.dynamic_batches(mesh.indices, cfg) if strategy in ("sort", "hash") else P.static_batches(len(mesh.indices), cfg)
    base = P.run_on_indices(strategy, mesh.indices, batches, cfg, P.position_shader(mesh, MATRIX), HashConfig(),
                            vertex_count=mesh.vertex_count)
    loaded = P.run_on_indices(strategy, mesh.indices, batches, cfg, P.position_shader(mesh, MATRIX, cycles=513), HashConfig(),
                              vertex_count=mesh.vertex_count)
    assert np.array_equal(base[0].as_array(), loaded[0].as_array())
    assert base[1].invocations == loaded[1].invocations
    assert np.array_equal(base[0].device_run.flat()["shaded"], loaded[0].device_run.flat()["shaded"])
    cost = P.estimate_cost(loaded[1], P.position_shader(mesh, MATRIX, cycles=513))
    assert cost.total_cycles == 513 * loaded[1].invocations


def test_pack_xyz(cuda_lib):
    """vr_pack_xyz: the stage's float4 records as the reference's float32[3] records (strategies.py:53-67)."""
    mesh = P.gen_grid(37, 29)
    cfg = BatchConfig()
    stream, _ = P.run_warp_voting(mesh, P.static_batches(len(mesh.indices), cfg), cfg, P.position_shader(mesh, MATRIX))
    run = stream.device_run
    for count in (run.invocations, run.invocations - 1, run.invocations - 2, run.invocations - 3, 1):
        xyz = run.shaded_xyz(count).cpu().numpy()
        assert xyz.shape == (count, 3) and np.array_equal(xyz, run.shaded4[:count, :3].cpu().numpy())
    # vr_pack_bytes: the local indices as bytes
    import torch
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for count in (run.indices, run.indices - 5, 17, 1):
        m8 = run.assembly_map_u8(count, flag=flag).cpu().numpy()
        assert np.array_equal(m8.astype(np.int32), run.flat()["assembly_map"][:count])
    assert int(flag.item()) == 0
    big = run.assembly_map.clone()
    big[3] = 300
    run.assembly_map = big
    run.assembly_map_u8(64, flag=flag)
    assert int(flag.item()) == 1
