"""CPU-only checks of the host mirror of the reference API and of the C-ABI boundary
(no compute calls: there is no GPU in the build container)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1805_08893_b200 as P
from paper_1805_08893_b200 import _native, build
from paper_1805_08893_b200.batching import Batch, BatchConfig, ConfigError
from paper_1805_08893_b200.strategies import HashConfig, ProbeStats, effective_workers

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestBatchConfig:  # reference tests/test_batching.py:17-42
    def test_defaults(self):
        cfg = BatchConfig()
        assert (cfg.batch_size, cfg.max_unique, cfg.max_indices, cfg.max_primitives) == (96, 256, 1023, 341)
        assert (cfg.warp_width, cfg.block_size, cfg.primitive_size) == (32, 256, 3)

    def test_validation(self):
        for bad in (dict(batch_size=97), dict(batch_size=0), dict(max_unique=2), dict(max_indices=2),
                    dict(block_size=0), dict(primitive_size=0)):
            with pytest.raises(ConfigError):
                BatchConfig(**bad)
        BatchConfig(max_unique=3)
        assert BatchConfig(primitive_size=1, max_unique=1).max_primitives == 1023
        with pytest.raises(ValueError):
            BatchConfig(warp_width=12)


class TestStaticBatches:  # reference tests/test_batching.py:44-68
    def test_cases(self):
        cfg = BatchConfig()
        assert P.static_batches(192, cfg) == [Batch(0, 96), Batch(96, 192)]
        assert P.static_batches(99, cfg) == [Batch(0, 96), Batch(96, 99)]
        assert P.static_batches(0, cfg) == []
        with pytest.raises(ConfigError):
            P.static_batches(100, cfg)
        batches = P.static_batches(606, BatchConfig(batch_size=12))
        assert batches[0].begin == 0 and batches[-1].end == 606
        assert all(a.end == b.begin for a, b in zip(batches, batches[1:]))


def test_offsets_roundtrip():  # reference tests/test_batching.py:123-131
    batches = [Batch(0, 96), Batch(96, 120), Batch(120, 300)]
    offs = P.batches_to_offsets(batches)
    assert list(offs) == [0, 96, 120, 300] and P.offsets_to_batches(offs) == batches
    assert len(P.batches_to_offsets([])) == 0 and P.offsets_to_batches(np.array([], dtype=np.int64)) == []


def test_hash_config():  # reference tests/test_strategies.py:151-157, :112-124
    for bad in (dict(table_size=12), dict(multiplier=2), dict(max_fast_probes=0), dict(multiplier=2**32 + 1)):
        with pytest.raises(ConfigError):
            HashConfig(**bad)
    h = HashConfig(table_size=8)
    assert (h.slot(5), h.slot(7), h.slot(3)) == (0, 2, 6)
    assert HashConfig(table_size=1).slot(12345) == 0


def test_probe_stats_merge():
    assert ProbeStats(1, 2, 3).merge(ProbeStats(4, 5, 2)) == ProbeStats(5, 7, 3)
    assert ProbeStats(1, 2, 3).total == 3


def test_worker_env_cap(monkeypatch):  # reference tests/test_strategies.py:282-289
    monkeypatch.setenv("VRLAB_THREADS", "2")
    assert effective_workers(8) == 2
    monkeypatch.setenv("VRLAB_THREADS", "junk")
    with pytest.raises(ConfigError):
        effective_workers(8)
    monkeypatch.delenv("VRLAB_THREADS")
    assert effective_workers(8) == 8


def test_warp_primitives():  # reference tests/test_warp.py
    from paper_1805_08893_b200.warp import WarpState, ballot, ffs, lane_bit, shfl
    assert shfl(WarpState((1, 2, 3, 4)), 2).lanes == (3, 3, 3, 3)
    assert ballot([True, False, True]) == 0b101 and ffs(0) == 0 and ffs(0b1000) == 4
    assert lane_bit(3, 4) == 8 and lane_bit(4, 4) == 0
    with pytest.raises(ValueError):
        WarpState((1, 2, 3))


def test_mesh_generators_match_oracle_restatement():
    import oracle as O
    m = P.gen_grid(9, 13)
    p, i = O.gen_grid(9, 13)
    assert np.array_equal(m.positions, p) and np.array_equal(m.indices, i)
    assert np.array_equal(P.shuffle_triangles(m, 4).indices, O.shuffle_triangles(i, 4))
    s = P.gen_icosphere(2)
    assert s.vertex_count == 10 * 16 + 2 and s.triangle_count == 20 * 16
    np.testing.assert_allclose(np.linalg.norm(s.positions, axis=1), 1.0, atol=1e-12)
    with pytest.raises(P.MeshError):
        P.IndexedMesh(positions=np.zeros((2, 3)), indices=np.array([0, 1, 5], dtype=np.uint32))


def test_golden_meshes_match_generators(golden_dir):
    """The corpus of tests/helpers.py:20-40 rebuilt with our generators equals the reference's."""
    data = np.load(os.path.join(golden_dir, "runs.npz"))
    rng = np.random.default_rng(100)
    for i in range(20):
        kind = i % 4
        if kind == 0:
            m = P.gen_grid(int(rng.integers(2, 11)), int(rng.integers(2, 11)))
        elif kind == 1:
            m = P.gen_icosphere(int(rng.integers(0, 3)))
        elif kind == 2:
            g = P.gen_grid(int(rng.integers(3, 11)), int(rng.integers(3, 11)))
            m = P.shuffle_triangles(g, int(rng.integers(0, 2**31)))
        else:
            s = P.gen_icosphere(int(rng.integers(1, 3)))
            m = P.shuffle_triangles(s, int(rng.integers(0, 2**31)))
        assert np.array_equal(m.indices, data[f"m{i}_indices"])
        assert np.array_equal(m.positions, data[f"m{i}_positions"])


def test_build_report_contract():  # reference tests/test_analytics.py:53-60
    with pytest.raises(AssertionError):
        P.build_report(scene="s", strategy="naive", indices=6, invocations=6, batches=1,
                       shade_counts=np.array([1, 1]))
    rep = P.build_report(scene="s", strategy="sort", indices=9, invocations=3, batches=1)
    assert rep.reuse_rate == 1 - 3 / 9
    assert set(rep.to_dict()) == {"scene", "strategy", "indices", "invocations", "reuse_rate", "batches"}
    assert P.build_report(scene="", strategy="x", indices=0, invocations=0, batches=0).reuse_rate == 0.0


# ---- boundary -----------------------------------------------------------------------------
def test_library_builds_and_exports_every_declared_symbol():
    build.build()
    header = open(os.path.join(ROOT, "include", "vrgeom.h")).read()
    declared = set(re.findall(r"\b(vr_[a-z_]+)\s*\(", header))
    assert declared, "no entry points parsed from include/vrgeom.h"
    assert declared == set(_native.exported_symbols())
    handle = ctypes.CDLL(build.LIB)
    for name in declared:
        assert hasattr(handle, name), f"{name} not exported"
    assert _native.lib().vr_abi_version() == _native.ABI_VERSION == 4
    assert _native.status_string(5).startswith("hash table full")


def test_sass_is_sm100():
    out = subprocess.run(["cuobjdump", "-lelf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_checks_through_abi():
    lib = _native.lib()
    ok = _native.BatchConfigC(96, 256, 1023, 32, 256, 3)
    assert lib.vr_check_batch_config(ctypes.byref(ok)) == 0
    for bad in ((97, 256, 1023, 32, 256, 3), (96, 2, 1023, 32, 256, 3), (96, 256, 1023, 12, 256, 3)):
        assert lib.vr_check_batch_config(ctypes.byref(_native.BatchConfigC(*bad))) == _native.VR_ERR_BAD_CONFIG
    assert lib.vr_check_hash_config(ctypes.byref(_native.HashConfigC(12, 3, 8))) == _native.VR_ERR_BAD_CONFIG
    assert lib.vr_static_batch_count(99, ctypes.byref(ok)) == 2


def test_no_cpu_fallback_without_device():
    """On a box without a GPU every compute entry point refuses loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeLibraryError):
        P.dynamic_batches(np.array([0, 1, 2], dtype=np.uint32), BatchConfig())
    with pytest.raises(_native.NativeLibraryError):
        P.sort_batch(np.array([0, 1, 2], dtype=np.uint32))
    m = P.gen_grid(3, 3)
    with pytest.raises(_native.NativeLibraryError):
        P.run_sorting(m, P.static_batches(len(m.indices), BatchConfig()), BatchConfig(), P.identity_shader())


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1805_08893_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "vr_oracle" not in text, f


def test_runner_validation_is_host_side():
    """Errors the reference raises before touching data need no GPU either."""
    ids = np.array([0, 1, 2], dtype=np.uint32)
    with pytest.raises(ConfigError):  # test_strategies.py:293-296
        P.run_on_indices("magic", ids, [Batch(0, 3)], BatchConfig(), P.identity_shader())
    with pytest.raises(ConfigError):  # test_strategies.py:298-301
        P.run_on_indices("naive", ids, [Batch(0, 6)], BatchConfig(), P.identity_shader())
    with pytest.raises(ConfigError):  # test_strategies.py:303-309
        P.run_on_indices("hash", ids, [Batch(0, 3)], BatchConfig(max_unique=256), P.identity_shader(),
                         HashConfig(table_size=128))
    # empty batch list is legal and needs no device (test_strategies.py:40-45, :183-190)
    stream, rep = P.run_on_indices("naive", np.array([], dtype=np.uint32), [], BatchConfig(), P.identity_shader())
    assert rep.invocations == 0 and len(stream) == 0
    stream, rep, stats = P.run_on_indices("hash", np.array([], dtype=np.uint32), [], BatchConfig(),
                                          P.identity_shader(), HashConfig())
    assert len(stream) == 0 and rep.invocations == 0 and stats.total == 0


def test_scene_corpus_is_the_config5_recipe():
    """rng = default_rng(2018), kind = k % 4 (grid, icosphere, shuffled grid, shuffled
    icosphere), sizes drawn before the shuffle seed.  Pinned on the first 40 draws; the 1000-draw totals
    (20 397 942 triangles, 10 319 577 vertices) are asserted by the GPU scale test."""
    from paper_1805_08893_b200.draws import scene_corpus
    ms = scene_corpus(40)
    assert sum(m.triangle_count for m in ms) == 799_986 and sum(m.vertex_count for m in ms) == 404_742
    assert [m.triangle_count for m in ms[:8]] == [22698, 5120, 12118, 5120, 12480, 20480, 16102, 5120]
    assert list(ms[2].indices[:6]) == [2815, 2889, 2816, 916, 989, 990]    # shuffled grid
    assert list(ms[3].indices[:6]) == [346, 1353, 1352, 274, 1062, 1067]  # shuffled icosphere
    again = scene_corpus(40)
    assert all(np.array_equal(a.indices, b.indices) for a, b in zip(ms, again))


def test_oracle_draws_helper_concatenates_per_mesh_runs():
    """The multi-draw parity tests compare against per-mesh oracle runs glued together; check the glue on
    two tiny meshes against a hand-built expectation."""
    import oracle as O
    from helpers import oracle_draws
    import paper_1805_08893_b200 as P
    a, b = P.gen_grid(3, 3), P.gen_grid(2, 4)
    got = oracle_draws(O, "sort", [a, b], shade=False)
    fa = O.run("sort", a.indices, [0], [len(a.indices)])
    fb = O.run("sort", b.indices, [0], [len(b.indices)])
    assert list(got["offsets"]) == [0, len(a.indices), len(a.indices) + len(b.indices)]
    assert np.array_equal(got["flat"]["unique_ids"], np.concatenate([fa.unique_ids, fb.unique_ids]))
    assert list(got["flat"]["round_uid_off"]) == [0, fa.invocations, fa.invocations + fb.invocations]
    assert got["per_draw"] == [(1, fa.invocations), (1, fb.invocations)]
    assert got["totals"]["invocations"] == fa.invocations + fb.invocations


def test_round2_entry_points_validate_without_a_device():
    """Host-side checks of the round-2 entry points (no compute: every one of them refuses or answers before it would
    touch a GPU)."""
    lib = _native.lib()
    cfg = _native.BatchConfigC(96, 256, 1023, 32, 256, 3)
    # every batch but the last holds >= min(max_unique - ps + 1, max_primitives * ps) indices (batching.py:106-118)
    assert lib.vr_dynamic_batch_bound(21591654, ctypes.byref(cfg), 0) == 21591654 // 254 + 2
    assert lib.vr_dynamic_batch_bound(21591654, ctypes.byref(cfg), 1000) == 21591654 // 254 + 1001
    one = _native.BatchConfigC(96, 256, 1023, 32, 256, 1)
    assert lib.vr_dynamic_batch_bound(300000, ctypes.byref(one), 0) == 300000 // 256 + 2
    assert lib.vr_dynamic_batch_bound(0, ctypes.byref(cfg), 0) == 0
    # ranges of the stream are whole groups of 64 chunks of max(1024, max_primitives) primitives
    assert lib.vr_dynamic_group_indices(ctypes.byref(cfg)) == 1024 * 64 * 3
    assert lib.vr_dynamic_group_count(21591654, ctypes.byref(cfg)) == -(-(-(-7197218 // 1024)) // 64)
    assert lib.vr_dynamic_table_words(21591654, ctypes.byref(cfg)) == 2 * (1023 // 3)
    # cache model: cache.py:85-86 alignment, cache.py:36-40 validation
    cc = _native.CacheConfigC(28, 1024, 256, 3)
    assert lib.vr_cache_workspace_bytes(9000, ctypes.byref(cc)) > 0
    assert lib.vr_cache_workspace_bytes(9001, ctypes.byref(cc)) == 0
    out = (ctypes.c_int64 * 4)()
    assert lib.vr_simulate_cache(None, 9001, ctypes.byref(cc), 0, None, out, None, 0, None) == _native.VR_ERR_UNALIGNED
    assert lib.vr_simulate_cache(None, 9000, ctypes.byref(_native.CacheConfigC(0, 1024, 256, 3)), 0, None, out, None, 0, None) \
        == _native.VR_ERR_BAD_CONFIG
    # walk client: walk.py:62-70 validation, device limit of 1024 candidate moves
    wc = _native.WalkConfigC()
    wc.grid_w, wc.grid_h, wc.max_move_distance, wc.kept_moves, wc.n_gaussians = 1, 256, 16, 8, 0
    st = (ctypes.c_int64 * 1)()
    assert lib.vr_walk_likelihoods(None, 0, ctypes.byref(wc), None, st, None) == _native.VR_ERR_BAD_CONFIG
    wc.grid_w, wc.max_move_distance = 256, 19
    assert lib.vr_walk_likelihoods(None, 0, ctypes.byref(wc), None, st, None) == _native.VR_ERR_UNSUPPORTED
    wc.max_move_distance, wc.kept_moves = 1, 6  # 5 candidate moves within distance 1
    assert lib.vr_walk_likelihoods(None, 0, ctypes.byref(wc), None, st, None) == _native.VR_ERR_BAD_CONFIG
    assert lib.vr_debug_reload_knobs() == 0
