"""Multi-draw scenes (BASELINE.json configs[4]): many meshes, each with
its own vertex buffer and its own greedy scan, packed into one stream and processed by one
sequence of kernels (paper_1805_08893_b200/draws.py).  The oracle goes the reference's way:
dynamic_batches + run_on_indices once per mesh; the device results must be the concatenation."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1805_08893_b200 as P
from helpers import MATRIX, assert_flat_equal, oracle_draws
from paper_1805_08893_b200 import draws as D
from paper_1805_08893_b200.batching import BatchConfig, ConfigError
from paper_1805_08893_b200.strategies import HashConfig

pytestmark = pytest.mark.gpu


def small_scene():
    """A corpus in the reference's test style plus the awkward draws: one triangle, smaller than
    a batch, empty, a draw whose ids collide numerically with its neighbours'."""
    ms = D.scene_corpus(22, seed=7, lo=6, hi=40, ico=(1, 4))
    one = P.IndexedMesh(positions=np.eye(3), indices=np.array([0, 1, 2], dtype=np.uint32))
    empty = P.IndexedMesh(positions=np.zeros((1, 3)), indices=np.zeros(0, dtype=np.uint32))
    tiny = P.gen_grid(2, 2)
    return ms[:5] + [one, empty, tiny] + ms[5:11] + [empty, empty, one] + ms[11:] + [tiny]


def check(strategy, meshes, cfg, hcfg=None, dynamic=True, counts=True):
    ds = D.pack_draws(meshes)
    offsets = D.dynamic_offsets_draws(ds, cfg) if dynamic else D.static_offsets_draws(ds, cfg)
    want = oracle_draws(O, strategy, meshes, dynamic=dynamic, batch_size=cfg.batch_size, max_unique=cfg.max_unique,
                        max_indices=cfg.max_indices, warp_width=cfg.warp_width,
                        table_size=hcfg.table_size if hcfg else 256,
                        max_fast_probes=hcfg.max_fast_probes if hcfg else 8, matrix=MATRIX)
    assert np.array_equal(offsets.cpu().numpy().astype(np.int64), want["offsets"]), "batch boundaries"
    run = D.run_draws(strategy, ds, offsets, cfg, hcfg, matrix=MATRIX, want_counts=counts)
    flat = run.flat()
    assert_flat_equal(flat, want["flat"], f"{strategy} dynamic={dynamic}")
    t = want["totals"]
    assert (run.invocations, run.rounds, run.indices) == (t["invocations"], t["rounds"], t["indices"])
    if strategy in ("hash", "phash"):
        assert run.probes == (t["probes_fast"], t["probes_slow"], t["probe_max_chain"])
    np.testing.assert_allclose(flat["shaded"][:, :3], want["shaded"], rtol=1e-5, atol=1e-5)
    if counts:
        assert np.array_equal(flat["shade_counts"], want["counts"])
    reports = D.per_draw_reports(run, ds, offsets, strategy)
    assert [(r.batches, r.invocations) for r in reports] == want["per_draw"]
    return run


@pytest.mark.parametrize("strategy", ["sort", "hash", "phash", "naive", "warp"])
def test_dynamic_batches_per_draw(cuda_lib, strategy):
    meshes = small_scene()
    hcfg = HashConfig() if strategy in ("hash", "phash") else None
    check(strategy, meshes, BatchConfig(), hcfg)
    # a tight budget: many batches per draw, boundaries everywhere
    small = BatchConfig(max_unique=24, max_indices=95)
    check(strategy, meshes, small, HashConfig(table_size=32) if hcfg else None)


@pytest.mark.parametrize("strategy", ["warp", "sort"])
def test_static_batches_per_draw(cuda_lib, strategy):
    """static_batches per mesh: the last batch of every draw is short; a batch never spans two draws."""
    cfg = BatchConfig(batch_size=96, max_unique=96)
    check(strategy, small_scene(), cfg, dynamic=False)


def test_one_draw_equals_the_single_mesh_path(cuda_lib):
    mesh = P.shuffle_triangles(P.gen_grid(90, 70), 3)
    cfg = BatchConfig()
    ds = D.pack_draws([mesh])
    a = D.dynamic_offsets_draws(ds, cfg).cpu().numpy()
    from paper_1805_08893_b200 import engine
    b = engine.dynamic_offsets_device(mesh.indices, cfg).cpu().numpy()
    assert np.array_equal(a, b)


def test_bad_draw_table(cuda_lib):
    import torch
    ds = D.pack_draws([P.gen_grid(8, 8), P.gen_grid(9, 9)])
    bad = ds.d_index_start.clone()
    bad[1] += 1  # not primitive-aligned
    ds.d_index_start = bad
    with pytest.raises(ConfigError):
        D.dynamic_offsets_draws(ds, BatchConfig())
    with pytest.raises(ConfigError):
        D.pack_draws([(np.array([0, 1, 5], dtype=np.uint32), np.zeros((3, 3)))])  # index outside its own buffer
