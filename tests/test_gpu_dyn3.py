"""Three-kernel sort / hash / phash path (csrc/vr_dyn3.cuh) against the oracle and against the general kernels:
every configuration the path accepts, error cases, table sizes below a bitmap word, multi-draw bases."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1805_08893_b200 as P
from helpers import MATRIX, assert_flat_equal, oracle_flat
from paper_1805_08893_b200 import _native as N
from paper_1805_08893_b200 import engine
from paper_1805_08893_b200.batching import BatchConfig
from paper_1805_08893_b200.strategies import HashConfig

pytestmark = pytest.mark.gpu

DYN3_PATH = 4


def _meshes():
    return {
        "strip": P.gen_grid(97, 113),
        "shuffled": P.shuffle_triangles(P.gen_grid(120, 77), 5),
        "sphere": P.gen_icosphere(4),
        "sphere-shuffled": P.shuffle_triangles(P.gen_icosphere(3), 11),
    }


def _run(strategy, mesh, offs, cfg, hc, *, fuse=True, shader="position", want_counts=True):
    import torch
    if shader == "position":
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                 matrix=MATRIX, vertex_count=mesh.vertex_count)
    else:
        spec = engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=mesh.vertex_count)
    o = torch.from_numpy(np.asarray(offs, dtype=np.int32)).cuda()
    return engine.run_device(strategy, engine.to_device_indices(mesh.indices), o[:-1], o[1:], len(offs) - 1,
                             len(mesh.indices), int(np.diff(offs).max()), cfg, hc, spec, want_counts=want_counts,
                             fuse=fuse)


CONFIGS = [
    # max_unique, max_indices, table_size, warp_width, max_fast_probes
    (256, 1023, 256, 32, 8),
    (256, 1023, 256, 4, 1),
    (256, 1023, 256, 64, 3),
    (64, 255, 64, 8, 2),
    (64, 255, 128, 16, 8),
    (16, 63, 16, 4, 2),
    (9, 30, 16, 32, 8),
    (255, 900, 256, 32, 300),
    (3, 3, 4, 4, 1),
]


@pytest.mark.parametrize("strategy", ["sort", "hash", "phash"])
@pytest.mark.parametrize("cfgi", range(len(CONFIGS)))
def test_dyn3_matches_oracle_and_general_kernels(cuda_lib, strategy, cfgi):
    mu, mi, ts, w, mfp = CONFIGS[cfgi]
    cfg = BatchConfig(max_unique=mu, max_indices=mi, warp_width=w)
    hc = HashConfig(table_size=ts, max_fast_probes=mfp)
    for name, mesh in _meshes().items():
        offs = O.dynamic_batches(mesh.indices, max_unique=mu, max_indices=mi)
        fr = O.run(strategy, mesh.indices, offs[:-1], offs[1:], max_unique=mu, warp_width=w, table_size=ts,
                   max_fast_probes=mfp)
        run = _run(strategy, mesh, offs, cfg, hc)
        assert run.kernel_path == DYN3_PATH, "expected the three-kernel path"
        got = run.flat()
        ctx = f"{strategy} {name} cfg{cfgi}"
        assert_flat_equal(got, oracle_flat(fr), ctx)
        assert run.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain), ctx
        assert (run.rounds, run.invocations, run.indices) == (fr.rounds, fr.invocations, fr.indices), ctx
        want = O.shade_positions(mesh.positions, fr.unique_ids, MATRIX)
        np.testing.assert_allclose(got["shaded"][:, :3], want, rtol=1e-5, atol=1e-5)
        assert np.array_equal(got["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count)), ctx
        old = _run(strategy, mesh, offs, cfg, hc, fuse=False)
        assert old.kernel_path == 0
        oldf = old.flat()
        assert_flat_equal(oldf, got, ctx + " vs general kernels")
        assert old.probes == run.probes
        assert np.array_equal(oldf["shaded"], got["shaded"])
        # identity shader: the expanded stream is the index buffer (tests/test_strategies.py:214-218)
        ident = _run(strategy, mesh, offs, cfg, hc, shader="identity", want_counts=False)
        ids = ident.expand_stream(False)
        assert np.array_equal(ids.cpu().numpy().view(np.uint32), mesh.indices), ctx


@pytest.mark.parametrize("strategy", ["sort", "hash", "phash"])
def test_dyn3_random_batches_with_duplicates(cuda_lib, strategy):
    """Arbitrary contiguous batch lists that honour the budget: ids drawn with heavy repetition, batch lengths
    1..341 triangles, so that groups with only duplicates, deferred duplicates and full tables all occur."""
    from helpers import random_batches
    import torch
    for seed, (mu, ts, w, mfp) in enumerate([(256, 256, 32, 8), (40, 64, 8, 2), (256, 256, 4, 1), (100, 128, 64, 4)]):
        parts = random_batches(150, seed, max_unique=mu)
        idx = np.concatenate(parts)
        offs = np.concatenate([[0], np.cumsum([len(p) for p in parts])])
        cfg = BatchConfig(max_unique=mu, max_indices=1023, warp_width=w)
        hc = HashConfig(table_size=ts, max_fast_probes=mfp)
        fr = O.run(strategy, idx, offs[:-1], offs[1:], max_unique=mu, warp_width=w, table_size=ts, max_fast_probes=mfp)
        spec = engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=100_000)
        o = torch.from_numpy(offs.astype(np.int32)).cuda()
        run = engine.run_device(strategy, engine.to_device_indices(idx), o[:-1], o[1:], len(offs) - 1, len(idx),
                                int(np.diff(offs).max()), cfg, hc, spec)
        assert run.kernel_path == DYN3_PATH
        assert_flat_equal(run.flat(), oracle_flat(fr), f"{strategy} seed {seed}")
        assert run.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain)


@pytest.mark.parametrize("strategy", ["sort", "hash", "phash"])
def test_dyn3_errors(cuda_lib, strategy):
    """strategies.py:451-455 (a batch above the unique budget) and :283-284 / :348-349 (table full): the first
    failing batch is reported with the reference's exception type."""
    mesh = P.shuffle_triangles(P.gen_grid(60, 60), 3)
    cfg = BatchConfig(max_unique=64, max_indices=255)
    hc = HashConfig(table_size=64)
    offs = O.dynamic_batches(mesh.indices, max_unique=64, max_indices=255)
    # merge batches 5 and 6: more than 64 distinct ids
    bad = np.delete(offs, 6)
    run = _run(strategy, mesh, bad, cfg, hc, want_counts=False)
    assert run.kernel_path == DYN3_PATH
    with pytest.raises((P.ConfigError, RuntimeError), match="batch 5\\)"):
        run.check()
    general = _run(strategy, mesh, bad, cfg, hc, want_counts=False, fuse=False)
    with pytest.raises((P.ConfigError, RuntimeError), match="batch 5\\)") as e_general:
        general.check()
    with pytest.raises(type(e_general.value)):
        run.check()
    # a batch that is not a primitive-aligned range
    bad2 = offs.copy()
    bad2[9] += 1
    run = _run(strategy, mesh, bad2, cfg, hc, want_counts=False)
    with pytest.raises(P.ConfigError, match="batch 8\\)"):
        run.check()


@pytest.mark.parametrize("strategy", ["naive", "warp", "sort", "hash", "phash"])
def test_output_queue_written_by_the_stage(cuda_lib, strategy):
    """vr_outputs.d_stream_xyz (strategies.py:456-463): the per-corner record queue written inside the stage
    (three-kernel sort/hash path: from the shaded records in shared memory) or by vr_run's closing kernel (other
    paths) equals the post-pass expansion (vr_expand_stream) and the float64 reference records."""
    import torch
    cfg, hc = BatchConfig(), HashConfig()
    for name, mesh in _meshes().items():
        dyn = strategy in ("sort", "hash", "phash")
        offs = O.dynamic_batches(mesh.indices) if dyn else O.static_batches(len(mesh.indices))
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                 matrix=MATRIX, vertex_count=mesh.vertex_count)
        o = torch.from_numpy(np.asarray(offs, dtype=np.int32)).cuda()
        variants = [dict()] if dyn else [dict(), dict(static=True)]
        if dyn:
            variants.append(dict(fuse=False))
        for kw in variants:
            args = (strategy, engine.to_device_indices(mesh.indices), o[:-1], o[1:], len(offs) - 1, len(mesh.indices),
                    int(np.diff(offs).max()), cfg, hc, spec)
            plain = engine.run_device(*args, **kw)
            want = plain.expand_stream(True).cpu().numpy()
            run = engine.run_device(*args, want_queue=True, **kw)
            if dyn and not kw:
                assert run.kernel_path == DYN3_PATH
            got = run.expand_stream(True).cpu().numpy()
            assert got.shape == (len(mesh.indices), 3) and np.array_equal(got, want), (strategy, name, kw)
            assert_flat_equal(run.flat(), plain.flat(), f"{strategy} {name} {kw}")
            pos = np.hstack([mesh.positions, np.ones((mesh.vertex_count, 1))]) @ MATRIX.T
            np.testing.assert_allclose(got, (pos[:, :3] / pos[:, 3:4])[mesh.indices], rtol=1e-5, atol=1e-5)
