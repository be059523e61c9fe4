"""Full-size configs (BASELINE.json configs[2], configs[3]): the oracle's goldens from
BASELINE.md plus size-independent properties (stream == input, tally sums, monotone offsets)."""
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


@pytest.fixture(scope="module")
def dragon_grid():
    mesh = P.gen_grid(1898, 1898)
    assert (mesh.vertex_count, mesh.triangle_count, len(mesh.indices)) == (3602404, 7197218, 21591654)
    return mesh


WARP_PATHS = {"generic": dict(), "static": dict(static=True, fuse=False), "fused": dict(static=True)}


@pytest.mark.parametrize("path", sorted(WARP_PATHS))
def test_config3_warp(cuda_lib, dragon_grid, path):
    """224 914 batches, 449 827 rounds, 8 100 190 invocations -- through the
    generic thread-per-batch kernel, the static-batch kernel and the fused kernel."""
    import torch
    mesh = dragon_grid
    cfg = BatchConfig()
    kw = WARP_PATHS[path]
    d_idx = engine.to_device_indices(mesh.indices)
    offs = engine.static_offsets_device(len(mesh.indices), cfg)
    nb = offs.numel() - 1
    spec = engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=mesh.vertex_count)
    run = engine.run_device("warp", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 96, cfg, None, spec,
                            want_counts=True, **kw).check()
    assert (nb, run.rounds, run.invocations) == (224914, 449827, 8100190)
    assert abs(1 - run.invocations / run.indices - 0.624846) < 1e-6
    assert np.array_equal(run.expand_stream(False).cpu().numpy().view(np.uint32), mesh.indices)
    assert int(run.shade_counts.sum().item()) == run.invocations
    if path == "fused":  # the persistent tile kernel: every output of the full run against the C oracle
        assert run.kernel_path == 3
        so = O.static_batches(len(mesh.indices))
        fr = O.run("warp", mesh.indices, so[:-1], so[1:])
        assert_flat_equal(run.flat(), oracle_flat(fr), "config 3, tile kernel")
        # ... and with the position shader: all 8 100 190 shaded vertices against the float64 oracle shader
        pspec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                  matrix=MATRIX, vertex_count=mesh.vertex_count)
        prun = engine.run_device("warp", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 96, cfg, None, pspec,
                                 want_counts=True, **kw).check()
        assert prun.kernel_path == 3
        pflat = prun.flat()
        assert_flat_equal(pflat, oracle_flat(fr), "config 3, tile kernel, position shader")
        want = O.shade_positions(mesh.positions, fr.unique_ids, MATRIX)
        assert pflat["shaded"].shape[0] == 8100190
        np.testing.assert_allclose(pflat["shaded"][:, :3], want, rtol=1e-5, atol=1e-5)
        assert np.array_equal(pflat["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count))
    # bit-exact against the oracle on a prefix and on a window in the middle of the stream
    for lo in (0, 3000 * 96 * 30):
        sub = mesh.indices[lo:lo + 96 * 3000 + 33]  # ragged last batch
        so = O.static_batches(len(sub))
        fr = O.run("warp", sub, so[:-1], so[1:])
        o = torch.from_numpy(so.astype(np.int32)).cuda()
        r = engine.run_device("warp", engine.to_device_indices(sub), o[:-1], o[1:], len(so) - 1, len(sub), 96,
                              cfg, None, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY), **kw)
        assert_flat_equal(r.flat(), oracle_flat(fr), f"{path} window {lo}")


@pytest.mark.parametrize("width", [4, 8, 16, 32, 64])
def test_warp_paths_agree_all_widths(cuda_lib, width):
    """Static-batch and fused kernels against the oracle for every warp width, positions shaded."""
    import torch
    mesh = P.shuffle_triangles(P.gen_grid(90, 70), 3) if width in (8, 32) else P.gen_grid(90, 70)
    for bs in (96, 24, 192):
        cfg = BatchConfig(batch_size=bs, warp_width=width)
        so = O.static_batches(len(mesh.indices), batch_size=bs)
        fr = O.run("warp", mesh.indices, so[:-1], so[1:], warp_width=width)
        want = O.shade_positions(mesh.positions, fr.unique_ids, MATRIX)
        o = torch.from_numpy(so.astype(np.int32)).cuda()
        for path, kw in WARP_PATHS.items():
            spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                     matrix=MATRIX, vertex_count=mesh.vertex_count)
            r = engine.run_device("warp", engine.to_device_indices(mesh.indices), o[:-1], o[1:], len(so) - 1,
                                  len(mesh.indices), bs, cfg, None, spec, want_counts=True, **kw)
            flat = r.flat()
            assert_flat_equal(flat, oracle_flat(fr), f"w={width} bs={bs} {path}")
            np.testing.assert_allclose(flat["shaded"][:, :3], want, rtol=1e-5, atol=1e-5)
            assert np.array_equal(flat["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count))


def test_config3_mesh_dynamic_sort(cuda_lib, dragon_grid):
    """dynamic 256/1023 on the strip-ordered mesh: 28 350 batches, 7 257 500 invocations."""
    mesh = dragon_grid
    cfg = BatchConfig()
    d_idx = engine.to_device_indices(mesh.indices)
    offs = engine.dynamic_offsets_device(d_idx, cfg)
    nb = offs.numel() - 1
    assert nb == 28350
    run = engine.run_device("sort", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 1023, cfg, None,
                            engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY)).check()
    assert run.invocations == 7257500
    assert np.array_equal(run.expand_stream(False).cpu().numpy().view(np.uint32), mesh.indices)
    h = offs.cpu().numpy().astype(np.int64)
    assert np.array_equal(h.astype(np.int64), O.dynamic_batches(mesh.indices))  # every boundary of the 21.6 M-index stream
    # the complete flat output (28 350 batches) against the oracle, then the shaded positions
    fr = O.run("sort", mesh.indices, h[:-1], h[1:])
    assert_flat_equal(run.flat(), oracle_flat(fr), "config 3 mesh, dynamic sort, full")
    pspec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                              matrix=MATRIX, vertex_count=mesh.vertex_count)
    prun = engine.run_device("sort", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 1023, cfg, None, pspec).check()
    pflat = prun.flat()
    assert_flat_equal(pflat, oracle_flat(fr), "config 3 mesh, dynamic sort, position shader")
    np.testing.assert_allclose(pflat["shaded"][:, :3], O.shade_positions(mesh.positions, fr.unique_ids, MATRIX),
                               rtol=1e-5, atol=1e-5)


def test_config4_shuffled_hash_and_sort(cuda_lib, dragon_grid):
    """84 672 batches, 21 591 005 invocations, probes 216 377 586 / chain 256."""
    mesh = P.shuffle_triangles(dragon_grid, 0)
    assert list(mesh.indices[:6]) == [3502237, 3504135, 3502238, 2050717, 2052615, 2050718]
    cfg = BatchConfig()
    d_idx = engine.to_device_indices(mesh.indices)
    offs = engine.dynamic_offsets_device(d_idx, cfg)
    nb = offs.numel() - 1
    assert nb == 84672
    h = offs.cpu().numpy().astype(np.int64)
    assert h[0] == 0 and h[-1] == len(mesh.indices) and (np.diff(h) > 0).all() and (np.diff(h) % 3 == 0).all()
    assert np.array_equal(h, O.dynamic_batches(mesh.indices))  # every boundary
    k = 3000
    pos4 = engine.to_device_positions4(mesh.positions)
    for strat in ("hash", "sort", "phash"):
        run = engine.run_device(strat, d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 1023, cfg,
                                HashConfig(), engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY)).check()
        assert run.invocations == 21591005
        if strat == "hash":
            assert run.probes == (216377586, 0, 256)
        assert np.array_equal(run.expand_stream(False).cpu().numpy().view(np.uint32), mesh.indices)
        # the COMPLETE flat output of all 84 672 batches and the probe statistics against the oracle
        full = O.run(strat, mesh.indices, h[:-1], h[1:])
        assert_flat_equal(run.flat(), oracle_flat(full), f"config4 {strat} full")
        if strat in ("hash", "phash"):
            assert run.probes == (full.probes_fast, full.probes_slow, full.probe_max_chain), strat
        # position shader on the shuffled stream (random gathers), every shaded vertex
        prun = engine.run_device(strat, d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 1023, cfg, HashConfig(),
                                 engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=MATRIX,
                                                   vertex_count=mesh.vertex_count)).check()
        got = prun.shaded4[:prun.invocations, :3].cpu().numpy()
        np.testing.assert_allclose(got, O.shade_positions(mesh.positions, full.unique_ids, MATRIX), rtol=1e-5, atol=1e-5)
        del full, got, prun
        sub_offs = h[:k + 1]
        fr = O.run(strat, mesh.indices, sub_offs[:-1], sub_offs[1:])
        sub = engine.run_device(strat, d_idx, offs[:k], offs[1:k + 1], k, int(sub_offs[-1]), 1023, cfg,
                                HashConfig(), engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY))
        assert_flat_equal(sub.flat(), oracle_flat(fr), f"config4 {strat} prefix")
        if strat in ("hash", "phash"):
            assert sub.probes == (fr.probes_fast, fr.probes_slow, fr.probe_max_chain)


def test_config5_multidraw_scene(cuda_lib):
    """BASELINE.json configs[4]: 1000 draws, 20 397 942 triangles, 10 319 577 vertices, dynamic 256/1023
    batches per draw, sort and hash dedup.  Everything is compared with the per-mesh oracle runs:
    boundaries, every round, every local index, statistics, per-vertex tallies."""
    from helpers import oracle_draws
    from paper_1805_08893_b200 import draws as D
    meshes = D.scene_corpus(1000)
    ds = D.pack_draws(meshes)
    assert (ds.triangles, int(ds.vertex_base[-1])) == (20_397_942, 10_319_577)
    cfg = BatchConfig()
    offsets = D.dynamic_offsets_draws(ds, cfg)
    for strategy in ("sort", "hash"):
        want = oracle_draws(O, strategy, meshes, matrix=MATRIX, shade=False)
        assert np.array_equal(offsets.cpu().numpy().astype(np.int64), want["offsets"])
        run = D.run_draws(strategy, ds, offsets, cfg, HashConfig(), matrix=MATRIX, want_counts=True)
        flat = run.flat()
        assert_flat_equal(flat, want["flat"], f"c5 {strategy}")
        t = want["totals"]
        assert (len(offsets) - 1, run.invocations, run.rounds) == (154_797, 39_026_006, 154_797)
        assert (run.invocations, run.rounds, run.indices) == (t["invocations"], t["rounds"], t["indices"])
        if strategy == "hash":
            assert run.probes == (t["probes_fast"], 0, t["probe_max_chain"]) and run.probes[0] == 328_902_576
        assert np.array_equal(flat["shade_counts"], want["counts"])
        # shaded positions: spot-check three draws against the float64 shader
        for d in (0, 501, 999):
            b0 = int(np.searchsorted(want["offsets"][:-1], ds.index_start[d]))
            b1 = int(np.searchsorted(want["offsets"][:-1], ds.index_start[d + 1]))
            ruo, bro = want["flat"]["round_uid_off"], want["flat"]["batch_round_off"]
            u0, u1 = int(ruo[bro[b0]]), int(ruo[bro[b1]])
            ref = O.shade_positions(meshes[d].positions, want["flat"]["unique_ids"][u0:u1], MATRIX)
            np.testing.assert_allclose(flat["shaded"][u0:u1, :3], ref, rtol=1e-5, atol=1e-5)


def test_sort_long_static_batches_both_kernels(cuda_lib):
    """configs[0]'s batch shape (static 768, up to 768 distinct ids) on a mesh with enough batches
    that the warp-per-batch sort kernel is chosen (>= 2048), and on a prefix that takes the CTA sort."""
    mesh = P.gen_grid(560, 560)
    cfg = BatchConfig(batch_size=768, max_unique=768, block_size=1024)
    for n_idx in (len(mesh.indices), 768 * 300):
        idx = mesh.indices[:n_idx]
        so = O.static_batches(n_idx, batch_size=768)
        assert (len(so) - 1 >= 2048) == (n_idx == len(mesh.indices))
        fr = O.run("sort", idx, so[:-1], so[1:], max_unique=768)
        d_idx = engine.to_device_indices(idx)
        offs = engine.static_offsets_device(n_idx, cfg)
        run = engine.run_device("sort", d_idx, offs[:-1], offs[1:], offs.numel() - 1, n_idx, 768, cfg, None,
                                engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY))
        assert_flat_equal(run.flat(), oracle_flat(fr), f"static-768 sort, {len(so) - 1} batches")


def test_config4_boundary_exchange_world8(cuda_lib, dragon_grid):
    """configs[3] 'sharded over 2/4/8 GPUs': the shuffled 7.2 M-triangle stream cut into 8 index ranges; every rank's
    range tables, one gather, every rank's offsets (shard.dynamic_offsets_exchange, the ranks run one after another
    here).  Their concatenation must be the 84 672 boundaries of the whole-stream scan."""
    import ctypes as C
    import torch
    from paper_1805_08893_b200 import shard
    mesh = P.shuffle_triangles(dragon_grid, 0)
    cfg = BatchConfig()
    d_idx = engine.to_device_indices(mesh.indices)
    whole = engine.dynamic_offsets_device(d_idx, cfg)
    lib = N.require_cuda()
    c = engine._cfg_c(cfg)
    n = len(mesh.indices)
    world = 8
    ng, words = lib.vr_dynamic_group_count(n, C.byref(c)), lib.vr_dynamic_table_words(n, C.byref(c))
    ws_bytes = lib.vr_dynamic_workspace_bytes(n, C.byref(c))
    ws, tables = [], []
    for r in range(world):
        ws.append(torch.empty(ws_bytes, dtype=torch.uint8, device="cuda"))
        glo, ghi = shard.shard_range(ng, r, world)
        t = torch.empty(words, dtype=torch.int32, device="cuda")
        engine.raise_status(lib.vr_dynamic_range_tables(engine._ptr(d_idx), n, C.byref(c), glo, ghi, engine._ptr(t),
                                                        engine._ptr(ws[r]), ws_bytes, engine._stream_ptr()))
        tables.append(t)
    gathered = torch.stack(tables)
    parts, seen = [], 0
    for r in range(world):
        local, base, total = shard.dynamic_offsets_exchange(d_idx, cfg, r, world, gather=lambda t: gathered, workspace=ws[r])
        assert base == seen and total == whole.numel() - 1 == 84672
        seen += local.numel() - 1
        parts.append(local[:-1])
        last = local[-1:]
    assert torch.equal(torch.cat(parts + [last]), whole)
