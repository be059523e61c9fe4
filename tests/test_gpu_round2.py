"""Round-2 parity additions: out-of-range vertex ids on every kernel path, static-looking batch lists that
do not start on an index quad, the stream dump format."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1805_08893_b200 as P
from helpers import MATRIX, assert_flat_equal, oracle_flat
from paper_1805_08893_b200 import _native as N
from paper_1805_08893_b200 import engine
from paper_1805_08893_b200.batching import Batch, BatchConfig
from paper_1805_08893_b200.strategies import HashConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["naive", "warp", "sort", "hash", "phash"])
@pytest.mark.parametrize("shader", ["position", "identity"])
def test_vertex_id_outside_buffer_every_strategy(cuda_lib, strategy, shader):
    """strategies.py:62-65: positions[vid] raises IndexError.  The generic kernels (K1 -> K2 -> K3), the unfused
    and the fused static warp kernels must report the first offending batch and neither gather nor tally out of
    bounds."""
    import torch
    mesh = P.gen_grid(90, 90)
    cfg = BatchConfig()
    idx = mesh.indices.copy()
    stat = strategy in ("naive", "warp")
    offs = O.static_batches(len(idx)) if stat else O.dynamic_batches(idx)
    bad_batch = 7
    idx[offs[bad_batch] + 4] = mesh.vertex_count + 11
    idx[offs[bad_batch + 9] + 1] = 0xFFFFFF00
    if not stat:
        offs = O.dynamic_batches(idx)
        bad_batch = int(np.searchsorted(offs, np.flatnonzero(idx >= mesh.vertex_count)[0], side="right") - 1)
    guard = torch.full((mesh.vertex_count + 4096,), 7, dtype=torch.int32, device="cuda")  # counts + canary behind them
    variants = [dict()]
    if strategy == "warp":
        variants += [dict(static=True, fuse=False), dict(static=True)]
    for kw in variants:
        guard.fill_(7)
        if shader == "position":
            spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                     matrix=MATRIX, vertex_count=mesh.vertex_count)
        else:
            spec = engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=mesh.vertex_count)
        o = torch.from_numpy(offs.astype(np.int32)).cuda()
        bufs = engine.RunBuffers()
        bufs.t["counts"] = guard[:mesh.vertex_count]  # the tally buffer, with the canary right behind it
        run = engine.run_device(strategy, engine.to_device_indices(idx), o[:-1], o[1:], len(offs) - 1, len(idx),
                                int(np.diff(offs).max()), cfg, HashConfig(), spec, want_counts=True, buffers=bufs, **kw)
        with pytest.raises(IndexError, match=f"batch {bad_batch}\\)"):
            run.check()
        torch.cuda.synchronize()
        assert int((guard[mesh.vertex_count:] != 7).sum()) == 0, "tally written out of bounds"
    # through the public API
    with pytest.raises(IndexError):
        batches = P.offsets_to_batches(offs)
        sh = P.position_shader(mesh, MATRIX) if shader == "position" else P.identity_shader()
        P.run_on_indices(strategy, idx, batches, cfg, sh, HashConfig(), vertex_count=mesh.vertex_count)


def test_equally_spaced_batches_off_quad_alignment(cuda_lib):
    """[Batch(3,99), Batch(99,195)] looks like static_batches shifted by one primitive; the
    position-aligned kernels need a 16-byte aligned start, so the list must take the general kernel instead of
    failing with 'batch is not a primitive-aligned range'."""
    mesh = P.gen_grid(30, 30)
    cfg = BatchConfig()
    for lists in ([Batch(3, 99), Batch(99, 195)], [Batch(3, 99)], [Batch(6, 102), Batch(102, 198), Batch(198, 240)],
                  [Batch(12, 108), Batch(108, 204)], [Batch(0, 96), Batch(96, 150)]):
        bb = np.array([b.begin for b in lists]), np.array([b.end for b in lists])
        for strat in ("warp", "naive", "sort"):
            out = P.run_on_indices(strat, mesh.indices, lists, cfg, P.identity_shader(), vertex_count=mesh.vertex_count)
            fr = O.run(strat, mesh.indices, bb[0], bb[1])
            assert_flat_equal(out[0].device_run.flat(), oracle_flat(fr), f"{strat} {lists}")
            assert np.array_equal(out[0].as_array(), np.concatenate([mesh.indices[b.begin:b.end] for b in lists]))


def test_stream_write_binary_roundtrip(cuda_lib, tmp_path):
    """strategies.py:150-152 / cli.py:340-345 --dump-stream: flat native-endian dump of the per-corner records."""
    mesh = P.shuffle_triangles(P.gen_grid(33, 21), 2)
    cfg = BatchConfig()
    dyn = P.dynamic_batches(mesh.indices, cfg)
    stream, _ = P.run_sorting(mesh, dyn, cfg, P.position_shader(mesh, MATRIX))
    path = tmp_path / "stream.bin"
    stream.write_binary(path)
    back = np.fromfile(path, dtype=np.float32).reshape(-1, 3)
    assert back.shape == (len(mesh.indices), 3) and np.array_equal(back, stream.as_array())
    pos = np.hstack([mesh.positions, np.ones((mesh.vertex_count, 1))]) @ MATRIX.T
    want = (pos[:, :3] / pos[:, 3:4]).astype(np.float32)[mesh.indices]
    np.testing.assert_allclose(back, want, rtol=1e-5, atol=1e-5)
    ident, _ = P.run_sorting(mesh, dyn, cfg, P.identity_shader())
    ident.write_binary(path)
    assert np.array_equal(np.fromfile(path, dtype=np.uint32), mesh.indices)


@pytest.mark.parametrize("case", ["static-warp", "dynamic-hash", "dynamic-sort", "static-naive"])
def test_sharded_runs_concatenate_to_the_unsharded_result(cuda_lib, case):
    """SURVEY.md 8e / strategies.py:465-483: one stream cut into whole batches per rank.  The shards of world =
    2, 3, 8 are run one after another on this GPU through shard.run_sharded (the code every rank runs); their
    ordered merge must equal the single-GPU result byte for byte, statistics and per-vertex tallies included."""
    from paper_1805_08893_b200 import shard
    import torch
    batching, strategy = case.split("-")
    mesh = P.shuffle_triangles(P.gen_grid(150, 131), 9) if batching == "dynamic" else P.gen_grid(150, 131)
    cfg = BatchConfig()
    hc = HashConfig()
    d_idx = engine.to_device_indices(mesh.indices)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=MATRIX, vertex_count=mesh.vertex_count)
    whole, plan1 = shard.run_sharded(strategy, d_idx, cfg, hc, spec, batching=batching, rank=0, world=1, want_counts=True)
    want = whole.flat()
    want_stats = whole.stats().copy()
    if strategy == "warp":
        assert whole.kernel_path == 3  # the persistent tile kernel
    for world in (2, 3, 8):
        flats, blocks, nb = [], [], 0
        for rank in range(world):
            run, plan = shard.run_sharded(strategy, d_idx, cfg, hc, spec, batching=batching, rank=rank, world=world,
                                          want_counts=True)
            assert plan.batch_lo == nb
            nb = plan.batch_hi
            flats.append(run.flat())
            s = run.stats_dev.clone()
            s[shard.STAT_BATCH_BASE] = plan.batch_lo
            blocks.append(s)
        assert nb == plan1.n_batches
        got = shard.concat_flats(flats)
        assert_flat_equal(got, want, f"{case} world {world}")
        assert np.array_equal(got["shaded"], want["shaded"])  # same kernels, same arithmetic: bit-identical
        assert np.array_equal(got["shade_counts"], want["shade_counts"])
        total = shard.merge_stats(torch.stack(blocks)).cpu().numpy()
        assert np.array_equal(total[:8], want_stats[:8]), (total, want_stats)


def test_sharded_error_names_the_stream_batch(cuda_lib):
    """The merged error word names the first failing batch of the STREAM, not of a shard."""
    from paper_1805_08893_b200 import shard
    import torch
    mesh = P.gen_grid(60, 60)
    idx = mesh.indices.copy()
    idx[96 * 55 + 7] = mesh.vertex_count + 1  # stream batch 55
    idx[96 * 40 + 7] = mesh.vertex_count + 2  # stream batch 40: the first one
    d_idx = engine.to_device_indices(idx)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=mesh.vertex_count)
    blocks = []
    for rank in range(4):
        run, plan = shard.run_sharded("warp", d_idx, BatchConfig(), None, spec, batching="static", rank=rank, world=4,
                                      want_counts=True)
        s = run.stats_dev.clone()
        s[shard.STAT_BATCH_BASE] = plan.batch_lo
        blocks.append(s)
    err = int(shard.merge_stats(torch.stack(blocks))[N.VR_STAT_ERROR])
    assert (err >> 8, err & 0xFF) == (40, N.VR_ERR_VERTEX_RANGE)


def test_sharded_multidraw_scene(cuda_lib):
    """configs[4] across ranks: whole draws per rank (LPT); the per-draw reports of all ranks together equal the
    per-draw reports of the single-GPU packed run."""
    from paper_1805_08893_b200 import draws as D
    from paper_1805_08893_b200 import shard
    meshes = D.scene_corpus(24, seed=5, lo=10, hi=40, ico=(1, 3))
    cfg = BatchConfig()
    ds = D.pack_draws(meshes)
    offs = D.dynamic_offsets_draws(ds, cfg)
    whole = D.run_draws("hash", ds, offs, cfg, HashConfig(), matrix=MATRIX)
    want = [(r.indices, r.invocations, r.batches) for r in D.per_draw_reports(whole, ds, offs, "hash")]
    for world in (2, 5):
        got = {}
        tot = np.zeros(8, dtype=np.int64)
        for rank in range(world):
            run, rds, roffs, mine = shard.run_draws_sharded("hash", meshes, cfg, HashConfig(), rank=rank, world=world,
                                                           matrix=MATRIX)
            for d, r in zip(mine, D.per_draw_reports(run, rds, roffs, "hash")):
                got[int(d)] = (r.indices, r.invocations, r.batches)
            st = run.stats()
            tot[:6] += st[:6]
            tot[6] = max(tot[6], st[6])
        assert [got[d] for d in range(len(meshes))] == want
        assert np.array_equal(tot[:7], whole.stats()[:7])


@pytest.mark.parametrize("cfgv", [(256, 1023, 3), (64, 255, 3), (256, 1023, 1), (40, 96, 3)])
def test_ranged_batch_formation_equals_the_whole_stream_scan(cuda_lib, cfgv):
    """SURVEY.md 8e option (ii): every rank scans its own range of the stream into an entry -> exit table, the tables
    are gathered (here: the ranks of a world run one after another on this GPU), every rank emits the batches that
    start in its range.  The concatenation must be vr_dynamic_batches' array, for any world size -- including
    worlds with more ranks than groups (empty ranges)."""
    from paper_1805_08893_b200 import shard
    import torch
    mu, mi, ps = cfgv
    cfg = BatchConfig(max_unique=mu, max_indices=mi, primitive_size=ps, batch_size=96 if ps == 3 else 97)
    mesh = P.shuffle_triangles(P.gen_grid(300, 290), 2) if mu != 64 else P.gen_grid(300, 290)
    idx = mesh.indices if ps == 3 else mesh.indices[:400_001]
    d_idx = engine.to_device_indices(idx)
    whole = engine.dynamic_offsets_device(d_idx, cfg).cpu().numpy()
    assert np.array_equal(whole, O.dynamic_batches(idx, primitive_size=ps, max_unique=mu, max_indices=mi))
    for world in (1, 2, 3, 5, 16):
        ws = [None] * world
        tables = []
        import ctypes as C
        lib = N.require_cuda()
        c = engine._cfg_c(cfg)
        n = len(idx)
        ng, words = lib.vr_dynamic_group_count(n, C.byref(c)), lib.vr_dynamic_table_words(n, C.byref(c))
        ws_bytes = lib.vr_dynamic_workspace_bytes(n, C.byref(c))
        for r in range(world):  # step 1 on every rank
            ws[r] = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
            glo, ghi = shard.shard_range(ng, r, world)
            t = torch.empty(words, dtype=torch.int32, device="cuda")
            engine.raise_status(lib.vr_dynamic_range_tables(engine._ptr(d_idx), n, C.byref(c), glo, ghi, engine._ptr(t),
                                                            engine._ptr(ws[r]), ws_bytes, engine._stream_ptr()))
            tables.append(t)
        gathered = torch.stack(tables)  # step 2: the all-gather
        parts, total_seen, next_base = [], None, 0
        for r in range(world):  # step 3 on every rank
            local, base, total = shard.dynamic_offsets_exchange(d_idx, cfg, r, world, gather=lambda t: gathered, workspace=ws[r])
            e, b, tot = shard.compose_tables(gathered.cpu().numpy(), r)
            assert (b, tot) == (base, total) == (next_base, len(whole) - 1), (world, r)
            local = local.cpu().numpy()
            next_base += len(local) - 1
            if len(local) > 1:
                parts.append(local[:-1])
                closing = local[-1]
        got = np.concatenate(parts + [[closing]])
        assert np.array_equal(got, whole), (cfgv, world)


def test_sharded_run_with_exchanged_boundaries(cuda_lib):
    """run_sharded(batching='exchange') at world 1 (no process group) equals the unsharded run."""
    from paper_1805_08893_b200 import shard
    mesh = P.shuffle_triangles(P.gen_grid(200, 180), 3)
    cfg, hc = BatchConfig(), HashConfig()
    d_idx = engine.to_device_indices(mesh.indices)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=MATRIX, vertex_count=mesh.vertex_count)
    a, plan_a = shard.run_sharded("hash", d_idx, cfg, hc, spec, batching="exchange", rank=0, world=1)
    b, plan_b = shard.run_sharded("hash", d_idx, cfg, hc, spec, batching="dynamic", rank=0, world=1)
    assert (plan_a.batch_lo, plan_a.batch_hi, plan_a.index_lo, plan_a.index_hi) == (plan_b.batch_lo, plan_b.batch_hi, plan_b.index_lo, plan_b.index_hi)
    assert_flat_equal(a.flat(), b.flat(), "exchange vs whole-stream scan")


@pytest.mark.parametrize("strategy", ["sort", "hash", "phash"])
def test_formation_to_stage_without_host_round_trip(cuda_lib, strategy):
    """vr_dynamic_batches -> vr_run_counted: the batch count stays on the device (the launch is sized for
    vr_dynamic_batch_bound); results, statistics and error reporting equal the synchronous path."""
    import ctypes as C
    cfg, hc = BatchConfig(), HashConfig()
    lib = N.require_cuda()
    for mesh in (P.gen_grid(140, 90), P.shuffle_triangles(P.gen_grid(120, 77), 5), P.gen_icosphere(4)):
        d_idx = engine.to_device_indices(mesh.indices)
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                                 matrix=MATRIX, vertex_count=mesh.vertex_count)
        offs = engine.dynamic_offsets_device(d_idx, cfg)
        want = engine.run_device(strategy, d_idx, offs[:-1], offs[1:], offs.numel() - 1, len(mesh.indices), 1023, cfg, hc, spec,
                                 want_counts=True)
        full, counts = engine.dynamic_offsets_device(d_idx, cfg, sync=False)
        bound = lib.vr_dynamic_batch_bound(len(mesh.indices), C.byref(engine._cfg_c(cfg)), 0)
        assert bound >= offs.numel() - 1
        run = engine.run_device(strategy, d_idx, None, None, 0, 0, 1023, cfg, hc, spec, want_counts=True, counted=(full, counts))
        assert run.kernel_path == 4
        got, ref = run.flat(), want.flat()
        assert run.n_batches == want.n_batches == offs.numel() - 1
        assert_flat_equal(got, ref, strategy)
        assert np.array_equal(got["shaded"], ref["shaded"]) and np.array_equal(got["shade_counts"], ref["shade_counts"])
        assert np.array_equal(run.stats()[:7], want.stats()[:7]) and run.probes == want.probes
    # the smallest budget: one triangle per batch, the bound is exact
    idx = np.array([0, 1, 2, 3, 3, 3, 4, 5, 6], dtype=np.uint32)
    tiny = BatchConfig(max_unique=3, max_indices=6, primitive_size=3)
    full, counts = engine.dynamic_offsets_device(idx, tiny, sync=False)
    run = engine.run_device(strategy, engine.to_device_indices(idx), None, None, 0, 0, 6, tiny, HashConfig(table_size=4),
                            engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=7), counted=(full, counts))
    assert run.flat()["round_prims"].tolist() == [1, 1, 1] and run.n_batches == 3
