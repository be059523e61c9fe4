"""The tile kernel of the static warp-voting path (csrc/vr_warp_rows.cuh): bulk-staged rows,
per-lane state machine, decoupled shading K tiles later, two-level offset scan, shade-only tail.  Everything is compared
bit-exactly with the CPU oracle; the kernel is reached through vr_run with VR_FLAG_STATIC and a
shader that states its vertex count (<= 2^24), exactly as bench.py does."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
import paper_1805_08893_b200 as P
from helpers import FLAT_KEYS, MATRIX, assert_flat_equal, oracle_flat
from paper_1805_08893_b200 import _native as N
from paper_1805_08893_b200 import engine
from paper_1805_08893_b200.batching import BatchConfig, ConfigError

pytestmark = pytest.mark.gpu


def tile_run(idx, cfg, spec, counts=False, lag=None):
    import torch
    d_idx = engine.to_device_indices(idx)
    so = O.static_batches(len(idx), batch_size=cfg.batch_size)
    o = torch.from_numpy(so.astype(np.int32)).cuda()
    old = os.environ.pop("VR_LAG", None)
    if lag is not None:
        os.environ["VR_LAG"] = str(lag)
    N.lib().vr_debug_reload_knobs()  # the knobs are read once per process
    try:
        run = engine.run_device("warp", d_idx, o[:-1], o[1:], len(so) - 1, len(idx), cfg.batch_size, cfg, None,
                                spec, want_counts=counts, static=True)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("VR_LAG", None)
        if old is not None:
            os.environ["VR_LAG"] = old
        N.lib().vr_debug_reload_knobs()
    assert run.kernel_path == 3 and run.launches == 2, "expected init + the persistent tile kernel"
    return run, so


def blob(flat):
    return b"".join(np.ascontiguousarray(flat[k]).tobytes() for k in FLAT_KEYS)


def test_lag_does_not_change_results(cuda_lib):
    """The tile a CTA's helpers shade (ticket - K) is a scheduling choice: K = 1, a few, more than the
    number of tiles (everything left to the shade-only tickets) and the default give identical bytes."""
    mesh = P.gen_grid(300, 217)
    cfg = BatchConfig()
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=MATRIX, vertex_count=mesh.vertex_count)
    so = O.static_batches(len(mesh.indices))
    fr = O.run("warp", mesh.indices, so[:-1], so[1:])
    want = O.shade_positions(mesh.positions, fr.unique_ids, MATRIX)
    blobs = []
    for lag in (1, 3, 64, 10 ** 6, None):
        run, _ = tile_run(mesh.indices, cfg, spec, counts=True, lag=lag)
        flat = run.flat()
        assert_flat_equal(flat, oracle_flat(fr), f"lag={lag}")
        np.testing.assert_allclose(flat["shaded"][:, :3], want, rtol=1e-5, atol=1e-5)
        assert np.array_equal(flat["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count))
        blobs.append(blob(flat) + flat["shaded"].tobytes())
    assert all(b == blobs[0] for b in blobs)


@pytest.mark.parametrize("width,bs", [(32, 96), (32, 192), (16, 120), (8, 48), (4, 24), (64, 192)])
def test_shuffled_and_random_ids(cuda_lib, width, bs):
    """Worst-case reuse (every index a new id: rows with ~batch_size claims, many rounds, tag wrap)
    and random ids with heavy repetition (degenerate triangles, long hit runs)."""
    rng = np.random.default_rng(width * 1000 + bs)
    cfg = BatchConfig(batch_size=bs, warp_width=width)
    cases = {
        "shuffled": P.shuffle_triangles(P.gen_grid(120, 97), 5).indices,
        "random-small-pool": rng.integers(0, 40, size=3 * 9001).astype(np.uint32),
        "random-large-pool": rng.integers(0, 1 << 24, size=3 * 7003).astype(np.uint32),
        "one-id": np.full(3 * 500, 7, dtype=np.uint32),
    }
    for name, idx in cases.items():
        vcount = int(idx.max()) + 1
        run, so = tile_run(idx, cfg, engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=vcount), counts=True)
        fr = O.run("warp", idx, so[:-1], so[1:], warp_width=width)
        assert_flat_equal(run.flat(), oracle_flat(fr), f"{name} w={width} bs={bs}")
        assert (run.invocations, run.rounds, run.indices) == (fr.invocations, fr.rounds, fr.indices)
        assert np.array_equal(run.expand_stream(False).cpu().numpy().view(np.uint32), idx)  # stream == input
        assert np.array_equal(run.flat()["shade_counts"], O.shade_counts(fr.unique_ids, vcount))


def test_attributes_pass_through(cuda_lib):
    import torch
    mesh = P.gen_icosphere(4)
    cfg = BatchConfig()
    attrs = (np.arange(mesh.vertex_count, dtype=np.uint32)[:, None] * np.array([3, 5], dtype=np.uint32)
             + np.array([1, 2], dtype=np.uint32)).astype(np.uint32)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=None, vertex_count=mesh.vertex_count,
                             attributes=torch.from_numpy(attrs.view(np.int32)).cuda())
    run, so = tile_run(mesh.indices, cfg, spec, counts=True)
    flat = run.flat()
    fr = O.run("warp", mesh.indices, so[:-1], so[1:])
    assert_flat_equal(flat, oracle_flat(fr), "icosphere")
    assert np.array_equal(flat["shaded_attr"].view(np.uint32), attrs[fr.unique_ids])
    assert np.array_equal(flat["shaded"][:, :3], mesh.positions[fr.unique_ids].astype(np.float32))  # plain cast is exact


def test_index_outside_vertex_buffer_is_an_error(cuda_lib):
    """The reference's position shader would raise on positions[vid]; the device path reports the first
    offending batch instead of gathering out of bounds."""
    mesh = P.gen_grid(64, 64)
    idx = mesh.indices.copy()
    idx[96 * 70 + 5] = mesh.vertex_count + 3  # batch 70, tile 1
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=MATRIX, vertex_count=mesh.vertex_count)
    run, _ = tile_run(idx, BatchConfig(), spec)
    with pytest.raises(IndexError, match="batch 70"):  # strategies.py:62-65 positions[vid]
        run.check()


def test_output_capacity_is_checked(cuda_lib):
    """Outputs smaller than the result: VR_ERR_CAPACITY, nothing written past the buffers."""
    import ctypes as C
    import torch
    mesh = P.gen_grid(100, 100)
    cfg = BatchConfig()
    lib = N.require_cuda()
    d_idx = engine.to_device_indices(mesh.indices)
    offs = engine.static_offsets_device(len(mesh.indices), cfg)
    nb = offs.numel() - 1
    cc = engine._cfg_c(cfg)
    ws = torch.empty(lib.vr_run_workspace_bytes(N.VR_WARP, len(mesh.indices), nb, C.byref(cc), None) + 256,
                     dtype=torch.uint8, device="cuda")
    cap = 1000  # far fewer than the ~22 000 invocations
    guard = 64
    uid = torch.full((cap + guard,), -7, dtype=torch.int32, device="cuda")
    shaded = torch.full((cap + guard, 4), -7.0, dtype=torch.float32, device="cuda")
    stats = torch.zeros(N.VR_STATS_WORDS, dtype=torch.int64, device="cuda")
    bro = torch.empty(nb + 1, dtype=torch.int32, device="cuda")
    ruo = torch.empty(4 * nb + 2, dtype=torch.int32, device="cuda")
    rp = torch.empty(4 * nb + 2, dtype=torch.int32, device="cuda")
    amap = torch.empty(len(mesh.indices) + 8, dtype=torch.int16, device="cuda")
    sh = N.ShaderC()
    sh.kind, sh.vertex_count, sh.has_matrix = N.VR_SHADER_POSITION, mesh.vertex_count, 0
    out = N.OutputsC(bro.data_ptr(), ruo.data_ptr(), rp.data_ptr(), uid.data_ptr(), amap.data_ptr(), shaded.data_ptr(),
                     None, None, stats.data_ptr(), cap, 4 * nb + 1)
    p4 = engine.to_device_positions4(mesh.positions)
    sh.d_positions4 = p4.data_ptr()
    st = lib.vr_run(N.VR_WARP | N.VR_FLAG_STATIC, d_idx.data_ptr(), d_idx.numel(), offs.data_ptr(),
                    offs.data_ptr() + 4, nb, len(mesh.indices), cfg.batch_size, C.byref(cc), None, C.byref(sh),
                    C.byref(out), ws.data_ptr(), ws.numel(), None)
    assert st == N.VR_OK
    torch.cuda.synchronize()
    err = int(stats[N.VR_STAT_ERROR].item())
    assert err != -1 and (err & 0xFF) == N.VR_ERR_CAPACITY
    assert bool((uid[cap:] == -7).all()) and bool((shaded[cap:] == -7.0).all())
