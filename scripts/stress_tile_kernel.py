#!/usr/bin/env python
"""Randomised stress of the persistent tile kernel against the CPU oracle: random grid sizes (ragged last
tile / group), random lags, shuffled and strip order, all (W, batch size) pairs the kernel takes.
python scripts/stress_tile_kernel.py [cases] [seed]"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import oracle as O
import paper_1805_08893_b200 as P
from helpers import assert_flat_equal, oracle_flat, MATRIX
from paper_1805_08893_b200 import engine, _native as N
from paper_1805_08893_b200.batching import BatchConfig

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
shapes = [(32, 96), (32, 192), (16, 120), (8, 48), (4, 24), (64, 192)]
for k in range(cases):
    w, bs = shapes[int(rng.integers(len(shapes)))]
    r, c = int(rng.integers(20, 420)), int(rng.integers(20, 420))
    mesh = P.gen_grid(r, c)
    if rng.random() < 0.4:
        mesh = P.shuffle_triangles(mesh, int(rng.integers(1 << 30)))
    cfg = BatchConfig(batch_size=bs, warp_width=w)
    lag = [None, 1, 2, 5, 33, 100, 700, 5000][int(rng.integers(8))]
    os.environ.pop("VR_LAG", None)
    if lag is not None:
        os.environ["VR_LAG"] = str(lag)
    N.lib().vr_debug_reload_knobs()  # the knobs are read once per process
    so = O.static_batches(len(mesh.indices), batch_size=bs)
    fr = O.run("warp", mesh.indices, so[:-1], so[1:], warp_width=w)
    offs = engine.static_offsets_device(len(mesh.indices), cfg)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions),
                             matrix=MATRIX, vertex_count=mesh.vertex_count)
    run = engine.run_device("warp", engine.to_device_indices(mesh.indices), offs[:-1], offs[1:], offs.numel() - 1,
                            len(mesh.indices), bs, cfg, None, spec, want_counts=True, static=True)
    flat = run.flat()
    assert run.kernel_path == 3
    assert_flat_equal(flat, oracle_flat(fr), f"case {k}: grid {r}x{c} w={w} bs={bs} lag={lag}")
    np.testing.assert_allclose(flat["shaded"][:, :3], O.shade_positions(mesh.positions, fr.unique_ids, MATRIX), rtol=1e-5, atol=1e-5)
    assert np.array_equal(flat["shade_counts"], O.shade_counts(fr.unique_ids, mesh.vertex_count))
print(f"{cases} random cases bit-exact")
