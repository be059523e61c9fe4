#!/bin/bash
# compute-sanitizer over small instances of every kernel family (memcheck + racecheck); logs in gpurun_out/
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import numpy as np, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1805_08893_b200 as P
from paper_1805_08893_b200 import engine, draws as D, _native as N
from paper_1805_08893_b200.batching import BatchConfig
from paper_1805_08893_b200.strategies import HashConfig
import torch
M = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]])
mesh = P.shuffle_triangles(P.gen_grid(70, 60), 1)
grid = P.gen_grid(120, 100)
cfg = BatchConfig()
# dynamic batching (tile link kernel) + sort / hash / phash, single mesh and multi-draw
for m in (mesh, grid):
    offs = engine.dynamic_offsets_device(m.indices, cfg)
    d_idx = engine.to_device_indices(m.indices)
    spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(m.positions), matrix=M, vertex_count=m.vertex_count)
    for strat in ("sort", "hash", "phash", "warp", "naive"):
        engine.run_device(strat, d_idx, offs[:-1], offs[1:], offs.numel() - 1, len(m.indices), 1023, cfg, HashConfig(), spec, want_counts=True).check()
        # the general kernels (K1 -> K2 -> K3) next to the three-kernel path
        engine.run_device(strat, d_idx, offs[:-1], offs[1:], offs.numel() - 1, len(m.indices), 1023, cfg, HashConfig(), spec, want_counts=True, fuse=False).check()
# small tables / group widths of the three-kernel path
small = BatchConfig(max_unique=16, max_indices=63, warp_width=4)
offs = engine.dynamic_offsets_device(mesh.indices, small)
for strat in ("sort", "hash", "phash"):
    engine.run_device(strat, engine.to_device_indices(mesh.indices), offs[:-1], offs[1:], offs.numel() - 1, len(mesh.indices), 63, small,
                      HashConfig(table_size=16, max_fast_probes=2), engine.ShaderSpec(kind=N.VR_SHADER_IDENTITY, vertex_count=mesh.vertex_count)).check()
# batch formation over ranges (3 ranks one after another), clients of the stage
from paper_1805_08893_b200 import shard
big = P.shuffle_triangles(P.gen_grid(300, 290), 2)
d_big = engine.to_device_indices(big.indices)
tabs, wss = [], []
import ctypes as C
lib = N.require_cuda()
cc = engine._cfg_c(cfg)
ng, words = lib.vr_dynamic_group_count(len(big.indices), C.byref(cc)), lib.vr_dynamic_table_words(len(big.indices), C.byref(cc))
wsb = lib.vr_dynamic_workspace_bytes(len(big.indices), C.byref(cc))
for r in range(3):
    wss.append(torch.empty(wsb, dtype=torch.uint8, device="cuda"))
    glo, ghi = shard.shard_range(ng, r, 3)
    t = torch.empty(words, dtype=torch.int32, device="cuda")
    engine.raise_status(lib.vr_dynamic_range_tables(engine._ptr(d_big), len(big.indices), C.byref(cc), glo, ghi, engine._ptr(t), engine._ptr(wss[r]), wsb, engine._stream_ptr()))
    tabs.append(t)
g = torch.stack(tabs)
for r in range(3):
    shard.dynamic_offsets_exchange(d_big, cfg, r, 3, gather=lambda t: g, workspace=wss[r])
# formation -> stage without the host (vr_run_counted) and the in-stage output queue
for strat in ("sort", "hash", "phash"):
    full, counts = engine.dynamic_offsets_device(mesh.indices, cfg, sync=False)
    spec_m = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions), matrix=M, vertex_count=mesh.vertex_count)
    engine.run_device(strat, engine.to_device_indices(mesh.indices), None, None, 0, 0, 1023, cfg, HashConfig(), spec_m, counted=(full, counts), want_queue=True).check()
offs_g = engine.static_offsets_device(len(grid.indices), cfg)
spec_g = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(grid.positions), matrix=M, vertex_count=grid.vertex_count)
engine.run_device("warp", engine.to_device_indices(grid.indices), offs_g[:-1], offs_g[1:], offs_g.numel() - 1, len(grid.indices), 96, cfg, None, spec_g, static=True, want_queue=True).check()
r = engine.run_device("naive", engine.to_device_indices(grid.indices), offs_g[:-1], offs_g[1:], offs_g.numel() - 1, len(grid.indices), 96, cfg, None, spec_g, want_queue=True).check()
r.assembly_map_u8(); r.shaded_xyz()
P.ideal_report(mesh)
P.simulate_parallel_cache(mesh.indices, P.CacheConfig(num_processors=3, wave_width=96, entries=64), miss_counts=np.zeros(mesh.vertex_count, dtype=np.int64))
P.run_walk(P.WalkConfig(grid=(40, 40), agents=500, max_move_distance=5, kept_moves=4, steps=2), "hash", BatchConfig(primitive_size=1, batch_size=576))
P.run_on_indices("sort", grid.indices, P.dynamic_batches(grid.indices, cfg), cfg, P.position_shader(grid, M, cycles=65))[0].device_run.shaded_xyz()
ds = D.pack_draws(D.scene_corpus(12, seed=3, lo=6, hi=30, ico=(1, 3)))
o = D.dynamic_offsets_draws(ds, cfg)
for strat in ("sort", "hash"):
    D.run_draws(strat, ds, o, cfg, HashConfig(), matrix=M, want_counts=True).check()
# the persistent tile kernel (two-level scan), several lags
so = engine.static_offsets_device(len(grid.indices), cfg)
spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(grid.positions), matrix=M, vertex_count=grid.vertex_count)
d_idx = engine.to_device_indices(grid.indices)
import os
for lag in ("3", "40", None):
    if lag: os.environ["VR_LAG"] = lag
    else: os.environ.pop("VR_LAG", None)
    N.lib().vr_debug_reload_knobs()
    r = engine.run_device("warp", d_idx, so[:-1], so[1:], so.numel() - 1, len(grid.indices), 96, cfg, None, spec, static=True).check()
    assert r.kernel_path == 3
torch.cuda.synchronize()
print("sanitize workload done")
PY
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool python /tmp/san.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done" gpurun_out/sanitize_$tool.log | tail -3
done
