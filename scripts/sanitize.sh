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
    r = engine.run_device("warp", d_idx, so[:-1], so[1:], so.numel() - 1, len(grid.indices), 96, cfg, None, spec, static=True).check()
    assert r.kernel_path == 3
torch.cuda.synchronize()
print("sanitize workload done")
PY
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool python /tmp/san.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done" gpurun_out/sanitize_$tool.log | tail -3
done
