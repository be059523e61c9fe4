#!/usr/bin/env python
"""Probe: do two independent stage runs overlap usefully on one GPU?  (Would pipelining kernel A of one part of the
batch list under kernel C of another pay?)  Two sort runs over the shuffled 7.2 M-triangle mesh with separate buffers:
back to back on one stream vs on two streams."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1805_08893_b200 as P
from paper_1805_08893_b200 import engine, _native as N
from paper_1805_08893_b200.batching import BatchConfig
from paper_1805_08893_b200.strategies import HashConfig

strategy = sys.argv[1] if len(sys.argv) > 1 else "sort"
mesh = P.shuffle_triangles(P.gen_grid(1898, 1898), 0)
cfg = BatchConfig()
M = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]])
d_idx = engine.to_device_indices(mesh.indices)
pos4 = engine.to_device_positions4(mesh.positions)
offs = engine.dynamic_offsets_device(d_idx, cfg)
nb = offs.numel() - 1
spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=M, vertex_count=mesh.vertex_count)
plans = [engine.run_device(strategy, d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 1023, cfg, HashConfig(), spec,
                           buffers=engine.RunBuffers(), plan_only=True) for _ in range(2)]
for p in plans:
    p.relaunch().check()
s = [torch.cuda.Stream(), torch.cuda.Stream()]
def timed(fn, reps=30):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def serial():
    plans[0].relaunch(); plans[1].relaunch()
def parallel():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event(); ev.record(cur)
    for k in range(2):
        s[k].wait_event(ev)
        with torch.cuda.stream(s[k]):
            plans[k].relaunch()
    for k in range(2):
        cur.wait_stream(s[k])
for _ in range(3): serial(); parallel()
print(f"{strategy}: two runs back to back {timed(serial):.4f} ms, on two streams {timed(parallel):.4f} ms")
