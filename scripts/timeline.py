#!/usr/bin/env python
"""Debugging aid: build libvrgeom with -DVR_TIMELINE into a scratch .so, run the headline workload once
and print per-phase durations of the tile kernel (median / p10 / p90 over tiles, microseconds)."""
import ctypes as C, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_08893_b200 import build as B, _native as N
lib_path = os.path.join(ROOT, "gpurun_out", "libvrgeom_timeline.so")
os.makedirs(os.path.dirname(lib_path), exist_ok=True)
flags = [f for f in B.NVCC_FLAGS if not f.startswith("--use_fast_math")]
subprocess.check_call(["/usr/local/cuda/bin/nvcc", *flags, "-DVR_TIMELINE", "-shared", "-o", lib_path] +
                      [os.path.join(B.CSRC, s) for s in B.SOURCES])
N.LIB_PATH = lib_path
import torch
import paper_1805_08893_b200 as P
from paper_1805_08893_b200 import engine
side = int(sys.argv[1]) if len(sys.argv) > 1 else 1898
mesh = P.gen_grid(side, side)
cfg = P.BatchConfig()
d_idx = engine.to_device_indices(mesh.indices)
pos4 = engine.to_device_positions4(mesh.positions)
offs = engine.static_offsets_device(len(mesh.indices), cfg)
nb = offs.numel() - 1
M = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]])
spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=M, vertex_count=mesh.vertex_count)
bufs = engine.RunBuffers()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    run = engine.run_device("warp", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 96, cfg, None, spec, buffers=bufs, static=True)
torch.cuda.synchronize()
run.check()
lib = N.lib()
MARKS, TILES = 6, 4096
buf = (C.c_ulonglong * (MARKS * 2 * TILES))()
lib.vr_debug_timeline.restype = C.c_int
got = lib.vr_debug_timeline(buf, MARKS * 2 * TILES)
a = np.frombuffer(buf, dtype=np.uint64).reshape(MARKS, 2, TILES).astype(np.int64)
nt = min(TILES, (nb + 63) // 64)
a = a[:, :, :nt]
t0 = a[0].min()
names = ["entry->ticket", "ticket->staged", "dedup", "lookback+amap", "shade"]
print(f"tiles {nt}, kernel span {(a[5].max() - t0) / 1e3:.1f} us")
for k in range(5):
    d = (a[k + 1] - a[k]).reshape(-1) / 1e3
    print(f"{names[k]:16s} median {np.median(d):7.2f}  p10 {np.percentile(d, 10):7.2f}  p90 {np.percentile(d, 90):7.2f}  mean {d.mean():7.2f} us")
life = (a[5] - a[0]).reshape(-1) / 1e3
print(f"{'lifetime':16s} median {np.median(life):7.2f}  p10 {np.percentile(life, 10):7.2f}  p90 {np.percentile(life, 90):7.2f}  mean {life.mean():7.2f} us")
start = (a[0][0] - t0) / 1e3
print("tile start times (us) at tile 0, 592, 1184, ...:", [round(float(start[i]), 1) for i in range(0, nt, 592)])
