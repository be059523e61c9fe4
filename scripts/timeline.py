#!/usr/bin/env python
"""Debugging aid: build libvrgeom with -DVR_TIMELINE into a scratch .so, run the headline workload and
print per-phase durations of the tile kernel (median / p10 / p90 over tiles, microseconds)."""
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
    if not os.environ.get("VR_NOFLUSH"): flush.zero_()
    run = engine.run_device("warp", d_idx, offs[:-1], offs[1:], nb, len(mesh.indices), 96, cfg, None, spec, buffers=bufs, static=True)
torch.cuda.synchronize()
run.check()
lib = N.lib()
MARKS, TILES = 12, 8192
buf = (C.c_ulonglong * (MARKS * 2 * TILES))()
lib.vr_debug_timeline.restype = C.c_int
got = lib.vr_debug_timeline(buf, MARKS * 2 * TILES)
a = np.frombuffer(buf, dtype=np.uint64).reshape(MARKS, 2, TILES).astype(np.int64)
nt = (nb + 63) // 64
t0 = a[0, 0, :nt].min()
def stat(name, d):
    d = d.reshape(-1) / 1e3
    print(f"  {name:28s} median {np.median(d):7.2f}  p10 {np.percentile(d, 10):7.2f}  p90 {np.percentile(d, 90):7.2f}  mean {d.mean():7.2f} us")
d = a[:, 0, :nt]
t0 = d[1].min()
print(f"tiles {nt}; dedup warp 0 (iterations of the persistent CTAs that own a tile); span to last publish {(d[5].max() - t0) / 1e3:.1f} us")
for k, nm in ((1, "ticket -> rows staged (wait)"), (2, "dedup"), (3, "barrier"), (4, "post (scratch, next staging, indices, publish)")):
    stat(nm, d[k + 1] - d[k])
stat("iteration", d[5] - d[1])
h = a[:, 1, :]
lag = int(os.environ.get("VR_LAG", 888))
sel = np.arange(lag, nt)  # iterations whose helpers shade a tile
print("helper warp 2 (shading tile i - K)")
stat("look-back + shading", h[6, sel] - h[7, sel])
stat("  wait aggregate", h[8, sel] - h[7, sel])
stat("  ids, gathers, look-back", h[9, sel] - h[8, sel])
stat("  stores + further steps", h[10, sel] - h[9, sel])
stat("  round tables", h[6, sel] - h[10, sel])
hs = a[:, 1, :nt + lag]
ends = hs[6][hs[6] > 0]
print(f"last shading ends {(ends.max() - t0) / 1e3:.1f} us after the first ticket; tail after the last publish {(ends.max() - d[5].max()) / 1e3:.1f} us")
