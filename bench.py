#!/usr/bin/env python
"""bench.py -- triangles/s through the geometry stage (BASELINE.json metric).

Headline workload (N=1): BASELINE.json configs[2] -- gen_grid(1898,1898) (3.6 M vertices, 7.2 M
triangles, strip order), warp-voting strategy, BatchConfig() defaults (96-index static batches,
warp 32), FP32 4x4 position shader.  One step = one pass of the whole stage (batch ranges ->
dedup -> shade once per unique vertex -> local-index triangles -> statistics) over that mesh.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference] [--no-others]

The JSON line also carries, under "others", the other strategies north_star grades (dynamic batches + sort /
hash / two-tier hash on the strip-ordered and on the shuffled mesh, the 1000-draw scene, configs[0]), each with
its own roofline fraction and -- for dynamic batches -- the figure including batch formation.

N>1 (torchrun, one rank per GPU): `value` is weak scaling -- every rank runs one whole mesh (vertex buffer
replicated), the statistics blocks are merged with one all-gather per timed run on a side stream.  The "sharded"
block is strong scaling: ONE configs[2] / configs[3] stream cut into whole batches per rank
(paper_1805_08893_b200/shard.py), and the 1000-draw scene split by whole draws (LPT).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MATRIX = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]], dtype=np.float64)
METRIC = "triangles/sec through vertex stage"
UNIT = "triangles/s"

# name -> (description, grid side, shuffle seed or None, strategy, batching, expected totals)
WORKLOADS = {
    "c3_warp": dict(desc="configs[2]: gen_grid(1898,1898) strip order, warp voting, static 96 / warp 32",
                    side=1898, shuffle=None, strategy="warp", batching="static",
                    expect=dict(batches=224914, rounds=449827, invocations=8100190)),
    "c3_dyn_sort": dict(desc="configs[2] mesh, dynamic 256/1023 batches, sort dedup",
                        side=1898, shuffle=None, strategy="sort", batching="dynamic",
                        expect=dict(batches=28350, rounds=28350, invocations=7257500)),
    "c3_dyn_hash": dict(desc="configs[2] mesh, dynamic 256/1023 batches, hash 256",
                        side=1898, shuffle=None, strategy="hash", batching="dynamic",
                        expect=dict(batches=28350, rounds=28350, invocations=7257500)),
    "c4_hash": dict(desc="configs[3]: shuffle_triangles(gen_grid(1898,1898), 0), dynamic 256/1023, hash 256",
                    side=1898, shuffle=0, strategy="hash", batching="dynamic",
                    expect=dict(batches=84672, rounds=84672, invocations=21591005, probes_fast=216377586)),
    "c4_sort": dict(desc="configs[3] mesh, dynamic 256/1023, sort dedup",
                    side=1898, shuffle=0, strategy="sort", batching="dynamic",
                    expect=dict(batches=84672, rounds=84672, invocations=21591005)),
    "c4_phash": dict(desc="configs[3] mesh, dynamic 256/1023, two-tier hash 256",
                     side=1898, shuffle=0, strategy="phash", batching="dynamic",
                     expect=dict(batches=84672, rounds=84672, invocations=21591005)),
    "c1_sort": dict(desc="configs[0]: gen_grid(256,256), static 768, sort dedup (launch-latency bound)",
                    side=256, shuffle=None, strategy="sort", batching="static768",
                    expect=dict(batches=509, rounds=509, invocations=131574)),
}
OTHERS = ("c3_dyn_sort", "c3_dyn_hash", "c4_hash", "c4_sort", "c4_phash", "c1_sort")

# configs[4]: oracle totals of the 1000-draw scene (scripts/c5_expect.py; dynamic 256/1023 per draw)
C5_EXPECT = {
    "sort": dict(batches=154797, rounds=154797, invocations=39026006),
    "hash": dict(batches=154797, rounds=154797, invocations=39026006, probes_fast=328902576),
}


def algorithmic_bytes(n_idx, n_inv, n_batches):
    """SURVEY.md 8(d) / BASELINE.md section 3: uint32 index read + float4 position read and float4
    shaded write per invocation + uint16 local-index write + 12 B of batch metadata."""
    return 4 * n_idx + 16 * n_inv + 16 * n_inv + 2 * n_idx + 12 * n_batches


def hbm_peak():
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region (NVML)."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40,
                 "sw_thermal_slowdown": 0x20, "hw_power_brake": 0x80}
        while not self.stop:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.nv:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


_MESHES = {}


def build_mesh(wl):
    import paper_1805_08893_b200 as P
    key = (wl["side"], wl["shuffle"])
    if key not in _MESHES:
        base = (wl["side"], None)
        if base not in _MESHES:
            _MESHES[base] = P.gen_grid(wl["side"], wl["side"])
        _MESHES[key] = _MESHES[base] if wl["shuffle"] is None else P.shuffle_triangles(_MESHES[base], wl["shuffle"])
    return _MESHES[key]


def workload_cfg(wl):
    import paper_1805_08893_b200 as P
    if wl["batching"] == "static768":
        return P.BatchConfig(batch_size=768, max_unique=768, block_size=1024)
    return P.BatchConfig()


# ---------------------------------------------------------------------------------------------
# reference arm / cpu baseline.  Two CPU implementations are timed and labelled:
#   kind "port"       oracle/vr_oracle.c -- a C restatement of the reference's algorithm, run on all host
#                     threads (ctypes releases the GIL).  This is the line's `value`: the strongest CPU arm.
#   kind "reference"  the UNMODIFIED reference package (pure Python + NumPy, oracle/_ref, installed by
#                     oracle/install_ref.py) through its own run_on_indices(..., workers=1) with
#                     position_shader and vertex_count, on a bounded prefix of the same workload
#                     (SURVEY.md 8d).  Extra workers do not help it (GIL).
# ---------------------------------------------------------------------------------------------
def oracle_step(wl, mesh, cfg, offsets, threads):
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor

    nb = len(offsets) - 1
    cuts = np.linspace(0, nb, threads + 1).astype(np.int64)

    def work(t):
        lo, hi = int(cuts[t]), int(cuts[t + 1])
        if hi <= lo:
            return 0, 0
        fr = O.run(wl["strategy"], mesh.indices, offsets[lo:hi], offsets[lo + 1:hi + 1],
                   max_unique=cfg.max_unique, warp_width=cfg.warp_width, table_size=cfg.block_size)
        O.shade_positions(mesh.positions, fr.unique_ids, MATRIX)
        return fr.invocations, fr.rounds

    if threads == 1:
        res = [work(0)]
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:  # ctypes releases the GIL
            res = list(pool.map(work, range(threads)))
    return sum(r[0] for r in res), sum(r[1] for r in res)


def host_offsets(wl, mesh, cfg):
    import oracle as O
    if wl["batching"].startswith("static"):
        return O.static_batches(len(mesh.indices), batch_size=cfg.batch_size)
    return O.dynamic_batches(mesh.indices, max_unique=cfg.max_unique, max_indices=cfg.max_indices)


def cpu_baseline(wl, mesh, cfg, threads, steps=1, warmup=0):
    offsets = host_offsets(wl, mesh, cfg)
    for _ in range(warmup):
        oracle_step(wl, mesh, cfg, offsets, threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        inv, _ = oracle_step(wl, mesh, cfg, offsets, threads)
    dt = (time.perf_counter() - t0) / steps
    assert inv == wl["expect"]["invocations"], (inv, wl["expect"])
    tris = mesh.triangle_count
    return {"value": tris / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"full workload ({tris} triangles) per step, {dt:.2f} s/step, C port of the reference "
                      f"(oracle/vr_oracle.c: dedup + float64 shader), batch formation excluded"}, dt


def unmodified_reference(wl, mesh, cfg, sample_tris, reps=1):
    """The reference's own run_on_indices on a prefix of the workload (oracle/_ref; None if not installed)."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.exists(os.path.join(ref_dir, "vrlab", "strategies.py")):
        return None
    sys.path.insert(0, ref_dir)
    try:
        import vrlab
    except Exception as exc:  # e.g. NumPy missing on the host
        return {"unavailable": f"import vrlab failed: {exc}"}
    finally:
        sys.path.remove(ref_dir)
    n = min(sample_tris, mesh.triangle_count) * 3
    idx = mesh.indices[:n]
    rcfg = vrlab.BatchConfig(batch_size=cfg.batch_size, max_unique=cfg.max_unique, max_indices=cfg.max_indices,
                             warp_width=cfg.warp_width, block_size=cfg.block_size)
    rmesh = vrlab.IndexedMesh(positions=mesh.positions, indices=mesh.indices)
    shader = vrlab.position_shader(rmesh, MATRIX)
    best, t_form = None, 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        if wl["batching"].startswith("static"):
            batches = vrlab.static_batches(n, rcfg)
        else:
            batches = vrlab.dynamic_batches(idx, rcfg)
        t1 = time.perf_counter()
        out = vrlab.run_on_indices(wl["strategy"], idx, batches, rcfg, shader,
                                   vrlab.HashConfig(table_size=cfg.block_size), vertex_count=mesh.vertex_count, workers=1)
        t2 = time.perf_counter()
        if best is None or t2 - t1 < best:
            best, t_form = t2 - t1, t1 - t0
    rep = out[1]
    return {"value": (n // 3) / best, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"first {n // 3} triangles of the workload through vrlab.run_on_indices(workers=1) with "
                      f"position_shader + vertex_count: {best:.2f} s (+ {t_form:.2f} s batch formation), "
                      f"{rep.invocations} invocations; unmodified reference package (oracle/_ref), Python + NumPy, "
                      f"host has {os.cpu_count()} cores, extra workers do not help (GIL)"}


def run_reference_arm(args, wl_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[wl_name]
    mesh = build_mesh(wl)
    cfg = workload_cfg(wl)
    threads = max(1, min(os.cpu_count() or 1, 64))
    base, dt = cpu_baseline(wl, mesh, cfg, threads, steps=args.steps, warmup=min(args.warmup, 1))
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 ids, f64 shader (CPU)", "data": "synthetic",
            "config": {"workload": wl["desc"], "strategy": wl["strategy"]},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    # the unmodified reference next to the port: configs[0] in full and a 28 800-triangle prefix of this workload
    ref = unmodified_reference(wl, mesh, cfg, 28800)
    if ref is not None:
        line["unmodified_reference"] = ref
        c1 = WORKLOADS["c1_sort"]
        r1 = unmodified_reference(c1, build_mesh(c1), workload_cfg(c1), 10 ** 9)
        if r1 is not None:
            r1["workload"] = c1["desc"]
            line["unmodified_reference_configs0"] = r1
    print(json.dumps(line))


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c3_warp", choices=sorted(WORKLOADS))
    ap.add_argument("--others", action="store_true", help="(default) also time the other strategies / configs")
    ap.add_argument("--no-others", action="store_true", help="headline workload only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="run the strong-scaling (sharded) block also at N=1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args, args.workload)
        return

    import torch
    import torch.distributed as dist

    import paper_1805_08893_b200 as P
    from paper_1805_08893_b200 import _native as N
    from paper_1805_08893_b200 import engine, shard
    from paper_1805_08893_b200.strategies import HashConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # launched by torchrun (any world size)
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    lib = N.require_cuda()
    peak, peak_src = hbm_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    side = torch.cuda.Stream(device=dev)  # statistics all-gather, off the critical path

    def max_over_ranks(ms):
        if not distributed or world == 1:
            return ms
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if distributed and world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed_steps(fn, steps, after=None):
        """K steps, each bracketed by CUDA events on the launching stream, L2 flushed in between (outside the
        events).  Returns (sum of the per-step device times in ms -- max over ranks --, wall seconds)."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        wall0 = time.perf_counter()
        for k in range(steps):
            flush.zero_()  # evict the previous step's lines from L2
            evs[k][0].record()
            fn()
            if after is not None:
                after(k == steps - 1)
            evs[k][1].record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        barrier()
        return max_over_ranks(float(sum(a.elapsed_time(b) for a, b in evs))), wall

    def stage_profile(fn, reps):
        """Per-kernel device times of one vr_run, in a separate untimed-for-the-metric pass."""
        lib.vr_profile_enable(1)
        stage_ms = np.zeros(N.VR_PROFILE_STAGES)
        buf = (C.c_float * 8)()
        for _ in range(reps):
            flush.zero_()
            fn()
            n = lib.vr_profile_read(buf, 8)
            stage_ms[:n] += np.array(buf[:n])
        torch.cuda.synchronize()
        lib.vr_profile_enable(0)
        return stage_ms / reps

    def shaded_sample_check(run, mesh, stride=997):
        """Parity gate on the FP32 shader: a strided sample of the shaded vertices against float64 NumPy
        (strategies.py:53-67), rtol 1e-5."""
        inv = run.invocations
        uid = run.unique_ids[:inv:stride].cpu().numpy().view(np.uint32)
        got = run.shaded4[:inv:stride].cpu().numpy()
        p = np.hstack([mesh.positions[uid], np.ones((len(uid), 1))]) @ MATRIX.T
        np.testing.assert_allclose(got[:, :3], p[:, :3] / p[:, 3:4], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(got[:, 3], p[:, 3], rtol=1e-5)

    def run_workload(name, steps, warmup, full):
        wl = WORKLOADS[name]
        mesh = build_mesh(wl)
        cfg = workload_cfg(wl)
        hcfg = HashConfig(table_size=cfg.block_size)
        tris, n_idx = mesh.triangle_count, len(mesh.indices)
        static = wl["batching"].startswith("static")
        # --- inputs resident in HBM before the timed region
        d_idx = engine.to_device_indices(mesh.indices, dev)
        pos4 = engine.to_device_positions4(mesh.positions, dev)
        t_form = None
        if static:
            offs = engine.static_offsets_device(n_idx, cfg, dev)
        else:
            ws_form = torch.empty(lib.vr_dynamic_workspace_bytes(n_idx, C.byref(engine._cfg_c(cfg))),
                                  dtype=torch.uint8, device=dev)
            offs = engine.dynamic_offsets_device(d_idx, cfg, workspace=ws_form)  # warm-up
        nb = offs.numel() - 1
        max_span = cfg.batch_size if static else max(cfg.batch_size, cfg.max_indices)
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=MATRIX,
                                 vertex_count=mesh.vertex_count)
        bufs = engine.RunBuffers()
        # buffers and arguments are prepared once; a step is one vr_run call (the host must not be what
        # the CUDA events around a 0.12 ms step measure)
        plan = engine.run_device(wl["strategy"], d_idx, offs[:-1], offs[1:], nb, n_idx, max_span, cfg,
                                 hcfg, spec, buffers=bufs, static=static, plan_only=True)
        step = plan.relaunch
        for _ in range(warmup):
            run = step()
        run.check()
        exp = wl["expect"]
        got = dict(batches=nb, rounds=run.rounds, invocations=run.invocations)
        if "probes_fast" in exp:
            got["probes_fast"] = run.probes[0]
        assert got == exp, f"parity gate failed: {got} != {exp}"
        shaded_sample_check(run, mesh)
        run._stats = None
        holder = {}

        def gather(last):
            # N>1: the ranks' 16-word statistics blocks are exchanged ONCE per timed run (one all-gather, inside the
            # last step's events): the path has no data-path collective, and a collective per
            # 0.12 ms step would measure the host's enqueue cost of the NCCL call (~0.1 ms), not the stage
            if not distributed or not last:
                return
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(side):
                side.wait_event(ev)
                holder["blocks"] = shard.gather_stats(plan.stats_dev)  # merged on the host after the loop
            if last:
                torch.cuda.current_stream().wait_stream(side)

        with ClockSampler(local) as clocks:
            total_ms, wall = timed_steps(step, steps, gather)
            # the same loop for >= 0.25 s so that the clock sampler sees the kernel under sustained load
            sus_steps = int(min(5000, max(steps, 250.0 / max(total_ms / steps + 0.05, 1e-3)))) if full else 0
            sus_ms = timed_steps(step, sus_steps)[0] if sus_steps else None
        stage_ms = stage_profile(step, max(3, min(steps, 20)))
        ms_per_step = total_ms / steps
        value = world * tris * steps / (total_ms * 1e-3)
        inv = run.check().invocations
        if distributed and "blocks" in holder:
            assert int(shard.merge_stats(holder["blocks"])[N.VR_STAT_INVOCATIONS]) == world * inv
        alg = algorithmic_bytes(n_idx, inv, nb)
        launches = lib.vr_last_launch_count()
        path = lib.vr_last_kernel_path()
        fused = path in (2, 3)  # init + one kernel that dedups, places and shades (4 = the three-kernel sort/hash path)
        dom = int(np.argmax(stage_ms))
        # per-kernel algorithmic bytes: dedup = index read + map write + metadata;
        # shade/finalize = staged id read is not algorithmic: position read + shaded write
        kernel_alg = {"dedup": 4 * n_idx + 2 * n_idx + 12 * nb, "shade_finalize": 32 * inv}
        dom_name = (N.KERNEL_PATH_NAMES.get(path) if fused else None) or N.PROFILE_STAGE_NAMES[dom]
        if path == 4:  # vr_dyn3.cuh: A (+ B) are timed as 'dedup', C as 'shade_finalize'
            dom_name = {"dedup": "dyn3 A: set dedup + offset sums (+ B: table replay)",
                        "shade_finalize": "dyn3 C: ranks + local indices + shading"}.get(N.PROFILE_STAGE_NAMES[dom], dom_name)
        traffic = None  # DRAM bytes per step of the dominant kernel, from the committed ncu --set full capture
        for tf in ("r2_traffic.json", "r1_traffic.json"):
            try:
                tj = json.load(open(os.path.join(ROOT, "profiles", tf)))
                ent = tj.get(name) if isinstance(tj.get(name), dict) else (tj if tj.get("workload") == name else None)
                if ent and fused:
                    traffic = ent["traffic_bytes_per_step"]
                    break
            except Exception:
                pass
        dom_alg = alg if fused else kernel_alg.get(N.PROFILE_STAGE_NAMES[dom], alg)
        res = {
            "value": value, "ms_per_step": ms_per_step, "wall_s": wall,
            "stage_ms": {N.PROFILE_STAGE_NAMES[i]: round(float(stage_ms[i]), 5) for i in range(N.VR_PROFILE_STAGES)},
            "roofline": {"bound": "hbm", "kernel": dom_name,
                         "achieved": dom_alg / (stage_ms[dom] * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": dom_alg / (stage_ms[dom] * 1e-3) / 1e9 / peak, "traffic": traffic,
                         "peak_source": peak_src, "algorithmic_bytes": dom_alg,
                         "share_of_step": float(stage_ms[dom] / max(ms_per_step, 1e-9))},
            "stage_roofline": {"algorithmic_bytes": alg, "bytes_per_triangle": alg / tris,
                               "achieved": alg / (ms_per_step * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                               "frac": alg / (ms_per_step * 1e-3) / 1e9 / peak},
            "invocations": inv, "shading_rate": inv / mesh.vertex_count, "reuse_rate": 1 - inv / n_idx,
            "batches": nb, "clocks": clocks.summary(), "kernel_path": path,
            "gpu_launches": steps * launches, "launches_per_step": launches, "fused": fused,
        }
        if sus_steps:
            res["sustained"] = {"steps": sus_steps, "ms_per_step": sus_ms / sus_steps,
                                "value": world * tris * sus_steps / (sus_ms * 1e-3)}
        if not static:
            # batch formation on the device (batching.py:87-125), and the stage including it: one more 4*I read
            form = lambda: engine.dynamic_offsets_device(d_idx, cfg, workspace=ws_form)
            f_steps = max(5, min(steps, 20))
            t_form = timed_steps(form, f_steps)[0] / f_steps

            def whole():  # no host round trip: the batch count stays on the device (vr_run_counted)
                o, cnt = engine.dynamic_offsets_device(d_idx, cfg, workspace=ws_form, sync=False)
                return engine.run_device(wl["strategy"], d_idx, None, None, 0, 0, max_span, cfg, hcfg, spec, buffers=bufs,
                                         counted=(o, cnt))
            chk = whole().check()
            assert (chk.n_batches, chk.invocations) == (nb, inv), "formation + stage without the host in between differs"
            whole()
            t_whole = timed_steps(whole, f_steps)[0] / f_steps
            alg_w = alg + 4 * n_idx
            res["batch_formation_ms"] = t_form
            res["incl_batch_formation"] = {"ms_per_step": t_whole, "value": world * tris / (t_whole * 1e-3),
                                           "algorithmic_bytes": alg_w, "frac": alg_w / (t_whole * 1e-3) / 1e9 / peak}
        if name in ("c3_warp", "c4_sort"):
            # the paper's stage output is the expanded per-corner queue (strategies.py:456-463), written
            # by the stage itself (kernel C of the sort/hash path) or by vr_run's closing kernel (tile kernel path),
            # with the queue in the denominator: + 12 B float32[3] record written per corner (and, for the closing
            # kernel, 2 B local index + 16 B record read)
            qplan = engine.run_device(wl["strategy"], d_idx, offs[:-1], offs[1:], nb, n_idx, max_span, cfg, hcfg, spec,
                                      buffers=engine.RunBuffers(), static=static, want_queue=True, plan_only=True)
            with_queue = qplan.relaunch  # the queue is an output of vr_run (vr_outputs.d_stream_xyz)
            with_queue().check()
            q_steps = max(5, min(steps, 20))
            t_q = timed_steps(with_queue, q_steps)[0] / q_steps
            alg_q = alg + n_idx * 12
            res["expanded_queue"] = {"ms_per_step": t_q, "value": world * tris / (t_q * 1e-3), "algorithmic_bytes": alg_q,
                                     "frac": alg_q / (t_q * 1e-3) / 1e9 / peak,
                                     "launches_per_step": lib.vr_last_launch_count(),
                                     "note": "stage incl. the per-corner record queue (float32[3] per corner, vr_outputs.d_stream_xyz)"}
        if not full:
            return res, None
        return res, run_e2e(wl, mesh, cfg, hcfg, offs, nb, max_span, static, inv, steps)

    def run_e2e(wl, mesh, cfg, hcfg, offs, nb, max_span, static, inv, steps):
        """End to end through host buffers, the way run_on_indices is used: every step copies the index buffer and
        the vertex buffer in from pinned host memory and copies the WHOLE result back (shaded vertices, unique
        ids, local-index triangles, round tables, statistics).  Three streams, two slots: the copy-in of step
        k+1 and the copy-out of step k-1 overlap the kernels of step k.  Result sizes are read from each step's
        statistics block (what DeviceRun.flat() does), so exactly the result crosses PCIe."""
        tris, n_idx, V = mesh.triangle_count, len(mesh.indices), mesh.vertex_count
        h_idx = torch.from_numpy(mesh.indices.view(np.int32).copy()).pin_memory()
        # the vertex buffer crosses PCIe as 3 floats per vertex and is packed to the float4 gather layout on
        # the device (what engine.to_device_positions4 does for any caller)
        h_pos = torch.from_numpy(np.ascontiguousarray(mesh.positions, dtype=np.float32)).pin_memory()
        s_in, s_run, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
        slots = []
        for j in range(2):
            d_idx = torch.empty(n_idx, dtype=torch.int32, device=dev)
            d_pos3 = torch.empty((V, 3), dtype=torch.float32, device=dev)
            p4 = torch.ones((V, 4), dtype=torch.float32, device=dev)
            spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=p4, matrix=MATRIX, vertex_count=V)
            plan = engine.run_device(wl["strategy"], d_idx, offs[:-1], offs[1:], nb, n_idx, max_span, cfg, hcfg, spec,
                                     buffers=engine.RunBuffers(), static=static, plan_only=True)
            slots.append(dict(d_idx=d_idx, d_pos3=d_pos3, p4=p4, plan=plan,
                              h_stats=torch.zeros(N.VR_STATS_WORDS, dtype=torch.int64).pin_memory(),
                              ev_in=torch.cuda.Event(), ev_run=torch.cuda.Event(), ev_out=torch.cuda.Event()))
        rounds_cap = int(slots[0]["plan"].round_prims.numel())
        inv_cap = int(inv * 1.05) + 1024
        for s in slots:  # the records cross PCIe in the reference's layout (float32[3]), packed on the device
            s["xyz"] = torch.empty((inv_cap, 3), dtype=torch.float32, device=dev)
            s["map8"] = torch.empty(n_idx + 16, dtype=torch.uint8, device=dev)  # ... and the local indices as bytes
            s["flag"] = torch.zeros(1, dtype=torch.int32, device=dev)
        host = dict(shaded=torch.empty((inv_cap, 3), dtype=torch.float32).pin_memory(),
                    uid=torch.empty(inv_cap, dtype=torch.int32).pin_memory(),
                    amap=torch.empty(n_idx, dtype=torch.uint8).pin_memory(), flag=torch.zeros(1, dtype=torch.int32).pin_memory(),
                    bro=torch.empty(nb + 1, dtype=torch.int32).pin_memory(),
                    ruo=torch.empty(rounds_cap + 1, dtype=torch.int32).pin_memory(),
                    rp=torch.empty(rounds_cap, dtype=torch.int32).pin_memory())
        d2h = [0]

        def copy_in_and_run(j):
            s = slots[j]
            with torch.cuda.stream(s_in):
                s_in.wait_event(s["ev_run"])  # the run that last read this input slot is done
                s["d_idx"].copy_(h_idx, non_blocking=True)
                s["d_pos3"].copy_(h_pos, non_blocking=True)
                s["ev_in"].record()
            with torch.cuda.stream(s_run):
                s_run.wait_event(s["ev_in"])
                s_run.wait_event(s["ev_out"])  # the previous result of this slot has left the device
                s["p4"][:, :3].copy_(s["d_pos3"])
                s["plan"].relaunch()
                s["h_stats"].copy_(s["plan"].stats_dev, non_blocking=True)
                s["ev_run"].record()

        def copy_out(j, full_result):
            s = slots[j]
            s["ev_run"].synchronize()  # host needs the result sizes (128 bytes) before it can size the copies
            st = s["h_stats"]
            assert int(st[N.VR_STAT_ERROR]) == -1 and int(st[N.VR_STAT_INVOCATIONS]) == inv
            u, r, m = int(st[N.VR_STAT_INVOCATIONS]), int(st[N.VR_STAT_ROUNDS]), int(st[N.VR_STAT_INDICES])
            d2h[0] = N.VR_STATS_WORDS * 8
            if not full_result:
                return
            p = s["plan"]
            with torch.cuda.stream(s_out):
                s_out.wait_event(s["ev_run"])
                host["shaded"][:u].copy_(p.shaded_xyz(u, s["xyz"]), non_blocking=True)
                host["uid"][:u].copy_(p.unique_ids[:u], non_blocking=True)
                host["amap"][:m].copy_(p.assembly_map_u8(m, s["map8"], s["flag"]), non_blocking=True)
                host["flag"].copy_(s["flag"], non_blocking=True)
                host["bro"].copy_(p.batch_round_off[:nb + 1], non_blocking=True)
                host["ruo"][:r + 1].copy_(p.round_uid_off[:r + 1], non_blocking=True)
                host["rp"][:r].copy_(p.round_prims[:r], non_blocking=True)
                s["ev_out"].record()
            d2h[0] += u * 12 + u * 4 + m * 1 + 4 + (nb + 1) * 4 + (r + 1) * 4 + r * 4

        def loop(k_steps, full_result):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            with torch.cuda.stream(s_in):
                e0.record()
            for k in range(k_steps + 1):
                if k < k_steps:
                    copy_in_and_run(k % 2)
                if k >= 1:
                    copy_out((k - 1) % 2, full_result)
            with torch.cuda.stream(s_out):
                s_out.wait_stream(s_run)
                e1.record()
            torch.cuda.synchronize()
            barrier()
            return max_over_ranks(e0.elapsed_time(e1))

        e2e_steps = max(5, min(steps, 20))
        out = {}
        for label, full_result in (("full_result", True), ("stats_only", False)):
            loop(3, full_result)
            ms = loop(e2e_steps, full_result)
            out[label] = {"value": world * tris * e2e_steps / (ms * 1e-3), "ms_per_step": ms / e2e_steps,
                          "d2h_bytes_per_step": int(d2h[0])}
        # the result that came back is the result: spot-check the host copies of the last full step
        uid = host["uid"][:inv:997].numpy().view(np.uint32)
        p = np.hstack([mesh.positions[uid], np.ones((len(uid), 1))]) @ MATRIX.T
        # (the last loop was stats-only, the host buffers still hold the last full-result step)
        np.testing.assert_allclose(host["shaded"][:inv:997, :3].numpy(), p[:, :3] / p[:, 3:4], rtol=1e-5, atol=1e-5)
        assert int(host["flag"][0]) == 0, "a local index did not fit a byte"
        return {"value": out["full_result"]["value"], "unit": UNIT,
                "h2d_bytes_per_step": int(h_idx.numel() * 4 + h_pos.numel() * 4),
                "d2h_bytes_per_step": out["full_result"]["d2h_bytes_per_step"], "steps": e2e_steps,
                "ms_per_step": out["full_result"]["ms_per_step"],
                "stats_only": out["stats_only"],
                "note": "pinned host index buffer (uint32) + vertex buffer (3 x fp32, packed to float4 on the device) copied in "
                        "every step; offsets resident; the whole result copied back to pinned host memory every step (shaded "
                        "vertices as the reference's float32[3] records and local-index triangles as bytes, both packed on the device; unique ids, round tables, statistics); copy-in, "
                        "kernels and copy-out of consecutive steps overlap on three streams (two device slots); "
                        "'stats_only' = same loop with only the 128-byte statistics block read back"}

    def run_multidraw(strategy, steps, warmup):
        """BASELINE.json configs[4]: 1000 draws, 20.4 M triangles, dynamic 256/1023 batches per
        draw, packed into one stream (paper_1805_08893_b200/draws.py).  Two figures: dedup + shade with the
        offsets precomputed (as the paper reports dynamic batching), and including batch formation."""
        from paper_1805_08893_b200 import draws as D
        cfg = P.BatchConfig()
        hcfg = HashConfig(table_size=cfg.block_size)
        meshes = D.scene_corpus(1000)
        if world > 1:  # whole draws per rank, LPT (shard.py)
            mine = shard.lpt_assign([m.triangle_count for m in meshes], world)[rank]
            meshes_r = [meshes[int(d)] for d in mine]
        else:
            meshes_r = meshes
        ds = D.pack_draws(meshes_r, dev)
        tris_all = sum(m.triangle_count for m in meshes)
        bufs = engine.RunBuffers()
        ws = torch.empty(lib.vr_dynamic_workspace_bytes(ds.indices.numel(), C.byref(engine._cfg_c(cfg))),
                         dtype=torch.uint8, device=dev)
        offs = D.dynamic_offsets_draws(ds, cfg, ws)
        vbase = D.batch_vertex_base(ds, offs)
        nb = offs.numel() - 1
        exp = C5_EXPECT[strategy]
        for _ in range(max(warmup, 1)):
            run = D.run_draws(strategy, ds, offs, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vbase)
        run.check()
        tot = shard.reduce_stats(run.stats_dev).cpu().numpy()
        got = dict(rounds=int(tot[N.VR_STAT_ROUNDS]), invocations=int(tot[N.VR_STAT_INVOCATIONS]),
                   batches=int(tot[N.VR_STAT_BATCHES]))
        if strategy == "hash":
            got["probes_fast"] = int(tot[N.VR_STAT_PROBES_FAST])
        assert got == exp, f"parity gate failed: {got} != {exp}"
        ms_run = timed_steps(lambda: D.run_draws(strategy, ds, offs, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vbase),
                             steps)[0] / steps

        def whole():
            o = D.dynamic_offsets_draws(ds, cfg, ws)
            vb = D.batch_vertex_base(ds, o, vbase)
            D.run_draws(strategy, ds, o, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vb)
        whole()
        ms_whole = timed_steps(whole, steps)[0] / steps
        inv = got["invocations"]
        n_idx_all = 3 * tris_all
        alg = algorithmic_bytes(n_idx_all, inv, got["batches"])
        return {"value": tris_all / (ms_run * 1e-3), "ms_per_step": ms_run,
                "value_incl_batch_formation": tris_all / (ms_whole * 1e-3), "ms_incl_batch_formation": ms_whole,
                "draws": len(meshes), "triangles": tris_all, "batches": got["batches"],
                "invocations": inv, "reuse_rate": 1 - inv / n_idx_all, "scaling": "strong" if world > 1 else None,
                "sharding": f"{world} ranks x whole draws (LPT)" if world > 1 else "one GPU",
                "stage_roofline": {"algorithmic_bytes": alg, "frac": alg / (ms_run * 1e-3) / 1e9 / (peak * world)},
                "incl_batch_formation_frac": (alg + 4 * n_idx_all) / (ms_whole * 1e-3) / 1e9 / (peak * world),
                "gpu_launches": steps * lib.vr_last_launch_count()}

    def run_sharded_stream(name, steps, warmup):
        """Strong scaling: ONE stream of the workload cut into whole batches per rank (shard.run_sharded); the
        full index stream and the vertex buffer are replicated, every rank dedups and shades its slice, the
        statistics blocks are merged by one all-gather.  Dynamic batches: reported with the offsets precomputed, and
        including batch formation -- by the boundary exchange (every rank scans its own range, one all-gather of
        small tables: SURVEY.md 8e option (ii)) and by the redundant whole-stream scan (option (i))."""
        wl = WORKLOADS[name]
        mesh = build_mesh(wl)
        cfg = workload_cfg(wl)
        hcfg = HashConfig(table_size=cfg.block_size)
        static = wl["batching"].startswith("static")
        d_idx = engine.to_device_indices(mesh.indices, dev)
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=engine.to_device_positions4(mesh.positions, dev),
                                 matrix=MATRIX, vertex_count=mesh.vertex_count)
        bufs = engine.RunBuffers()
        offs = None if static else engine.dynamic_offsets_device(d_idx, cfg)
        plan_run, plan = shard.run_sharded(wl["strategy"], d_idx, cfg, hcfg, spec, batching="static" if static else "offsets",
                                           offsets=offs, rank=rank, world=world, buffers=bufs, plan_only=True)
        step = plan_run.relaunch if plan_run is not None else (lambda: None)
        for _ in range(warmup):
            step()
        tot = shard.global_stats(plan_run, plan, device=dev).cpu().numpy()
        exp = wl["expect"]
        got = dict(batches=int(tot[N.VR_STAT_BATCHES]), rounds=int(tot[N.VR_STAT_ROUNDS]),
                   invocations=int(tot[N.VR_STAT_INVOCATIONS]))
        if "probes_fast" in exp:
            got["probes_fast"] = int(tot[N.VR_STAT_PROBES_FAST])
        assert got == exp and int(tot[N.VR_STAT_ERROR]) == -1, f"sharded parity gate failed: {got} != {exp}"
        ms = timed_steps(step, steps)[0] / steps
        tris = mesh.triangle_count
        alg = algorithmic_bytes(len(mesh.indices), got["invocations"], got["batches"])
        res = {"workload": wl["desc"], "scaling": "strong", "value": tris / (ms * 1e-3), "ms_per_step": ms,
               "batches_per_rank": plan.n_batches, "frac_of_n_x_peak": alg / (ms * 1e-3) / 1e9 / (peak * world)}
        if not static:
            f_steps = max(5, min(steps, 20))
            for label, mode in (("incl_boundary_exchange", "exchange"), ("incl_redundant_boundary_scan", "dynamic")):
                # batch formation inside the step: "exchange" = every rank scans its own range, one all-gather of
                # 2.7 KB tables (SURVEY.md 8e option (ii)); "dynamic" = every rank scans the whole stream (option (i))
                def whole():
                    shard.run_sharded(wl["strategy"], d_idx, cfg, hcfg, spec, batching=mode, rank=rank, world=world, buffers=bufs)
                whole()
                ms_w = timed_steps(whole, f_steps)[0] / f_steps
                res[label] = {"ms_per_step": ms_w, "value": tris / (ms_w * 1e-3),
                              "frac_of_n_x_peak": (alg + 4 * len(mesh.indices)) / (ms_w * 1e-3) / 1e9 / (peak * world)}
        return res

    def run_shader_load(steps, warmup):
        """PAPER.md:661 / :696-714: where reuse pays.  The stage on the configs[2] mesh with a synthetic shader load of
        0 / 256 / 1024 dependent FMAs per invocation: no reuse (naive, 3 invocations per triangle) against static
        warp-voting batches and dynamic sort batches."""
        wl = WORKLOADS["c3_warp"]
        mesh = build_mesh(wl)
        cfg = P.BatchConfig()
        hcfg = HashConfig(table_size=cfg.block_size)
        n_idx = len(mesh.indices)
        d_idx = engine.to_device_indices(mesh.indices, dev)
        pos4 = engine.to_device_positions4(mesh.positions, dev)
        stat = engine.static_offsets_device(n_idx, cfg, dev)
        dyn = engine.dynamic_offsets_device(d_idx, cfg)
        out = {}
        for cycles in (0, 256, 1024):
            spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=MATRIX,
                                     vertex_count=mesh.vertex_count, extra_cycles=cycles)
            row = {}
            for strat, offs, static in (("naive", stat, True), ("warp", stat, True), ("sort", dyn, False)):
                nb = offs.numel() - 1
                plan = engine.run_device(strat, d_idx, offs[:-1], offs[1:], nb, n_idx,
                                         cfg.batch_size if static else max(cfg.batch_size, cfg.max_indices), cfg, hcfg, spec,
                                         buffers=engine.RunBuffers(), static=static, plan_only=True)
                for _ in range(warmup):
                    run = plan.relaunch()
                run.check()
                ms = timed_steps(plan.relaunch, steps)[0] / steps
                row[strat] = {"ms_per_step": ms, "value": mesh.triangle_count / (ms * 1e-3), "invocations": run.invocations}
            row["speedup_warp_vs_naive"] = row["naive"]["ms_per_step"] / row["warp"]["ms_per_step"]
            row["speedup_sort_vs_naive"] = row["naive"]["ms_per_step"] / row["sort"]["ms_per_step"]
            out[f"cycles_{cycles}"] = row
        return out

    def run_clients(steps):
        """SURVEY.md 8f rows on the device: ideal counts and the LRU cache model on the configs[2] mesh, one step of the
        random-walk client (walk.py defaults: 300 000 agents, 256 x 256 grid, radius 16, 8 moves kept)."""
        from paper_1805_08893_b200 import walk as W
        mesh = build_mesh(WORKLOADS["c3_warp"])
        d_idx = engine.to_device_indices(mesh.indices, dev)
        out = {}
        ms = timed_steps(lambda: engine.ideal_counts(d_idx, mesh.vertex_count), 5)[0] / 5
        referenced, _ = engine.ideal_counts(d_idx, mesh.vertex_count)
        out["ideal_report"] = {"ms": ms, "invocations": referenced, "reuse_rate": 1 - referenced / len(mesh.indices)}
        t0 = time.perf_counter()
        rep = P.simulate_parallel_cache(d_idx, P.CacheConfig())
        out["lru_cache_28x1024x256"] = {"wall_s": time.perf_counter() - t0, "hit_rate": rep.hit_rate, "misses": rep.misses}
        wcfg = W.WalkConfig(steps=1)
        pos = W._to_device_positions(W.initial_positions(wcfg))
        bcfg = P.BatchConfig(primitive_size=1, batch_size=576)
        for strat in ("sort", "hash"):
            W._step_device(pos, wcfg, 0, strat, bcfg, None, "walk")  # warm-up
            t = timed_steps(lambda: W._step_device(pos, wcfg, 0, strat, bcfg, None, "walk"), 5)[0] / 5
            _, rep = W._step_device(pos, wcfg, 0, strat, bcfg, None, "walk")
            out[f"walk_step_{strat}"] = {"ms": t, "agents": wcfg.agents, "evaluations": rep.invocations,
                                         "reuse_rate": rep.reuse_rate, "agents_per_s": wcfg.agents / (t * 1e-3)}
        d_cells = W._pack_device(pos)
        t = timed_steps(lambda: W._likelihoods_device(d_cells, wcfg), 3)[0] / 3
        out["walk_step_no_reuse_likelihoods_ms"] = t
        return out

    res, e2e = run_workload(args.workload, args.steps, args.warmup, True)
    others = {}
    if not args.no_others:
        o_steps = max(10, min(args.steps, 20))
        for name in OTHERS:
            if name != args.workload:
                others[name] = run_workload(name, o_steps, args.warmup, False)[0]
        for strat in ("sort", "hash"):
            others[f"c5_multidraw_{strat}"] = run_multidraw(strat, o_steps, args.warmup)
        if world == 1:
            others["shader_load"] = run_shader_load(max(5, min(args.steps, 10)), args.warmup)
            others["clients"] = run_clients(5)
    sharded = {}
    if world > 1 or args.sharded:
        s_steps = max(10, min(args.steps, 20))
        for name in ("c3_warp", "c4_hash", "c4_sort"):
            sharded[name] = run_sharded_stream(name, s_steps, args.warmup)
    wl = WORKLOADS[args.workload]
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 ids / fp32 positions", "data": "synthetic",
        "config": {"workload": wl["desc"], "strategy": wl["strategy"],
                   "l2": "flushed between steps (256 MiB memset outside the per-step CUDA events); "
                   "step working set 391 MB > 126 MB L2", "sharding": f"{world} x one mesh per GPU, vertex buffer replicated"},
        "roofline": res["roofline"], "stage_roofline": res["stage_roofline"], "stage_ms": res["stage_ms"],
        "e2e": e2e, "gpu_launches": res["gpu_launches"], "clocks": res["clocks"], "sustained": res.get("sustained"),
        "shading_rate": res["shading_rate"], "reuse_rate": res["reuse_rate"], "invocations": res["invocations"],
        "batches": res["batches"], "batch_formation_ms": res.get("batch_formation_ms"),
        "kernel_path": res["kernel_path"], "expanded_queue": res.get("expanded_queue"),
    }
    if others:
        line["others"] = others
    if sharded:
        line["sharded"] = sharded
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mesh = build_mesh(wl)
        base, _ = cpu_baseline(wl, mesh, workload_cfg(wl), 1)
        line["cpu_baseline"] = base
        ref = unmodified_reference(wl, mesh, workload_cfg(wl), 28800)
        if ref is not None:
            line["cpu_baseline_unmodified_reference"] = ref
    if rank == 0:
        print(json.dumps(line))
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
