#!/usr/bin/env python
"""bench.py -- triangles/s through the geometry stage (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[2] -- gen_grid(1898,1898) (3.6 M vertices, 7.2 M
triangles, strip order), warp-voting strategy, BatchConfig() defaults (96-index static batches,
warp 32), FP32 4x4 position shader.  One step = one pass of the whole stage (batch ranges ->
dedup -> shade once per unique vertex -> local-index triangles -> statistics) over that mesh.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

N>1 (torchrun, one rank per GPU): weak scaling -- every rank owns one whole draw of the workload
(its contiguous shard of an N-draw index stream), the vertex buffer is replicated, and the only
collective is the NCCL reduction of the statistics block after each step.
"""
from __future__ import annotations

import argparse
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
    "c3_dyn_sort": dict(desc="configs[2] mesh, dynamic 256/1023 batches (precomputed), sort dedup",
                        side=1898, shuffle=None, strategy="sort", batching="dynamic",
                        expect=dict(batches=28350, rounds=28350, invocations=7257500)),
    "c4_hash": dict(desc="configs[3]: shuffle_triangles(gen_grid(1898,1898), 0), dynamic 256/1023, hash 256",
                    side=1898, shuffle=0, strategy="hash", batching="dynamic",
                    expect=dict(batches=84672, rounds=84672, invocations=21591005, probes_fast=216377586)),
    "c4_phash": dict(desc="configs[3] mesh, dynamic 256/1023, two-tier hash 256 (elements replayed in the reference's order, probes of an element in parallel)",
                     side=1898, shuffle=0, strategy="phash", batching="dynamic",
                     expect=dict(batches=84672, rounds=84672, invocations=21591005)),
    "c4_sort": dict(desc="configs[3] mesh, dynamic 256/1023, sort dedup",
                    side=1898, shuffle=0, strategy="sort", batching="dynamic",
                    expect=dict(batches=84672, rounds=84672, invocations=21591005)),
    "c1_sort": dict(desc="configs[0]: gen_grid(256,256), static 768, sort dedup (launch-latency bound)",
                    side=256, shuffle=None, strategy="sort", batching="static768",
                    expect=dict(batches=509, rounds=509, invocations=131574)),
}


# configs[4]: oracle totals of the 1000-draw scene (scripts/c5_expect.py; dynamic 256/1023 per draw)
C5_EXPECT = {
    "sort": dict(batches=154797, rounds=154797, invocations=39026006),
    "hash": dict(batches=154797, rounds=154797, invocations=39026006, probes_fast=328902576),
}


def algorithmic_bytes(n_idx, n_inv, n_batches):
    """SURVEY.md 8(d) / BASELINE.md section 3: uint32 index read + float4 position read and float4
    shaded write per invocation + uint16 local-index write + 12 B of batch metadata."""
    return 4 * n_idx + 16 * n_inv + 16 * n_inv + 2 * n_idx + 12 * n_batches


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


def build_mesh(wl):
    import paper_1805_08893_b200 as P
    mesh = P.gen_grid(wl["side"], wl["side"])
    if wl["shuffle"] is not None:
        mesh = P.shuffle_triangles(mesh, wl["shuffle"])
    return mesh


def workload_cfg(wl):
    import paper_1805_08893_b200 as P
    if wl["batching"] == "static768":
        return P.BatchConfig(batch_size=768, max_unique=768, block_size=1024)
    return P.BatchConfig()


# ---------------------------------------------------------------------------------------------
# reference arm / cpu baseline: the CPU oracle (a C port of the reference's algorithm; the
# reference itself is pure Python and does not travel to the GPU box)
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
    ap.add_argument("--others", action="store_true", help="also time the other workloads (reported under 'others')")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = N.require_cuda()

    def run_workload(name, steps, warmup, full):
        wl = WORKLOADS[name]
        mesh = build_mesh(wl)
        cfg = workload_cfg(wl)
        hcfg = HashConfig(table_size=cfg.block_size)
        tris, n_idx = mesh.triangle_count, len(mesh.indices)
        # --- inputs resident in HBM before the timed region
        d_idx = engine.to_device_indices(mesh.indices, dev)
        pos4 = engine.to_device_positions4(mesh.positions, dev)
        t_form = None
        if wl["batching"].startswith("static"):
            offs = engine.static_offsets_device(n_idx, cfg, dev)
        else:
            engine.dynamic_offsets_device(d_idx, cfg)  # warm-up
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            offs = engine.dynamic_offsets_device(d_idx, cfg)
            e1.record()
            torch.cuda.synchronize()
            t_form = e0.elapsed_time(e1)
        nb = offs.numel() - 1
        max_span = max(cfg.batch_size, cfg.max_indices) if wl["batching"] == "dynamic" else cfg.batch_size
        spec = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos4, matrix=MATRIX,
                                 vertex_count=mesh.vertex_count)
        bufs = engine.RunBuffers()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

        # buffers and arguments are prepared once; a step is one vr_run call (the host must not be what
        # the CUDA events around a 0.12 ms step measure)
        plan = engine.run_device(wl["strategy"], d_idx, offs[:-1], offs[1:], nb, n_idx, max_span, cfg,
                                 hcfg, spec, buffers=bufs, static=wl["batching"].startswith("static"), plan_only=True)

        def step():
            return plan.relaunch()

        for _ in range(warmup):
            run = step()
        run.check()
        exp = wl["expect"]
        got = dict(batches=nb, rounds=run.rounds, invocations=run.invocations)
        if "probes_fast" in exp:
            got["probes_fast"] = run.probes[0]
        assert got == exp, f"parity gate failed: {got} != {exp}"
        run._stats = None

        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            wall0 = time.perf_counter()
            for k in range(steps):
                flush.zero_()  # evict the previous step's lines from L2 (outside the event pair)
                evs[k][0].record()
                run = step()
                if world > 1:
                    run.reduced = shard.reduce_stats(run.stats_dev)
                evs[k][1].record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - wall0
        if world > 1:
            dist.barrier()
        # per-kernel times in a second, untimed-for-the-metric pass: the extra CUDA events between the
        # kernels of one vr_run are measurement overhead and stay out of `value`
        lib.vr_profile_enable(1)
        stage_ms = np.zeros(N.VR_PROFILE_STAGES)
        buf = (C.c_float * 8)()
        prof_steps = max(3, min(steps, 20))
        for k in range(prof_steps):
            flush.zero_()
            run = step()
            n = lib.vr_profile_read(buf, 8)
            stage_ms[:n] += np.array(buf[:n])
        torch.cuda.synchronize()
        lib.vr_profile_enable(0)
        step_ms = np.array([a.elapsed_time(b) for a, b in evs])
        total_ms = float(step_ms.sum())
        if world > 1:
            t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        stage_ms /= prof_steps
        ms_per_step = total_ms / steps
        value = world * tris * steps / (total_ms * 1e-3)
        inv = run.check().invocations
        alg = algorithmic_bytes(n_idx, inv, nb)
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak, peak_src = (peaks["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)") if "hbm_gbs" in peaks \
            else (6650.0, "fallback (B200_PROFILING.md)")
        launches = lib.vr_last_launch_count()
        path = lib.vr_last_kernel_path()
        fused = path >= 2  # init + one kernel that dedups, places and shades
        dom = int(np.argmax(stage_ms))
        # per-kernel algorithmic bytes: dedup = index read + map write + metadata;
        # shade/finalize = staged id read is not algorithmic: position read + shaded write
        kernel_alg = {"dedup": 4 * n_idx + 2 * n_idx + 12 * nb, "shade_finalize": 32 * inv}
        dom_name = ("persistent tile kernel (stage + dedup + decoupled look-back/shade)" if path == 3
                    else "fused dedup+offsets+shade" if fused else N.PROFILE_STAGE_NAMES[dom])
        traffic = None  # DRAM bytes per step of the dominant kernel(s), from the committed ncu --set full capture
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))
            if tj.get("workload") == name and path == 3:
                traffic = tj["traffic_bytes_per_step"]
        except Exception:
            pass
        dom_alg = alg if fused else kernel_alg.get(dom_name, alg)
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
            "batches": nb, "batch_formation_ms": t_form, "clocks": clocks.summary(),
            "gpu_launches": steps * launches, "fused": fused,
        }
        if not full:
            return res, None
        # --- end to end through host buffers: pinned H2D of the step's inputs, D2H of its statistics
        h_idx = torch.from_numpy(mesh.indices.view(np.int32).copy()).pin_memory()
        # the vertex buffer crosses PCIe as 3 floats per vertex and is packed to the float4 gather layout on
        # the device (what engine.to_device_positions4 does for any caller)
        h_pos = torch.from_numpy(np.ascontiguousarray(mesh.positions, dtype=np.float32)).pin_memory()
        h_stats = torch.empty(N.VR_STATS_WORDS, dtype=torch.int64).pin_memory()
        d_idx2, pos42 = torch.empty_like(d_idx), torch.ones_like(pos4)
        d_pos3 = torch.empty((mesh.vertex_count, 3), dtype=torch.float32, device=dev)
        spec2 = engine.ShaderSpec(kind=N.VR_SHADER_POSITION, positions4=pos42, matrix=MATRIX,
                                  vertex_count=mesh.vertex_count)
        e2e_steps = max(3, min(steps, 20))

        plan2 = engine.run_device(wl["strategy"], d_idx2, offs[:-1], offs[1:], nb, n_idx, max_span, cfg, hcfg,
                                  spec2, buffers=bufs, static=wl["batching"].startswith("static"), plan_only=True)

        def e2e_step():
            d_idx2.copy_(h_idx, non_blocking=True)
            d_pos3.copy_(h_pos, non_blocking=True)
            pos42[:, :3].copy_(d_pos3)
            r = plan2.relaunch()
            h_stats.copy_(r.stats_dev, non_blocking=True)
            return r

        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(e2e_steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        assert int(h_stats[N.VR_STAT_INVOCATIONS]) == inv
        e2e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": world * tris * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h_idx.numel() * 4 + h_pos.numel() * 4),
               "d2h_bytes_per_step": int(h_stats.numel() * 8), "steps": e2e_steps,
               "note": "pinned host index buffer (uint32) + vertex buffer (3 x fp32, packed to float4 on the device) copied in every step; offsets resident; "
                       "statistics block read back; shaded vertices/triangles stay on the GPU for the next stage"}
        return res, e2e

    def run_multidraw(strategy, steps, warmup):
        """BASELINE.json configs[4]: 1000 draws, 20.4 M triangles, dynamic 256/1023 batches per
        draw, packed into one stream (paper_1805_08893_b200/draws.py).  Two figures: dedup + shade with the
        offsets precomputed (as the paper reports dynamic batching), and including batch formation."""
        from paper_1805_08893_b200 import draws as D
        cfg = __import__("paper_1805_08893_b200").BatchConfig()
        hcfg = HashConfig(table_size=cfg.block_size)
        ds = D.pack_draws(D.scene_corpus(1000), dev)
        tris = ds.triangles
        bufs = engine.RunBuffers()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ws = torch.empty(lib.vr_dynamic_workspace_bytes(ds.indices.numel(), C.byref(engine._cfg_c(cfg))),
                         dtype=torch.uint8, device=dev)
        offs = D.dynamic_offsets_draws(ds, cfg, ws)
        vbase = D.batch_vertex_base(ds, offs)
        nb = offs.numel() - 1
        exp = C5_EXPECT[strategy]
        for _ in range(max(warmup, 1)):
            run = D.run_draws(strategy, ds, offs, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vbase)
        run.check()
        got = dict(batches=nb, rounds=run.rounds, invocations=run.invocations)
        if strategy == "hash":
            got["probes_fast"] = run.probes[0]
        assert got == exp, f"parity gate failed: {got} != {exp}"

        def timed(fn):
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            torch.cuda.synchronize()
            for k in range(steps):
                flush.zero_()
                evs[k][0].record()
                fn()
                evs[k][1].record()
            torch.cuda.synchronize()
            return float(np.mean([a.elapsed_time(b) for a, b in evs]))

        ms_run = timed(lambda: D.run_draws(strategy, ds, offs, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vbase))

        def whole():
            o = D.dynamic_offsets_draws(ds, cfg, ws)  # (reads the batch count back: one host round trip)
            vb = D.batch_vertex_base(ds, o, vbase)
            D.run_draws(strategy, ds, o, cfg, hcfg, matrix=MATRIX, buffers=bufs, vbase=vb)
        whole()
        ms_whole = timed(whole)
        inv = run.invocations
        alg = algorithmic_bytes(ds.indices.numel(), inv, nb)
        return {"value": tris / (ms_run * 1e-3), "ms_per_step": ms_run,
                "value_incl_batch_formation": tris / (ms_whole * 1e-3), "ms_incl_batch_formation": ms_whole,
                "draws": ds.n_draws, "triangles": tris, "vertices": int(ds.vertex_base[-1]), "batches": nb,
                "invocations": inv, "reuse_rate": 1 - inv / ds.indices.numel(),
                "stage_roofline": {"algorithmic_bytes": alg, "frac": alg / (ms_run * 1e-3) / 1e9 / 6557.1},
                "gpu_launches": steps * lib.vr_last_launch_count()}

    import ctypes as C
    res, e2e = run_workload(args.workload, args.steps, args.warmup, True)
    others = {}
    if args.others:
        for name in WORKLOADS:
            if name != args.workload:
                r, _ = run_workload(name, max(10, args.steps // 5), args.warmup, False)
                others[name] = r
        for strat in ("sort", "hash"):
            others[f"c5_multidraw_{strat}"] = run_multidraw(strat, max(10, args.steps // 5), args.warmup)
    wl = WORKLOADS[args.workload]
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 ids / fp32 positions", "data": "synthetic",
        "config": {"workload": wl["desc"], "strategy": wl["strategy"], "triangles_per_gpu": build_mesh(wl).triangle_count
                   if False else None, "l2": "flushed between steps (256 MiB memset outside the per-step CUDA events); "
                   "step working set 391 MB > 126 MB L2", "sharding": f"{world} x one draw per GPU, vertex buffer replicated"},
        "roofline": res["roofline"], "stage_roofline": res["stage_roofline"], "stage_ms": res["stage_ms"],
        "e2e": e2e, "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
        "shading_rate": res["shading_rate"], "reuse_rate": res["reuse_rate"], "invocations": res["invocations"],
        "batches": res["batches"], "batch_formation_ms": res["batch_formation_ms"],
    }
    line["config"].pop("triangles_per_gpu")
    if others:
        line["others"] = others
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mesh = build_mesh(wl)
        base, _ = cpu_baseline(wl, mesh, workload_cfg(wl), 1)
        line["cpu_baseline"] = base
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
