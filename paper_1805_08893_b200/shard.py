"""Multi-GPU sharding of the geometry stage.

Batches are independent (SPEC: "batches may be processed concurrently and results concatenated
in batch order"), so ONE index stream is cut into contiguous ranges of WHOLE batches, one range
per rank, with the vertex buffer replicated.  No collective sits on the data path; the only
exchange is one all-gather of the 16-word statistics blocks, merged locally the way the reference's
ordered merge does (strategies.py:472-483: SUM for the counters, MAX for the longest probe chain, the
first failing batch in stream order for the error).

  static batches   cut points are multiples of batch_size: closed form, no communication
                   (`plan_static`);
  dynamic batches  a cut must fall on a true greedy boundary, known only after the scan.  Option (ii) of
                   SURVEY.md 8e (`dynamic_offsets_exchange`, batching="exchange"): every rank scans ITS
                   range of the stream into a table "entry offset -> (exit offset, batches)", ONE all-gather
                   of those tables (2.7 KB per rank) composes them, and every rank emits the batches that
                   start in its range -- the batch formation scales with the ranks, and this all-gather is
                   the path's one real exchange step.  Option (i) (batching="dynamic"): every rank runs
                   the index-only boundary scan over the whole stream redundantly and takes its slice of
                   batches (`plan_from_offsets`); kept for configurations the ranged kernels do not take;
  multi-draw       whole draws per rank, longest-processing-time bin packing (`lpt_assign`), every rank
                   packs and runs its own draws (`run_draws_sharded`).

`run_sharded` is the per-rank entry point; `concat_flats` is the reference's ordered merge of the
per-shard results and is what the tests compare with the unsharded run."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N

SUM_WORDS = (N.VR_STAT_INDICES, N.VR_STAT_INVOCATIONS, N.VR_STAT_BATCHES, N.VR_STAT_ROUNDS,
             N.VR_STAT_PROBES_FAST, N.VR_STAT_PROBES_SLOW)
MAX_WORDS = (N.VR_STAT_PROBE_MAX_CHAIN,)
STAT_BATCH_BASE = 8  # spare word of the statistics block: first batch of the rank's shard (for the error merge)


def shard_range(n_items: int, rank: int, world: int):
    """Balanced contiguous split: the first n % world ranks get one extra item."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_batches(offsets, rank: int, world: int):
    """Offsets array (n_batches+1) -> this rank's sub-array (whole batches, contiguous)."""
    nb = max(len(offsets) - 1, 0)
    lo, hi = shard_range(nb, rank, world)
    return offsets[lo:hi + 1] if hi > lo else offsets[:0]


def lpt_assign(sizes, world: int):
    """Whole draws to ranks, largest first onto the least-loaded rank (ties: lowest rank).
    Returns a list of index arrays, each in ascending draw order."""
    sizes = np.asarray(sizes, dtype=np.int64)
    load = np.zeros(world, dtype=np.int64)
    owner = np.zeros(len(sizes), dtype=np.int64)
    for d in np.argsort(-sizes, kind="stable"):
        r = int(np.argmin(load))
        owner[d] = r
        load[r] += sizes[d]
    return [np.flatnonzero(owner == r) for r in range(world)]


# ---------------------------------------------------------------------------------------------
# statistics: one collective
# ---------------------------------------------------------------------------------------------
def merge_stats(blocks) -> torch.Tensor:
    """[world, VR_STATS_WORDS] per-rank blocks (tensor or array) -> the block of the whole stream, a CPU int64
    tensor (strategies.py:472-483).  The error word of a rank holds (batch within its shard << 8 | status); word
    STAT_BATCH_BASE holds the shard's first batch, so the merged word names the first failing batch of the STREAM."""
    b = blocks.detach().cpu().numpy() if isinstance(blocks, torch.Tensor) else np.asarray(blocks)
    b = b.reshape(-1, N.VR_STATS_WORDS).astype(np.int64)
    out = np.zeros(N.VR_STATS_WORDS, dtype=np.int64)
    for w in SUM_WORDS:
        out[w] = b[:, w].sum()
    for w in MAX_WORDS:
        out[w] = b[:, w].max()
    err = b[:, N.VR_STAT_ERROR]
    glob = (((err >> 8) + b[:, STAT_BATCH_BASE]) << 8) | (err & 0xFF)
    bad = glob[err >= 0]
    out[N.VR_STAT_ERROR] = bad.min() if len(bad) else -1
    return torch.from_numpy(out)


def gather_stats(stats: torch.Tensor, group=None, batch_base: int = 0) -> torch.Tensor:
    """The ONE collective of a sharded run: all-gather of the ranks' statistics blocks -> [world, VR_STATS_WORDS]
    on the device of `stats` (NCCL for CUDA tensors, gloo for CPU tensors); asynchronous on the current stream.
    Merge with `merge_stats` when the host wants the numbers."""
    s = stats.clone()
    s[STAT_BATCH_BASE] = batch_base
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return s.unsqueeze(0)
    world = dist.get_world_size(group)
    out = torch.empty((world, s.numel()), dtype=s.dtype, device=s.device)
    dist.all_gather(list(out.unbind(0)), s, group=group)
    return out


def reduce_stats(stats: torch.Tensor, group=None, batch_base: int = 0) -> torch.Tensor:
    """One statistics block per rank -> the block of the whole job on every rank (CPU tensor): one all-gather
    of VR_STATS_WORDS int64 and a host-side merge."""
    return merge_stats(gather_stats(stats, group, batch_base))


# ---------------------------------------------------------------------------------------------
# one stream, whole batches per rank
# ---------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class ShardPlan:
    """This rank's contiguous range of whole batches of one stream."""

    rank: int
    world: int
    batch_lo: int
    batch_hi: int
    index_lo: int
    index_hi: int
    static: bool

    @property
    def n_batches(self) -> int:
        return self.batch_hi - self.batch_lo

    @property
    def span(self) -> int:
        return self.index_hi - self.index_lo


def plan_static(index_count: int, cfg, rank: int, world: int) -> ShardPlan:
    """static_batches (batching.py:76-84): cut points at multiples of batch_size, no communication."""
    nb = -(-index_count // cfg.batch_size) if index_count > 0 else 0
    lo, hi = shard_range(nb, rank, world)
    return ShardPlan(rank, world, lo, hi, min(lo * cfg.batch_size, index_count), min(hi * cfg.batch_size, index_count), True)


def plan_from_offsets(offsets, rank: int, world: int) -> ShardPlan:
    """Any offsets array (batching.py:128-137), e.g. the dynamic boundaries every rank computed for the whole
    stream: this rank's slice of whole batches.  Reads two entries of a device array (16 bytes)."""
    nb = max(int(offsets.shape[0]) - 1, 0)
    lo, hi = shard_range(nb, rank, world)
    if nb == 0:
        return ShardPlan(rank, world, 0, 0, 0, 0, False)
    if isinstance(offsets, torch.Tensor):
        ends = offsets[[lo, hi]].cpu()
        a, b = int(ends[0]), int(ends[1])
    else:
        a, b = int(offsets[lo]), int(offsets[hi])
    return ShardPlan(rank, world, lo, hi, a, b, False)


def compose_tables(tables, rank: int):
    """Host restatement of range_entry_kernel: tables[q] = (exit[cap], count[cap]) of rank q's range; the chain
    enters range 0 at offset 0.  Returns (entry offset into range `rank`, number of its first batch, total batches)."""
    t = np.asarray(tables)
    world, cap = t.shape[0], t.shape[1] // 2
    e = base = 0
    entry = (0, 0)
    for q in range(world):
        if q == rank:
            entry = (e, base)
        base += int(t[q, cap + e])
        e = int(t[q, e])
    return entry[0], entry[1], base


def dynamic_offsets_exchange(d_indices: torch.Tensor, cfg, rank: int, world: int, group=None, gather=None,
                             workspace: torch.Tensor | None = None):
    """batching.py:87-125 over a stream sharded by index range (include/vrgeom.h, vr_dynamic_range_*): this rank's
    offsets array (the batches that start in its range; positions in the whole buffer), the global number of its
    first batch and the batch count of the whole stream.  `gather(table) -> [world, words]` replaces the NCCL
    all-gather (tests run the ranks of a world one after another on one GPU)."""
    import ctypes as C
    from . import engine

    lib = N.require_cuda()
    n = int(d_indices.numel())
    dev = d_indices.device
    c = engine._cfg_c(cfg)
    if n % cfg.primitive_size != 0:
        from .batching import ConfigError
        raise ConfigError(f"index count {n} is not primitive-aligned")
    n_groups = int(lib.vr_dynamic_group_count(n, C.byref(c)))
    words = int(lib.vr_dynamic_table_words(n, C.byref(c)))
    glo, ghi = shard_range(n_groups, rank, world)
    ws_bytes = lib.vr_dynamic_workspace_bytes(n, C.byref(c))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    table = torch.empty(words, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_dynamic_range_tables(engine._ptr(d_indices), n, C.byref(c), glo, ghi, engine._ptr(table),
                                                        engine._ptr(workspace), ws_bytes, engine._stream_ptr()))
    if gather is not None:
        tables = gather(table)
    elif dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        tables = torch.empty((world, words), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(tables, table, group=group)  # the one exchange step of the path
    else:
        tables = table.unsqueeze(0)
    tables = tables.contiguous()
    group_prims = int(lib.vr_dynamic_group_indices(C.byref(c))) // cfg.primitive_size
    cap_out = min(n // cfg.primitive_size, (ghi - glo) * group_prims) + 2
    offs = torch.empty(cap_out, dtype=torch.int32, device=dev)
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        engine.raise_status(lib.vr_dynamic_range_offsets(engine._ptr(d_indices), n, C.byref(c), glo, ghi, engine._ptr(tables),
                                                         world, rank, engine._ptr(offs), engine._ptr(counts),
                                                         engine._ptr(workspace), ws_bytes, engine._stream_ptr()))
    cnt, status, base, total = (int(v) for v in counts.cpu())
    if status:
        engine.raise_status(status)
    return offs[:cnt + 1], base, total


def run_sharded(strategy: str, d_indices: torch.Tensor, cfg, hcfg=None, shader=None, *, batching: str = "static",
                offsets: torch.Tensor | None = None, rank: int | None = None, world: int | None = None,
                want_counts: bool = False, buffers=None, group=None, plan_only: bool = False):
    """This rank's share of ONE index stream: (DeviceRun over the rank's batches, ShardPlan).

    `d_indices` is the whole stream (replicated, like the vertex buffer: 4 B per index is what a rank needs
    to find dynamic boundaries on its own).  batching = "static" | "exchange" (dynamic batches, every rank scans
    its own range, one all-gather of tables) | "dynamic" (dynamic batches, redundant whole-stream scan) | "offsets"
    (a precomputed device offsets array for the whole stream).  The DeviceRun's outputs are relative to the shard: batch 0
    is stream batch plan.batch_lo, the assembly map starts at index plan.index_lo."""
    from . import engine

    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_idx = int(d_indices.numel())
    dev = d_indices.device
    if batching == "exchange":
        local, base, _total = dynamic_offsets_exchange(d_indices, cfg, rank, world, group)
        nb = int(local.numel()) - 1
        max_span = max(cfg.batch_size, cfg.max_indices - cfg.max_indices % cfg.primitive_size)
        if nb <= 0:
            return None, ShardPlan(rank, world, base, base, 0, 0, False)
        ends = local[[0, nb]].cpu()
        plan = ShardPlan(rank, world, base, base + nb, int(ends[0]), int(ends[1]), False)
        run = engine.run_device(strategy, d_indices, local[:-1], local[1:], nb, plan.span, max_span, cfg, hcfg, shader,
                                want_counts=want_counts, buffers=buffers, contiguous=True, plan_only=plan_only)
        return run, plan
    if batching == "static":
        plan = plan_static(n_idx, cfg, rank, world)
        offs = engine.static_offsets_device(n_idx, cfg, dev) if offsets is None else offsets
        max_span = cfg.batch_size
    else:
        if offsets is None:
            if batching != "dynamic":
                raise ValueError("batching='offsets' needs the offsets array")
            offs = engine.dynamic_offsets_device(d_indices, cfg)  # redundant on every rank: SURVEY 8e option (i)
        else:
            offs = offsets
        plan = plan_from_offsets(offs, rank, world)
        max_span = max(cfg.batch_size, cfg.max_indices - cfg.max_indices % cfg.primitive_size)
    if plan.n_batches == 0:
        return None, plan
    lo, hi = plan.batch_lo, plan.batch_hi
    # the position-aligned (tile) kernels want a 16-byte aligned first index
    static = plan.static and plan.index_lo % 4 == 0
    run = engine.run_device(strategy, d_indices, offs[lo:hi], offs[lo + 1:hi + 1], hi - lo, plan.span, max_span, cfg,
                            hcfg, shader, want_counts=want_counts, buffers=buffers, contiguous=True, static=static,
                            plan_only=plan_only)
    return run, plan


def global_stats(run, plan: ShardPlan, group=None, device=None) -> torch.Tensor:
    """Statistics of the whole stream from the per-rank runs (one all-gather).  A rank with no batches
    contributes an empty block."""
    if run is None:
        s = torch.zeros(N.VR_STATS_WORDS, dtype=torch.int64, device=device or "cpu")
        s[N.VR_STAT_ERROR] = -1
    else:
        s = run.stats_dev
    return reduce_stats(s, group, batch_base=plan.batch_lo)


def concat_flats(flats) -> dict:
    """The reference's ordered merge (strategies.py:472-483) of per-shard flattened results, in rank order:
    streams are concatenated, round / unique-id offsets are rebased."""
    out = {"batch_round_off": [np.zeros(1, dtype=np.int64)], "round_uid_off": [np.zeros(1, dtype=np.int64)],
           "round_prims": [], "unique_ids": [], "assembly_map": []}
    extra = {}
    r_base = u_base = 0
    for f in flats:
        if f is None:
            continue
        out["batch_round_off"].append(np.asarray(f["batch_round_off"][1:], dtype=np.int64) + r_base)
        out["round_uid_off"].append(np.asarray(f["round_uid_off"][1:], dtype=np.int64) + u_base)
        r_base += int(f["batch_round_off"][-1])
        u_base += int(f["round_uid_off"][-1])
        for k in ("round_prims", "unique_ids", "assembly_map"):
            out[k].append(np.asarray(f[k]))
        for k in ("shaded", "shaded_attr"):
            if k in f:
                extra.setdefault(k, []).append(f[k])
        if "shade_counts" in f:  # per-vertex tallies add up (vertex buffer replicated)
            extra["shade_counts"] = f["shade_counts"] if "shade_counts" not in extra else extra["shade_counts"] + f["shade_counts"]
    res = {k: (np.concatenate(v) if v else np.zeros(0, dtype=np.int64)) for k, v in out.items()}
    for k, v in extra.items():
        res[k] = np.concatenate(v) if isinstance(v, list) else v
    return res


# ---------------------------------------------------------------------------------------------
# multi-draw scenes: whole draws per rank
# ---------------------------------------------------------------------------------------------
def run_draws_sharded(strategy: str, meshes, cfg, hcfg=None, *, rank: int, world: int, matrix=None,
                      want_counts: bool = False, buffers=None, device=None):
    """BASELINE.json configs[4] across ranks: this rank packs the draws `lpt_assign` gives it (ascending draw
    order), forms their dynamic batches and runs them.  Returns (DeviceRun or None, DrawSet or None, offsets,
    draw ids).  Every draw restarts the greedy scan, so no boundary couples two ranks."""
    from . import draws as D

    mine = lpt_assign([len(m.indices) // cfg.primitive_size for m in meshes], world)[rank]
    if len(mine) == 0:
        return None, None, None, mine
    ds = D.pack_draws([meshes[int(d)] for d in mine], device)
    offs = D.dynamic_offsets_draws(ds, cfg)
    run = D.run_draws(strategy, ds, offs, cfg, hcfg, matrix=matrix, want_counts=want_counts, buffers=buffers)
    return run, ds, offs, mine
