"""N>1 host logic on CPU: world_size-2 gloo processes shard a batch list, each computes its
shard's statistics with the oracle standing in for the device, and the reduced block must
equal the single-process result."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_08893_b200 import _native as N
from paper_1805_08893_b200 import shard


def test_shard_range_partitions():
    for n in (0, 1, 7, 224914):
        for world in (1, 2, 3, 8):
            cuts = [shard.shard_range(n, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
            sizes = [hi - lo for lo, hi in cuts]
            assert max(sizes) - min(sizes) <= 1


def test_shard_batches_whole_batches():
    offs = np.array([0, 96, 192, 288, 300], dtype=np.int64)
    parts = [shard.shard_batches(offs, r, 3) for r in range(3)]
    assert [list(p) for p in parts] == [[0, 96, 192], [192, 288], [288, 300]]
    assert len(shard.shard_batches(offs[:1], 0, 2)) == 0


def test_lpt_assign_balances():
    sizes = np.array([50, 10, 40, 30, 20, 60, 5])
    parts = shard.lpt_assign(sizes, 3)
    assert sorted(np.concatenate(parts).tolist()) == list(range(7))
    loads = [int(sizes[p].sum()) for p in parts]
    assert max(loads) - min(loads) <= 15
    assert all((np.diff(p) > 0).all() for p in parts)


def test_merge_stats_names_the_first_failing_batch_of_the_stream():
    """rank-local error words carry shard-relative batch numbers; the merge adds the shard's first
    batch before taking the minimum, sums the counters and takes the max of the chain length."""
    blocks = torch.zeros((3, N.VR_STATS_WORDS), dtype=torch.int64)
    blocks[:, N.VR_STAT_ERROR] = -1
    blocks[:, N.VR_STAT_INVOCATIONS] = torch.tensor([5, 7, 11])
    blocks[:, N.VR_STAT_PROBE_MAX_CHAIN] = torch.tensor([3, 9, 4])
    blocks[:, shard.STAT_BATCH_BASE] = torch.tensor([0, 100, 200])
    out = shard.merge_stats(blocks)
    assert int(out[N.VR_STAT_INVOCATIONS]) == 23 and int(out[N.VR_STAT_PROBE_MAX_CHAIN]) == 9
    assert int(out[N.VR_STAT_ERROR]) == -1
    blocks[2, N.VR_STAT_ERROR] = (1 << 8) | N.VR_ERR_HASH_FULL       # stream batch 201
    blocks[1, N.VR_STAT_ERROR] = (50 << 8) | N.VR_ERR_OVER_BUDGET    # stream batch 150: earlier in the stream
    out = shard.merge_stats(blocks)
    assert int(out[N.VR_STAT_ERROR]) == (150 << 8) | N.VR_ERR_OVER_BUDGET


def test_concat_flats_is_the_ordered_merge():
    """strategies.py:472-483: per-shard results concatenated in rank order == the unsharded result (oracle on
    both sides: this checks the host-side merge and the shard plans, the GPU test checks the device runs)."""
    import oracle as O
    from helpers import assert_flat_equal, oracle_flat
    _, idx = O.gen_grid(50, 37)
    offs = O.dynamic_batches(idx, max_unique=32, max_indices=127)
    whole = O.run("hash", idx, offs[:-1], offs[1:], max_unique=32, table_size=32)
    for world in (1, 2, 3, 8, 500):
        flats, nb = [], 0
        for r in range(world):
            plan = shard.plan_from_offsets(offs, r, world)
            assert plan.batch_lo == nb and (plan.index_lo, plan.index_hi) == (offs[plan.batch_lo], offs[plan.batch_hi])
            nb = plan.batch_hi
            if plan.n_batches == 0:
                flats.append(None)
                continue
            mine = offs[plan.batch_lo:plan.batch_hi + 1]
            flats.append(oracle_flat(O.run("hash", idx, mine[:-1], mine[1:], max_unique=32, table_size=32)))
        assert nb == len(offs) - 1
        assert_flat_equal(shard.concat_flats(flats), oracle_flat(whole), f"world {world}")
    so = O.static_batches(len(idx))
    from paper_1805_08893_b200.batching import BatchConfig
    for world in (2, 3, 7):
        plans = [shard.plan_static(len(idx), BatchConfig(), r, world) for r in range(world)]
        assert plans[0].index_lo == 0 and plans[-1].index_hi == len(idx)
        assert all(a.index_hi == b.index_lo and a.batch_hi == b.batch_lo for a, b in zip(plans, plans[1:]))
        assert all(p.index_lo == so[p.batch_lo] and p.index_hi == so[p.batch_hi] for p in plans)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, idx = O.gen_grid(40, 40)
    offs = O.dynamic_batches(idx, max_unique=32, max_indices=127)
    mine = shard.shard_batches(offs, rank, world)
    stats = torch.zeros(N.VR_STATS_WORDS, dtype=torch.int64)
    stats[N.VR_STAT_ERROR] = -1
    if len(mine):
        fr = O.run("hash", idx, mine[:-1], mine[1:], max_unique=32, table_size=32)
        stats[N.VR_STAT_INDICES] = fr.indices
        stats[N.VR_STAT_INVOCATIONS] = fr.invocations
        stats[N.VR_STAT_BATCHES] = len(mine) - 1
        stats[N.VR_STAT_ROUNDS] = fr.rounds
        stats[N.VR_STAT_PROBES_FAST] = fr.probes_fast
        stats[N.VR_STAT_PROBE_MAX_CHAIN] = fr.probe_max_chain
    lo, _ = shard.shard_range(len(offs) - 1, rank, world)
    total = shard.reduce_stats(stats, batch_base=lo)
    if rank == 0:
        q.put(total.tolist())
    dist.destroy_process_group()


def test_two_rank_statistics_match_single_process():
    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, idx = O.gen_grid(40, 40)
    offs = O.dynamic_batches(idx, max_unique=32, max_indices=127)
    fr = O.run("hash", idx, offs[:-1], offs[1:], max_unique=32, table_size=32)
    assert total[N.VR_STAT_INDICES] == fr.indices and total[N.VR_STAT_INVOCATIONS] == fr.invocations
    assert total[N.VR_STAT_BATCHES] == len(offs) - 1 and total[N.VR_STAT_ROUNDS] == fr.rounds
    assert total[N.VR_STAT_PROBES_FAST] == fr.probes_fast
    assert total[N.VR_STAT_PROBE_MAX_CHAIN] == fr.probe_max_chain
    assert total[N.VR_STAT_ERROR] == -1


def _draw_worker(rank, world, port, q):
    """Multi-draw scene sharded by whole draws: every rank runs the per-mesh path over the
    draws lpt_assign gives it; the reduced statistics must equal the single-process scene."""
    import oracle as O
    from paper_1805_08893_b200.draws import scene_corpus
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    meshes = scene_corpus(14, seed=5, lo=6, hi=24, ico=(1, 3))
    mine = shard.lpt_assign([m.triangle_count for m in meshes], world)[rank]
    stats = torch.zeros(N.VR_STATS_WORDS, dtype=torch.int64)
    stats[N.VR_STAT_ERROR] = -1
    for d in mine:
        idx = meshes[int(d)].indices
        offs = O.dynamic_batches(idx, max_unique=32, max_indices=127)
        fr = O.run("hash", idx, offs[:-1], offs[1:], max_unique=32, table_size=32)
        stats[N.VR_STAT_INDICES] += fr.indices
        stats[N.VR_STAT_INVOCATIONS] += fr.invocations
        stats[N.VR_STAT_BATCHES] += len(offs) - 1
        stats[N.VR_STAT_ROUNDS] += fr.rounds
        stats[N.VR_STAT_PROBES_FAST] += fr.probes_fast
        stats[N.VR_STAT_PROBE_MAX_CHAIN] = max(int(stats[N.VR_STAT_PROBE_MAX_CHAIN]), fr.probe_max_chain)
    total = shard.reduce_stats(stats)
    if rank == 0:
        q.put((total.tolist(), [int(x) for x in mine]))
    dist.destroy_process_group()


def test_two_rank_draw_sharding_matches_single_process():
    import oracle as O
    from paper_1805_08893_b200.draws import scene_corpus
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_draw_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, mine0 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    meshes = scene_corpus(14, seed=5, lo=6, hi=24, ico=(1, 3))
    parts = shard.lpt_assign([m.triangle_count for m in meshes], world)
    assert sorted(int(x) for p in parts for x in p) == list(range(14)) and mine0 == [int(x) for x in parts[0]]
    loads = [sum(meshes[int(d)].triangle_count for d in p) for p in parts]
    assert max(loads) - min(loads) <= max(m.triangle_count for m in meshes)  # LPT bound
    want = dict(i=0, v=0, b=0, r=0, p=0, c=0)
    for m in meshes:
        offs = O.dynamic_batches(m.indices, max_unique=32, max_indices=127)
        fr = O.run("hash", m.indices, offs[:-1], offs[1:], max_unique=32, table_size=32)
        want["i"] += fr.indices; want["v"] += fr.invocations; want["b"] += len(offs) - 1
        want["r"] += fr.rounds; want["p"] += fr.probes_fast; want["c"] = max(want["c"], fr.probe_max_chain)
    assert (total[N.VR_STAT_INDICES], total[N.VR_STAT_INVOCATIONS], total[N.VR_STAT_BATCHES]) == (want["i"], want["v"], want["b"])
    assert (total[N.VR_STAT_ROUNDS], total[N.VR_STAT_PROBES_FAST], total[N.VR_STAT_PROBE_MAX_CHAIN]) == (want["r"], want["p"], want["c"])
    assert total[N.VR_STAT_ERROR] == -1


def _exchange_worker(rank, world, port, q):
    """SURVEY.md 8e option (ii) on the host: this rank scans ITS range of the stream into the table "entry offset ->
    (exit offset, batches)" (the oracle's greedy splitter, restarted at every start primitive of the range, stands in
    for the device's stage A), ONE all-gather of the tables, shard.compose_tables gives the true entry, the rank
    emits the batches that start in its range."""
    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, idx = O.gen_grid(31, 29)
    idx = O.shuffle_triangles(idx, 5) if hasattr(O, "shuffle_triangles") else idx
    mu, mi, ps = 24, 95, 3
    cap = mi // ps
    T = len(idx) // ps
    s_lo, s_hi = shard.shard_range(T, rank, world)

    def next_of(s):  # end of the greedy batch that starts at primitive s (batching.py:101-123)
        return s + int(O.dynamic_batches(idx[ps * s:ps * min(T, s + cap + 1)], max_unique=mu, max_indices=mi)[1]) // ps

    nxt = {s: next_of(s) for s in range(s_lo, s_hi)}
    table = torch.zeros(2 * cap, dtype=torch.int32)
    for o in range(cap):
        s, cnt = s_lo + o, 0
        while s < s_hi:
            s, cnt = nxt[s], cnt + 1
        table[o], table[cap + o] = s - s_hi, cnt
    gathered = [torch.zeros_like(table) for _ in range(world)]
    dist.all_gather(gathered, table)  # the exchange
    entry, base, total = shard.compose_tables(torch.stack(gathered).numpy(), rank)
    mine, s = [], s_lo + entry
    while s < s_hi:
        mine.append(ps * s)
        s = nxt[s]
    assert len(mine) == int(table[cap + entry])
    out = [None] * world
    dist.all_gather_object(out, (base, total, mine))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_two_and_three_rank_boundary_exchange_matches_the_sequential_scan():
    import oracle as O
    _, idx = O.gen_grid(31, 29)
    idx = O.shuffle_triangles(idx, 5) if hasattr(O, "shuffle_triangles") else idx
    want = O.dynamic_batches(idx, max_unique=24, max_indices=95)
    for world in (2, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        out = q.get(timeout=180)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        offs, seen = [], 0
        for base, total, mine in out:
            assert base == seen and total == len(want) - 1
            offs += mine
            seen += len(mine)
        assert np.array_equal(np.array(offs + [len(idx)]), want)
