"""Pins the CPU oracle (oracle/vr_oracle.c) against the reference: its hand traces / KATs and
the fixtures generated from the unmodified reference (tests/golden/make_golden.py).  CPU only."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

import oracle as O
from helpers import FLAT_KEYS, assert_flat_equal, load_json, load_npz, oracle_flat

REFERENCE = "/root/reference/pkg/src"


# ---- the reference's own known-answer tests ----------------------------------------------
def test_warp_trace_duplicates_within_fetch():  # test_strategies.py:49-58
    rounds, inv, _ = O.warp_vote_batch([0, 1, 2, 0, 2, 3], 4)
    assert inv == 4 and rounds == [((0, 1, 2, 3), (0, 1, 2, 0, 2, 3), 2)]


def test_warp_trace_discard_and_reshade():  # test_strategies.py:60-67
    rounds, inv, _ = O.warp_vote_batch([0, 1, 2, 3, 4, 5], 4)
    assert inv == 7
    assert [r[0] for r in rounds] == [(0, 1, 2, 3), (3, 4, 5)]
    assert [r[2] for r in rounds] == [1, 1]


def test_warp_wide_and_all_equal():  # test_strategies.py:69-77
    rounds, inv, _ = O.warp_vote_batch([10, 20, 30], 32)
    assert inv == 3 and rounds[0][2] == 1
    rounds, inv, _ = O.warp_vote_batch([9] * 6, 4)
    assert inv == 1


def test_warp_width_below_primitive():  # test_strategies.py:79-81
    with pytest.raises(O.OracleError) as e:
        O.warp_vote_batch([0, 1, 2, 3, 4], 4, primitive_size=5)
    assert e.value.kind == "ConfigError"


def test_sort_spec_example():  # test_strategies.py:92-97
    rounds, inv, _ = O.sort_batch([5, 5, 7, 3, 7, 3])
    assert rounds == [((3, 5, 7), (1, 1, 2, 0, 2, 0), 2)] and inv == 3


def test_hash_kat():  # test_strategies.py:112-124: h(5)=0, h(7)=2, h(3)=6
    rounds, inv, _, probes = O.hash_batch([5, 5, 7, 3, 7, 3], table_size=8)
    assert rounds[0][0] == (5, 7, 3) and rounds[0][1] == (0, 0, 1, 2, 1, 2)
    assert inv == 3 and probes == (6, 0, 1)


def test_hash_table_full():  # test_strategies.py:146-149
    ids = np.arange(9, dtype=np.uint32).repeat(3)[:27]
    with pytest.raises(O.OracleError) as e:
        O.hash_batch(ids, table_size=8)
    assert e.value.kind == "RuntimeError"


def test_phash_engineered_collisions():  # test_strategies.py:170-181
    ids = np.repeat(np.array([0, 5, 13, 18, 26, 34], dtype=np.uint32), 3)
    rp, inv, _, probes = O.parallel_hash_batch(ids, 4, table_size=8, max_fast_probes=2)
    rh, _, _, _ = O.hash_batch(ids, table_size=8)
    assert probes[1] > 0 and inv == 6
    corners = lambda rounds: [r[0][s] for r in rounds for s in r[1]]
    assert corners(rp) == corners(rh)


def test_dynamic_examples():  # test_batching.py:71-97
    d = lambda ids, **k: list(O.dynamic_batches(np.array(ids, dtype=np.uint32), **k))
    assert d([0, 1, 2, 0, 2, 3, 4, 5, 6], max_unique=4) == [0, 6, 9]
    assert d([0, 1, 2, 3, 4, 5], max_unique=6) == [0, 6]
    assert d([0, 1, 2, 1, 2, 3], max_unique=4) == [0, 6]  # tie keeps the triangle
    offs = d(list(range(30)), max_unique=256, max_indices=9)
    assert offs[:2] == [0, 9] and max(np.diff(offs)) <= 9
    assert d([]) == []
    with pytest.raises(O.OracleError):
        d([0, 1])


def test_static_examples():  # test_batching.py:44-66
    assert list(O.static_batches(192)) == [0, 96, 192]
    assert list(O.static_batches(99)) == [0, 96, 99]
    assert list(O.static_batches(0)) == []
    with pytest.raises(O.OracleError):
        O.static_batches(100)


# ---- fixtures generated from the reference -----------------------------------------------
def test_kernels_golden():
    data, meta = load_npz("kernels.npz"), load_json("kernels.json")
    for case in meta:
        k = case["id"]
        ids = data[f"k{k}_ids"]
        for strat in O.STRATEGIES:
            fr = O.run(strat, ids, [0], [len(ids)], max_unique=2**31 - 1, warp_width=case["warp_width"],
                       table_size=case["table_size"], max_fast_probes=case["max_fast_probes"])
            want = {name: data[f"k{k}_{strat}_{name}"] for name in FLAT_KEYS}
            assert_flat_equal(oracle_flat(fr), want, f"case {k} {strat}")
            assert fr.invocations == case[strat]["invocations"]
            if strat in ("hash", "phash"):
                assert [fr.probes_fast, fr.probes_slow, fr.probe_max_chain] == case[strat]["probes"]


def test_dynamic_golden():
    data, meta = load_npz("dynamic.npz"), load_json("dynamic.json")
    for case in meta:
        k = case["id"]
        got = O.dynamic_batches(data[f"d{k}_ids"], primitive_size=case.get("primitive_size", 3),
                                max_unique=case["max_unique"], max_indices=case["max_indices"])
        assert np.array_equal(got, data[f"d{k}_offsets"]), f"dynamic case {k}"


def test_runs_golden():
    data, meta = load_npz("runs.npz"), load_json("runs.json")
    matrix = np.array(meta["matrix"])
    for m in meta["meshes"]:
        i, cfg, hc = m["id"], m["cfg"], m["hash"]
        idx, pos = data[f"m{i}_indices"], data[f"m{i}_positions"]
        stat = O.static_batches(len(idx), batch_size=cfg["batch_size"])
        dyn = O.dynamic_batches(idx, max_unique=cfg["max_unique"], max_indices=cfg["max_indices"])
        assert np.array_equal(stat, data[f"m{i}_static"]) and np.array_equal(dyn, data[f"m{i}_dynamic"])
        for strat in O.STRATEGIES:
            offs = stat if strat in ("naive", "warp") else dyn
            fr = O.run(strat, idx, offs[:-1], offs[1:], max_unique=cfg["max_unique"],
                       warp_width=cfg["warp_width"], table_size=hc["table_size"],
                       max_fast_probes=hc["max_fast_probes"])
            want = {name: data[f"m{i}_{strat}_{name}"] for name in FLAT_KEYS}
            assert_flat_equal(oracle_flat(fr), want, f"mesh {i} {strat}")
            rep = m["runs"][strat]
            assert fr.invocations == rep["invocations"] and fr.indices == rep["indices"]
            assert fr.reuse_rate == rep["reuse_rate"]
            if strat in ("hash", "phash"):
                assert (fr.probes_fast, fr.probes_slow, fr.probe_max_chain) == (
                    rep["probes_fast"], rep["probes_slow"], rep["probe_max_chain"])
            shaded = O.shade_positions(pos, fr.unique_ids, matrix)
            ids, stream = O.expand_stream(fr, shaded=shaded)
            assert np.array_equal(ids, idx)  # test_strategies.py:214-218 stream == input
            np.testing.assert_allclose(stream, data[f"m{i}_{strat}_stream"], rtol=1e-6, atol=1e-7)
            assert np.array_equal(O.shade_counts(fr.unique_ids, len(pos)), data[f"m{i}_{strat}_counts"])


def test_grid256_table():
    """configs 1/2 on gen_grid(256,256)."""
    _, idx = O.gen_grid(256, 256)
    assert len(idx) == 390150
    for row in load_json("grid256.json"):
        B = row["B"]
        if row["batching"] == "static":
            offs = O.static_batches(len(idx), batch_size=3 * B)
            mu = 3 * B
        else:
            offs = O.dynamic_batches(idx, max_unique=B, max_indices=4 * B - 1)
            mu = B
        fr = O.run(row["strategy"], idx, offs[:-1], offs[1:], max_unique=mu, warp_width=32,
                   table_size=row["table_size"], outputs=False)
        assert len(offs) - 1 == row["batches"], row
        assert (fr.rounds, fr.invocations) == (row["rounds"], row["invocations"]), row
        if row["strategy"] == "hash":
            assert (fr.probes_fast, fr.probe_max_chain) == (row["probes_fast"], row["probe_max_chain"]), row


def test_over_budget_is_config_error():  # test_strategies.py:315-320
    ids = np.array([0, 1, 2, 3, 4, 5], dtype=np.uint32)
    with pytest.raises(O.OracleError) as e:
        O.run("sort", ids, [0], [6], max_unique=3)
    assert e.value.kind == "ConfigError" and e.value.batch == 0


# ---- the reference itself, when it is mounted (build container only) ---------------------
@pytest.mark.skipif(not os.path.isdir(REFERENCE), reason="reference tree not mounted")
def test_against_live_reference():
    sys.path.insert(0, REFERENCE)
    try:
        import vrlab
        from vrlab.batching import BatchConfig, batches_to_offsets, dynamic_batches
        from vrlab.strategies import warp_vote_batch, hash_batch, HashConfig
    finally:
        sys.path.remove(REFERENCE)
    rng = np.random.default_rng(99)
    for trial in range(25):
        n = 3 * int(rng.integers(1, 200))
        ids = rng.integers(0, int(rng.integers(2, 300)), size=n).astype(np.uint32)
        w = int(rng.choice([4, 8, 16, 32, 64]))
        r = warp_vote_batch(ids, w)
        rounds, inv, _ = O.warp_vote_batch(ids, w)
        assert [(x.unique_ids, x.assembly_map, x.primitives_emitted) for x in r.rounds] == rounds
        ts = 512
        rh, st = hash_batch(ids, HashConfig(table_size=ts))
        oh = O.hash_batch(ids, table_size=ts)
        assert [(x.unique_ids, x.assembly_map, x.primitives_emitted) for x in rh.rounds] == oh[0]
        assert (st.fast, st.slow, st.max_chain) == oh[3]
        mu = int(rng.integers(3, 40))
        ref = batches_to_offsets(dynamic_batches(ids, BatchConfig(max_unique=mu, max_indices=60)))
        assert np.array_equal(ref, O.dynamic_batches(ids, max_unique=mu, max_indices=60))
    p, i = O.gen_grid(19, 7)
    m = vrlab.gen_grid(19, 7)
    assert np.array_equal(p, m.positions) and np.array_equal(i, m.indices)
    assert np.array_equal(O.shuffle_triangles(i, 3), vrlab.shuffle_triangles(m, 3).indices)
