"""Shared helpers of the parity tests."""
from __future__ import annotations

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
FLAT_KEYS = ("batch_round_off", "round_uid_off", "round_prims", "unique_ids", "assembly_map")
MATRIX = np.array([[1, 0, 0, .5], [0, 2, 0, 0], [0, 0, 1, 0], [0, 0, .1, 1]], dtype=np.float64)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def oracle_flat(fr) -> dict:
    """oracle.FlatRun -> dict with the golden key names."""
    return {k: getattr(fr, k) for k in FLAT_KEYS}


def assert_flat_equal(got: dict, want: dict, ctx=""):
    """Bit-exact comparison of a flattened DedupResult list."""
    for k in FLAT_KEYS:
        g, w = np.asarray(got[k]).astype(np.int64), np.asarray(want[k]).astype(np.int64)
        assert g.shape == w.shape, f"{ctx}: {k} shape {g.shape} != {w.shape}"
        if not np.array_equal(g, w):
            bad = int(np.argmax(g != w))
            raise AssertionError(f"{ctx}: {k} differs first at {bad}: got {g[bad]}, want {w[bad]}")


def random_batches(count, seed, max_unique=256, max_tris=341):
    """Random id arrays honouring the dynamic-batch bound (same recipe as the reference's
    tests/helpers.py:43-51)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        pool = rng.choice(100_000, size=int(rng.integers(1, max_unique + 1)), replace=False)
        tris = int(rng.integers(1, max_tris + 1))
        out.append(rng.choice(pool, size=3 * tris).astype(np.uint32))
    return out


def next_pow2(x):
    p = 1
    while p < x:
        p *= 2
    return p


def oracle_draws(O, strategy, meshes, *, dynamic=True, batch_size=96, max_unique=256, max_indices=1023,
                 warp_width=32, table_size=256, max_fast_probes=8, matrix=None, shade=True):
    """The reference's way through a multi-draw scene: dynamic_batches / static_batches and
    run_on_indices once per mesh (strategies.py:404-415), concatenated in draw order."""
    offs, bro, ruo, rp, uid, amap, shaded, counts = [], [0], [0], [], [], [], [], []
    tot = dict(rounds=0, invocations=0, indices=0, probes_fast=0, probes_slow=0, probe_max_chain=0)
    per_draw = []
    ipos = 0
    for m in meshes:
        idx = np.asarray(m.indices, dtype=np.uint32)
        if dynamic:
            so = O.dynamic_batches(idx, max_unique=max_unique, max_indices=max_indices)
        else:
            so = O.static_batches(len(idx), batch_size=batch_size)
        if len(so) == 0:
            per_draw.append((0, 0))
            counts.append(np.zeros(m.vertex_count, dtype=np.int64))
            continue
        fr = O.run(strategy, idx, so[:-1], so[1:], max_unique=max_unique, warp_width=warp_width,
                   table_size=table_size, max_fast_probes=max_fast_probes)
        offs.append(so[:-1] + ipos)
        bro.extend((fr.batch_round_off[1:] + bro[-1]).tolist())
        ruo.extend((fr.round_uid_off[1:] + ruo[-1]).tolist())
        rp.append(fr.round_prims)
        uid.append(fr.unique_ids)
        amap.append(fr.assembly_map)
        if shade:
            shaded.append(O.shade_positions(m.positions, fr.unique_ids, matrix))
        counts.append(O.shade_counts(fr.unique_ids, m.vertex_count))
        for k in ("rounds", "invocations", "indices", "probes_fast", "probes_slow"):
            tot[k] += getattr(fr, k)
        tot["probe_max_chain"] = max(tot["probe_max_chain"], fr.probe_max_chain)  # ProbeStats.merge
        per_draw.append((len(so) - 1, fr.invocations))
        ipos += len(idx)
    cat = lambda parts, dt: np.concatenate(parts).astype(dt) if parts else np.zeros(0, dtype=dt)
    total_idx = sum(len(m.indices) for m in meshes)
    flat = {
        "batch_round_off": np.asarray(bro, dtype=np.int64),
        "round_uid_off": np.asarray(ruo, dtype=np.int64),
        "round_prims": cat(rp, np.int32),
        "unique_ids": cat(uid, np.uint32),
        "assembly_map": cat(amap, np.int32),
    }
    offsets = np.concatenate([cat(offs, np.int64), [total_idx]]) if offs else np.zeros(0, dtype=np.int64)
    return dict(flat=flat, offsets=offsets, totals=tot, per_draw=per_draw,
                shaded=np.concatenate(shaded) if shaded else np.zeros((0, 3), np.float32),
                counts=cat(counts, np.int64))
