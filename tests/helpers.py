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
