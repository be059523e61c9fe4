"""oracle/clients.py (random-walk client, LRU cache model, ideal counts) pinned against fixtures generated from the
unmodified reference by tests/golden/make_golden.py (walk.npz, cache.json).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import load_json, load_npz
from oracle import clients as OC

WALK_CASES = ("default_small", "radius16", "uniform_field", "one_peak")


def walk_case(g, name):
    gw, gh, agents, dist, kept, steps, seed = (int(v) for v in g[f"{name}/cfg"])
    gaussians = [tuple(row) for row in g[f"{name}/gaussians"]]
    return dict(grid=(gw, gh), agents=agents, dist=dist, kept=kept, steps=steps, seed=seed, gaussians=gaussians)


@pytest.mark.parametrize("name", WALK_CASES)
def test_walk_oracle_matches_reference(name):
    g = load_npz("walk.npz")
    c = walk_case(g, name)
    for cell, want in zip(g[f"{name}/cells"], g[f"{name}/tables"]):
        got = OC.cell_moves(int(cell), c["grid"], c["dist"], c["kept"], c["gaussians"])
        assert np.array_equal(got, want), (name, int(cell))  # bit-exact: same arithmetic, same summation
    uni = g[f"{name}/uniforms"]
    for t in range(uni.shape[0]):
        for a in (0, 1, 17, c["agents"] - 1):
            assert OC.uniform(c["seed"], t, a) == uni[t, a]
    traj = g[f"{name}/trajectory"]
    pos = traj[0].copy()
    for t in range(min(c["steps"], 2)):
        pos = OC.walk_step(pos, c["grid"], c["dist"], c["kept"], c["gaussians"], c["seed"], t)
        assert np.array_equal(pos, traj[t + 1]), (name, t)


def test_walk_known_answers():
    """tests/test_walk.py:31-34 pack examples, :113-119 choose_move proportions."""
    assert (3 << 16) | 5 == 196613
    moves = np.array([[0, 0, 0.5], [1, 0, 0.25], [0, 1, 0.25]])
    assert [OC.pick_move(moves, u) for u in (0.0, 0.49, 0.5, 0.74, 0.75, 0.999999)] == [0, 0, 1, 1, 2, 2]


def test_cache_oracle_matches_reference():
    import paper_1805_08893_b200 as P
    meshes = {"grid40x31": P.gen_grid(40, 31), "grid40x31s": P.shuffle_triangles(P.gen_grid(40, 31), 4),
              "sphere3": P.gen_icosphere(3), "grid9x9": P.gen_grid(9, 9)}
    for case in load_json("cache.json"):
        mesh = meshes[case["mesh"]]
        if "ideal_invocations" in case:
            n, counts = OC.ideal_counts(mesh.indices, mesh.vertex_count)
            assert n == case["ideal_invocations"] and 1.0 - n / len(mesh.indices) == case["ideal_rate"]
            continue
        miss = np.zeros(mesh.vertex_count, dtype=np.int64)
        hits, misses, rate = OC.simulate_cache(mesh.indices, case["procs"], case["wave"], case["entries"], miss_counts=miss)
        assert (hits, misses, rate) == (case["hits"], case["misses"], case["hit_rate"]), case
        assert int(miss.sum()) == case["miss_counts_sum"]
        assert int((miss * (np.arange(len(miss)) % 9973 + 1)).sum()) == case["miss_counts_crc"]


def test_cache_hand_trace():
    """tests/test_cache.py:57-64: entries = 2 over [0,1,0,2,1]: only the second 0 hits; :44-50: one wave as wide
    as the buffer never hits."""
    assert OC.lru_chunk([0, 1, 0, 2, 1], 1, 2)[0:2] == (1, 4)
    idx = np.tile(np.arange(6), 5)
    assert OC.lru_chunk(idx, len(idx), 64) == (0, len(idx))
