"""ctypes front-end of oracle/vr_oracle.c (TEST INFRASTRUCTURE ONLY).

The function names and result shapes follow the reference
(`/root/reference/pkg/src/vrlab/strategies.py`, `batching.py`) so that the
parity tests read like the reference's own tests:

* per-batch kernels return ``(rounds, invocations, indices_consumed)`` with
  ``rounds = [(unique_ids, assembly_map, primitives_emitted), ...]``
  (strategies.py:114-129), hashing kernels additionally ``(fast, slow, max_chain)``
  (strategies.py:94-111);
* ``run`` returns a :class:`FlatRun` -- the flattened ``DedupResult`` list the
  CUDA path is compared against array for array.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vr_oracle.c")
_SO = os.path.join(_HERE, "libvr_oracle.so")

STRATEGIES = ("naive", "warp", "sort", "hash", "phash")  # strategies.py:387
FIBONACCI_MULTIPLIER = 2654435769  # strategies.py:33

ERRORS = {
    1: ("ConfigError", "dynamic-strategy batch holds more unique ids than max_unique"),
    2: ("RuntimeError", "hash table full before all unique ids were inserted"),
    3: ("RuntimeError", "warp voting made no progress; primitive exceeds warp capacity"),
    4: ("ConfigError", "warp width below primitive size cannot make progress"),
    5: ("ConfigError", "index count is not primitive-aligned"),
    6: ("ConfigError", "primitive has more unique indices than max_unique"),
    7: ("MemoryError", "oracle allocation failed"),
}


class OracleError(Exception):
    def __init__(self, code: int, batch: int = -1):
        kind, msg = ERRORS.get(code, ("Error", "unknown"))
        super().__init__(f"{kind}: {msg} (batch {batch})")
        self.code = code
        self.kind = kind
        self.batch = batch


def build(force: bool = False) -> str:
    """Compile vr_oracle.c with gcc (seconds).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _SO, _SRC],
            cwd=_HERE,
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_run.restype = C.c_int
        _lib.orc_batch.restype = C.c_int
        _lib.orc_dynamic_batches.restype = C.c_int
        _lib.orc_static_batches.restype = C.c_int
        _lib.orc_shade_positions.restype = None
        _lib.orc_shade_counts.restype = None
        _lib.orc_expand_stream.restype = None
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def inv_bound(strategy: str, n_idx: int, n_batches: int, ps: int, w: int) -> int:
    if strategy == "warp":
        return n_idx * w // max(1, w - ps + 1) + n_batches * ps + w
    return n_idx + 1


@dataclass
class FlatRun:
    """Flattened list of DedupResult (strategies.py:114-129), batch order."""

    batch_round_off: np.ndarray  # int64[n_batches+1]
    round_uid_off: np.ndarray  # int64[rounds+1]
    round_prims: np.ndarray  # int32[rounds]
    unique_ids: np.ndarray  # uint32[invocations]
    assembly_map: np.ndarray  # int32[consumed]
    rounds: int
    invocations: int
    indices: int
    probes_fast: int
    probes_slow: int
    probe_max_chain: int

    @property
    def reuse_rate(self) -> float:  # analytics.py:92
        return 1.0 - self.invocations / self.indices if self.indices > 0 else 0.0


def run(strategy: str, indices, begins, ends, *, primitive_size=3, max_unique=256, warp_width=32,
        table_size=256, multiplier=FIBONACCI_MULTIPLIER, max_fast_probes=8,
        outputs: bool = True) -> FlatRun:
    """run_on_indices (strategies.py:404-502) without the shader; see shade_positions."""
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    bb = np.ascontiguousarray(begins, dtype=np.int64)
    be = np.ascontiguousarray(ends, dtype=np.int64)
    nb = len(bb)
    s = STRATEGIES.index(strategy)
    span = int((be - bb).sum()) if nb else 0
    max_inv = inv_bound(strategy, span, nb, primitive_size, warp_width)
    if strategy in ("hash", "phash"):
        max_inv = max(max_inv, nb * table_size + 1)
    max_rounds = span // primitive_size + nb + 1
    bro = np.zeros(nb + 1, dtype=np.int64)
    totals = np.zeros(8, dtype=np.int64)
    if outputs:
        ruo = np.zeros(max_rounds + 1, dtype=np.int64)
        rp = np.zeros(max_rounds, dtype=np.int32)
        uid = np.zeros(max_inv, dtype=np.uint32)
        amap = np.zeros(span + 1, dtype=np.int32)
    else:
        ruo = rp = uid = amap = None
    st = lib().orc_run(
        C.c_int(s), _p(idx), C.c_int64(len(idx)), _p(bb), _p(be), C.c_int64(nb),
        C.c_int32(primitive_size), C.c_int32(max_unique), C.c_int32(warp_width),
        C.c_uint32(table_size), C.c_uint32(multiplier), C.c_int32(max_fast_probes),
        _p(bro), _p(ruo), _p(rp), _p(uid), _p(amap), _p(totals),
    )
    if st != 0:
        raise OracleError(st, int(totals[6]))
    r, inv = int(totals[0]), int(totals[1])
    empty = np.zeros(0)
    return FlatRun(
        batch_round_off=bro,
        round_uid_off=ruo[: r + 1].copy() if outputs else empty,
        round_prims=rp[:r].copy() if outputs else empty,
        unique_ids=uid[:inv].copy() if outputs else empty,
        assembly_map=amap[: int(totals[7])].copy() if outputs else empty,
        rounds=r, invocations=inv, indices=int(totals[2]),
        probes_fast=int(totals[3]), probes_slow=int(totals[4]), probe_max_chain=int(totals[5]),
    )


def _batch(strategy, ids, ps, w=32, table_size=256, multiplier=FIBONACCI_MULTIPLIER, mfp=8):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    n = len(ids)
    if strategy == "warp" and w not in (4, 8, 16, 32, 64):  # warp.py:32-35
        raise ValueError("warp width must be one of (4, 8, 16, 32, 64)")
    fr = run(strategy, ids, [0] if n else [], [n] if n else [], primitive_size=ps,
             max_unique=2**31 - 1, warp_width=w, table_size=table_size, multiplier=multiplier,
             max_fast_probes=mfp)
    rounds = []
    m = 0
    for r in range(fr.rounds):
        a, b = int(fr.round_uid_off[r]), int(fr.round_uid_off[r + 1])
        k = int(fr.round_prims[r]) * ps
        rounds.append((tuple(int(v) for v in fr.unique_ids[a:b]),
                       tuple(int(v) for v in fr.assembly_map[m:m + k]),
                       int(fr.round_prims[r])))
        m += k
    return rounds, fr


def naive_batch(ids, primitive_size=3):
    rounds, fr = _batch("naive", ids, primitive_size)
    return rounds, fr.invocations, len(ids)


def warp_vote_batch(ids, warp_width, primitive_size=3):
    rounds, fr = _batch("warp", ids, primitive_size, w=warp_width)
    return rounds, fr.invocations, len(ids)


def sort_batch(ids, primitive_size=3):
    rounds, fr = _batch("sort", ids, primitive_size)
    return rounds, fr.invocations, len(ids)


def hash_batch(ids, table_size=256, multiplier=FIBONACCI_MULTIPLIER, primitive_size=3):
    if len(ids) == 0:  # reference emits one empty round (strategies.py:370-380)
        return [((), (), 0)], 0, 0, (0, 0, 0)
    rounds, fr = _batch("hash", ids, primitive_size, table_size=table_size, multiplier=multiplier)
    return rounds, fr.invocations, len(ids), (fr.probes_fast, fr.probes_slow, fr.probe_max_chain)


def parallel_hash_batch(ids, warp_width, table_size=256, multiplier=FIBONACCI_MULTIPLIER,
                        max_fast_probes=8, primitive_size=3):
    if len(ids) == 0:
        return [((), (), 0)], 0, 0, (0, 0, 0)
    rounds, fr = _batch("phash", ids, primitive_size, w=warp_width, table_size=table_size,
                        multiplier=multiplier, mfp=max_fast_probes)
    return rounds, fr.invocations, len(ids), (fr.probes_fast, fr.probes_slow, fr.probe_max_chain)


def dynamic_batches(indices, *, primitive_size=3, max_unique=256, max_indices=1023) -> np.ndarray:
    """batching.py:87-125 -> flat int64 offsets (batching.py:128-137); empty input -> length 0."""
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    n = len(idx)
    out = np.zeros(n // max(1, primitive_size) + 2, dtype=np.int64)
    nb = C.c_int64(0)
    st = lib().orc_dynamic_batches(_p(idx), C.c_int64(n), C.c_int32(primitive_size),
                                   C.c_int32(max_unique), C.c_int32(max_indices), _p(out),
                                   C.byref(nb))
    if st != 0:
        raise OracleError(st)
    return out[: nb.value + 1].copy() if nb.value else np.zeros(0, dtype=np.int64)


def static_batches(index_count: int, *, primitive_size=3, batch_size=96) -> np.ndarray:
    """batching.py:76-84 -> flat int64 offsets."""
    out = np.zeros(index_count // batch_size + 3, dtype=np.int64)
    nb = C.c_int64(0)
    st = lib().orc_static_batches(C.c_int64(index_count), C.c_int32(primitive_size),
                                  C.c_int32(batch_size), _p(out), C.byref(nb))
    if st != 0:
        raise OracleError(st)
    return out[: nb.value + 1].copy() if nb.value else np.zeros(0, dtype=np.int64)


def shade_positions(positions, unique_ids, matrix=None) -> np.ndarray:
    """position_shader (strategies.py:53-67) applied to a unique-id list -> float32[n,3]."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    uid = np.ascontiguousarray(unique_ids, dtype=np.uint32)
    m = None if matrix is None else np.ascontiguousarray(matrix, dtype=np.float64).reshape(16)
    out = np.zeros((len(uid), 3), dtype=np.float32)
    lib().orc_shade_positions(_p(pos), _p(m), _p(uid), C.c_int64(len(uid)), _p(out))
    return out


def shade_counts(unique_ids, vertex_count: int) -> np.ndarray:
    """np.bincount tally of strategies.py:485-489."""
    uid = np.ascontiguousarray(unique_ids, dtype=np.uint32)
    out = np.zeros(vertex_count, dtype=np.int64)
    lib().orc_shade_counts(_p(uid), C.c_int64(len(uid)), _p(out))
    return out


def expand_stream(fr: FlatRun, primitive_size=3, shaded=None):
    """Per-corner record stream of strategies.py:456-463 (ids, and positions if `shaded`)."""
    n = len(fr.assembly_map)
    ids = np.zeros(n, dtype=np.uint32)
    pos = None
    sh = None
    if shaded is not None:
        sh = np.ascontiguousarray(shaded, dtype=np.float32)
        pos = np.zeros((n, 3), dtype=np.float32)
    lib().orc_expand_stream(_p(fr.batch_round_off), _p(fr.round_uid_off), _p(fr.round_prims),
                            _p(fr.assembly_map), C.c_int64(fr.rounds), C.c_int32(primitive_size),
                            _p(sh), _p(fr.unique_ids), _p(pos), _p(ids))
    return ids, pos


# ---------------------------------------------------------------------------
# Input generators restated from mesh.py (vectorised; bit-identical, see
# tests/test_oracle_golden.py).  Inputs only -- not part of the timed path.
# ---------------------------------------------------------------------------
def gen_grid(rows: int, cols: int):
    """mesh.py:229-247: positions float64[V,3], indices uint32[3T] in row-major strip order."""
    ys, xs = np.mgrid[0:rows, 0:cols]
    positions = np.column_stack(
        [xs.ravel().astype(np.float64), ys.ravel().astype(np.float64), np.zeros(rows * cols)])
    r, c = np.mgrid[0:rows - 1, 0:cols - 1]
    v00 = (r * cols + c).ravel().astype(np.int64)
    v01, v10 = v00 + 1, v00 + cols
    v11 = v10 + 1
    faces = np.stack([v00, v10, v01, v01, v10, v11], axis=1).reshape(-1)
    return positions, faces.astype(np.uint32)


def shuffle_triangles(indices, seed: int, primitive_size: int = 3):
    """mesh.py:250-256: default_rng(seed).shuffle(tris, axis=0)."""
    tris = np.asarray(indices).reshape(-1, primitive_size).copy()
    np.random.default_rng(seed).shuffle(tris, axis=0)
    return tris.reshape(-1)
