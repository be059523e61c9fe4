"""Input side of the hot path: the indexed-mesh container and the synthetic generators
BASELINE.json's configs name.  Host-side NumPy only; nothing here is timed.

Mirrors `vrlab/mesh.py` (/root/reference/pkg/src/vrlab/mesh.py): `IndexedMesh` :34-88,
`VertexShadingCounts` :91-108, `gen_icosphere` :190-221, `gen_grid` :229-247,
`shuffle_triangles` :250-256.  OBJ/PLY I/O is out of scope.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

INVALID_INDEX = 0xFFFFFFFF  # mesh.py:11-13: reserved sentinel


class MeshError(ValueError):
    """Invalid mesh data or construction parameters (mesh.py:22-23)."""


@dataclass(frozen=True)
class IndexedMesh:
    """positions (V,3) float64, indices (3T,) uint32, optional opaque attributes (mesh.py:34-88)."""

    positions: np.ndarray
    indices: np.ndarray
    attributes: np.ndarray | None = None
    primitive_size: int = 3

    def __post_init__(self):
        pos = np.ascontiguousarray(self.positions, dtype=np.float64)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise MeshError(f"positions must be (V, 3), got {pos.shape}")
        idx = np.ascontiguousarray(self.indices, dtype=np.uint32)
        if idx.ndim != 1:
            raise MeshError("indices must be a flat array")
        if self.primitive_size != 3:
            raise MeshError("meshes are triangle lists (primitive_size 3)")
        if len(idx) % 3 != 0:
            raise MeshError(f"index count {len(idx)} is not a multiple of 3")
        if len(idx) > 0:
            if len(pos) < 1:
                raise MeshError("non-empty index buffer with no vertices")
            top = int(idx.max())
            if top >= len(pos):
                raise MeshError(f"index {top} out of range for {len(pos)} vertices")
            if top >= INVALID_INDEX:
                raise MeshError("vertex index collides with reserved sentinel")
        if self.attributes is not None and len(self.attributes) != len(pos):
            raise MeshError("attributes must have one record per vertex")
        pos.flags.writeable = False
        idx.flags.writeable = False
        object.__setattr__(self, "positions", pos)
        object.__setattr__(self, "indices", idx)

    @property
    def vertex_count(self) -> int:
        return len(self.positions)

    @property
    def triangle_count(self) -> int:
        return len(self.indices) // 3

    def triangles(self) -> np.ndarray:
        return self.indices.reshape(-1, 3)


@dataclass(frozen=True)
class VertexShadingCounts:
    """Per-vertex shader invocation tallies of one run (mesh.py:91-108)."""

    counts: np.ndarray

    def __post_init__(self):
        c = np.ascontiguousarray(self.counts, dtype=np.int64)
        if c.ndim != 1:
            raise MeshError("counts must be a flat array")
        if len(c) and c.min() < 0:
            raise MeshError("negative shading count")
        c.flags.writeable = False
        object.__setattr__(self, "counts", c)

    @property
    def total(self) -> int:
        return int(self.counts.sum())


def gen_grid(rows: int, cols: int) -> IndexedMesh:
    """Regular z=0 grid, triangles (v00,v10,v01),(v01,v10,v11) in row-major strip order
    (mesh.py:229-247).  Vectorised; bit-identical to the reference loop."""
    if rows < 2 or cols < 2:
        raise MeshError("grid needs rows, cols >= 2")
    ys, xs = np.mgrid[0:rows, 0:cols]
    positions = np.column_stack(
        [xs.ravel().astype(np.float64), ys.ravel().astype(np.float64), np.zeros(rows * cols)])
    r, c = np.mgrid[0:rows - 1, 0:cols - 1]
    v00 = (r * cols + c).ravel().astype(np.int64)
    v01, v10 = v00 + 1, v00 + cols
    v11 = v10 + 1
    faces = np.stack([v00, v10, v01, v01, v10, v11], axis=1).reshape(-1)
    return IndexedMesh(positions=positions, indices=faces.astype(np.uint32))


_T = (1.0 + math.sqrt(5.0)) / 2.0
_ICO_VERTS = [
    (-1, _T, 0), (1, _T, 0), (-1, -_T, 0), (1, -_T, 0),
    (0, -1, _T), (0, 1, _T), (0, -1, -_T), (0, 1, -_T),
    (_T, 0, -1), (_T, 0, 1), (-_T, 0, -1), (-_T, 0, 1),
]
_ICO_FACES = [
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
]


def _unit(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


def gen_icosphere(subdivisions: int) -> IndexedMesh:
    """Unit icosphere, 10*4^s+2 vertices / 20*4^s triangles, midpoints shared per edge in
    first-use order (mesh.py:190-221)."""
    if not 0 <= subdivisions <= 8:
        raise MeshError("subdivisions must be in [0, 8]")
    verts = [_unit(v) for v in _ICO_VERTS]
    faces = list(_ICO_FACES)
    for _ in range(subdivisions):
        cache: dict = {}
        nxt = []
        for a, b, c in faces:
            mids = []
            for p, q in ((a, b), (b, c), (c, a)):
                key = (p, q) if p < q else (q, p)
                m = cache.get(key)
                if m is None:
                    vp, vq = verts[p], verts[q]
                    verts.append(_unit(((vp[0] + vq[0]) / 2, (vp[1] + vq[1]) / 2, (vp[2] + vq[2]) / 2)))
                    m = cache[key] = len(verts) - 1
                mids.append(m)
            ab, bc, ca = mids
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nxt
    return IndexedMesh(positions=np.array(verts, dtype=np.float64),
                       indices=np.array(faces, dtype=np.uint32).reshape(-1))


def shuffle_triangles(mesh: IndexedMesh, seed: int) -> IndexedMesh:
    """Seeded permutation of triangle order (mesh.py:250-256)."""
    tris = mesh.triangles().copy()
    np.random.default_rng(seed).shuffle(tris, axis=0)
    return IndexedMesh(positions=mesh.positions, indices=tris.reshape(-1), attributes=mesh.attributes)
