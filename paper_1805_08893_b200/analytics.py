"""Reuse statistics contract of the hot path (host mirror of `vrlab/analytics.py`,
/root/reference/pkg/src/vrlab/analytics.py:20-50 `ReuseReport`, :74-102 `build_report`).
`ideal_report` :105-119 runs on the device.  Tables and CSV/JSON writers are out of scope."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import VertexShadingCounts


@dataclass(frozen=True)
class ReuseReport:
    """Invocation accounting for one strategy on one scene (analytics.py:20-50)."""

    scene: str
    strategy: str
    indices: int
    invocations: int
    reuse_rate: float
    batches: int
    per_vertex: VertexShadingCounts | None = None
    probe_stats: object | None = None

    @property
    def shading_rate(self) -> float | None:
        """invocations / vertex -- BASELINE.json's second metric."""
        if self.per_vertex is None or len(self.per_vertex.counts) == 0:
            return None
        return self.invocations / len(self.per_vertex.counts)

    def to_dict(self) -> dict:
        out = {"scene": self.scene, "strategy": self.strategy, "indices": self.indices,
               "invocations": self.invocations, "reuse_rate": self.reuse_rate, "batches": self.batches}
        if self.probe_stats is not None:
            out["probes_fast"] = self.probe_stats.fast
            out["probes_slow"] = self.probe_stats.slow
            out["probe_max_chain"] = self.probe_stats.max_chain
        return out


def build_report(*, scene: str, strategy: str, indices: int, invocations: int, batches: int,
                 shade_counts: np.ndarray | None = None, probe_stats=None) -> ReuseReport:
    """analytics.py:74-102: reuse_rate = 1 - invocations/indices; per-vertex tallies must add up."""
    per_vertex = None
    if shade_counts is not None:
        per_vertex = VertexShadingCounts(shade_counts)
        if per_vertex.total != invocations:
            raise AssertionError(
                f"per-vertex tallies sum to {per_vertex.total}, expected {invocations} invocations")
    reuse = 1.0 - invocations / indices if indices > 0 else 0.0
    return ReuseReport(scene=scene, strategy=strategy, indices=indices, invocations=invocations,
                       reuse_rate=reuse, batches=batches, per_vertex=per_vertex, probe_stats=probe_stats)


def ideal_report(mesh, scene: str = "") -> ReuseReport:
    """Reuse ceiling: one invocation per referenced vertex (analytics.py:105-119), counted on the device
    (vr_ideal_counts)."""
    from . import engine

    if len(mesh.indices) == 0:
        raise ValueError("empty index buffer")
    referenced, counts = engine.ideal_counts(engine.to_device_indices(mesh.indices), mesh.vertex_count)
    return build_report(scene=scene, strategy="ideal", indices=len(mesh.indices), invocations=referenced,
                        batches=1, shade_counts=counts.cpu().numpy().astype(np.int64))


@dataclass(frozen=True)
class CostEstimate:
    """analytics.py:53-71: abstract cost = invocations x ShaderFn.cycles."""

    invocations: int
    cycles_per_invocation: int
    total_cycles: int


def estimate_cost(report: ReuseReport, shader) -> CostEstimate:
    return CostEstimate(invocations=report.invocations, cycles_per_invocation=shader.cycles,
                        total_cycles=report.invocations * shader.cycles)
