"""Warp-collective semantics used by the voting strategy.

Host-side definitions mirroring `vrlab/warp.py` (/root/reference/pkg/src/vrlab/warp.py:14-76).
On the device these ARE the hardware intrinsics (`__shfl_sync`, `__ballot_sync`, `__ffs`) at
width 32; the functions below only pin the semantics (widths 4..64, the clamp of `lane_bit`)
that the CUDA kernels reproduce in closed form (csrc/vr_run.cu, csrc/vr_warp32.cu).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

DEFAULT_WIDTH = 32
ALLOWED_WIDTHS = (4, 8, 16, 32, 64)  # warp.py:14


def check_width(width: int) -> int:
    """warp.py:32-35."""
    if width not in ALLOWED_WIDTHS:
        raise ValueError(f"warp width must be one of {ALLOWED_WIDTHS}")
    return width


@dataclass(frozen=True)
class WarpState:
    """One 32-bit register per lane (warp.py:17-29)."""

    lanes: tuple

    def __post_init__(self):
        check_width(len(self.lanes))

    @property
    def width(self) -> int:
        return len(self.lanes)


def shfl(state: WarpState, src_lane: int) -> WarpState:
    """Broadcast of one lane's value (warp.py:38-44)."""
    if not 0 <= src_lane < state.width:
        raise ValueError(f"source lane {src_lane} out of range for width {state.width}")
    return WarpState((state.lanes[src_lane],) * state.width)


def ballot(predicates: Sequence[bool]) -> int:
    """Lane mask of true predicates (warp.py:47-55)."""
    return sum(1 << i for i, p in enumerate(predicates) if p)


def ffs(mask: int) -> int:
    """1-based lowest set bit, 0 when empty (warp.py:58-66)."""
    return (mask & -mask).bit_length() if mask else 0


def lane_bit(fill: int, width: int) -> int:
    """1 << fill, 0 at or past the warp width (warp.py:69-76)."""
    return 0 if fill >= width else 1 << fill
