"""Quadtree section ids and partitioning (API of rhseg/sections.py:21-79).

On the device path the partition is implicit: leaf section s of a side x side
grid reads its window of the HBM-resident cube directly (leaf_init_kernel), so
`partition` here only serves callers that want the host-side task list."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import IndivisibleImage
from .image import HyperImage


@dataclass(frozen=True, order=True)
class SectionId:
    level: int
    row: int
    col: int

    def __str__(self) -> str:
        return f"L{self.level}[{self.row},{self.col}]"

    def parent(self) -> "SectionId":
        return SectionId(self.level - 1, self.row // 2, self.col // 2)

    def children(self) -> list["SectionId"]:
        """NW, NE, SW, SE (sections.py:33-38)."""
        return [SectionId(self.level + 1, 2 * self.row + k // 2, 2 * self.col + k % 2) for k in range(4)]


@dataclass
class SectionTask:
    section_id: SectionId
    origin: tuple
    edge: int
    image: HyperImage | None = None


def section_side(level: int) -> int:
    return 1 << (level - 1)


def total_sections(levels: int) -> int:
    return sum(section_side(l) ** 2 for l in range(1, levels + 1))


def check_divisible(edge: int, levels: int) -> int:
    if levels < 1:
        raise ValueError(f"levels must be >= 1, got {levels}")
    side = section_side(levels)
    if edge % side:
        raise IndivisibleImage(f"edge {edge} not divisible by {side} (levels={levels})")
    return edge // side


def partition(image: HyperImage, levels: int) -> list[SectionTask]:
    """Leaf tasks, row-major, with sub-cube payloads (sections.py:57-79)."""
    sub = check_divisible(image.edge, levels)
    side = section_side(levels)
    return [
        SectionTask(SectionId(levels, r, c), (r * sub, c * sub), sub, image.subimage(r * sub, c * sub, sub))
        for r in range(side)
        for c in range(side)
    ]


def log_order(levels: int) -> list[SectionId]:
    """Level L down to 1, row-major within a level (recursive.py:95-104)."""
    return [
        SectionId(level, r, c)
        for level in range(levels, 0, -1)
        for r in range(section_side(level))
        for c in range(section_side(level))
    ]
