"""Quadtree section ids and partitioning (API of rhseg/sections.py:21-79).

On the device path the partition is implicit: leaf section s of a side x side
grid reads its window of the HBM-resident cube directly (leaf_init_kernel), so
`partition` here only serves callers that want the host-side task list."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import IndivisibleImage, ShapeMismatch
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


def stitch(quadrants, connectivity: int = 8):
    """sections.py:103-163 as a host helper on RegionGraph objects (the device path
    stitches whole levels in stitch_kernel): NW, NE, SW, SE children renumbered densely
    (each child's live ids ascending, children in order), sums and counts carried over
    exactly, and every pixel adjacency across the two internal seams linked."""
    from .graph import Region, RegionGraph, neighbor_offsets

    if len(quadrants) != 4:
        raise ShapeMismatch(f"stitch needs exactly 4 quadrants, got {len(quadrants)}")
    e, bands = quadrants[0].width, quadrants[0].bands
    for g in quadrants:
        if g.width != e or g.height != e:
            raise ShapeMismatch("quadrants differ in size")
        if g.bands != bands:
            raise ShapeMismatch("quadrants differ in band count")
    neighbor_offsets(connectivity)  # validates
    n = 2 * e
    out = RegionGraph(n, n, bands)
    grid = np.empty((n, n), np.int64)
    base = 0
    for k, g in enumerate(quadrants):
        ids = np.array(sorted(g.regions), np.int64)
        orow, ocol = (k // 2) * e, (k % 2) * e
        local = np.asarray(g.pixel_assignment, np.int64).reshape(e, e)
        grid[orow:orow + e, ocol:ocol + e] = base + np.searchsorted(ids, local)
        remap = {int(r): base + i for i, r in enumerate(ids.tolist())}
        for rid, i in remap.items():
            reg = g.regions[rid]
            p = np.asarray(reg.pixels, np.int64)
            out.regions[i] = Region(i, reg.pixel_count, reg.band_sums.copy(), {remap[a] for a in reg.adjacency},
                                    ((orow + p // e) * n + ocol + p % e).tolist())
        base += len(ids)
    out.pixel_assignment = grid.reshape(-1).copy()
    # seams: column e-1 | e and row e-1 | e, plus both diagonals across each under 8-connectivity
    pairs = [(grid[:, e - 1], grid[:, e]), (grid[e - 1, :], grid[e, :])]
    if connectivity == 8:
        pairs += [(grid[:-1, e - 1], grid[1:, e]), (grid[:-1, e], grid[1:, e - 1]),
                  (grid[e - 1, :-1], grid[e, 1:]), (grid[e - 1, 1:], grid[e, :-1])]
    for a, b in pairs:
        m = a != b
        for x, y in zip(a[m].tolist(), b[m].tolist()):
            out.regions[x].adjacency.add(y)
            out.regions[y].adjacency.add(x)
    return out
