"""Multi-GPU decomposition of a wavefront pass.

A pass is one chain of warp-strips; across GPUs the chain simply continues:
GPU g owns a contiguous *row slab* of strips, and the bottom DP row of slab g
(H and F for every column, index 0 = left border) is the top border of slab
g+1.  On NVLink the device kernels stream that row through peer-mapped memory
strip block by strip block (publication protocol of DESIGN.md §3.2); the host
logic here — partitioning, the row handed over, the final merge of per-slab
bests with the reference's tie rules (engine.py:247-259) — is shared by the
device path and by the world-size-2 gloo test (tests/test_multigpu_gloo.py),
which checks that a slab-split pass reproduces the single pass exactly.
"""
from __future__ import annotations

from dataclasses import dataclass

TRACK_NONE, TRACK_MIN, TRACK_MAX = 0, 1, 2


@dataclass(frozen=True)
class Slab:
    rank: int
    row0: int  # first DP row owned (cell row index)
    row1: int  # one past the last

    @property
    def rows(self) -> int:
        return self.row1 - self.row0


def slab_partition(n1: int, world: int, strip_rows: int = 1024) -> list[Slab]:
    """Split n1 rows into `world` contiguous slabs of whole strips, as even as
    possible (the last slab takes the ragged remainder).  Every rank gets at
    least one row when n1 >= world."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if n1 < 1:
        raise ValueError("cannot partition an empty pass")
    strips = -(-n1 // strip_rows)
    bounds = []
    for g in range(world + 1):
        k = (strips * g) // world
        bounds.append(min(n1, k * strip_rows))
    if strips < world:  # fewer strips than ranks: split rows directly
        bounds = [(n1 * g) // world for g in range(world + 1)]
    return [Slab(g, bounds[g], bounds[g + 1]) for g in range(world)]


def merge_best(results: list[tuple[int, int, int]], track: int) -> tuple[int, int, int]:
    """Combine per-slab (score, i, j) with absolute rows; i < 0 means none.
    TRACK_MIN: max score, ties to the smallest (i, j), only positive scores;
    TRACK_MAX: max score, ties to the largest (i, j)."""
    best = None
    for s, i, j in results:
        if i < 0:
            continue
        if track == TRACK_MIN and s <= 0:
            continue
        if best is None:
            best = (s, i, j)
            continue
        bs, bi, bj = best
        if track == TRACK_MIN:
            take = s > bs or (s == bs and (i, j) < (bi, bj))
        else:
            take = s > bs or (s == bs and (i, j) > (bi, bj))
        if take:
            best = (s, i, j)
    if best is None:
        return (0, -1, -1) if track == TRACK_MIN else (-(2 ** 61), -1, -1)
    return best


def handoff_bytes(n2: int) -> int:
    """Bytes one slab boundary moves over NVLink: (H, F) int32 per column."""
    return 8 * n2
