"""Phase 1: forward local score pass with upper-bound pruning (phase1.py).

The whole pass is one persistent device launch (csrc/swb_kernels.cuh): local
borders, clamp at zero, TRACK_MIN (best positive cell, ties to the
lexicographically smallest (i, j)), and block pruning with the reference's
bound evaluated per 32-column warp tile against a device-global running best.
"""
from __future__ import annotations

from dataclasses import dataclass

from .engine import TRACK_MIN, PassResult, Session
from .model import Coord


@dataclass(frozen=True)
class ScoredEndpoint:
    score: int
    end: Coord


def prune_verdict(best_so_far: int, max_substitution_score: int, len1: int, len2: int,
                  input_max: int, origin: Coord) -> bool:
    """The pruning bound (phase1.py:24-41): no path through a tile whose
    best entering H is input_max can reach best_so_far.  The device kernel
    applies max(input_max, 0) + max_sub * min(rows left, cols left) < best."""
    remaining = min(len1 - origin.i, len2 - origin.j)
    return input_max + max_substitution_score * remaining < best_so_far


def best_local(S: Session, prune: bool = True) -> tuple[ScoredEndpoint, PassResult]:
    """Optimal local score and endpoint over the full matrix (phase1.py:44-85).
    When the session's tile bound maps are on, the pass also records an upper
    bound of H per tile for phases 2 and 3."""
    res = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                      track=TRACK_MIN, prune=prune, bound_write=1 if S.bounds else 0)])[0]
    if res.best_score <= 0:
        return ScoredEndpoint(0, Coord(0, 0)), res
    return ScoredEndpoint(res.best_score, Coord(res.best_i + 1, res.best_j + 1)), res
