"""Phase 2: reverse start-point pass (phase2.py).

The restricted pass runs over the reversed prefixes ending at the phase-1
endpoint, addressed as reversed slices of the device-resident sequences (no
host copies).  Band arithmetic is host-side integer math identical to the
reference (Ukkonen corridor widened to the indel budget).
"""
from __future__ import annotations

import logging
import math
import os
from dataclasses import dataclass

from .engine import TRACK_MAX, Session, bound_slack
from .errors import StartNotFound
from .model import Coord, ScoringScheme

logger = logging.getLogger(__name__)


@dataclass(frozen=True)
class BandSpec:
    t: int
    m_prime: int
    p: int
    lo: int
    hi: int
    degenerate: bool = False


def compute_band(score: int, n_short: int, m_long: int, scheme: ScoringScheme) -> BandSpec:
    """Corridor for a known-score alignment ending at the origin (phase2.py:45-64)."""
    if score < 1:
        raise ValueError("banding needs a positive known score")
    if n_short > m_long:
        raise ValueError("n_short must not exceed m_long")
    t = score // scheme.max_substitution_score
    degenerate = t > n_short
    if degenerate:
        logger.warning("degenerate band: deformation %d exceeds short length %d; clamping",
                       t, n_short)
        t = n_short
    m_prime = min(n_short + (n_short - t) // scheme.gap_extend, m_long)
    p = max(0, math.ceil(0.5 * (2 * n_short - t - m_prime)))
    return BandSpec(t, m_prime, p, -p, p + (m_long - n_short), degenerate)


def indel_budget(score: int, n_short: int, scheme: ScoringScheme) -> int:
    return max(0, (scheme.max_substitution_score * n_short - score) // scheme.gap_extend)


def applied_interval(band: BandSpec, score: int, n_short: int,
                     scheme: ScoringScheme) -> tuple[int, int]:
    g = indel_budget(score, n_short, scheme)
    return min(band.lo, -g), max(band.hi, g)


def oriented_interval(band: BandSpec, score: int, rows: int, cols: int,
                      scheme: ScoringScheme) -> tuple[int, int]:
    """Longer-minus-shorter corridor -> this pass's (row - col) units
    (phase2.py:155-163)."""
    lo, hi = applied_interval(band, score, min(rows, cols), scheme)
    return (lo, hi) if rows >= cols else (-hi, -lo)


def restricted_search(S: Session, rows: tuple, cols: tuple, target: int, interval,
                      preopen_vgap: bool = False, track: int = TRACK_MAX,
                      gap_tolerant: bool = False, bounds: bool = False,
                      maps: tuple[int, int] = (1, 2)) -> tuple[int, int]:
    """Origin-anchored pass returning the cell that attains `target`
    (phase2.py:82-138).  rows/cols are (offset, length, reversed) slices.
    With bounds, the pass skips blocks the tile map maps[0] proves useless and
    records its own bounds in map maps[1] (1 forward, 2 reverse; DESIGN.md
    §3.6): a reversed search (phase 2) reads the forward map of the local pass
    and writes the reverse map, a forward search from a known start (split
    mode) reads the reverse map and writes the forward one."""
    if gap_tolerant or preopen_vgap:
        border = "continue" if preopen_vgap else "free"
    else:
        border = "restricted"
    # prune kind 2: blocks from which no path can reach `target` are skipped
    # (sound: every cell attaining target keeps its exact value).
    # bounds: the phase-1 tile map bounds what the rest of the path (up to the
    # start) can add, and this pass records its own tile map for phase 3 (§3.6).
    extra = {}
    if bounds and S.bounds and S.target_prune:
        extra = dict(bound_read=maps[0], bound_write=maps[1], bound_offset=bound_slack(S.scheme))
    res = S.run([dict(rows=rows, cols=cols, border=border, clamp=False, track=track,
                      band=interval, prune=2 if S.target_prune else 0,
                      prune_target=target, **extra)])[0]
    if res.best_i < 0 or res.best_score != target:
        found = res.best_score if res.best_i >= 0 else "none"
        if os.environ.get("SWB_DUMP_ON_FAIL"):  # per-strip record of the failed launch
            print(f"restricted pass {rows} x {cols} band {interval} target {target}: "
                  f"{res} launches {S.ctx.launch_count}\n{S.ctx.debug_strips().tolist()}\n"
                  f"claims {S.ctx.debug_claims(S.ctx.launch_count - 1).tolist()}", flush=True)
        raise StartNotFound(f"no cell attains the known score {target} (best found: {found}); "
                            "this indicates an internal bug")
    return res.best_i, res.best_j


def locate_start(S: Session, end: Coord, score: int, band: BandSpec | None) -> Coord:
    """Smallest (i, j) where an optimal alignment ending at `end` begins
    (phase2.py:141-165)."""
    if score < 1:
        raise ValueError("locate_start needs a positive score")
    interval = None
    if band is not None:
        interval = oriented_interval(band, score, end.i, end.j, S.scheme)
    ri, rj = restricted_search(S, (0, end.i, 1), (0, end.j, 1), score, interval, bounds=True)
    return Coord(end.i - ri - 1, end.j - rj - 1)
