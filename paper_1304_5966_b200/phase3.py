"""Phase 3: Myers-Miller reconstruction, level-synchronous on the device.

The reference recurses depth-first (phase3.solve_rect, phase3.py:250-286) and
runs two global passes per split.  Every split of one recursion level is
independent, so this module walks the recursion tree breadth-first: all
splits of a level go to the device in ONE swb_crossings call (both half passes
of every subproblem share one persistent launch; the middle-row combination
and _pick_crossing run on the device), and all leaves go to ONE swb_leaves
call at the end.  The tree, the child expected scores and vgap flags, the leaf
predicate and therefore the leaves and their order are exactly the
reference's, so the path is identical.  Host bookkeeping is vectorised numpy
over structured arrays.
"""
from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from .engine import SUBPROBLEM_DTYPE, Session
from .errors import DiscontiguousParts, ScoreMismatch
from .model import AlignmentPath, AlignmentSummary, Coord, Op, ScoringScheme, score_of_path

logger = logging.getLogger(__name__)

DEFAULT_LEAF_LIMIT = 128 * 128


@dataclass(frozen=True)
class Subproblem:
    start: Coord
    end: Coord
    expected: int
    start_vgap: bool = False
    end_vgap: bool = False

    @property
    def rows(self) -> int:
        return self.end.i - self.start.i

    @property
    def cols(self) -> int:
        return self.end.j - self.start.j


def band_interval(rows: int, cols: int, score: int, scheme: ScoringScheme) -> tuple[int, int]:
    """Admissible (row - col) corridor of a known-score global alignment
    (phase3.py:83-98)."""
    d = rows - cols
    denom = scheme.max_substitution_score + 2 * scheme.gap_extend
    g = (scheme.max_substitution_score * (rows + cols) - 2 * score) // denom
    g = min(max(g, abs(d)), rows + cols)
    pad = (g - abs(d)) // 2
    return min(0, d) - pad, max(0, d) + pad


def _as_array(subs: list[Subproblem], use_bounds: bool = False) -> np.ndarray:
    """Device form; prefix/suffix (scores before start and after end) start at
    0 for the root, which is the whole alignment."""
    a = np.zeros(len(subs), dtype=SUBPROBLEM_DTYPE)
    for t, s in enumerate(subs):
        a[t] = (s.start.i, s.start.j, s.end.i, s.end.j, s.expected, int(s.start_vgap),
                int(s.end_vgap), int(use_bounds), 0, 0, 0)
    return a


def find_crossing(S: Session, sub: Subproblem, band: bool = True) -> tuple[Coord, int, int, bool]:
    """Single-subproblem form of the batched crossing (phase3.py:136-190)."""
    if sub.rows < 2:
        raise ValueError("crossing needs at least two rows")
    res, cells = S.ctx.crossings(S.cs, S.s1, S.s2, _as_array([sub]), band)
    S.cells += cells
    r = res[0]
    if r["status"]:
        raise ScoreMismatch(f"middle-row combination reached {int(r['upper'])}, "
                            f"expected {sub.expected}")
    return Coord(int(r["mid_i"]), int(r["mid_j"])), int(r["upper"]), int(r["lower"]), \
        bool(r["gap_join"])


def _is_leaf(level: np.ndarray, leaf_limit: int) -> np.ndarray:
    rows = level["ei"] - level["si"]
    cols = level["ej"] - level["sj"]
    return (rows * cols <= leaf_limit) | (rows <= 1) | (cols <= 1)


def _split_level(S: Session, level: np.ndarray, band: bool) -> np.ndarray:
    """Replace every subproblem of `level` by its two children, in order
    (upper child first), via one batched device call."""
    meter = getattr(S, "meter", None)
    state = int((8 * (level["ej"] - level["sj"] + 1) + 2 * (level["ei"] - level["si"])).sum())
    if meter is not None:  # both halves' row buffers and final rows, lane state
        meter.add(state)
    try:
        res, cells = S.ctx.crossings(S.cs, S.s1, S.s2, level, band)
    finally:
        if meter is not None:
            meter.release(state)
    S.cells += cells
    bad = np.flatnonzero(res["status"])
    if bad.size:
        t = int(bad[0])
        raise ScoreMismatch(f"middle-row combination reached {int(res['upper'][t])}, "
                            f"expected {int(level['expected'][t])}")
    go = S.scheme.gap_open
    kids = np.zeros(2 * level.shape[0], dtype=SUBPROBLEM_DTYPE)
    up, dn = kids[0::2], kids[1::2]
    up["si"], up["sj"] = level["si"], level["sj"]
    up["ei"], up["ej"] = res["mid_i"], res["mid_j"]
    up["expected"] = res["upper"]
    up["start_vgap"] = level["start_vgap"]
    up["end_vgap"] = res["gap_join"]
    dn["si"], dn["sj"] = res["mid_i"], res["mid_j"]
    dn["ei"], dn["ej"] = level["ei"], level["ej"]
    dn["expected"] = res["lower"] + go * res["gap_join"].astype(np.int64)
    dn["start_vgap"] = res["gap_join"]
    dn["end_vgap"] = level["end_vgap"]
    # optimal-path scores before / after each child (the children's expected
    # scores partition the parent's), for tile-bound pruning
    up["use_bounds"] = dn["use_bounds"] = level["use_bounds"]
    up["prefix"] = level["prefix"]
    up["suffix"] = level["suffix"] + dn["expected"]
    dn["prefix"] = level["prefix"] + up["expected"]
    dn["suffix"] = level["suffix"]
    return kids


def collect_leaves(S: Session, root: np.ndarray, leaf_limit: int, band: bool,
                   stats: dict | None = None) -> np.ndarray:
    """Breadth-first Myers-Miller recursion; returns the leaves in path order."""
    frontier = root
    done = np.zeros(frontier.shape[0], dtype=bool)
    levels = 0
    while True:
        leaf = done | _is_leaf(frontier, leaf_limit)
        if leaf.all():
            if stats is not None:
                stats["mm_levels"] = stats.get("mm_levels", 0) + levels
                stats["mm_leaves"] = stats.get("mm_leaves", 0) + int(frontier.shape[0])
            return frontier
        inner = np.flatnonzero(~leaf)
        if stats is not None:
            import time
            t0, c0 = time.perf_counter(), S.cells
        kids = _split_level(S, frontier[inner], band)
        if stats is not None:
            sub = frontier[inner]
            area = int(((sub["ei"] - sub["si"]) * (sub["ej"] - sub["sj"])).sum())
            stats.setdefault("mm_level_stats", []).append(
                {"subs": int(inner.size), "area": area, "cells": int(S.cells - c0),
                 "wall_s": round(time.perf_counter() - t0, 4),
                 "kernel_ms": round(float(getattr(S.ctx, "last_kernel_ms", 0.0)), 3)})
        # splice: every inner node becomes two consecutive entries
        width = np.where(leaf, 1, 2)
        pos = np.concatenate(([0], np.cumsum(width)[:-1]))
        nxt = np.zeros(int(width.sum()), dtype=SUBPROBLEM_DTYPE)
        nxt_done = np.zeros(nxt.shape[0], dtype=bool)
        keep = np.flatnonzero(leaf)
        nxt[pos[keep]] = frontier[keep]
        nxt_done[pos[keep]] = True
        nxt[pos[inner]] = kids[0::2]
        nxt[pos[inner] + 1] = kids[1::2]
        frontier, done = nxt, nxt_done
        levels += 1


def solve_leaves(S: Session, leaves: np.ndarray, band: bool) -> np.ndarray:
    """phase3._solve_leaf (phase3.py:200-247) for every leaf, concatenated."""
    sc = S.scheme
    rows = leaves["ei"] - leaves["si"]
    cols = leaves["ej"] - leaves["sj"]
    parts: list = [None] * leaves.shape[0]
    # degenerate rectangles are closed-form (phase3.py:209-222)
    for t in np.flatnonzero((rows == 0) | (cols == 0)).tolist():
        r, c = int(rows[t]), int(cols[t])
        exp = int(leaves["expected"][t])
        svg, evg = bool(leaves["start_vgap"][t]), bool(leaves["end_vgap"][t])
        if r == 0 and c == 0:
            if exp != 0:
                raise ScoreMismatch("empty rectangle with nonzero expected score")
            parts[t] = np.empty(0, dtype=np.uint8)
        elif r == 0:
            if svg or evg:
                raise ScoreMismatch("vertical gap flags on a rectangle with no rows")
            if exp != -(sc.gap_open + c * sc.gap_extend):
                raise ScoreMismatch("pure insert run does not reproduce expected score")
            parts[t] = np.full(c, Op.INSERT, dtype=np.uint8)
        else:
            fee = 0 if svg else sc.gap_open
            if exp != -(fee + r * sc.gap_extend):
                raise ScoreMismatch("pure delete run does not reproduce expected score")
            parts[t] = np.full(r, Op.DELETE, dtype=np.uint8)
    real = np.flatnonzero((rows > 0) & (cols > 0))
    if real.size:
        sel = np.ascontiguousarray(leaves[real])
        ops, offsets, counts, scores = S.ctx.leaves(S.cs, S.s1, S.s2, sel, band)
        bad = np.flatnonzero((counts < 0) | (scores != sel["expected"]))
        if bad.size:
            t = int(bad[0])
            raise ScoreMismatch(
                f"leaf solve reached {int(scores[t])}, expected {int(sel['expected'][t])} "
                f"({int(rows[real[t]])}x{int(cols[real[t]])} rectangle at "
                f"{Coord(int(sel['si'][t]), int(sel['sj'][t]))})")
        for q, t in enumerate(real.tolist()):
            o = int(offsets[q])
            parts[t] = ops[o:o + int(counts[q])]
    if not parts:
        return np.empty(0, dtype=np.uint8)
    return np.concatenate(parts).astype(np.uint8, copy=False)


def solve_rect(S: Session, sub: Subproblem, leaf_limit: int = DEFAULT_LEAF_LIMIT,
               band: bool = True, stats: dict | None = None) -> np.ndarray:
    """Full op sequence of one known-score rectangle (phase3.py:250-286)."""
    import time
    t0 = time.perf_counter()
    leaves = collect_leaves(S, _as_array([sub], getattr(S, "bounds", False)), leaf_limit, band,
                            stats)
    t1 = time.perf_counter()
    ops = solve_leaves(S, leaves, band)
    if stats is not None:
        stats["t_crossings"] = stats.get("t_crossings", 0.0) + (t1 - t0)
        stats["t_leaves"] = stats.get("t_leaves", 0.0) + (time.perf_counter() - t1)
    return ops


def solve_rects(S: Session, subs: list[Subproblem], leaf_limit: int = DEFAULT_LEAF_LIMIT,
                band: bool = True, stats: dict | None = None) -> np.ndarray:
    """solve_rect for consecutive rectangles of one path (split mode's two
    halves of a midpoint alignment): one breadth-first recursion over all of
    them, so every level's crossings of every rectangle share a launch.  The
    leaves stay in path order, so the result is the concatenation of the
    rectangles' op sequences."""
    leaves = collect_leaves(S, _as_array(subs, getattr(S, "bounds", False)), leaf_limit, band,
                            stats)
    return solve_leaves(S, leaves, band)


def reconstruct(S: Session, summary: AlignmentSummary, leaf_limit: int = DEFAULT_LEAF_LIMIT,
                band: bool = True, stats: dict | None = None) -> AlignmentPath:
    """Full path for a summary from phases 1 and 2 (phase3.py:289-312)."""
    if summary.score == 0:
        return AlignmentPath.empty()
    ops = solve_rect(S, Subproblem(summary.start, summary.end, summary.score), leaf_limit, band,
                     stats)
    path = AlignmentPath(summary.start, ops)
    achieved = score_of_path(path, _Seq(S.codes1), _Seq(S.codes2), S.scheme)
    if achieved != summary.score:
        raise ScoreMismatch(f"reconstructed path scores {achieved}, expected {summary.score}")
    return path


class _Seq:
    """Minimal Sequence stand-in for score_of_path over raw code arrays."""

    def __init__(self, codes):
        self.codes = codes

    def __len__(self):
        return int(self.codes.size)


def join_paths(parts: list[AlignmentPath]) -> AlignmentPath:
    """Concatenate coordinate-contiguous sub-paths (phase3.py:315-327)."""
    if not parts:
        return AlignmentPath.empty()
    for a, b in zip(parts, parts[1:]):
        if a.end != b.start:
            raise DiscontiguousParts(f"part ends at {a.end} but next starts at {b.start}")
    return AlignmentPath(parts[0].start, np.concatenate([p.ops for p in parts]))
