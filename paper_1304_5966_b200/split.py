"""Dual-half scoring with the paper's Figure-1 middle-row combine (split.py).

The upper-forward and lower-reversed local passes run as two jobs of ONE
persistent device launch (on one B200 the "two cards" of the paper are two
job chains sharing the SMs; across GPUs, multigpu.split_align_distributed
gives each half its own GPU group).  Their final rows meet at the middle row
exactly like a Myers-Miller split; the three candidate optima are classified
with the reference's tie order and each case is finished with the
phase-2/phase-3 device operators.

Fast path: both halves run on the packed 16x2 kernel with
phase-1 pruning against a running best SHARED by the two halves, each half's
bound counting the rows of the other half (rows_after), so every cell of an
optimal alignment — upper, lower or through the middle row — keeps its exact
value, while cells that cannot reach the optimum become fill.  The combine is
exact wherever it matters: a column whose true sum hh or ff equals the
optimum lies on an optimal path; any other column can only be
under-estimated, which cannot change the classification (ties included).  The
halves also record tile bound maps (upper: forward map, lower: reverse map of
the reversed local pass = a bound on the best path leaving a cell), so the
finishing restricted searches and Myers-Miller passes skip tiles as in
split=1.
"""
from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from . import phase2, phase3
from .engine import TRACK_MAX, TRACK_MIN, Session
from .errors import ScoreMismatch
from .model import AlignmentPath, AlignmentSummary, Coord, score_of_path

logger = logging.getLogger(__name__)


@dataclass
class MidCombine:
    upper_score: int
    upper_end: Coord
    lower_score: int
    lower_start: Coord
    mid_score: int
    mid_col: int
    gap_join: bool
    upper_seg: int
    lower_seg: int


def classify_midcase(mc: MidCombine) -> str:
    """Argmax of the three candidates; ties upper > midpoint > lower (split.py:55-61)."""
    if mc.upper_score >= mc.mid_score and mc.upper_score >= mc.lower_score:
        return "upper"
    return "midpoint" if mc.mid_score >= mc.lower_score else "lower"


def pick_crossing(hh: np.ndarray, ff: np.ndarray) -> tuple[int, int, bool]:
    """phase3._pick_crossing (phase3.py:123-133): best, smallest column, plain
    join before gap join at the same column."""
    best = max(int(hh.max()), int(ff.max()))
    big = np.iinfo(np.int64).max
    jh = int(np.argmax(hh == best)) if (hh == best).any() else big
    jf = int(np.argmax(ff == best)) if (ff == best).any() else big
    return (best, jh, False) if jh <= jf else (best, jf, True)


def _search_interval(score, rows, cols, scheme, band):
    if not band:
        return None
    bspec = phase2.compute_band(score, min(rows, cols), max(rows, cols), scheme)
    return phase2.oriented_interval(bspec, score, rows, cols, scheme)


def split_align(S: Session, leaf_limit: int = phase3.DEFAULT_LEAF_LIMIT, band: bool = True,
                report: dict | None = None, fast: bool = True
                ) -> tuple[AlignmentSummary, AlignmentPath]:
    """split.split_align (split.py:84-182).  fast=False runs the two halves as
    the reference does (no pruning, no tile maps)."""
    import time
    from .multigpu import Boundary
    t0 = time.perf_counter()
    n1, n2 = S.n1, S.n2
    mid = n1 // 2
    best = None
    if fast:
        S.reset_bounds()
        best = Boundary(S.ctx, 1)  # its progress word: the running best of both halves
    try:
        specs = half_specs(n1, n2, mid, best.progress if best else 0)
        res = S.run(specs if mid >= 1 else specs[1:])
    finally:
        if best is not None:
            best.free()
    res_up, res_dn = (res[0], res[1]) if mid >= 1 else (None, res[0])
    t1 = time.perf_counter()
    out = combine_and_finish(S, res_up, res_dn, mid, leaf_limit, band, report)
    if report is not None:
        report.update(phase_seconds=(t1 - t0, time.perf_counter() - t1),
                      halves_cells=(res_up.cells_executed if res_up else 0) + res_dn.cells_executed)
    return out


def half_specs(n1: int, n2: int, mid: int, shared_best: int) -> list[dict]:
    """Session.run() specs of the upper-forward and lower-reversed local passes
    (split.py:64-81, :103-122).  With a shared best (fast path) both prune
    against the running best of the two, each counting the other half's rows
    (rows_after), and they record the forward / reverse tile maps."""
    up = dict(rows=(0, mid, 0), cols=(0, n2, 0), border="local", clamp=True, track=TRACK_MIN,
              want_final=True)
    dn = dict(rows=(mid, n1 - mid, 1), cols=(0, n2, 1), border="local", clamp=True,
              track=TRACK_MIN, want_final=True)
    if shared_best:
        up.update(prune=True, shared_best=shared_best, rows_after=n1 - mid, bound_write=1)
        dn.update(prune=True, shared_best=shared_best, rows_after=mid, bound_write=2)
    return [up, dn]


def combine_and_finish(S: Session, res_up, res_dn, mid: int, leaf_limit: int, band: bool,
                       report: dict | None) -> tuple[AlignmentSummary, AlignmentPath]:
    """Middle-row combine of the two halves' results (split.py:124-149) and the
    three-case finish (split.py:150-182); shared with the multi-GPU split."""
    n1, n2 = S.n1, S.n2
    go = S.scheme.gap_open
    if res_up is not None:
        upper_score = max(0, res_up.best_score)
        upper_end = Coord(res_up.best_i + 1, res_up.best_j + 1) if upper_score > 0 else Coord(0, 0)
        hh = res_up.final_row_h + res_dn.final_row_h[::-1]
        ff = res_up.final_row_f + res_dn.final_row_f[::-1] + go
        mid_score, jc, gap_join = pick_crossing(hh, ff)
        if gap_join:
            upper_seg, lower_seg = int(res_up.final_row_f[jc]), int(res_dn.final_row_f[n2 - jc])
        else:
            upper_seg, lower_seg = int(res_up.final_row_h[jc]), int(res_dn.final_row_h[n2 - jc])
    else:
        upper_score, upper_end = 0, Coord(0, 0)
        mid_score, jc, gap_join, upper_seg, lower_seg = 0, 0, False, 0, 0
    lower_score = max(0, res_dn.best_score)
    lower_start = (Coord(n1 - (res_dn.best_i + 1), n2 - (res_dn.best_j + 1))
                   if lower_score > 0 else Coord(0, 0))
    mc = MidCombine(upper_score, upper_end, lower_score, lower_start, int(mid_score), int(jc),
                    bool(gap_join), upper_seg, lower_seg)
    case = classify_midcase(mc)
    if report is not None:
        report.update(case=case, upper_score=mc.upper_score, lower_score=mc.lower_score,
                      mid_score=mc.mid_score, upper_rows=(0, mid), lower_rows=(mid, n1),
                      upper_cells=res_up.cells_executed if res_up else 0,
                      lower_cells=res_dn.cells_executed)
    logger.debug("split case %s (upper=%d lower=%d mid=%d)", case, mc.upper_score,
                 mc.lower_score, mc.mid_score)
    if case == "upper":
        if mc.upper_score == 0:
            return AlignmentSummary.empty(), AlignmentPath.empty()
        return _finish_upper(S, mc, leaf_limit, band)
    if case == "lower":
        return _finish_lower(S, mc, leaf_limit, band)
    return _finish_midpoint(S, mc, mid, leaf_limit, band)


def _finish_upper(S, mc, leaf_limit, band):
    score, end = mc.upper_score, mc.upper_end
    bspec = phase2.compute_band(score, min(end), max(end), S.scheme) if band else None
    start = phase2.locate_start(S, end, score, bspec)
    summary = AlignmentSummary(score, start, end)
    return summary, phase3.reconstruct(S, summary, leaf_limit, band)


def _finish_lower(S, mc, leaf_limit, band):
    score, start = mc.lower_score, mc.lower_start
    rows, cols = S.n1 - start.i, S.n2 - start.j
    iv = _search_interval(score, rows, cols, S.scheme, band)
    ci, cj = phase2.restricted_search(S, (start.i, rows, 0), (start.j, cols, 0), score, iv,
                                      track=TRACK_MIN, bounds=True, maps=(2, 1))
    summary = AlignmentSummary(score, start, Coord(start.i + ci + 1, start.j + cj + 1))
    return summary, phase3.reconstruct(S, summary, leaf_limit, band)


def _finish_midpoint(S, mc, mid, leaf_limit, band):
    jc, gap = mc.mid_col, mc.gap_join
    go = S.scheme.gap_open
    cross = Coord(mid, jc)
    upper_target = mc.upper_seg + (go if gap else 0)
    lower_expected = mc.lower_seg + (go if gap else 0)
    parts = []
    if not gap and mc.upper_seg == 0:
        ustart = cross
    else:
        iv = _search_interval(upper_target, mid, jc, S.scheme, band) if upper_target >= 1 else None
        ri, rj = phase2.restricted_search(S, (0, mid, 1), (0, jc, 1), upper_target, iv,
                                          preopen_vgap=gap, track=TRACK_MAX, gap_tolerant=True,
                                          bounds=True, maps=(1, 2))
        ustart = Coord(mid - ri - 1, jc - rj - 1)
        parts.append(phase3.Subproblem(ustart, cross, mc.upper_seg, start_vgap=False,
                                       end_vgap=gap))
    rows, cols = S.n1 - mid, S.n2 - jc
    iv = (_search_interval(lower_expected, rows, cols, S.scheme, band)
          if lower_expected >= 1 else None)
    ci, cj = phase2.restricted_search(S, (mid, rows, 0), (jc, cols, 0), lower_expected, iv,
                                      preopen_vgap=gap, track=TRACK_MIN, gap_tolerant=True,
                                      bounds=True, maps=(2, 1))
    lend = Coord(mid + ci + 1, jc + cj + 1)
    parts.append(phase3.Subproblem(cross, lend, lower_expected, start_vgap=gap, end_vgap=False))
    # both rectangles in one breadth-first recursion (= join_paths of the two)
    path = AlignmentPath(ustart, phase3.solve_rects(S, parts, leaf_limit, band))
    summary = AlignmentSummary(mc.mid_score, ustart, lend)
    if path.end != lend:
        raise ScoreMismatch(f"joined midpoint path ends at {path.end}, expected {lend}")
    achieved = score_of_path(path, phase3._Seq(S.codes1), phase3._Seq(S.codes2), S.scheme)
    if achieved != summary.score:
        raise ScoreMismatch(f"joined midpoint path scores {achieved}, expected {summary.score}")
    return summary, path
