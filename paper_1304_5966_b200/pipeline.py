"""Entry points: align() and score_only() (reference pipeline.py:25-126).

Same signatures, return types, report keys and exceptions as the reference;
every DP pass, crossing and leaf runs on the B200 through libswb.so.
"""
from __future__ import annotations

import logging
import time
from dataclasses import dataclass

from . import phase1, phase2, phase3
from . import split as split_mod
from .engine import DEFAULT_BLOCK_COLS, DEFAULT_BLOCK_ROWS, Session, get_context
from .model import AlignmentPath, AlignmentSummary, ScoringScheme, Sequence, validate_scheme

logger = logging.getLogger(__name__)


@dataclass
class AlignConfig:
    """pipeline.AlignConfig (pipeline.py:25-43) plus the device ordinal.
    workers / block dims / concurrent_leaves / meter are validated and kept for
    API parity; the device decomposition does not depend on them (results are
    invariant to them in the reference too, SURVEY.md §0 finding 1)."""

    workers: int = 1
    block_rows: int = DEFAULT_BLOCK_ROWS
    block_cols: int = DEFAULT_BLOCK_COLS
    leaf_limit: int = phase3.DEFAULT_LEAF_LIMIT
    prune: bool = True
    band: bool = True
    split: int = 1
    concurrent_leaves: bool = False
    meter: object = None
    device: int = 0

    def __post_init__(self):
        if self.split not in (1, 2):
            raise ValueError("split must be 1 or 2")
        if self.workers < 1 or self.leaf_limit < 1:
            raise ValueError("workers and leaf_limit must be positive")
        if self.block_rows < 1 or self.block_cols < 1:
            raise ValueError("block dims must be positive")


def _report_phase1(report, scored, p1, S):
    if report is not None:
        report.update(score=scored.score, total_blocks=p1.total_blocks,
                      pruned_blocks=p1.pruned_blocks,
                      pruned_fraction=p1.pruned_blocks / max(1, p1.total_blocks),
                      cells_executed=p1.cells_executed, kernel_ms=p1.kernel_ms, kernel=p1.kernel,
                      rows_per_lane=p1.rows_per_lane)


def align(seq1: Sequence, seq2: Sequence, scheme: ScoringScheme,
          config: AlignConfig | None = None,
          report: dict | None = None) -> tuple[AlignmentSummary, AlignmentPath]:
    """Optimal local alignment: summary plus full path (pipeline.py:46-100)."""
    cfg = config or AlignConfig()
    if len(seq1) < 1 or len(seq2) < 1:
        raise ValueError("alignment inputs must be non-empty")
    scheme = validate_scheme(scheme)
    with Session(get_context(cfg.device), seq1.codes, seq2.codes, scheme) as S:
        S.meter = cfg.meter
        if cfg.split == 2:
            out = split_mod.split_align(S, cfg.leaf_limit, cfg.band, report)
            if report is not None:
                report.update(device_kernel_ms=S.kernel_ms, device_cells=S.cells)
            return out
        t0 = time.perf_counter()
        S.reset_bounds()  # tile bound maps for phases 2 and 3
        scored, p1 = phase1.best_local(S, cfg.prune)
        _report_phase1(report, scored, p1, S)
        return finish(S, scored, cfg, report, t0)


def finish(S: Session, scored: phase1.ScoredEndpoint, cfg: AlignConfig, report: dict | None,
           t0: float) -> tuple[AlignmentSummary, AlignmentPath]:
    """Phases 2 and 3 after a phase-1 endpoint (pipeline.py:75-100); shared by
    align() and multigpu.align_distributed()."""
    t1 = time.perf_counter()
    if scored.score == 0:
        return AlignmentSummary.empty(), AlignmentPath.empty()
    band = None
    if cfg.band:
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), S.scheme)
    start = phase2.locate_start(S, scored.end, scored.score, band)
    t2 = time.perf_counter()
    summary = AlignmentSummary(scored.score, start, scored.end)
    path = phase3.reconstruct(S, summary, cfg.leaf_limit, cfg.band, stats=report)
    t3 = time.perf_counter()
    if report is not None:
        report.update(device_kernel_ms=S.kernel_ms, device_cells=S.cells,
                      phase_seconds=(t1 - t0, t2 - t1, t3 - t2))
    return summary, path


def score_only(seq1: Sequence, seq2: Sequence, scheme: ScoringScheme,
               config: AlignConfig | None = None,
               report: dict | None = None) -> phase1.ScoredEndpoint:
    """Phase 1 alone: optimal local score and endpoint (pipeline.py:103-126)."""
    cfg = config or AlignConfig()
    if len(seq1) < 1 or len(seq2) < 1:
        raise ValueError("alignment inputs must be non-empty")
    scheme = validate_scheme(scheme)
    with Session(get_context(cfg.device), seq1.codes, seq2.codes, scheme) as S:
        scored, p1 = phase1.best_local(S, cfg.prune)
        _report_phase1(report, scored, p1, S)
        return scored
