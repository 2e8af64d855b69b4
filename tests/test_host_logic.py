"""Host-side logic of the device pipeline, tested on CPU.

The level-synchronous Myers-Miller driver (phase3.collect_leaves /
solve_leaves) and the split classification are pure host bookkeeping around
the device operators.  Here the device operators are replaced by a stub that
answers from the CPU oracle (test infrastructure only — the product path has
no CPU fallback), so the breadth-first splicing, child expected scores, vgap
flags, leaf predicate and path order can be checked against the reference's
depth-first recursion (phase3.py:250-286, restated in oracle/pipeline.py)."""
import numpy as np
import pytest

import oracle
from oracle import pipeline as opl
from helpers import dna_scheme, golden_inputs, mutate_codes, oracle_scheme, random_codes
from paper_1304_5966_b200 import Coord, phase2, phase3, split
from paper_1304_5966_b200.engine import CROSSING_DTYPE, SUBPROBLEM_DTYPE
from paper_1304_5966_b200.model import AlignmentSummary


class OracleCtx:
    """Answers swb_crossings / swb_leaves from the CPU oracle."""

    def __init__(self, c1, c2, osch):
        self.c1, self.c2, self.osch = c1, c2, osch
        self.calls = 0

    def crossings(self, cs, s1, s2, subs, band):
        self.calls += 1
        out = np.zeros(subs.shape[0], dtype=CROSSING_DTYPE)
        for t, s in enumerate(subs):
            sub = ((int(s["si"]), int(s["sj"])), (int(s["ei"]), int(s["ej"])), int(s["expected"]),
                   bool(s["start_vgap"]), bool(s["end_vgap"]))
            (mi, mj), up, lo, gap = opl._crossing(sub, self.c1, self.c2, self.osch, band, 1)
            out[t] = (mi, mj, up, lo, int(gap), 0)
        return out, 0

    def leaves(self, cs, s1, s2, subs, band):
        n = subs.shape[0]
        rows = subs["ei"] - subs["si"]
        cols = subs["ej"] - subs["sj"]
        cap = rows + cols
        offsets = np.zeros(n, dtype=np.int64)
        offsets[1:] = np.cumsum(cap)[:-1]
        ops = np.zeros(int(cap.sum()) + 1, dtype=np.uint8)
        counts = np.zeros(n, dtype=np.int64)
        scores = np.zeros(n, dtype=np.int64)
        for t, s in enumerate(subs):
            r, c, e = int(rows[t]), int(cols[t]), int(s["expected"])
            lo, hi = opl._mm_band(r, c, e, self.osch) if band else (-(r + c), r + c)
            sc, o = oracle.leaf_solve(self.c1[s["si"]:s["ei"]], self.c2[s["sj"]:s["ej"]], self.osch,
                                      bool(s["start_vgap"]), bool(s["end_vgap"]), lo, hi)
            scores[t] = sc
            counts[t] = -1 if o is None else o.size
            if o is not None:
                ops[offsets[t]:offsets[t] + o.size] = o
        return ops, offsets, counts, scores


class FakeSession:
    def __init__(self, c1, c2, scheme):
        self.codes1, self.codes2, self.scheme = c1, c2, scheme
        self.n1, self.n2 = c1.size, c2.size
        self.ctx = OracleCtx(c1, c2, oracle_scheme(scheme))
        self.cs = self.s1 = self.s2 = None
        self.cells = 0
        self.kernel_ms = 0.0


@pytest.mark.parametrize("seed,leaf_limit", [(1, 16), (2, 64), (3, 300), (4, 4), (5, 1024)])
def test_bfs_reconstruction_equals_dfs(seed, leaf_limit):
    rng = np.random.default_rng(seed)
    a = random_codes(rng, 700)
    b = mutate_codes(rng, a, 0.2)
    scheme = dna_scheme()
    osch = oracle_scheme(scheme)
    score, start, end, ops = oracle.align(a, b, osch, leaf_limit=leaf_limit)
    S = FakeSession(a, b, scheme)
    summ = AlignmentSummary(score, Coord(*start), Coord(*end))
    stats = {}
    path = phase3.reconstruct(S, summ, leaf_limit=leaf_limit, stats=stats)
    assert np.array_equal(path.ops, ops)
    assert stats["mm_leaves"] >= 1


def test_bfs_with_vgap_flags_from_goldens(golden_small):
    # instances whose reference path crosses split rows inside gaps
    hit = 0
    for rec in golden_small[:400]:
        s1, s2, scheme = golden_inputs(rec)
        want = rec["align_leaf"]
        if want["score"] == 0:
            continue
        S = FakeSession(s1.codes, s2.codes, scheme)
        summ = AlignmentSummary(want["score"], Coord(*want["start"]), Coord(*want["end"]))
        path = phase3.reconstruct(S, summ, leaf_limit=rec["leaf_limit_small"])
        from paper_1304_5966_b200 import path_to_cigar
        assert path_to_cigar(path) == want["cigar"]
        hit += 1
    assert hit > 100


def test_band_helpers_match_reference_formulas():
    scheme = dna_scheme()
    for rows, cols, score in [(10, 12, 5), (100, 80, 40), (7, 7, 7), (1000, 990, 100)]:
        assert phase3.band_interval(rows, cols, score, scheme) == opl._mm_band(rows, cols, score,
                                                                               oracle_scheme(scheme))
    # compute_band worked example (test_phase2.py:22-47 style): C1 numbers, SURVEY §8a P2-1
    b = phase2.compute_band(4842, 10000, 10000, scheme)
    assert (b.t, b.m_prime, b.p) == (4842, 10000, 2579)
    lo, hi = phase2.applied_interval(b, 4842, 10000, scheme)
    assert lo <= b.lo and hi >= b.hi


def test_classify_midcase_ties():
    mk = lambda u, m, l: split.MidCombine(u, Coord(0, 0), l, Coord(0, 0), m, 0, False, 0, 0)
    assert split.classify_midcase(mk(5, 5, 5)) == "upper"
    assert split.classify_midcase(mk(4, 5, 5)) == "midpoint"
    assert split.classify_midcase(mk(4, 4, 5)) == "lower"
    assert split.classify_midcase(mk(0, 0, 0)) == "upper"


def test_pick_crossing_tie_rules():
    hh = np.array([1, 5, 3, 5], dtype=np.int64)
    ff = np.array([5, 0, 0, 0], dtype=np.int64)
    assert split.pick_crossing(hh, ff) == (5, 0, True)
    ff2 = np.array([0, 5, 0, 0], dtype=np.int64)
    assert split.pick_crossing(hh, ff2) == (5, 1, False)


def test_leaf_predicate_and_splice_order():
    lvl = np.zeros(3, dtype=SUBPROBLEM_DTYPE)
    lvl["ei"] = [1, 200, 10]
    lvl["ej"] = [500, 300, 10]
    assert phase3._is_leaf(lvl, 16384).tolist() == [True, False, True]


class RecordingCtx(OracleCtx):
    def __init__(self, *a):
        super().__init__(*a)
        self.seen = []

    def crossings(self, cs, s1, s2, subs, band):
        self.seen.append(subs.copy())
        return super().crossings(cs, s1, s2, subs, band)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_prefix_suffix_partition_the_score(seed):
    """Tile-bound pruning needs, for every Myers-Miller
    subproblem, the optimal path's score before its start (prefix) and after
    its end (suffix): prefix + expected + suffix must equal the total at every
    level, and the leaves' prefixes must be the running sums of their
    expected scores in path order."""
    rng = np.random.default_rng(seed)
    a = random_codes(rng, 900)
    b = mutate_codes(rng, a, 0.15)
    scheme = dna_scheme()
    osch = oracle_scheme(scheme)
    score, start, end, ops = oracle.align(a, b, osch, leaf_limit=64)
    S = FakeSession(a, b, scheme)
    S.ctx = RecordingCtx(a, b, osch)
    S.bounds = True
    root = phase3._as_array([phase3.Subproblem(Coord(*start), Coord(*end), score)], True)
    leaves = phase3.collect_leaves(S, root, 64, True)
    assert len(S.ctx.seen) >= 3
    for level in S.ctx.seen:
        assert (level["use_bounds"] == 1).all()
        assert (level["prefix"] + level["expected"] + level["suffix"] == score).all()
    assert (leaves["prefix"] + leaves["expected"] + leaves["suffix"] == score).all()
    run = np.concatenate(([0], np.cumsum(leaves["expected"])[:-1]))
    assert np.array_equal(leaves["prefix"], run)
    path = phase3.reconstruct(S, AlignmentSummary(score, Coord(*start), Coord(*end)), leaf_limit=64)
    assert np.array_equal(path.ops, ops)
