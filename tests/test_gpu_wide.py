"""The int64 pass kernel (csrc/swb_wide.cu): passes whose dynamic range does
not fit the int32 kernels run on it instead of being refused, as the
reference computes in int64 (kernels.py:14).

* Option wide_log2 lowers the int32 limits so EVERY pass of an alignment runs
  on the int64 kernel; the golden records must still come out byte-equal.
* A scheme with scores and gap costs in the 10^5 range makes the passes
  exceed the int32 range for real; results equal the int64 CPU oracle.
"""
import numpy as np
import pytest

import oracle
from helpers import golden_inputs, mutate_codes, oracle_scheme, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Alphabet, ScoringScheme, Sequence, path_to_cigar
from paper_1304_5966_b200.engine import get_context

pytestmark = pytest.mark.gpu


@pytest.fixture
def all_wide():
    ctx = get_context(0)
    ctx.set_option("wide_log2", 4)
    try:
        yield ctx
    finally:
        ctx.set_option("wide_log2", 28)


def _summ(summary, path):
    return {"score": summary.score, "start": list(summary.start), "end": list(summary.end),
            "cigar": path_to_cigar(path)}


def test_goldens_on_the_wide_kernel(all_wide, golden_small, golden_medium, golden_protein):
    rep = {}
    for rec in golden_small[::5] + golden_medium + golden_protein[::4]:
        s1, s2, scheme = golden_inputs(rec)
        sc = swb.score_only(s1, s2, scheme, report=rep)
        assert {"score": sc.score, "end": list(sc.end)} == rec["score_only"]
        assert rep["kernel"] == "wide64"
        for tag, cfg in (("align", AlignConfig()),
                         ("align_leaf", AlignConfig(leaf_limit=rec["leaf_limit_small"])),
                         ("align_split", AlignConfig(split=2))):
            got = _summ(*swb.align(s1, s2, scheme, cfg))
            assert got == rec[tag], (tag, rec.get("tag"), got, rec[tag])


def test_final_rows_on_the_wide_kernel(all_wide):
    """Final rows (int64, sentinel drift included) equal the oracle's for
    every border family (engine.py:340-401)."""
    from paper_1304_5966_b200.engine import Session, TRACK_MAX, TRACK_MIN, TRACK_NONE
    rng = np.random.default_rng(5)
    a = random_codes(rng, 1500)
    b = mutate_codes(rng, a, 0.2)[:1300]
    scheme = ScoringScheme.match_mismatch(Alphabet.dna(wildcard=False), 2, -3, 4, 1)
    osch = oracle_scheme(scheme)
    for border, clamp, track in (("local", True, TRACK_MIN), ("restricted", False, TRACK_MAX),
                                 ("free", False, TRACK_NONE), ("continue", False, TRACK_MIN),
                                 ("charge", False, TRACK_MAX)):
        with Session(get_context(0), a, b, scheme) as S:
            r = S.run([dict(rows=(0, a.size, 0), cols=(0, b.size, 0), border=border, clamp=clamp,
                            track=track, want_final=True)])[0]
        assert r.kernel == "wide64"
        ref = oracle.run_wavefront(a, b, osch, border, clamp, track)
        assert np.array_equal(r.final_row_h, ref.final_h), border
        assert np.array_equal(r.final_row_f, ref.final_f), border
        if track != TRACK_NONE:
            assert (r.best_score, r.best_i, r.best_j) == (ref.best, ref.bi, ref.bj), border


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_scores_beyond_int32_range(seed):
    """match +100000 / mismatch -80000 / gap 50000 + 20000k: every pass of a
    3 kbp alignment exceeds the int32 kernels' range (the previous build
    raised ValueError / ERANGE here); the result equals the int64 oracle."""
    rng = np.random.default_rng(seed)
    a = random_codes(rng, 3000)
    b = mutate_codes(rng, a, 0.15)
    b = np.concatenate([random_codes(rng, 200), b, random_codes(rng, 150)])
    alpha = Alphabet.dna(wildcard=False)
    scheme = ScoringScheme.match_mismatch(alpha, 100000, -80000, 50000, 20000)
    s1, s2 = Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha)
    want = oracle.align(a, b, oracle_scheme(scheme))
    rep = {}
    summary, path = swb.align(s1, s2, scheme, report=rep)
    assert rep["kernel"] == "wide64"
    assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3]
    assert np.array_equal(path.ops, want[3])
    summary2, _ = swb.align(s1, s2, scheme, AlignConfig(split=2))
    assert summary2.score == summary.score
