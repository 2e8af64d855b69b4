"""Full-size properties (BASELINE configs C2 scale) that need no CPU oracle:
pruning invariance, decomposition invariance (split=2 vs split=1 scores,
row slabs vs one pass), reversal symmetry of the local score, and path
self-consistency (re-score == score, path end == end) of a full alignment."""
import numpy as np
import pytest

from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Sequence
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.multigpu import SLAB_STRIP_ROWS, run_slabs_sequential, slab_partition

pytestmark = pytest.mark.gpu

SCHEME = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)


def seqs(a, b):
    return Sequence.from_codes("a", a, SCHEME.alphabet), Sequence.from_codes("b", b, SCHEME.alphabet)


@pytest.fixture(scope="module")
def c2_pair():
    return synthetic_pair(1_000_000, seed=1002)


def test_c2_prune_invariance_and_slabs(c2_pair):
    a, b = c2_pair
    s1, s2 = seqs(a, b)
    on = swb.score_only(s1, s2, SCHEME, AlignConfig(prune=True))
    off = swb.score_only(s1, s2, SCHEME, AlignConfig(prune=False))
    assert (on.score, on.end) == (off.score, off.end)
    assert on.score > 0.4 * a.size
    with Session(get_context(0), a, b, SCHEME) as S:
        merged, _ = run_slabs_sequential(S, slab_partition(S.n1, 4, SLAB_STRIP_ROWS))
    assert merged == (on.score, on.end.i - 1, on.end.j - 1)


def test_c2_reversal_symmetry(c2_pair):
    a, b = c2_pair
    fwd = swb.score_only(*seqs(a, b), SCHEME)
    rev = swb.score_only(*seqs(a[::-1].copy(), b[::-1].copy()), SCHEME)
    assert fwd.score == rev.score


def test_unrelated_scores_small_and_symmetric():
    a, b = synthetic_pair(1_000_000, seed=1004, homologous=False)
    r1 = swb.score_only(*seqs(a, b), SCHEME)
    r2 = swb.score_only(*seqs(b, a), SCHEME)
    assert r1.score == r2.score  # swap symmetry of the local score (test_oracle.py:92-100)
    assert 5 < r1.score < 60


def test_full_align_self_consistent_and_split_equal():
    a, b = synthetic_pair(300_000, seed=1003)
    s1, s2 = seqs(a, b)
    summ, path = swb.align(s1, s2, SCHEME)
    assert swb.score_of_path(path, s1, s2, SCHEME) == summ.score
    assert path.start == summ.start and path.end == summ.end
    sc = swb.score_only(s1, s2, SCHEME)
    assert (sc.score, sc.end) == (summ.score, summ.end)
    summ2, path2 = swb.align(s1, s2, SCHEME, AlignConfig(split=2))
    assert summ2.score == summ.score
    assert swb.score_of_path(path2, s1, s2, SCHEME) == summ2.score
    # leaf-limit changes the path, never the score or the endpoints' validity
    summ3, path3 = swb.align(s1, s2, SCHEME, AlignConfig(leaf_limit=256))
    assert (summ3.score, summ3.start, summ3.end) == (summ.score, summ.start, summ.end)
    assert swb.score_of_path(path3, s1, s2, SCHEME) == summ.score
