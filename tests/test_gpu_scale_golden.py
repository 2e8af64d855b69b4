"""Parity at BASELINE scale against the unmodified reference.

tests/golden/golden_scale.json.gz was produced by running the reference
(`wavealign`, /root/reference/pkg/src) on the bench's own synthetic pairs
(tests/golden/make_golden_scale.py; 8 workers, 37 min for C2):

  C2         align on the full 1 Mbp x 1 Mbp pair (seed 1002); its phase 1 is
             score_only (reference pipeline.py:74 vs :103-126), so the headline
             pass's (score, end) is pinned, and start / CIGAR pin phases 2-3
  C3w, C5w   align on the first 200 kbp x 200 kbp of the C3 / C5 pairs
  C3w_split  align(split=2) on the C3 window (split.py:84-182)
  C4w        score_only on the first 1 Mbp x 1 Mbp of the C4 unrelated pair

Every device configuration that can carry the pass is checked against the
same record: packed 16x2 and 32-bit kernels, pruning on and off, and 1 / 2 /
4 / 8 row slabs chained on one GPU.  Bar: bit-exact score, start, end, CIGAR.
"""
import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Sequence
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.multigpu import (SLAB_STRIP_ROWS, run_slabs_concurrent,
                                          run_slabs_sequential, run_split_slabs_concurrent,
                                          slab_partition)

pytestmark = pytest.mark.gpu

GOLDEN = {r["name"]: r for r in json.load(gzip.open(
    Path(__file__).resolve().parent / "golden" / "golden_scale.json.gz", "rt"))}
SCHEME = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)  # the bench's alphabet


def pair(name):
    g = GOLDEN[name]
    a, b = synthetic_pair(g["n"], seed=g["seed"], homologous=g["homologous"])
    if g["window"]:
        a, b = a[:g["window"][0]], b[:g["window"][1]]
    assert (a.size, b.size) == (g["n1"], g["n2"])
    return (Sequence.from_codes("target", a, SCHEME.alphabet),
            Sequence.from_codes("query", b, SCHEME.alphabet), a, b)


@pytest.fixture(scope="module")
def c2():
    return pair("C2")


def _opt(name, value):
    get_context(0).set_option(name, value)


@pytest.mark.parametrize("x2,blk", [(1, 32), (1, 64), (0, 0)])
@pytest.mark.parametrize("prune", [True, False])
def test_c2_score_pass(c2, x2, blk, prune):
    """Packed kernel with 32- and 64-step blocks (x2_blk), and the 32-bit kernel."""
    s1, s2, _, _ = c2
    g = GOLDEN["C2"]
    _opt("x2", x2)
    _opt("x2_blk", blk)
    try:
        rep = {}
        r = swb.score_only(s1, s2, SCHEME, AlignConfig(prune=prune), report=rep)
    finally:
        _opt("x2", 1)
        _opt("x2_blk", 0)
    assert (r.score, list(r.end)) == (g["score"], g["end"])
    assert rep["kernel"] == ("packed16x2" if x2 else "lane32")


@pytest.mark.parametrize("nslabs", [1, 2, 4, 8])
def test_c2_row_slabs(c2, nslabs):
    """The multi-GPU decomposition, slabs chained on one GPU."""
    _, _, a, b = c2
    g = GOLDEN["C2"]
    with Session(get_context(0), a, b, SCHEME) as S:
        merged, _ = run_slabs_sequential(S, slab_partition(S.n1, nslabs, SLAB_STRIP_ROWS))
    assert (merged[0], [merged[1] + 1, merged[2] + 1]) == (g["score"], g["end"])


@pytest.mark.parametrize("nslabs", [2, 4, 8])
@pytest.mark.parametrize("prune,share", [(True, True), (True, False), (False, False)])
def test_c2_row_slabs_concurrent(c2, nslabs, prune, share):
    """The N-rank boundary protocol with every rank running at once: all slabs
    in one launch, each consuming its predecessor through the ext path, with
    and without the running best shared between slabs."""
    _, _, a, b = c2
    g = GOLDEN["C2"]
    pruned = []
    for _ in range(3):
        with Session(get_context(0), a, b, SCHEME) as S:
            merged, res = run_slabs_concurrent(S, slab_partition(S.n1, nslabs, SLAB_STRIP_ROWS),
                                               prune, share)
        assert (merged[0], [merged[1] + 1, merged[2] + 1]) == (g["score"], g["end"])
        assert all(r.kernel == "packed16x2" for r in res)
        pruned.append(sum(r.pruned_blocks for r in res))
    if not prune:
        assert max(pruned) == 0


def test_c2_row_slabs_concurrent_blk64(c2):
    """The slab boundary protocol with 64-step packed blocks."""
    _, _, a, b = c2
    g = GOLDEN["C2"]
    _opt("x2_blk", 64)
    try:
        with Session(get_context(0), a, b, SCHEME) as S:
            merged, res = run_slabs_concurrent(S, slab_partition(S.n1, 4, SLAB_STRIP_ROWS), True, True)
    finally:
        _opt("x2_blk", 0)
    assert (merged[0], [merged[1] + 1, merged[2] + 1]) == (g["score"], g["end"])


def test_shared_best_prunes_more(c2):
    """Slabs below the alignment's start prune with the whole pass's best when
    it is shared (swb_pass_desc.shared_best) and far less on their own."""
    _, _, a, b = c2
    out = {}
    for share in (False, True):
        with Session(get_context(0), a, b, SCHEME) as S:
            _, res = run_slabs_concurrent(S, slab_partition(S.n1, 8, SLAB_STRIP_ROWS), True, share)
        out[share] = sum(r.pruned_blocks for r in res)
    assert out[True] > out[False]


def _check_align(name, cfg=None):
    s1, s2, _, _ = pair(name)
    g = GOLDEN[name]
    summ, path = swb.align(s1, s2, SCHEME, cfg)
    assert (summ.score, list(summ.start), list(summ.end)) == (g["score"], g["start"], g["end"])
    assert swb.path_to_cigar(path) == g["cigar"]


def test_c2_full_align(c2):
    _check_align("C2")


@pytest.mark.parametrize("name", ["C3w", "C5w"])
def test_window_align(name):
    _check_align(name)


@pytest.mark.parametrize("blk", [0, 64])
def test_c3_window_split2(blk):
    """split=2's halves on the packed FINAL kernels, 64-step blocks forced too."""
    _opt("x2_blk", blk)
    try:
        _check_align("C3w_split", AlignConfig(split=2))
    finally:
        _opt("x2_blk", 0)


@pytest.mark.parametrize("name", ["C3w", "C5w"])
def test_window_align_blk64(name):
    _opt("x2_blk", 64)
    try:
        _check_align(name)
    finally:
        _opt("x2_blk", 0)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c3_window_split2_gpu_groups(world):
    """The Figure-1 split across `world` GPUs (upper half on ranks [0, G/2),
    lower half on [G/2, G), row slabs within each group, one shared running
    best), emulated in one launch: byte-equal to the reference's split=2."""
    s1, s2, a, b = pair("C3w_split")
    g = GOLDEN["C3w_split"]
    with Session(get_context(0), a, b, SCHEME) as S:
        summ, path = run_split_slabs_concurrent(S, world)
    assert (summ.score, list(summ.start), list(summ.end)) == (g["score"], g["start"], g["end"])
    assert swb.path_to_cigar(path) == g["cigar"]


def test_c4_window_score():
    s1, s2, _, _ = pair("C4w")
    g = GOLDEN["C4w"]
    r = swb.score_only(s1, s2, SCHEME)
    assert (r.score, list(r.end)) == (g["score"], g["end"])


def test_both_strands_single_gpu():
    """align_both_strands finds an inverted copy on the minus strand and
    equals align() on (seq1, seq2) and (seq1, revcomp(seq2))."""
    from paper_1304_5966_b200.multigpu import align_both_strands, reverse_complement_codes
    a, b = synthetic_pair(60_000, seed=77)
    b = np.concatenate([b[:20_000], reverse_complement_codes(a[30_000:50_000], SCHEME.alphabet)])
    s1 = Sequence.from_codes("t", a, SCHEME.alphabet)
    s2 = Sequence.from_codes("q", b, SCHEME.alphabet)
    both = align_both_strands(s1, s2, SCHEME)
    fwd = swb.align(s1, s2, SCHEME)
    rc = Sequence.from_codes("q_rc", reverse_complement_codes(b, SCHEME.alphabet), SCHEME.alphabet)
    rev = swb.align(s1, rc, SCHEME)
    assert both["+"][0] == fwd[0] and np.array_equal(both["+"][1].ops, fwd[1].ops)
    assert both["-"][0] == rev[0] and np.array_equal(both["-"][1].ops, rev[1].ops)
    assert both["-"][0].score >= 19_000  # the inverted 20 kbp copy, exact
