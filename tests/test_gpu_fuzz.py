"""Randomised parity sweep of the CUDA path against the pinned oracle.

Many small pairs, each with its own random scheme: general (asymmetric,
mostly negative) substitution matrices over 4-, 5- (with the 'N' wildcard),
20-, 24- and 32-code alphabets, gap_open 0..12, gap_extend 1..6, lengths 1..4000
(ragged, often far from the 32/64-column tile edges), and every
configuration the reference's pipeline offers (split=1/2, small leaf
limits, band off, prune off).  Complements the fixed cases of
test_gpu_parity.py the way the reference's randomised oracle tests
do (pkg/tests/test_oracle.py:75-90, random_scheme in support.py).  Bar: bit-exact score, start, end and path.
"""
import numpy as np
import pytest

import oracle
from helpers import mutate_codes, oracle_scheme
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Alphabet, ScoringScheme, Sequence

pytestmark = pytest.mark.gpu

_ALPHAS = (Alphabet.dna(wildcard=False), Alphabet.dna(wildcard=True), Alphabet.protein(),
           Alphabet("protein", "ARNDCQEGHILKMFPSTWYVBZX*"),          # BLOSUM62 order, K=24
           Alphabet("custom", "ABCDEFGHIJKLMNOPQRSTUVWXYZ012345"))  # K=32, the device limit


def _random_scheme(rng):
    alpha = _ALPHAS[int(rng.integers(0, len(_ALPHAS)))]
    k = len(alpha)
    m = rng.integers(-6, 2, size=(k, k)).astype(np.int64)
    m[np.arange(k), np.arange(k)] = rng.integers(1, 7, size=k)
    if alpha.wildcard is not None:
        w = alpha.index(alpha.wildcard)
        m[w, :] = 0
        m[:, w] = 0
    go, ge = int(rng.integers(0, 13)), int(rng.integers(1, 7))
    return ScoringScheme(alpha, m, go, ge, int(m.max()))


def _random_len(rng):
    return int(rng.integers(1, 601)) if rng.random() < 0.85 else int(rng.integers(601, 4001))


def _random_pair(rng, k):
    n1 = _random_len(rng)
    a = rng.integers(0, k, size=n1, dtype=np.uint8)
    kind = int(rng.integers(0, 3))
    if kind == 0:      # unrelated
        b = rng.integers(0, k, size=_random_len(rng), dtype=np.uint8)
    else:              # homologous, with random flanks
        b = mutate_codes(rng, a, 0.05 + 0.25 * rng.random(), k=k)
        lf, rf = int(rng.integers(0, 80)), int(rng.integers(0, 80))
        b = np.concatenate([rng.integers(0, k, size=lf, dtype=np.uint8), b,
                            rng.integers(0, k, size=rf, dtype=np.uint8)])
    if rng.random() < 0.5:
        a, b = b, a
    return a, b


_CONFIGS = ({}, {"split": 2}, {"leaf_limit": 64}, {"band": False}, {"prune": False},
            {"leaf_limit": 1000, "split": 2})


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_align_vs_oracle(seed):
    rng = np.random.default_rng(9000 + seed)
    for case in range(40):
        scheme = _random_scheme(rng)
        k = len(scheme.alphabet)
        a, b = _random_pair(rng, k)
        cfg_kw = _CONFIGS[case % len(_CONFIGS)]
        osch = oracle_scheme(scheme)
        want = oracle.align(a, b, osch, **cfg_kw)
        s1 = Sequence.from_codes("a", a, scheme.alphabet)
        s2 = Sequence.from_codes("b", b, scheme.alphabet)
        summary, path = swb.align(s1, s2, scheme, AlignConfig(**cfg_kw))
        tag = (seed, case, a.size, b.size, k, scheme.gap_open, scheme.gap_extend, cfg_kw)
        assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3], tag
        assert np.array_equal(path.ops, want[3]), tag
        # split=2 may report a different co-optimal end (split.py:84-182), so
        # score_only is checked against the oracle's own score pass
        prune = bool(case % 2)
        ws, we, _ = oracle.score_only(a, b, osch, prune=prune)
        sc = swb.score_only(s1, s2, scheme, AlignConfig(prune=prune))
        assert (sc.score, tuple(sc.end)) == (ws, we), tag


def test_fuzz_zero_score_pairs():
    """No positive-scoring pair can form: empty summary and path on every
    entry point (pipeline.py:75-82 returns AlignmentSummary.empty())."""
    rng = np.random.default_rng(77)
    alpha = Alphabet.dna(wildcard=False)
    m = np.full((4, 4), -2, dtype=np.int64)
    m[0, 0] = 3                       # only A/A scores positive
    scheme = ScoringScheme(alpha, m, 4, 1, 3)
    for n1, n2 in ((1, 1), (37, 900), (700, 65), (1500, 1499)):
        a = rng.integers(1, 4, size=n1, dtype=np.uint8)     # no A in seq1
        b = rng.integers(0, 4, size=n2, dtype=np.uint8)
        want = oracle.align(a, b, oracle_scheme(scheme))
        assert want[0] == 0
        s1, s2 = Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha)
        for cfg_kw in ({}, {"split": 2}):
            summary, path = swb.align(s1, s2, scheme, AlignConfig(**cfg_kw))
            assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3], cfg_kw
            assert len(path) == 0
        assert swb.score_only(s1, s2, scheme).score == 0


def test_protein_record_85_repeated(golden_protein):
    """Golden protein record 85 (1171 x 144, a 12-residue local hit): its
    phase-2 pass (3 strips, 49 columns) used to fault or return a wrong start
    after a zero-score DNA alignment had run in the same process.  Root cause
    (DESIGN.md §7): lanes read the producer's live end at slightly different
    times, so some lanes took the early exit while the others ran the block and
    their shuffles paired with the exited lanes' (shfl.sync matches any
    shfl.sync of the same mask), which ran a strip twice and corrupted its
    values.  The sequence below is the reproducer (tools/repro_zero_protein.py
    a1), with every live-range feature on, repeated."""
    from helpers import golden_inputs
    from paper_1304_5966_b200.engine import get_context
    ctx = get_context(0)
    assert ctx.get_option("live_big") == 3 and ctx.get_option("live_ranges") == 3
    rng = np.random.default_rng(77)
    alpha = Alphabet.dna(wildcard=False)
    m = np.full((4, 4), -2, dtype=np.int64)
    m[0, 0] = 3
    zscheme = ScoringScheme(alpha, m, 4, 1, 3)
    for n1, n2 in ((1, 1), (37, 900)):
        a = rng.integers(1, 4, size=n1, dtype=np.uint8)
        b = rng.integers(0, 4, size=n2, dtype=np.uint8)
    swb.align(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha), zscheme)
    rec = golden_protein[85]
    s1, s2, scheme = golden_inputs(rec)
    for _ in range(30):
        assert swb.score_only(s1, s2, scheme).score == rec["score_only"]["score"]
        summary, path = swb.align(s1, s2, scheme)
        assert summary.score == rec["align"]["score"]
        assert list(summary.start) == rec["align"]["start"]
        assert list(summary.end) == rec["align"]["end"]
        assert swb.path_to_cigar(path) == rec["align"]["cigar"]
