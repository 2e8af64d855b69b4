"""The packed 16x2 phase-1 kernel (swb_x2.cuh) against the 32-bit kernel and
the oracle: identical (score, end) on homologous, unrelated, repetitive and
ragged inputs, with and without pruning."""
import numpy as np
import pytest

import oracle
from helpers import dna_scheme, mutate_codes, oracle_scheme, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Sequence
from paper_1304_5966_b200.engine import get_context

pytestmark = pytest.mark.gpu


def _both(a, b, scheme, prune=True):
    """[packed kernel, 32-bit kernel] (score, end); the packed kernel runs with
    32- and 64-step blocks (x2_blk) and must agree with itself."""
    ctx = get_context(0)
    s1 = Sequence.from_codes("a", a, scheme.alphabet)
    s2 = Sequence.from_codes("b", b, scheme.alphabet)
    out = []
    default = ctx.get_option("x2")
    try:
        for flag, blk in ((1, 32), (1, 64), (0, 0)):
            ctx.set_option("x2", flag)
            ctx.set_option("x2_blk", blk)
            rep = {}
            r = swb.score_only(s1, s2, scheme, AlignConfig(prune=prune), report=rep)
            out.append((r.score, tuple(r.end)))
    finally:
        ctx.set_option("x2", default)
        ctx.set_option("x2_blk", 0)
    assert out[0] == out[1], ("x2_blk 32 vs 64", out)
    return [out[0], out[2]]


@pytest.mark.parametrize("seed,n1,n2,kind", [
    (1, 3000, 2800, "hom"), (2, 70_000, 65_000, "hom"), (3, 50_000, 52_000, "unrel"),
    (4, 1025, 4000, "hom"), (5, 2049, 64, "unrel"), (6, 40_000, 40_000, "rep"),
    (7, 129, 100_000, "hom"), (8, 200_000, 150_000, "hom")])
def test_x2_matches_32bit(seed, n1, n2, kind):
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n1)
    if kind == "hom":
        b = mutate_codes(rng, a, 0.12)[:n2]
        if b.size < n2:
            b = np.concatenate([b, random_codes(rng, n2 - b.size)])
    elif kind == "rep":
        unit = random_codes(rng, 7)
        a = np.tile(unit, n1 // 7 + 1)[:n1]
        b = mutate_codes(rng, a, 0.05)[:n2]
    else:
        b = random_codes(rng, n2)
    for prune in (True, False):
        x2, ref = _both(a, b, dna_scheme(), prune)
        assert x2 == ref, (seed, prune, x2, ref)


@pytest.mark.parametrize("args", [(2, -1, 3, 2), (5, -2, 0, 4), (1, -3, 5, 2), (3, -5, 10, 1)])
def test_x2_schemes_vs_oracle(args):
    rng = np.random.default_rng(sum(args))
    a = random_codes(rng, 6000)
    b = mutate_codes(rng, a, 0.2)
    scheme = dna_scheme(None, *args)
    x2, ref = _both(a, b, scheme)
    want = oracle.score_only(a, b, oracle_scheme(scheme))
    assert x2 == ref == (want[0], want[1])


@pytest.mark.parametrize("n1,n2", [(512, 64), (1024, 64), (1100, 64), (2049, 64), (600, 40),
                                   (300, 3), (64, 1), (130, 95), (4000, 96)])
def test_x2_narrow_after_32bit_launch(n1, n2):
    """Regression: narrow passes leave ring slots past n2 unstaged; their content
    (left over from earlier launches) must never reach an active half."""
    rng = np.random.default_rng(n1 * 1000 + n2)
    a = random_codes(rng, n1)
    b = random_codes(rng, n2)
    want = oracle.score_only(a, b, oracle_scheme(dna_scheme()))
    for _ in range(3):
        ref, x2 = _both(a, b, dna_scheme(), prune=False)[::-1]
        assert x2 == ref == (want[0], want[1]), (x2, ref, want[:2])


@pytest.mark.parametrize("n,seed", [(20000, 2), (5000, 4)])
def test_x2_invariant_to_shape(n, seed):
    """Every rows-per-lane, launch shape and pruning setting of the packed
    kernel gives the 32-bit kernel's (score, end)."""
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n)
    b = mutate_codes(rng, a, 0.12)[:n]
    sc = dna_scheme()
    ctx = get_context(0)
    saved = {k: ctx.get_option(k) for k in ("x2", "x2_R", "max_ctas_per_sm", "x2_blk")}
    s1 = Sequence.from_codes("a", a, sc.alphabet)
    s2 = Sequence.from_codes("b", b, sc.alphabet)
    res = set()
    try:
        for x2, R, ctas in ((0, 0, 0), (1, 8, 0), (1, 10, 0), (1, 12, 0), (1, 14, 0), (1, 16, 0),
                            (1, 8, 1), (1, 14, 2)):
            ctx.set_option("x2", x2)
            ctx.set_option("x2_R", R)
            ctx.set_option("max_ctas_per_sm", ctas)
            for blk in ((32, 64) if x2 else (0,)):
                ctx.set_option("x2_blk", blk)
                for prune in (True, False):
                    r = swb.score_only(s1, s2, sc, AlignConfig(prune=prune))
                    res.add((r.score, tuple(r.end)))
    finally:
        for k, v in saved.items():
            ctx.set_option(k, v)
    assert len(res) == 1, res


@pytest.mark.parametrize("seed,n1,n2,frac", [(21, 3000, 2900, 0.02), (22, 60_000, 58_000, 0.001),
                                             (23, 1100, 40_000, 0.3)])
def test_x2_wildcard_rows(seed, n1, n2, frac):
    """The default DNA alphabet ('N' = code 4 scores 0 against everything):
    rows holding N run the packed kernel's WILD variant; same (score, end) as
    the 32-bit kernel and the oracle, and the full alignment matches too."""
    from paper_1304_5966_b200 import Alphabet
    rng = np.random.default_rng(seed)
    alpha = Alphabet.dna()
    scheme = swb.ScoringScheme.match_mismatch(alpha, 1, -3, 5, 2)
    a = random_codes(rng, n1)
    b = mutate_codes(rng, a, 0.1)[:n2]
    if b.size < n2:
        b = np.concatenate([b, random_codes(rng, n2 - b.size)])
    for arr in (a, b):
        arr[rng.random(arr.size) < frac] = 4
        st = int(rng.integers(0, arr.size - 50))
        arr[st:st + 50] = 4
    got = _both(a, b, scheme)
    assert got[0] == got[1]
    rep = {}
    swb.score_only(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha), scheme,
                   report=rep)
    assert rep["kernel"] == "packed16x2"
    if n1 * n2 <= 2e8:
        want = oracle.align(a, b, oracle_scheme(scheme))
        summ, path = swb.align(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha),
                               scheme)
        assert (summ.score, tuple(summ.start), tuple(summ.end)) == want[:3]
        assert np.array_equal(path.ops, want[3])
