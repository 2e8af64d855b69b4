"""Tile bound maps, static Myers-Miller strip ranges and live column ranges of
restricted passes only skip work: score, start, end and
the path are identical with every combination switched on or off, on sizes
where the ranges leave strips empty (the buffer-reuse hazard they exposed)."""
import numpy as np
import pytest

from helpers import dna_scheme, mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context

pytestmark = pytest.mark.gpu

OPTS = ("bound_maps", "mm_static", "mm_dyn", "live_ranges", "chain_cta", "chain_wait")


def _align(a, b, scheme, **opts):
    ctx = get_context(0)
    saved = {k: ctx.get_option(k) for k in OPTS}
    try:
        for k, v in opts.items():
            ctx.set_option(k, v)
        s1 = swb.Sequence.from_codes("a", a, scheme.alphabet)
        s2 = swb.Sequence.from_codes("b", b, scheme.alphabet)
        summ, path = swb.align(s1, s2, scheme)
        return summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes()
    finally:
        for k, v in saved.items():
            ctx.set_option(k, v)


@pytest.mark.parametrize("seed,n", [(0, 120_000), (1, 120_000), (2, 150_000), (3, 60_000)])
def test_bounds_and_ranges_exact(seed, n):
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n)
    b = mutate_codes(rng, a, 0.1)
    sc = dna_scheme()
    ref = _align(a, b, sc, bound_maps=0, live_ranges=0)
    assert _align(a, b, sc, bound_maps=1, mm_static=1, mm_dyn=1, live_ranges=3) == ref
    assert _align(a, b, sc, bound_maps=1, mm_static=1, mm_dyn=0, live_ranges=1) == ref
    assert _align(a, b, sc, bound_maps=1, mm_static=0, mm_dyn=1, live_ranges=2) == ref


def test_bounds_with_other_schemes():
    rng = np.random.default_rng(9)
    a = random_codes(rng, 80_000)
    b = mutate_codes(rng, a, 0.2)
    for args in ((2, -1, 3, 2), (3, -5, 10, 1)):
        sc = dna_scheme(None, *args)
        assert _align(a, b, sc, bound_maps=1, live_ranges=3) == _align(a, b, sc, bound_maps=0,
                                                                       live_ranges=0)


@pytest.mark.parametrize("seed,n,rate", [(10, 9_000, 0.1), (11, 33_000, 0.2), (12, 130_000, 0.1),
                                         (13, 70_000, 0.02)])
def test_chain_chunks_exact(seed, n, rate):
    """Chain chunks (4 strips per CTA, shared-memory ring with
    a global fallback, lazy global release) and acquire polling change only
    the schedule: identical results with each switched off, on strip counts
    that are not multiples of 4 and with levels of many short jobs."""
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n)
    b = mutate_codes(rng, a, rate)[: n - 777]
    sc = dna_scheme()
    ref = _align(a, b, sc, chain_cta=0, chain_wait=0)
    assert _align(a, b, sc, chain_cta=1, chain_wait=1) == ref
    assert _align(a, b, sc, chain_cta=1, chain_wait=0) == ref
    assert _align(a, b, sc, chain_cta=1, live_ranges=0) == ref
