"""Row-slab (multi-GPU) pass on one GPU, slabs run one after another through
the ext_in / ext_out boundary path: the merged result must equal
the single pass exactly."""
import numpy as np
import pytest

from helpers import dna_scheme, mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.multigpu import SLAB_STRIP_ROWS, run_slabs_sequential, slab_partition

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,kind", [(2, "hom"), (3, "unrel"), (4, "hom"), (8, "hom")])
def test_sequential_slabs_match_single_pass(world, kind):
    rng = np.random.default_rng(world)
    a = random_codes(rng, 60_000)
    b = random_codes(rng, 45_000) if kind == "unrel" else mutate_codes(rng, a, 0.1)[:50_000]
    scheme = dna_scheme()
    ctx = get_context(0)
    with Session(ctx, a, b, scheme) as S:
        single = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                             track=1, prune=True)])[0]
        slabs = slab_partition(S.n1, world, SLAB_STRIP_ROWS)
        merged, per = run_slabs_sequential(S, slabs)
    assert merged == (single.best_score, single.best_i, single.best_j)
    assert sum(r.cells_executed for r in per) > 0


def test_slab_public_api_equivalence():
    rng = np.random.default_rng(77)
    a = random_codes(rng, 30_000)
    b = mutate_codes(rng, a, 0.15)
    scheme = dna_scheme()
    s1 = swb.Sequence.from_codes("a", a, scheme.alphabet)
    s2 = swb.Sequence.from_codes("b", b, scheme.alphabet)
    ref = swb.score_only(s1, s2, scheme)
    with Session(get_context(0), a, b, scheme) as S:
        merged, _ = run_slabs_sequential(S, slab_partition(S.n1, 3, SLAB_STRIP_ROWS))
    assert merged == (ref.score, ref.end.i - 1, ref.end.j - 1)


@pytest.mark.parametrize("x2", [1, 0])
def test_slab_prune_bound_counts_rows_below(x2):
    """A strong alignment that ends inside slab 0 must not let slab 0 prune the
    start of a stronger one that continues into slab 1 (rows_after)."""
    rng = np.random.default_rng(2024)
    n1 = 61_440
    a = random_codes(rng, n1)
    b = random_codes(rng, 52_000)
    b[:20_000] = a[:20_000]                    # X: ends in slab 0, score 20000
    b[20_000:20_000 + 31_720] = a[29_720:]     # Y: starts 1000 rows above the slab cut
    scheme = dna_scheme()
    ctx = get_context(0)
    default = ctx.get_option("x2")
    ctx.set_option("x2", x2)
    try:
        with Session(ctx, a, b, scheme) as S:
            single = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local",
                                 clamp=True, track=1, prune=True)])[0]
            slabs = slab_partition(S.n1, 2, SLAB_STRIP_ROWS)
            assert slabs[0].row1 == 30_720
            merged, per = run_slabs_sequential(S, slabs)
    finally:
        ctx.set_option("x2", default)
    assert single.best_score >= 31_720
    assert merged == (single.best_score, single.best_i, single.best_j)
    assert {r.kernel for r in per} == {"packed16x2" if x2 else "lane32"}


@pytest.mark.parametrize("world", [2, 4])
def test_slabs_x2_equal_32bit(world):
    rng = np.random.default_rng(100 + world)
    a = random_codes(rng, 80_000)
    b = mutate_codes(rng, a, 0.12)[:70_000]
    ctx = get_context(0)
    default = ctx.get_option("x2")
    out = []
    try:
        for flag in (1, 0):
            ctx.set_option("x2", flag)
            with Session(ctx, a, b, dna_scheme()) as S:
                merged, per = run_slabs_sequential(S, slab_partition(S.n1, world, SLAB_STRIP_ROWS))
            out.append(merged)
    finally:
        ctx.set_option("x2", default)
    assert out[0] == out[1]
