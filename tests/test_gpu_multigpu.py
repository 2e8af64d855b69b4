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
