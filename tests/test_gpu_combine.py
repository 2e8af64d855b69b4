"""The chunked Myers-Miller middle-row combine (combine_part_kernel +
combine_final_kernel, swb_mm.cu) against the one-CTA-per-subproblem
combine_kernel it replaced (diagnostic proto 15): identical crossings, hence
identical paths, on pairs whose top levels span many 16 384-column chunks,
including gap joins (large gap-open) and unrelated flanks."""
import numpy as np
import pytest

from helpers import dna_scheme, mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import Sequence
from paper_1304_5966_b200.engine import get_context

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,n,rate,args", [
    (1, 120_000, 0.10, (1, -3, 5, 2)),
    (2, 300_000, 0.15, (1, -3, 5, 2)),
    (3, 80_000, 0.20, (2, -1, 12, 1)),
    (4, 50_000, 0.05, (5, -2, 0, 4)),
])
def test_chunked_combine_matches_single_cta(seed, n, rate, args):
    rng = np.random.default_rng(seed)
    core = random_codes(rng, n)
    a = np.concatenate([random_codes(rng, 5000), core, random_codes(rng, 3000)])
    b = np.concatenate([random_codes(rng, 2000), mutate_codes(rng, core, rate), random_codes(rng, 4000)])
    sc = dna_scheme(None, *args)
    s1 = Sequence.from_codes("a", a, sc.alphabet)
    s2 = Sequence.from_codes("b", b, sc.alphabet)
    ctx = get_context(0)
    old = ctx.get_option("proto")
    out = []
    try:
        for proto in (old, 15):
            ctx.set_option("proto", proto)
            summ, path = swb.align(s1, s2, sc)
            out.append((summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes()))
    finally:
        ctx.set_option("proto", old)
    assert out[0] == out[1]
