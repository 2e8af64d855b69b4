"""Packed kernel: identical (score, end) for every rows-per-lane and launch shape."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import dna_scheme, random_codes, mutate_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = dna_scheme()
for n, seed in ((20000, 2), (60000, 3), (5000, 4)):
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n); b = mutate_codes(rng, a, 0.12)[:n]
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    res = {}
    for x2, R, ctas in ((0, 0, 0), (1, 8, 0), (1, 10, 0), (1, 12, 0), (1, 14, 0), (1, 16, 0), (1, 8, 1), (1, 14, 2)):
        ctx.set_option("x2", x2); ctx.set_option("x2_R", R); ctx.set_option("max_ctas_per_sm", ctas)
        for prune in (True, False):
            r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
            res[(x2, R, ctas, prune)] = (r.score, tuple(r.end))
    vals = set(res.values())
    print(n, "consistent" if len(vals) == 1 else "INCONSISTENT", vals if len(vals) > 1 else list(vals)[0], flush=True)
    if len(vals) > 1:
        for k, v in res.items(): print("   ", k, v)
ctx.set_option("x2", 1); ctx.set_option("x2_R", 0); ctx.set_option("max_ctas_per_sm", 0)
