"""Search small seeded cases where live ranges + static ranges break phase 3."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
fails = 0
for n in (20_000, 120_000, 400_000):
    for seed in range(4):
        rng = np.random.default_rng(seed)
        a = random_codes(rng, n); b = mutate_codes(rng, a, 0.1)
        s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
        res = []
        for live in (0, 3):
            ctx.set_option("live_ranges", live)
            try:
                summ, path = swb.align(s1, s2, sc)
                res.append((summ.score, tuple(summ.start), path.ops.tobytes()))
            except Exception as e:
                res.append(type(e).__name__)
        ok = all(r == res[0] for r in res)
        if not ok:
            fails += 1
            print("FAIL n", n, "seed", seed, [r if isinstance(r, str) else r[:2] for r in res], flush=True)
print("fails", fails)
ctx.set_option("live_ranges", 3)
