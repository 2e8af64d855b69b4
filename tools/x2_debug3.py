import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import dna_scheme, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = dna_scheme()
rng = np.random.default_rng(1)
a = random_codes(rng, 512); b = random_codes(rng, 64)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
def run(flag, tag):
    ctx.set_option("x2", flag)
    r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=False))
    print(tag, flag, r.score, tuple(r.end), flush=True)
for t in range(3): run(1, "x2-first")
run(0, "ref")
for t in range(3): run(1, "x2-after-ref")
# big 32-bit job then x2
rng2 = np.random.default_rng(9)
A = random_codes(rng2, 50000); B = random_codes(rng2, 50000)
ctx.set_option("x2", 0)
swb.score_only(swb.Sequence.from_codes("a", A, sc.alphabet), swb.Sequence.from_codes("b", B, sc.alphabet), sc)
for t in range(2): run(1, "x2-after-big-ref")
ctx.set_option("x2", 1)
swb.score_only(swb.Sequence.from_codes("a", A, sc.alphabet), swb.Sequence.from_codes("b", B, sc.alphabet), sc)
for t in range(2): run(1, "x2-after-big-x2")
