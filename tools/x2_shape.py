"""Packed kernel launch-shape sweep on the C2 pair: (rows per lane, CTAs per SM)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from bench import synthetic_pair
from helpers import dna_scheme
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = dna_scheme()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synthetic_pair(n, seed=1002)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
for R, ctas in ((0, 0), (14, 2), (12, 3), (10, 3), (8, 3), (8, 4), (10, 4)):
    ctx.set_option("x2_R", R); ctx.set_option("max_ctas_per_sm", ctas)
    out = []
    for prune in (True, False):
        best = 1e9
        for _ in range(2):
            rep = {}
            r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
            best = min(best, ctx.last_kernel_ms)
        out.append(best)
    print(f"R={R} ctas={ctas}: prune {out[0]:.1f} ms  full {out[1]:.1f} ms  score={r.score}", flush=True)
ctx.set_option("x2_R", 0); ctx.set_option("max_ctas_per_sm", 0)
