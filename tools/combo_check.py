"""Full align under option combinations (debugging exactness)."""
import itertools, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
a, b = synthetic_pair(n, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ref = None
for live, static, dyn, rep in itertools.product((1,), (0, 1), (0, 1), range(1)):
    maps = 1
    ctx.set_option("live_ranges", live); ctx.set_option("mm_static", static); ctx.set_option("mm_dyn", dyn)
    try:
        summ, path = swb.align(s1, s2, sc)
        key = (summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes())
        ref = ref or key
        print("live", live, "static", static, "dyn", dyn, "ok", key == ref, summ.start, flush=True)
    except Exception as e:
        print("live", live, "static", static, "dyn", dyn, "FAIL", type(e).__name__, str(e)[:100], flush=True)
for k, v in (("live_ranges", 1), ("mm_static", 1), ("bound_maps", 1)):
    ctx.set_option(k, v)
