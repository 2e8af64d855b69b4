"""Phase-2 time vs rows per lane (bound-pruned restricted pass) and live ranges."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
a, b = synthetic_pair(n, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ref = None
for p2r, live in ((16, 0), (16, 0), (16, 3), (8, 3), (24, 3)):
    ctx.set_option("p2_R", p2r); ctx.set_option("live_ranges", live)
    rep = {}
    t0 = time.perf_counter()
    summ, path = swb.align(s1, s2, sc, report=rep)
    dt = time.perf_counter() - t0
    key = (summ.score, tuple(summ.start), path.ops.tobytes()); ref = ref or key
    print(f"p2_R={p2r} live={live}: wall {dt:.2f} phases {[round(x, 2) for x in rep['phase_seconds']]} same {key == ref}", flush=True)
ctx.set_option("p2_R", 8); ctx.set_option("live_ranges", 0)
