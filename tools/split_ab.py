"""A/B of one context option on split=2 full alignment of the C3 pair:
split_ab.py OPTION V1,V2 [REPS] [N]"""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
opt, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = int(sys.argv[4]) if len(sys.argv) > 4 else 5_000_000
a, b = synthetic_pair(n, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx = get_context(0)
old = ctx.get_option(opt)
swb.align(s1, s2, sc, swb.AlignConfig(split=2))
for _ in range(reps):
    for v in vals:
        ctx.set_option(opt, v)
        rep = {}
        t0 = time.perf_counter()
        summ, path = swb.align(s1, s2, sc, swb.AlignConfig(split=2), report=rep)
        print(json.dumps({opt: v, "s": round(time.perf_counter() - t0, 3),
                          "phase_s": [round(x, 3) for x in rep.get("phase_seconds", ())],
                          "score": summ.score, "start": list(summ.start)}), flush=True)
ctx.set_option(opt, old)
