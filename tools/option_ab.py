"""A/B of one context option on the full alignment (phase seconds):
    option_ab.py N OPTION V1,V2[,...] [REPS]"""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n, opt = int(sys.argv[1]), sys.argv[2]
vals = [int(v) for v in sys.argv[3].split(",")]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
a, b = synthetic_pair(n, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx = get_context(0)
old = ctx.get_option(opt)
swb.align(s1, s2, sc)
ref = None
for v in vals * reps:
    ctx.set_option(opt, v)
    rep = {}
    t0 = time.perf_counter()
    summ, path = swb.align(s1, s2, sc, report=rep)
    dt = time.perf_counter() - t0
    key = (summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes())
    ref = ref or key
    print(json.dumps({opt: v, "wall_s": round(dt, 3), "phase_s": [round(x, 3) for x in rep["phase_seconds"]],
                      "same_result": key == ref}), flush=True)
ctx.set_option(opt, old)
