"""A/B of one context option on a packed score pass (kernel ms):
opt_score.py OPTION V1,V2 [REPS] [N] [unrelated]"""
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
opt, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1_000_000
hom = not (len(sys.argv) > 5 and sys.argv[5] == "unrelated")
a, b = synthetic_pair(n, seed=(1002 if n == 1_000_000 else 1003) if hom else 1004, homologous=hom)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
old = ctx.get_option(opt)
swb.score_only(s1, s2, sc)
res = {v: [] for v in vals}
for _ in range(reps):
    for v in vals:
        ctx.set_option(opt, v)
        r = swb.score_only(s1, s2, sc)
        res[v].append(round(ctx.last_kernel_ms, 1))
ctx.set_option(opt, old)
for v in vals:
    print(f"{opt}={v}: {res[v]} mean {sum(res[v]) / len(res[v]):.1f} ms (score {r.score})", flush=True)
