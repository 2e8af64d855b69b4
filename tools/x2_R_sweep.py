"""C2 score pass with the packed kernel at each rows-per-lane (pruning on):
x2_R_sweep.py R1,R2,... [REPS]"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from bench import synthetic_pair
from helpers import dna_scheme
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = dna_scheme()
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
hom = (sys.argv[4] != "unrelated") if len(sys.argv) > 4 else True
a, b = synthetic_pair(n, seed=1002 if hom else 1004, homologous=hom)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
Rs = [int(x) for x in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for _ in range(reps):
    for R in Rs:
        ctx.set_option("x2_R", R)
        rep = {}
        r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=True), report=rep)
        t = ctx.debug_times().astype(np.float64)
        t0 = t[:, 0].min()
        en = (t[:, 1] - t0) / 1e6
        print(f"R={R} kernel {ctx.last_kernel_ms:.1f} ms items={len(t)} score={r.score} end={r.end} "
              f"rpl={rep.get('rows_per_lane')} end[0]={en[0]:.1f} end[mid]={en[len(t)//2]:.1f} "
              f"pruned={rep.get('pruned_fraction', 0):.3f}", flush=True)
ctx.set_option("x2_R", 0)
