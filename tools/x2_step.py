"""Single-warp step time of the packed kernel (one item of 64R rows, long row,
no producer): the per-column cost of the warp on a chain's critical path.
x2_step.py [NCOLS] [R,...]"""
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
nc = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
Rs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (14,)
for hom in (True, False):
    a, b = synthetic_pair(nc, seed=7, homologous=hom)
    for R in Rs:
        ctx.set_option("x2_R", R)
        s1 = swb.Sequence.from_codes("a", a[:64 * R], sc.alphabet)
        s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
        ms = []
        for _ in range(3):
            rep = {}
            swb.score_only(s1, s2, sc, swb.AlignConfig(prune=False), report=rep)
            ms.append(ctx.last_kernel_ms)
        t = min(ms) * 1e-3 / (b.size + 63)
        print(f"R={R} {'homologous' if hom else 'unrelated '} {min(ms):8.2f} ms {t * 1e9:6.1f} ns/step "
              f"{t * 1.965e9:5.0f} cyc/step kernel={rep.get('kernel')} rpl={rep.get('rows_per_lane')}", flush=True)
ctx.set_option("x2_R", 0)
