"""A/B: packed 16x2 kernel vs 32-bit kernel on the C2 pair and an unrelated pair."""
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
for hom in (True, False):
    a, b = synthetic_pair(n, seed=1002 if hom else 1004, homologous=hom)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    for prune in (True, False):
        if not hom and prune:
            continue
        for flag, R in ((0, 0), (1, 0), (1, 8), (1, 12), (1, 16)):
            ctx.set_option("x2", flag); ctx.set_option("x2_R", R)
            best = 1e9
            for _ in range(3):
                r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
                best = min(best, ctx.last_kernel_ms)
            print(f"hom={hom} prune={prune} x2={flag} R={R}: {best:.1f} ms "
                  f"{a.size * b.size / best / 1e6:.0f} GCUPS  score={r.score}", flush=True)
ctx.set_option("x2", 1); ctx.set_option("x2_R", 0)
