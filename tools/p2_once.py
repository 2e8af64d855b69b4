"""Phase 1 then ONE phase-2 pass (ncu target: `-k pass_kernel -c 1`):
p2_once.py [N]"""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
a, b = synthetic_pair(n, seed=1003)
ctx = get_context(0)
with Session(ctx, a, b, sc) as S:
    S.reset_bounds()
    scored, _ = phase1.best_local(S, True)
    e = scored.end
    band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
    t0 = time.perf_counter()
    start = phase2.locate_start(S, e, scored.score, band)
    print(f"phase 2 {time.perf_counter() - t0:.3f} s kernel {ctx.last_kernel_ms:.1f} ms start {start}", flush=True)
