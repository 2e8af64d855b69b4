"""Phase 3 with static ranges when the reverse map is empty (all tiles unknown)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, phase3
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.model import AlignmentSummary
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
a, b = synthetic_pair(n, seed=1003)
for mode in ("rev-empty", "both-empty"):
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        if mode == "both-empty":
            S.bounds = False
            scored, _ = phase1.best_local(S, True)
            S.bounds = True
        else:
            scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        interval = phase2.oriented_interval(band, scored.score, e.i, e.j, sc)
        ri, rj = phase2.restricted_search(S, (0, e.i, 1), (0, e.j, 1), scored.score, interval, bounds=False)
        start = swb.Coord(e.i - ri - 1, e.j - rj - 1)
        try:
            path = phase3.reconstruct(S, AlignmentSummary(scored.score, start, e), band=True)
            print(mode, "ok", start, path.ops.size, flush=True)
        except Exception as ex:
            print(mode, "FAIL", type(ex).__name__, str(ex)[:120], flush=True)
