"""Restricted-pass results with and without live column ranges."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
for n in [int(x) for x in sys.argv[1:]] or [300_000]:
    a, b = synthetic_pair(n, seed=1003)
    with Session(ctx, a, b, sc) as S:
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        interval = phase2.oriented_interval(band, scored.score, e.i, e.j, sc)
        for prune in (0, 2):
            out = []
            for live in (0, 1):
                ctx.set_option("live_ranges", live)
                r = S.run([dict(rows=(0, e.i, 1), cols=(0, e.j, 1), border="restricted", clamp=False,
                                track=TRACK_MAX, band=interval, prune=prune, prune_target=scored.score)])[0]
                out.append((r.best_score, r.best_i, r.best_j, r.cells_executed, round(r.kernel_ms, 1)))
            print(n, "prune", prune, out, "SAME" if out[0][:3] == out[1][:3] else "DIFF", flush=True)
ctx.set_option("live_ranges", 1)
