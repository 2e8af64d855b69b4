"""Compare phase-2 reverse tile maps with and without live column ranges."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
a, b = synthetic_pair(n, seed=1003)
maps = {}
for live in (0, 1):
    ctx.set_option("live_ranges", live)
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        st = phase2.locate_start(S, e, scored.score, band)
        maps[live] = (ctx.bounds_map(1).astype(np.int64), ctx.bounds_map(2).astype(np.int64), st)
        print("live", live, "start", st, flush=True)
f0, r0, _ = maps[0]; f1, r1, _ = maps[1]
print("fwd equal", np.array_equal(f0, f1))
both = (r0 >= 0) & (r1 >= 0)
print("rev written: live0", int((r0 >= 0).sum()), "live1", int((r1 >= 0).sum()), "both", int(both.sum()))
lower = both & (r1 < r0)
print("tiles where live1 < live0:", int(lower.sum()))
nc = (b.size + 1023) // 1024
for k in np.flatnonzero(lower)[:10]:
    print("  tile", divmod(int(k), nc), "live0", int(r0[k]) - (1 << 30), "live1", int(r1[k]) - (1 << 30))
only0 = (r0 >= 0) & (r1 < 0)
print("written only without live:", int(only0.sum()), " only with live:", int(((r1 >= 0) & (r0 < 0)).sum()))
ctx.set_option("live_ranges", 1)
d = np.flatnonzero(f0 != f1)
nr = (a.size + 1023) // 1024
print("fwd diffs", d.size, "of", f0.size, "nr", nr, "nc", nc)
for k in d[:12]:
    print("  tile", divmod(int(k), nc), "live0", int(f0[k]) - (1 << 30) if f0[k] >= 0 else -1,
          "live1", int(f1[k]) - (1 << 30) if f1[k] >= 0 else -1)
