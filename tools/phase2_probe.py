"""Phase-2 pass anatomy: cells, kernel time, per-strip timeline (5 Mbp by default)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
a, b = synthetic_pair(n, seed=1003)
ctx = get_context(0)
with Session(ctx, a, b, sc) as S:
    r = swb.score_only(swb.Sequence.from_codes("a", a, sc.alphabet), swb.Sequence.from_codes("b", b, sc.alphabet), sc)
    e = r.end
    band = phase2.compute_band(r.score, min(e.i, e.j), max(e.i, e.j), sc)
    interval = phase2.oriented_interval(band, r.score, e.i, e.j, sc)
    print("score", r.score, "end", e, "interval", interval, flush=True)
    for prune in (2, 0):
        t0 = time.perf_counter()
        res = S.run([dict(rows=(0, e.i, 1), cols=(0, e.j, 1), border="restricted", clamp=False,
                          track=TRACK_MAX, band=interval, prune=prune, prune_target=r.score)])[0]
        dt = time.perf_counter() - t0
        t = ctx.debug_times().astype(np.float64)
        t0n = t[:, 0].min()
        st, en, wt = (t[:, 0] - t0n) / 1e6, (t[:, 1] - t0n) / 1e6, t[:, 2] / 1e6
        act = en - st
        print(f"prune={prune}: wall {dt:.3f}s kernel {res.kernel_ms:.1f} ms cells {res.cells_executed:.3e} "
              f"({res.cells_executed / res.kernel_ms / 1e6:.0f} GCUPS exec) R={res.rows_per_lane} kernel={res.kernel} "
              f"strips={len(t)} busy={(act - wt).sum() / (en.max() * len(t)):.3f} "
              f"tiles exec/pruned/banded {res.executed_blocks}/{res.pruned_blocks}/{res.banded_out_blocks} best=({res.best_score},{res.best_i},{res.best_j})", flush=True)
        q = np.linspace(0, len(t) - 1, 9).astype(int)
        print("   start", np.round(st[q], 1), "\n   end  ", np.round(en[q], 1), "\n   wait ", np.round(wt[q], 1), flush=True)
