"""Phase-2 anatomy at large n (phase 1 with tile maps first)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX, bound_slack
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
a, b = synthetic_pair(n, seed=1005 if n >= 32_000_000 else 1003)
ctx = get_context(0)
with Session(ctx, a, b, sc) as S:
    S.reset_bounds()
    t0 = time.perf_counter()
    scored, p1 = phase1.best_local(S, True)
    print(f"phase1 {time.perf_counter() - t0:.1f} s score {scored.score}", flush=True)
    e = scored.end
    band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
    interval = phase2.oriented_interval(band, scored.score, e.i, e.j, sc)
    t0 = time.perf_counter()
    res = S.run([dict(rows=(0, e.i, 1), cols=(0, e.j, 1), border="restricted", clamp=False,
                      track=TRACK_MAX, band=interval, prune=2, prune_target=scored.score,
                      bound_read=1, bound_write=2, bound_offset=bound_slack(sc))])[0]
    dt = time.perf_counter() - t0
    t = ctx.debug_times().astype(np.float64)
    t0n = t[:, 0].min()
    st, en, wt = (t[:, 0] - t0n) / 1e6, (t[:, 1] - t0n) / 1e6, t[:, 2] / 1e6
    act = en - st
    print(f"phase2 pass {dt:.2f} s kernel {res.kernel_ms:.0f} ms cells {res.cells_executed:.3e} R={res.rows_per_lane} "
          f"strips {len(t)} active mean {act.mean():.2f} ms wait mean {wt.mean():.2f} "
          f"tiles exec/pruned/total {res.executed_blocks}/{res.pruned_blocks}/{res.total_blocks}", flush=True)
    q = np.linspace(0, len(t) - 1, 11).astype(int)
    print("  start", np.round(st[q], 1)); print("  end  ", np.round(en[q], 1)); print("  act-wait", np.round((act - wt)[q], 3))
    d = np.diff(en); print("  median end diff ms", float(np.median(d)))
