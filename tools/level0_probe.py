"""Timeline of the Myers-Miller level-0 crossing launch with tile bounds (C3 by default)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, phase3
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.model import AlignmentSummary
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
a, b = synthetic_pair(n, seed=1003)
ctx = get_context(0)


def timeline(tag):
    t = ctx.debug_times().astype(np.float64)
    np.save(ROOT / "gpurun_out" / (tag.replace(" ", "_").replace("=", "") + ".npy"), t)
    t0n = t[:, 0].min()
    st, en, wt = (t[:, 0] - t0n) / 1e6, (t[:, 1] - t0n) / 1e6, t[:, 2] / 1e6
    act = en - st
    print(f"{tag}: items {len(t)} span {en.max():.1f} ms active mean {act.mean():.2f} max {act.max():.2f} "
          f"wait mean {wt.mean():.2f}", flush=True)
    q = np.linspace(0, len(t) - 1, 9).astype(int)
    print("   start", np.round(st[q], 1), "\n   end  ", np.round(en[q], 1), "\n   wait ", np.round(wt[q], 2), flush=True)


with Session(ctx, a, b, sc) as S:
    S.reset_bounds()
    scored, p1 = phase1.best_local(S, True)
    e = scored.end
    band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
    t0 = time.perf_counter()
    start = phase2.locate_start(S, e, scored.score, band)
    print(f"phase 2 {time.perf_counter() - t0:.3f} s", flush=True)
    timeline("phase2")
    root = phase3._as_array([phase3.Subproblem(start, e, scored.score)], True)
    for R, cc in [(int(x), 1) for x in sys.argv[2:]] or ((0, 1), (0, 0), (8, 1), (16, 1)):
        ctx.set_option("rows_per_lane", R)
        ctx.set_option("chain_cta", cc)
        t0 = time.perf_counter()
        res, cells = ctx.crossings(S.cs, S.s1, S.s2, root, True)
        print(f"level0 R={R} chain_cta={cc}: {time.perf_counter() - t0:.3f} s cells {cells:.3e} kernel {ctx.last_kernel_ms:.1f} ms", flush=True)
        timeline(f"level0 R={R} cc={cc}")
    ctx.set_option("rows_per_lane", 0)
