"""Single-warp step time of the lane kernel (one strip of 32R rows, long row):
the per-column cost that bounds chain-shaped passes (phase 2, top Myers-Miller
levels).  lane_step.py [NCOLS]"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX, TRACK_MIN, TRACK_NONE
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
nc = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
ctx = get_context(0)
a, b = synthetic_pair(nc, seed=7)
ctx.set_option("x2", 0)
Rs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (2, 8, 16)
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ("local/min", "restricted/max", "local/none")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
for R in Rs:
    a2 = a[:32 * R]
    with Session(ctx, a2, b, sc) as S:
        ctx.set_option("rows_per_lane", R)
        for border, track, name in (("local", TRACK_MIN, "local/min"), ("restricted", TRACK_MAX, "restricted/max"),
                                    ("local", TRACK_NONE, "local/none")):
            if (border == "local" and R < 8) or name not in modes:
                continue
            ms = []
            for _ in range(reps):
                r = S.run([dict(rows=(0, a2.size, 1), cols=(0, b.size, 1), border=border, clamp=track == TRACK_MIN, track=track, prune=0)])[0]
                ms.append(r.kernel_ms)
            t = min(ms) * 1e-3 / (b.size + 31)
            print(f"R={R:2d} {name:15s} {min(ms):8.2f} ms  {t * 1e9:6.1f} ns/step  {t * 1.965e9:6.0f} cyc/step "
                  f"{t * 1.965e9 / R:5.1f} cyc/row-step  kernel={r.kernel}", flush=True)
ctx.set_option("rows_per_lane", 0)
ctx.set_option("x2", 1)
