"""A/B of one context option on the phase-1 score pass (packed kernel):
C2 homologous and an unrelated pair; ms per pass (CUDA events), results equal.
    x2_opt_ab.py OPTION V1,V2 [N] [REPS]"""
import json
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import TRACK_MIN, Session, get_context

opt, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
ctx = get_context(0)
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
for kind in ("homologous", "unrelated"):
    a, b = synthetic_pair(n, seed=1002 if kind == "homologous" else 1004, homologous=kind == "homologous")
    with Session(ctx, a, b, sc) as S:
        spec = [dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                     track=TRACK_MIN, prune=True)]
        ref = None
        for v in vals:
            ctx.set_option(opt, v)
            S.run(spec)
            ms = []
            for _ in range(reps):
                ctx.flush_l2()
                ctx.timer_start()
                r = S.run(spec)[0]
                ms.append(ctx.timer_stop())
            key = (r.best_score, r.best_i, r.best_j)
            ref = ref or key
            print(json.dumps({"kind": kind, opt: v, "ms_min": round(min(ms), 2),
                              "ms_mean": round(sum(ms) / len(ms), 2), "same": key == ref,
                              "kernel": r.kernel, "R": r.rows_per_lane}), flush=True)
