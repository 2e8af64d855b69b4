"""Anatomy of the chain-shaped phase-2 pass (C-config pair): per-strip start
lag, active time, executed / skipped blocks and column range, from
swb_debug_strips.   chain_anatomy.py [N] [OPT=V ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
ctx = get_context(0)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
a, b = synthetic_pair(n, seed=1003)
with Session(ctx, a, b, sc) as S:
    S.reset_bounds()
    scored, _ = phase1.best_local(S, True)
    e = scored.end
    band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
    for rep in range(2):
        t0 = time.perf_counter()
        phase2.locate_start(S, e, scored.score, band)
        wall = time.perf_counter() - t0
    d = ctx.debug_strips()
cb, ce, ex, sk = d[:, 1], d[:, 2], d[:, 4], d[:, 5]
t0s, t1s = d[:, 12].astype(np.float64), d[:, 13].astype(np.float64)
ran = ex + sk > 0
tmin = t0s[ran].min()
starts = (t0s - tmin) / 1e3
ends = (t1s - tmin) / 1e3
idx = np.flatnonzero(ran)
lag = np.diff(starts[idx])
act = (ends - starts)[idx]
width = (ce - cb)[idx]
out = {"n": n, "wall_s": round(wall, 3), "kernel_ms": round(ctx.last_kernel_ms, 1),
       "strips": int(d.shape[0]), "strips_ran": int(idx.size),
       "span_us": round(float(ends[idx].max()), 1),
       "lag_us_median": round(float(np.median(lag)), 2), "lag_us_mean": round(float(lag.mean()), 2),
       "active_us_median": round(float(np.median(act)), 2),
       "width_cols_median": int(np.median(width)), "exec_blocks_median": int(np.median(ex[idx])),
       "skip_blocks_median": int(np.median(sk[idx])),
       "us_per_exec_block": round(float(act.sum() / max(1, ex[idx].sum())), 3)}
print(json.dumps(out), flush=True)
