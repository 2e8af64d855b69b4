"""Banded vs unbanded per-step cost with a handful of strips (no contention)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402
from paper_1304_5966_b200.engine import Session  # noqa: E402

sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = swb.get_context(0)
a, b = synthetic_pair(2_000_000, seed=5)
for spec in sys.argv[1:]:
    rows, band, R = [int(x) for x in spec.split(":")]
    ctx.set_option("rows_per_lane", R)
    ctx.set_option("reset_debug", 0)
    with Session(ctx, a[:rows], b, sc) as S:
        sp = [dict(rows=(0, rows, 0), cols=(0, S.n2, 0), border="free", clamp=False, track=0,
                   band=None if band == 0 else (-band, band))]
        S.run(sp)
        ctx.set_option("reset_debug", 0)
        res = S.run(sp)[0]
        tm = ctx.debug_times()
    t0 = tm[:, 0].min()
    per = [(int(x[1] - x[0]) / 1e6) for x in tm]
    steps = res.cells_executed / rows
    print(json.dumps({"spec": spec, "ms": round(res.kernel_ms, 2), "cells": res.cells_executed,
                      "strip_ms": [round(p, 2) for p in per[:6]],
                      "us_per_step": round(res.kernel_ms * 1e3 / max(steps, 1), 4)}), flush=True)
