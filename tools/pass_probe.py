"""Single-pass timing for any border / tracking / band: pass_probe.py SPEC...
SPEC = n:border:track[:band=W][:R=r]  (homologous pair, n x n)"""
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
for spec in sys.argv[1:]:
    n, border, track, *opt = spec.split(":")
    n, track = int(n), int(track)
    band = None
    R = 0
    for o in opt:
        if o.startswith("band="):
            w = int(o[5:])
            band = (-w, w)
        if o.startswith("R="):
            R = int(o[2:])
    claim = 0
    for o in opt:
        if o.startswith("claim="):
            claim = int(o[6:])
    ctx.set_option("rows_per_lane", R)
    ctx.set_option("claim_mode", claim)
    ctx.set_option("reset_debug", 0)
    a, b = synthetic_pair(n, seed=5)
    with Session(ctx, a, b, sc) as S:
        sp = [dict(rows=(0, a.size, 0), cols=(0, b.size, 0), border=border,
                   clamp=border == "local", track=track, band=band)]
        S.run(sp)
        ctx.set_option("reset_debug", 0)
        res = S.run(sp)[0]
        dbg = ctx.debug_stats()
        tm = ctx.debug_times()
        np.save(ROOT / "gpurun_out" / f"times_{spec.replace(':', '_').replace('=', '')}.npy", tm)
    print(json.dumps({"spec": spec, "kernel_ms": round(res.kernel_ms, 2),
                      "cells": res.cells_executed,
                      "gcups_exec": round(res.cells_executed / res.kernel_ms / 1e6, 1),
                      "wait_frac": round(dbg["wait_cycles"] / max(1, dbg["strip_cycles"]), 3),
                      "best": [res.best_score, res.best_i, res.best_j]}), flush=True)
