"""A/B of the tile bound maps on full alignments: identical
results, phase times and per-level stats."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
for n in [int(x) for x in sys.argv[1:]] or [1_000_000]:
    a, b = synthetic_pair(n, seed=1003)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    ref = None
    for on in (0, 1):
        ctx.set_option("bound_maps", on)
        rep = {}
        t0 = time.perf_counter()
        summ, path = swb.align(s1, s2, sc, report=rep)
        dt = time.perf_counter() - t0
        key = (summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes())
        ref = ref or key
        lv = [(x["subs"], x["cells"], x["wall_s"]) for x in rep.get("mm_level_stats", [])][:8]
        print(json.dumps({"n": n, "bound_maps": on, "wall_s": round(dt, 3),
                          "phase_s": [round(x, 3) for x in rep["phase_seconds"]],
                          "cells": rep.get("device_cells"), "same": key == ref, "levels": lv}), flush=True)
ctx.set_option("bound_maps", 1)
