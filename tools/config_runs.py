"""Large BASELINE configs on one GPU: C4 (10 Mbp x 10 Mbp unrelated, score pass)
and C5 (32 Mbp x 32 Mbp homologous, full alignment), one JSON line each.
    python tools/config_runs.py c4 c5"""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context

sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)  # the bench alphabet
ctx = get_context(0)
for which in sys.argv[1:]:
    if which in ("c4", "c3s", "c5s"):
        if which == "c4":
            a, b = synthetic_pair(10_000_000, seed=1004, homologous=False)
        elif which == "c5s":
            a, b = synthetic_pair(32_000_000, seed=1005)
        else:
            a, b = synthetic_pair(5_000_000, seed=1003)
        s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
        rep = {}
        t0 = time.perf_counter()
        r = swb.score_only(s1, s2, sc, report=rep)
        dt = time.perf_counter() - t0
        name = {"c4": "C4 10 Mbp x 10 Mbp unrelated (seed 1004), score_only",
                "c3s": "C3 5 Mbp homologous (seed 1003), score_only",
                "c5s": "C5 32 Mbp homologous (seed 1005), score_only"}[which]
        print(json.dumps({"config": name, "n1": int(a.size),
                          "n2": int(b.size), "score": r.score, "end": list(r.end), "wall_s": round(dt, 3),
                          "gcups_e2e": round(a.size * b.size / dt / 1e9, 1),
                          **{k: v for k, v in rep.items() if isinstance(v, (int, float, str))}}), flush=True)
    elif which in ("c5", "c3"):
        n = 32_000_000 if which == "c5" else 5_000_000
        a, b = synthetic_pair(n, seed=1005 if which == "c5" else 1003)
        s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
        rep = {}
        t0 = time.perf_counter()
        summ, path = swb.align(s1, s2, sc, report=rep)
        dt = time.perf_counter() - t0
        ok = swb.score_of_path(path, s1, s2, sc) == summ.score and path.start == summ.start and path.end == summ.end
        print(json.dumps({"config": f"{which.upper()} {n // 1_000_000} Mbp homologous full align, 1 GPU",
                          "n1": int(a.size), "n2": int(b.size), "score": summ.score, "start": list(summ.start),
                          "end": list(summ.end), "ops": int(path.ops.size), "path_rescored_equal": bool(ok),
                          "wall_s": round(dt, 3),
                          "phase_seconds": [round(x, 3) for x in rep.get("phase_seconds", [])],
                          "mm_levels": rep.get("mm_levels"), "device_cells": rep.get("device_cells")}), flush=True)
