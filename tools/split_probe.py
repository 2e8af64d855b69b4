"""split=2 against split=1 on C-config pairs: wall time, phase report, results.
Usage: split_probe.py [N ...]"""
import json
import sys
import time
sys.path.insert(0, '/root/repo')
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
for n in [int(x) for x in sys.argv[1:]] or (1_000_000, 5_000_000):
    a, b = synthetic_pair(n, seed=1003)
    s1, s2 = swb.Sequence.from_codes("a", a, sc.alphabet), swb.Sequence.from_codes("b", b, sc.alphabet)
    swb.align(s1, s2, sc, swb.AlignConfig(split=2))
    out = {}
    from paper_1304_5966_b200 import split as split_mod
    from paper_1304_5966_b200.engine import Session, get_context
    modes = [(1, None), (2, True)] + ([(2, False)] if n <= 1_000_000 else [])
    for split, mode in modes:
        rep = {}
        t0 = time.perf_counter()
        if split == 1:
            summ, path = swb.align(s1, s2, sc, swb.AlignConfig(split=1), report=rep)
        else:
            with Session(get_context(0), a, b, sc) as S:
                summ, path = split_mod.split_align(S, report=rep, fast=mode)
        dt = time.perf_counter() - t0
        out[split] = (summ.score, tuple(summ.start), tuple(summ.end))
        print(json.dumps({"n": n, "split": split, "mode": mode, "s": round(dt, 3), "score": summ.score,
                          "start": list(summ.start), "end": list(summ.end),
                          "case": rep.get("case"), "kernel_ms": round(rep.get("device_kernel_ms", 0), 1),
                          "phase_s": [round(x, 3) for x in rep.get("phase_seconds", ())],
                          "halves_ms": round(rep.get("halves_kernel_ms", 0), 1),
                          "halves_cells": rep.get("halves_cells"), "p1_cells": rep.get("cells_executed"),
                          "rescored": swb.score_of_path(path, s1, s2, sc) == summ.score}), flush=True)
