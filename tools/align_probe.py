"""Full alignment timing by phase: align_probe.py N [N ...] (homologous pairs)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402

sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
check = "--check" in sys.argv
for arg in [x for x in sys.argv[1:] if not x.startswith("--")]:
    n = int(arg)
    a, b = synthetic_pair(n, seed=1003)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet)
    s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    if n <= 200_000:
        swb.align(s1, s2, sc)  # warm-up
    rep = {}
    t0 = time.perf_counter()
    summ, path = swb.align(s1, s2, sc, report=rep)
    dt = time.perf_counter() - t0
    out = {"n1": int(a.size), "n2": int(b.size), "score": summ.score, "start": list(summ.start),
           "end": list(summ.end), "ops": int(path.ops.size), "wall_s": round(dt, 3),
           "gcups_e2e": round(a.size * b.size / dt / 1e9, 1),
           **{k: (round(v, 3) if isinstance(v, float) else v) for k, v in rep.items()
              if k in ("phase_seconds", "mm_levels", "mm_leaves", "t_crossings", "t_leaves",
                       "device_kernel_ms", "kernel_ms", "pruned_fraction", "mm_level_stats")}}
    if "phase_seconds" in out:
        out["phase_seconds"] = [round(x, 3) for x in rep["phase_seconds"]]
    if check:
        import oracle
        want = oracle.align(a, b, oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2))
        out["oracle_equal"] = bool((summ.score, tuple(summ.start), tuple(summ.end)) == want[:3]
                                   and np.array_equal(path.ops, want[3]))
    print(json.dumps(out), flush=True)
