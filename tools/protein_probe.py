"""Protein (BLOSUM62, 24 symbols) throughput: score pass and full alignment."""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from conftest import load_golden
from helpers import golden_inputs, mutate_codes, random_codes
import paper_1304_5966_b200 as swb
_, _, sc = golden_inputs(load_golden("golden_protein.json.gz")[0])
for n in [int(x) for x in sys.argv[1:]] or [100_000, 1_000_000]:
    rng = np.random.default_rng(7)
    a = random_codes(rng, n, 20); b = mutate_codes(rng, a, 0.3, 20)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    swb.score_only(s1, s2, sc)
    rep = {}
    t0 = time.perf_counter(); r = swb.score_only(s1, s2, sc, report=rep); dt = time.perf_counter() - t0
    out = {"n": n, "gap": [sc.gap_open, sc.gap_extend], "score": r.score, "score_pass_s": round(dt, 3),
           "gcups": round(a.size * b.size / dt / 1e9, 1), "pruned_fraction": rep.get("pruned_fraction")}
    if n <= 2_000_000:
        t0 = time.perf_counter(); summ, path = swb.align(s1, s2, sc); out["align_s"] = round(time.perf_counter() - t0, 3)
        out["path_ok"] = bool(swb.score_of_path(path, s1, s2, sc) == summ.score)
    print(json.dumps(out), flush=True)
