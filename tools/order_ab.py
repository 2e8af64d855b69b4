"""A/B of the multi-job claim order (strip-major item map vs job-major) on a full align."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synthetic_pair(n, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ref = None
for jm in (1, 0, 1, 0):
    ctx.set_option("job_major", jm)
    rep = {}
    t0 = time.perf_counter()
    summ, path = swb.align(s1, s2, sc, report=rep)
    dt = time.perf_counter() - t0
    key = (summ.score, tuple(summ.start), tuple(summ.end), path.ops.tobytes())
    ref = ref or key
    lv = [(x["subs"], x["wall_s"], x["kernel_ms"]) for x in rep.get("mm_level_stats", [])]
    print(json.dumps({"job_major": jm, "wall_s": round(dt, 3), "phase_s": [round(x, 3) for x in rep["phase_seconds"]],
                      "same": key == ref, "levels": lv}), flush=True)
ctx.set_option("job_major", 0)
