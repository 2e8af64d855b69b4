"""Break down the end-to-end score_only call (upload, pass, release)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MIN  # noqa: E402

a, b = synthetic_pair(1_000_000, seed=1002)
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet)
s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx = get_context(0)
for it in range(4):
    t0 = time.perf_counter()
    S = Session(ctx, a, b, sc)
    t1 = time.perf_counter()
    r = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                    track=TRACK_MIN, prune=True)])[0]
    t2 = time.perf_counter()
    S.close()
    t3 = time.perf_counter()
    t4 = time.perf_counter()
    swb.score_only(s1, s2, sc)
    t5 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  pass {1e3*(t2-t1):.1f} ms (kernel {r.kernel_ms:.1f})  "
          f"release {1e3*(t3-t2):.1f} ms  score_only {1e3*(t5-t4):.1f} ms", flush=True)
