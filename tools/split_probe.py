import sys, time, json
sys.path.insert(0, '/root/repo')
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
for n in (1_000_000, 5_000_000):
    a, b = synthetic_pair(n, seed=1003)
    s1, s2 = swb.Sequence.from_codes("a", a, sc.alphabet), swb.Sequence.from_codes("b", b, sc.alphabet)
    swb.align(s1, s2, sc, swb.AlignConfig(split=2))
    for split in (1, 2):
        t0 = time.perf_counter(); summ, path = swb.align(s1, s2, sc, swb.AlignConfig(split=split)); dt = time.perf_counter() - t0
        print(json.dumps({"n": n, "split": split, "s": round(dt, 3), "score": summ.score, "start": list(summ.start), "end": list(summ.end)}), flush=True)
