"""Default DNA alphabet (with the 'N' wildcard, code 4) on the packed kernel:
C2-size score pass without N, with N runs in both sequences, and the same
input on the 32-bit lane kernel (x2 off) for comparison.  wild_ab.py [N]"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synthetic_pair(n, seed=1002)
rng = np.random.default_rng(5)
aN, bN = a.copy(), b.copy()
for arr in (aN, bN):  # N runs (assembly gaps) and scattered N
    for st in rng.integers(0, arr.size - 200, 20):
        arr[st:st + int(rng.integers(1, 200))] = 4
    arr[rng.integers(0, arr.size, arr.size // 1000)] = 4
ctx = get_context(0)
for label, alpha, x, y in (("dna4", swb.Alphabet.dna(wildcard=False), a, b),
                           ("dna5 no N", swb.Alphabet.dna(), a, b),
                           ("dna5 with N", swb.Alphabet.dna(), aN, bN)):
    sc = swb.ScoringScheme.match_mismatch(alpha, 1, -3, 5, 2)
    s1, s2 = swb.Sequence.from_codes("a", x, alpha), swb.Sequence.from_codes("b", y, alpha)
    outs = {}
    for x2 in (1, 0):
        ctx.set_option("x2", x2)
        ms = []
        for _ in range(3):
            rep = {}
            r = swb.score_only(s1, s2, sc, report=rep)
            ms.append(rep["kernel_ms"])
        outs[x2] = (r.score, tuple(r.end))
        print(f"{label:12s} x2={x2} score {r.score} end {tuple(r.end)} kernel {min(ms):8.1f} ms "
              f"{x.size * y.size / min(ms) / 1e9:7.1f} TCUPS kernel={rep.get('kernel')}", flush=True)
    print(f"{label:12s} packed == lane: {outs[1] == outs[0]}", flush=True)
ctx.set_option("x2", 1)
