"""Tall-narrow pairs (n1 ~ 1000-1600, n2 ~ 30-200) with random schemes over
DNA and protein alphabets, checked against the oracle: exercises restricted
passes whose strips start late and exit early.
    narrow_sweep.py KIND(dna|protein) CASES SEED"""
import os, sys
import numpy as np
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "tests")]
import oracle
from helpers import mutate_codes, oracle_scheme
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import Alphabet, ScoringScheme, Sequence
kind, cases, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(seed)
alpha = Alphabet.dna(wildcard=False) if kind == "dna" else Alphabet("protein", "ARNDCQEGHILKMFPSTWYVBZX*")
k = len(alpha)
bad = 0
for c in range(cases):
    m = rng.integers(-4, 2, size=(k, k)).astype(np.int64)
    m[np.arange(k), np.arange(k)] = rng.integers(2, 12, size=k)
    sch = ScoringScheme(alpha, m, int(rng.integers(0, 12)), int(rng.integers(1, 5)), int(m.max()))
    n2 = int(rng.integers(30, 200))
    core = rng.integers(0, k, size=n2, dtype=np.uint8)
    b = mutate_codes(rng, core, 0.2, k=k)
    a = np.concatenate([rng.integers(0, k, size=int(rng.integers(300, 800)), dtype=np.uint8), core,
                        rng.integers(0, k, size=int(rng.integers(300, 800)), dtype=np.uint8)])
    if rng.random() < 0.3:
        a, b = b, a
    want = oracle.align(a, b, oracle_scheme(sch))
    s, p = swb.align(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha), sch)
    ok = (s.score, tuple(s.start), tuple(s.end)) == want[:3] and np.array_equal(p.ops, want[3])
    bad += not ok
    if not ok:
        print("MISMATCH", c, a.size, b.size, flush=True)
print(kind, "cases", cases, "bad", bad, flush=True)
