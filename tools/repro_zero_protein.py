"""Reproducer: zero-score DNA pairs, then the protein goldens, in one process.
Usage: python tools/repro_zero_protein.py [which zero calls, e.g. 'a0 s0 o0 a1 ...'] """
import gzip, json, os, sys
import numpy as np
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "tests")]
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Alphabet, ScoringScheme, Sequence
from helpers import golden_inputs

from paper_1304_5966_b200.engine import get_context
for kv in filter(None, os.environ.get("OPTS", "").split(",")):
    k, v = kv.split("=")
    get_context(0).set_option(k, int(v))
steps = sys.argv[1].split() if len(sys.argv) > 1 else None
rng = np.random.default_rng(77)
alpha = Alphabet.dna(wildcard=False)
m = np.full((4, 4), -2, dtype=np.int64)
m[0, 0] = 3
scheme = ScoringScheme(alpha, m, 4, 1, 3)
for k, (n1, n2) in enumerate(((1, 1), (37, 900), (700, 65), (1500, 1499))):
    a = rng.integers(1, 4, size=n1, dtype=np.uint8)
    b = rng.integers(0, 4, size=n2, dtype=np.uint8)
    s1, s2 = Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha)
    for tag, fn in ((f"a{k}", lambda: swb.align(s1, s2, scheme)),
                    (f"s{k}", lambda: swb.align(s1, s2, scheme, AlignConfig(split=2))),
                    (f"o{k}", lambda: swb.score_only(s1, s2, scheme))):
        if steps is None or tag in steps:
            fn()
            print("ran", tag, flush=True)
recs = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden_protein.json.gz")))
first = int(os.environ.get("FIRST", 0))
only = os.environ.get("ONLY")
nrec = len(recs)
recs = recs * int(os.environ.get("REPEAT", 1))
for i, rec in enumerate(recs):
    i = i % nrec
    if i < first or (only and str(i) not in only.split(',')):
        continue
    s1, s2, sch = golden_inputs(rec)
    sc = swb.score_only(s1, s2, sch)
    print("protein", i, sc.score, rec["score_only"]["score"], flush=True)
    swb.align(s1, s2, sch)
    swb.align(s1, s2, sch, AlignConfig(split=2))
print("done")
