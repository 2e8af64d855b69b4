"""One score pass (one pass_kernel launch) for ncu / compute-sanitizer."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import dna_scheme, mutate_codes, random_codes  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
unrel = len(sys.argv) > 2 and sys.argv[2] == "unrelated"
rng = np.random.default_rng(1002)
a = random_codes(rng, n)
b = random_codes(rng, n) if unrel else mutate_codes(rng, a, 0.10)
sc = dna_scheme()
s1 = swb.Sequence.from_codes("a", a, sc.alphabet)
s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
import os
if "X2" in os.environ:
    swb.get_context(0).set_option("x2", int(os.environ["X2"]))
rep = {}
r = swb.score_only(s1, s2, sc, report=rep)
print(r, rep)
