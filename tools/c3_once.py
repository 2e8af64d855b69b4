"""One full alignment of the C3 pair (ncu launch-list target)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
a, b = synthetic_pair(5_000_000, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
rep = {}
summ, path = swb.align(s1, s2, sc, report=rep)
print(summ, rep.get("phase_seconds"))
