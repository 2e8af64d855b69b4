import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
a, b = synthetic_pair(5_000_000, seed=1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
swb.align(s1, s2, sc)
pr = cProfile.Profile(); pr.enable()
swb.align(s1, s2, sc)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
