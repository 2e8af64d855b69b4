"""Randomised full-alignment parity sweep against the CPU oracle (all device
features at their defaults): schemes, sizes, input kinds."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import oracle
from helpers import dna_scheme, mutate_codes, oracle_scheme, random_codes
import paper_1304_5966_b200 as swb
rng0 = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
fails = 0
SIZES = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [3000, 12000, 40000, 90000]
t0 = time.time()
for t in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    rng = np.random.default_rng(rng0.integers(1 << 30))
    args = [(1, -3, 5, 2), (2, -1, 3, 2), (5, -2, 0, 4), (3, -5, 10, 1), (1, -1, 2, 1), (4, -4, 6, 3)][t % 6]
    sc = dna_scheme(None, *args)
    n = int(rng.choice(SIZES))
    kind = t % 4
    a = random_codes(rng, n)
    if kind == 0:
        b = mutate_codes(rng, a, float(rng.choice([0.05, 0.15, 0.3])))
    elif kind == 1:
        b = random_codes(rng, int(n * rng.uniform(0.5, 1.2)))
    elif kind == 2:  # embedded homolog with flanks
        core = mutate_codes(rng, a[n // 4: 3 * n // 4], 0.1)
        b = np.concatenate([random_codes(rng, n // 3), core, random_codes(rng, n // 5)])
    else:  # repeats
        unit = random_codes(rng, int(rng.integers(2, 12)))
        a = np.tile(unit, n // unit.size + 1)[:n]
        b = mutate_codes(rng, a, 0.08)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    summ, path = swb.align(s1, s2, sc)
    want = oracle.align(a, b, oracle_scheme(sc))
    ok = (summ.score, tuple(summ.start), tuple(summ.end)) == (want[0], tuple(want[1]), tuple(want[2])) \
        and np.array_equal(path.ops, want[3])
    if not ok:
        fails += 1
        print("FAIL", t, args, n, kind, (summ.score, tuple(summ.start), tuple(summ.end)), want[:3], flush=True)
print("cases", t + 1, "fails", fails, f"{time.time() - t0:.0f} s", flush=True)
