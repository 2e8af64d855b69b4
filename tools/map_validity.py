"""Check the tile bound maps against an optimal path: for every path cell c,
fwd map >= prefix score up to c and rev map >= suffix score from c."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2
from paper_1304_5966_b200.engine import Session, get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
import numpy as _np
sys.path.insert(0, str(ROOT / 'tests'))
from helpers import mutate_codes, random_codes
_rng = _np.random.default_rng(0)
a = random_codes(_rng, n); b = mutate_codes(_rng, a, 0.1)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx.set_option("live_ranges", 0)
summ, path = swb.align(s1, s2, sc)
# per-cell prefix scores along the path (cells consumed by = / X / D / I ops)
go, ge = sc.gap_open, sc.gap_extend
i, j = summ.start.i, summ.start.j
cells, pre = [], []
score, prev = 0, None
for op in path.ops.tolist():
    if op in (0, 1):
        score += int(sc.matrix[a[i], b[j]]); c = (i, j); i += 1; j += 1
    elif op == 2:
        score -= ge + (go if prev != 2 else 0); c = (i - 1, j); j += 1
    else:
        score -= ge + (go if prev != 3 else 0); c = (i, j - 1); i += 1
    prev = op
    cells.append(c); pre.append(score)
pre = np.array(pre); total = pre[-1]
assert total == summ.score
ci = np.array([max(x[0], 0) for x in cells]); cj = np.array([max(x[1], 0) for x in cells])
nc = (b.size + 1023) // 1024
for live in (0, 1):
    ctx.set_option("live_ranges", live)
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        phase2.locate_start(S, e, scored.score, band)
        fm = ctx.bounds_map(1).astype(np.int64); rm = ctx.bounds_map(2).astype(np.int64)
    k = (ci >> 10) * nc + (cj >> 10)
    f = np.where(fm[k] < 0, 1 << 40, fm[k] - (1 << 30)); r = np.where(rm[k] < 0, 1 << 40, rm[k] - (1 << 30))
    suf = total - pre + np.array([int(sc.matrix[a[x], b[y]]) if x < a.size and y < b.size else 0 for x, y in cells])
    badf = np.flatnonzero(f < pre - 20); badr = np.flatnonzero(r < suf - 40)
    from paper_1304_5966_b200.engine import bound_slack
    K = bound_slack(sc)
    marg = f + r - (total - K)
    t = int(np.argmin(marg))
    print("   min margin f+r-(target-K):", int(marg.min()), "at", cells[t], "f-pre", int(f[t] - pre[t]),
          "r-suf", int(r[t] - suf[t]), "K", K, "frac<0", float((marg < 0).mean()), flush=True)
    print("live", live, "path cells", len(cells), "fwd violations", badf.size, "rev violations", badr.size, flush=True)
    for t in badr[:8]:
        print("   rev cell", cells[t], "tile", (cells[t][0] >> 10, cells[t][1] >> 10), "map", int(r[t]), "suffix", int(suf[t]))
    for t in badf[:5]:
        print("   fwd cell", cells[t], "map", int(f[t]), "prefix", int(pre[t]))
ctx.set_option("live_ranges", 1)
