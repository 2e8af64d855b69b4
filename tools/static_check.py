"""Replicate the level-0 static strip ranges in numpy and check that the
final path's cells lie inside them (upper half forward, lower half reversed)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, phase3
from paper_1304_5966_b200.engine import Session, get_context, bound_slack
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 120_000
rng = np.random.default_rng(0)
a = random_codes(rng, n); b = mutate_codes(rng, a, 0.1)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx.set_option("live_ranges", 0)
summ, path = swb.align(s1, s2, sc)
ops = path.ops
# path cells: DP coordinates after each op (i, j) = cells consumed
i, j = summ.start.i, summ.start.j
pts = [(i, j)]
for op in ops.tolist():
    if op in (0, 1): i += 1; j += 1
    elif op == 2: j += 1
    else: i += 1
    pts.append((i, j))
pts = np.array(pts)
K = bound_slack(sc)
if len(sys.argv) > 2:   # si sj ei ej expected
    si, sj, ei, ej, X = (int(x) for x in sys.argv[2:7])
    S_, T_ = swb.Coord(si, sj), swb.Coord(ei, ej)
else:
    S_, T_, X = summ.start, summ.end, summ.score
rows, cols = T_.i - S_.i, T_.j - S_.j
midr = rows // 2
lo_b, hi_b = phase3.band_interval(rows, cols, X, sc)
print("sub", S_, T_, "X", X, "band", lo_b, hi_b, flush=True)
nc = (b.size + 1023) >> 10
for live in (0, 1):
    ctx.set_option("live_ranges", live)
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        phase2.locate_start(S, e, scored.score, band)
        fm = ctx.bounds_map(1).astype(np.int64); rm = ctx.bounds_map(2).astype(np.int64)
    def useful(rt, ct):
        k = rt * nc + ct
        return (fm[k] < 0) | (rm[k] < 0) | (fm[k] + rm[k] - 2 * (1 << 30) + K >= summ.score)
    Rr = 8
    bad = 0
    # upper pass: forward rows S.i + r (r < midr), cols S.j + c
    for half in ("up", "dn"):
        n1 = midr if half == "up" else rows - midr
        if half == "up":
            blo, bhi = lo_b, hi_b
            r0f, rdir, c0f, cdir = S_.i, 1, S_.j, 1
        else:
            blo, bhi = rows - cols - hi_b, rows - cols - lo_b
            r0f, rdir, c0f, cdir = T_.i - 1, -1, T_.j - 1, -1
        for s in range((n1 + 32 * Rr - 1) // (32 * Rr)):
            pr0 = s * 32 * Rr; pr1 = min(pr0 + 32 * Rr, n1) - 1
            cb = max(0, pr0 - bhi); ce = min(cols, pr1 - blo + 1)
            if cb >= ce: continue
            fr = sorted((r0f + rdir * pr0, r0f + rdir * pr1)); rts = range(max(fr[0], 0) >> 10, (fr[1] >> 10) + 1)
            fc = sorted((c0f + cdir * cb, c0f + cdir * (ce - 1))); cts = np.arange(max(fc[0], 0) >> 10, (fc[1] >> 10) + 1)
            u = np.zeros(cts.size, dtype=bool)
            for rt in rts:
                u |= useful(rt, cts)
            if not u.any():
                lo_p, hi_p = ce, ce
            else:
                fmin, fmax = cts[u].min(), cts[u].max()
                flo, fhi = fmin << 10, ((fmax + 1) << 10) - 1
                lo, hi = (flo - c0f, fhi - c0f) if cdir > 0 else (c0f - fhi, c0f - flo)
                lo_p, hi_p = max(cb, lo), min(ce, hi + 1)
            # path cells in these rows (pass coordinates)
            if half == "up":
                sel = (pts[:, 0] - 1 - S_.i >= pr0) & (pts[:, 0] - 1 - S_.i <= pr1)
                pc = pts[sel, 1] - 1 - S_.j
            else:
                sel = (T_.i - pts[:, 0] >= pr0) & (T_.i - pts[:, 0] <= pr1)
                pc = T_.j - pts[sel, 1]
            pc = pc[(pc >= 0) & (pc < cols)]
            if pc.size == 0:
                continue
            out = pc[(pc < lo_p) | (pc >= hi_p)]
            if out.size:
                bad += 1
                if bad <= 5:
                    print(f"  live {live} {half} strip {s} range [{lo_p},{hi_p}) band [{cb},{ce}) path cols {pc.min()}..{pc.max()} outside {out.size}")
    print("live", live, "strips with path outside range:", bad, flush=True)
ctx.set_option("live_ranges", 3)
