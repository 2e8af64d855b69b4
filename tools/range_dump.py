"""Dump the kernel's per-strip column ranges for the failing level-1 subproblem
(proto 9) and check the final path against them."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, phase3
from paper_1304_5966_b200.engine import Session, get_context
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = 120_000
rng = np.random.default_rng(0)
a = random_codes(rng, n); b = mutate_codes(rng, a, 0.1)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
ctx.set_option("live_ranges", 0)
summ, path = swb.align(s1, s2, sc)
i, j = summ.start.i, summ.start.j
pts = [(i, j)]
for op in path.ops.tolist():
    if op in (0, 1): i += 1; j += 1
    elif op == 2: j += 1
    else: i += 1
    pts.append((i, j))
pts = np.array(pts)
sub = np.zeros(1, dtype=phase3.SUBPROBLEM_DTYPE)
sub[0] = (0, 0, 60000, 59937, 27775, 0, 0, 1, 0, 0, 28012)
for live in (0, 3):
    ctx.set_option("live_ranges", live)
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        phase2.locate_start(S, e, scored.score, band)
        ctx.set_option("proto", 9)
        res, cells = ctx.crossings(S.cs, S.s1, S.s2, sub, True)
        t = ctx.debug_times()
        ctx.set_option("proto", 2)
    print("live", live, "status", int(res["status"][0]), "upper", int(res["upper"][0]), "strips", len(t), flush=True)
    rng_cb = (t[:, 2] >> 32).astype(np.int64); rng_ce = (t[:, 2] & 0xffffffff).astype(np.int64)
    # strips: upper pass first (job 0) then lower (job 1), 256 rows each (R=8)
    nup = (30000 + 255) // 256
    bad = 0
    for k in range(len(t)):
        if k < nup:
            s = k; pr0, pr1 = s * 256, min(s * 256 + 256, 30000) - 1
            sel = (pts[:, 0] - 1 >= pr0) & (pts[:, 0] - 1 <= pr1); pc = pts[sel, 1] - 1
        else:
            s = k - nup; pr0, pr1 = s * 256, min(s * 256 + 256, 30000) - 1
            sel = (60000 - pts[:, 0] >= pr0) & (60000 - pts[:, 0] <= pr1); pc = 59937 - pts[sel, 1]
        pc = pc[(pc >= 0) & (pc < 59937)]
        if pc.size == 0: continue
        out = pc[(pc < rng_cb[k]) | (pc >= rng_ce[k])]
        if out.size:
            bad += 1
            if bad <= 6:
                print(f"   strip {k} range [{rng_cb[k]},{rng_ce[k]}) path {pc.min()}..{pc.max()} outside {out.size}")
    print("   strips with path outside:", bad, flush=True)
ctx.set_option("live_ranges", 3)
