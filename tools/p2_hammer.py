"""Hammer the phase-2 restricted pass (late start + early exit + tile bound
maps, shared-table kernel) with the protein goldens in random order, random
zero-score DNA aligns in between to vary scratch contents; on a wrong pass
result dump the per-strip record (swb_debug_strips).
Usage: p2_hammer.py ITERS SEED   (env OPTS=name=v,...)"""
import gzip, json, os, sys
import numpy as np
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "tests")]
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, Alphabet, ScoringScheme, Sequence
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX, bound_slack
from helpers import golden_inputs

iters, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
ctx = get_context(0)
for kv in filter(None, os.environ.get("OPTS", "").split(",")):
    k, v = kv.split("=")
    ctx.set_option(k, int(v))
recs = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden_protein.json.gz")))
alpha = Alphabet.dna(wildcard=False)
m = np.full((4, 4), -2, dtype=np.int64); m[0, 0] = 3
zscheme = ScoringScheme(alpha, m, 4, 1, 3)
bad = 0
for it in range(iters):
    if rng.random() < 0.5:
        n1, n2 = int(rng.integers(1, 2000)), int(rng.integers(1, 2000))
        a = rng.integers(1, 4, size=n1, dtype=np.uint8); b = rng.integers(0, 4, size=n2, dtype=np.uint8)
        fn = [swb.align, swb.score_only][int(rng.integers(0, 2))]
        fn(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha), zscheme)
    ri = int(rng.integers(0, len(recs)))
    s1, s2, sch = golden_inputs(recs[ri])
    if rng.random() < 0.5:
        swb.score_only(s1, s2, sch)
    with Session(ctx, s1.codes, s2.codes, sch) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        if scored.score == 0:
            continue
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sch)
        interval = phase2.oriented_interval(band, scored.score, e.i, e.j, sch)
        res = S.run([dict(rows=(0, e.i, 1), cols=(0, e.j, 1), border="restricted", clamp=False,
                          track=TRACK_MAX, band=interval, prune=2, prune_target=scored.score,
                          bound_read=1, bound_write=2, bound_offset=bound_slack(sch))])[0]
        want = recs[ri]["align"]
        ok = res.best_score == scored.score and (e.i - res.best_i - 1, e.j - res.best_j - 1) == tuple(want["start"])
        if not ok:
            bad += 1
            print(f"WRONG it {it} rec {ri}: target {scored.score} at {tuple(e)} band {interval} -> "
                  f"best {res.best_score} ({res.best_i},{res.best_j}) R {res.rows_per_lane} exec "
                  f"{res.executed_blocks} skip {res.pruned_blocks} total {res.total_blocks}\n"
                  f"  strips (cb_static cb ce exit exec skip alo ahi key i j has):\n  "
                  + str(ctx.debug_strips()).replace("\n", "\n  "), flush=True)
print("iters", iters, "bad", bad, flush=True)
