"""Phase-2 pass of golden protein record 85 under option variants (the
fault / wrong-start case of DESIGN.md §7): prints the pass result, tile
counters and, with proto 9, each strip's final column range.
Usage: p2_fault_probe.py [REPS] [prefix]   (prefix: run the zero-score a1 align first)"""
import gzip, json, os, sys
import numpy as np
sys.path[:0] = [os.path.join(os.path.dirname(__file__), ".."), os.path.join(os.path.dirname(__file__), "..", "tests")]
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, Alphabet, ScoringScheme, Sequence
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MAX, bound_slack
from helpers import golden_inputs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = get_context(0)
if len(sys.argv) > 2 and sys.argv[2] == "prefix":
    rng = np.random.default_rng(77)
    alpha = Alphabet.dna(wildcard=False)
    m = np.full((4, 4), -2, dtype=np.int64); m[0, 0] = 3
    scheme = ScoringScheme(alpha, m, 4, 1, 3)
    for k, (n1, n2) in enumerate(((1, 1), (37, 900))):
        a = rng.integers(1, 4, size=n1, dtype=np.uint8); b = rng.integers(0, 4, size=n2, dtype=np.uint8)
        if k == 1:
            swb.align(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha), scheme)
recs = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden_protein.json.gz")))
s1, s2, sch = golden_inputs(recs[int(os.environ.get("REC", 85))])
if len(sys.argv) > 2 and sys.argv[2] == "prefix":
    for k, v in dict(live_big=3).items():
        ctx.set_option(k, v)
    swb.score_only(s1, s2, sch)
    print("prefix done", flush=True)
variants = [dict(live_big=lb, bound_maps=bm, proto=pr) for pr in (2, 9) for bm in (1, 0) for lb in (3, 1, 2, 0)]
for v in variants:
    for k, val in v.items():
        ctx.set_option(k, val)
    for rep in range(reps):
        with Session(ctx, s1.codes, s2.codes, sch) as S:
            S.reset_bounds()
            scored, _ = phase1.best_local(S, True)
            e = scored.end
            band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sch)
            interval = phase2.oriented_interval(band, scored.score, e.i, e.j, sch)
            extra = dict(bound_read=1, bound_write=2, bound_offset=bound_slack(sch)) if v["bound_maps"] else {}
            res = S.run([dict(rows=(0, e.i, 1), cols=(0, e.j, 1), border="restricted", clamp=False,
                              track=TRACK_MAX, band=interval, prune=2, prune_target=scored.score, **extra)])[0]
            ok = res.best_score == scored.score
            line = (f"{v} rep {rep}: target {scored.score} at {e} band {interval} -> best {res.best_score} "
                    f"({res.best_i},{res.best_j}) R {res.rows_per_lane} tiles exec {res.executed_blocks} "
                    f"pruned {res.pruned_blocks} total {res.total_blocks} {'OK' if ok else 'WRONG'}")
            if not ok or os.environ.get("DUMP"):
                line += "\n  strips (cb_static cb ce exit exec skip alo ahi runs sm cta warp t0 key i j has):\n  " + \
                    str(ctx.debug_strips()).replace("\n", "\n  ")
            if v["proto"] == 9 or not ok:
                t = ctx.debug_times()
                line += " ranges " + str([(int(x) >> 32, int(x) & 0xffffffff) for x in t[:, 2]])
            print(line, flush=True)
ctx.set_option("proto", 2)
