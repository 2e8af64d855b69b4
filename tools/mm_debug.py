"""Run phase 3 level by level with live ranges on and report the first
failing subproblem (debug aid for the tile-bound static ranges)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import phase1, phase2, phase3
from paper_1304_5966_b200.engine import Session, get_context
from paper_1304_5966_b200.model import AlignmentSummary
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
ctx = get_context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 120_000
rng = np.random.default_rng(0)
a = random_codes(rng, n); b = mutate_codes(rng, a, 0.1)
for live in (0, 3):
    ctx.set_option("live_ranges", live)
    with Session(ctx, a, b, sc) as S:
        S.reset_bounds()
        scored, _ = phase1.best_local(S, True)
        e = scored.end
        band = phase2.compute_band(scored.score, min(e.i, e.j), max(e.i, e.j), sc)
        start = phase2.locate_start(S, e, scored.score, band)
        frontier = phase3._as_array([phase3.Subproblem(start, e, scored.score)], True)
        done = np.zeros(1, dtype=bool)
        for level in range(40):
            leaf = done | phase3._is_leaf(frontier, phase3.DEFAULT_LEAF_LIMIT)
            if leaf.all():
                print("live", live, "ok levels", level, flush=True)
                break
            inner = np.flatnonzero(~leaf)
            sub = frontier[inner]
            res, cells = ctx.crossings(S.cs, S.s1, S.s2, sub, True)
            badi = np.flatnonzero(res["status"])
            if badi.size:
                t = int(badi[0])
                print("live", live, "FAIL level", level, "sub", sub[t].tolist(), "reached", int(res["upper"][t]), flush=True)
                break
            kids = phase3._split_level(S, sub, True)
            width = np.where(leaf, 1, 2)
            pos = np.concatenate(([0], np.cumsum(width)[:-1]))
            nxt = np.zeros(int(width.sum()), dtype=frontier.dtype)
            nd = np.zeros(nxt.shape[0], dtype=bool)
            keep = np.flatnonzero(leaf)
            nxt[pos[keep]] = frontier[keep]; nd[pos[keep]] = True
            nxt[pos[inner]] = kids[0::2]; nxt[pos[inner] + 1] = kids[1::2]
            frontier, done = nxt, nd
        if live == 0:
            np.save(ROOT / "gpurun_out" / "frontier0.npy", frontier)
ctx.set_option("live_ranges", 3)
