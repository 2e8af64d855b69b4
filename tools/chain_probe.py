"""Timing probe for the score pass: kernel time vs strip count (chain length)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import dna_scheme, mutate_codes, random_codes  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402

sc = dna_scheme()
ctx = swb.get_context(0)
for spec in sys.argv[1:]:
    n1, n2, kind, *opt = spec.split(":")
    n1, n2 = int(n1), int(n2)
    prune = "noprune" not in opt
    ctas = 0
    for o in opt:
        if o.startswith("ctas="):
            ctas = int(o[5:])
    ctx.set_option("max_ctas_per_sm", ctas)
    proto = 2
    rpl = 0
    claim = 0
    for o in opt:
        if o.startswith("claim="):
            claim = int(o[6:])
        if o.startswith("R="):
            rpl = int(o[2:])
        if o.startswith("proto="):
            proto = int(o[6:])
    ctx.set_option("proto", proto)
    ctx.set_option("rows_per_lane", rpl)
    ctx.set_option("claim_mode", claim)
    rng = np.random.default_rng(7)
    a = random_codes(rng, n1)
    if kind == "hom":
        b = mutate_codes(rng, random_codes(rng, n2) if n2 > n1 else a, 0.1)[:n2]
        if b.size < n2:
            b = np.concatenate([b, random_codes(rng, n2 - b.size)])
    else:
        b = random_codes(rng, n2)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet)
    s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    cfg = swb.AlignConfig(prune=prune)
    swb.score_only(s1, s2, sc, cfg)
    rep = {}
    ctx.set_option("reset_debug", 0)
    r = swb.score_only(s1, s2, sc, cfg, report=rep)
    dbg = ctx.debug_stats()
    ms = rep["kernel_ms"]
    strips = (n1 + 1023) // 1024
    print(json.dumps({"spec": spec, "score": r.score, "end": list(r.end), "kernel_ms": round(ms, 3),
                      "strips": strips, "us_per_step": round(ms * 1e3 / (n2 + 64 * strips), 4),
                      "gcups": round(n1 * n2 / ms / 1e6, 2),
                      "gcups_exec": round(rep["cells_executed"] / ms / 1e6, 2),
                      "pruned": round(rep["pruned_fraction"], 3),
                      "wait_frac": round(dbg["wait_cycles"] / max(1, dbg["strip_cycles"]), 3)}), flush=True)
