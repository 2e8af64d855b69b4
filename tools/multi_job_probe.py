"""Independent passes in one launch: per-warp speed vs chain length.
usage: multi_job_probe.py JOBS:ROWS ...  (ROWS per job, 20000 columns)"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import dna_scheme, random_codes  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402
from paper_1304_5966_b200.engine import Session, TRACK_MIN, TRACK_NONE  # noqa: E402

sc = dna_scheme()
ctx = swb.get_context(0)
rng = np.random.default_rng(3)
a = random_codes(rng, 1 << 20)
b = random_codes(rng, 20000)
for spec in sys.argv[1:]:
    k, rows, *opt = spec.split(":")
    k, rows = int(k), int(rows)
    track = TRACK_NONE if "none" in opt else TRACK_MIN
    local = "global" not in opt
    if not local and track == TRACK_MIN:
        track = TRACK_NONE
    with Session(ctx, a, b, sc) as S:
        specs = [dict(rows=(rows * t, rows, 0), cols=(0, 20000, 0),
                      border="local" if local else "free", clamp=local, track=track)
                 for t in range(k)]
        S.run(specs)
        ctx.set_option("reset_debug", 0)
        res = S.run(specs)
        dbg = ctx.debug_stats()
        tm = ctx.debug_times()
        t0 = tm[:, 0].min()
        timeline = [[round((x[0] - t0) / 1e6, 3), round((x[1] - t0) / 1e6, 3), round(x[2] / 1e6, 3)]
                    for x in tm[:8]]
        strips = k * ((rows + 1023) // 1024)
        print(json.dumps({"spec": spec, "kernel_ms": round(res[0].kernel_ms, 3),
                          "us_per_step": round(res[0].kernel_ms * 1e3 / 20000, 4),
                          "strip_ms_avg": round(dbg["strip_cycles"] / strips / 1.965e6, 3),
                          "wait_frac": round(dbg["wait_cycles"] / max(1, dbg["strip_cycles"]), 4),
                          "timeline_ms": timeline}),
              flush=True)
