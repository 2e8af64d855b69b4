"""Quick device probe: integer/DPX peak + score pass throughput at a few sizes.

    python tools/perf_probe.py [n] [--rows-per-lane R] [--ctas K]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

from helpers import dna_scheme, mutate_codes, random_codes  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402
from paper_1304_5966_b200 import Sequence, get_context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sizes", nargs="*", type=int, default=[100_000, 1_000_000])
    ap.add_argument("--rows-per-lane", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--unrelated", action="store_true")
    ap.add_argument("--noprune", action="store_true")
    ap.add_argument("--peak", action="store_true")
    args = ap.parse_args()
    ctx = get_context(0)
    if args.peak:
        print(json.dumps({"int_peak": ctx.measure_int_peak()}))
    ctx.set_option("rows_per_lane", args.rows_per_lane)
    ctx.set_option("max_ctas_per_sm", args.ctas)
    scheme = dna_scheme()
    for n in args.sizes:
        rng = np.random.default_rng(1002)
        a = random_codes(rng, n)
        b = random_codes(rng, n) if args.unrelated else mutate_codes(rng, a, 0.10)
        s1 = Sequence.from_codes("a", a, scheme.alphabet)
        s2 = Sequence.from_codes("b", b, scheme.alphabet)
        cfg = swb.AlignConfig(prune=not args.noprune)
        swb.score_only(s1, s2, scheme, cfg)  # warm-up
        rep = {}
        t0 = time.perf_counter()
        r = swb.score_only(s1, s2, scheme, cfg, report=rep)
        t1 = time.perf_counter()
        cells = a.size * b.size
        print(json.dumps({"n1": int(a.size), "n2": int(b.size), "score": r.score, "end": list(r.end),
                          "wall_s": t1 - t0, "kernel_ms": rep["kernel_ms"],
                          "gcups_full_kernel": cells / (rep["kernel_ms"] * 1e-3) / 1e9,
                          "gcups_exec_kernel": rep["cells_executed"] / (rep["kernel_ms"] * 1e-3) / 1e9,
                          "pruned_fraction": rep["pruned_fraction"]}), flush=True)


if __name__ == "__main__":
    main()
