"""Single-warp step time of the packed kernel: a short, wide pass (few items,
one warp per SM sub-partition) is a pure chain, time / columns = step time."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import dna_scheme, mutate_codes, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MIN
ctx = get_context(0)
sc = dna_scheme()
rng = np.random.default_rng(5)
n2 = 1_000_000
b = random_codes(rng, n2)
for R in (8, 14, 16):
    for kind in ("unrelated", "copy"):
        n1 = 64 * R * 4
        a = random_codes(rng, n1) if kind == "unrelated" else b[:n1].copy()
        ctx.set_option("x2_R", R)
        with Session(ctx, a, b, sc) as S:
            for _ in range(2):
                r = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                                track=TRACK_MIN, prune=False)])[0]
        ms = r.kernel_ms
        print(f"R={R} {kind}: {ms:.1f} ms for {n2} columns -> {ms * 1e6 / (n2 + 4 * 96):.1f} ns/step "
              f"({ms * 1e6 / (n2 + 384) * 1.965:.0f} cycles), items {r.total_blocks and (n1 // (64 * R))}", flush=True)
ctx.set_option("x2_R", 0)
