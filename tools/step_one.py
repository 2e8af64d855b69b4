"""One chain-bound packed pass (4 items, one warp per sub-partition) for ncu."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from helpers import dna_scheme, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import Session, get_context, TRACK_MIN
ctx = get_context(0)
sc = dna_scheme()
rng = np.random.default_rng(5)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 14
b = random_codes(rng, 200_000)
a = random_codes(rng, 64 * R * 4)
ctx.set_option("x2_R", R)
with Session(ctx, a, b, sc) as S:
    r = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                    track=TRACK_MIN, prune=False)])[0]
print(r.kernel_ms)
