"""One banded free pass (TRACK_NONE) for ncu: n x n, band +-w."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_pair  # noqa: E402
import paper_1304_5966_b200 as swb  # noqa: E402
from paper_1304_5966_b200.engine import Session  # noqa: E402

n = int(sys.argv[1])
w = int(sys.argv[2])
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(wildcard=False), 1, -3, 5, 2)
a, b = synthetic_pair(n, seed=5)
with Session(swb.get_context(0), a, b, sc) as S:
    r = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="free", clamp=False, track=0,
                    band=(-w, w) if w else None)])[0]
print(r.kernel_ms, r.cells_executed)
