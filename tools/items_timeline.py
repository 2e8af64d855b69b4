"""Per-item timeline of one packed score pass on a BASELINE pair: busy
fraction, wait, and per-round statistics (items in claim order, one round =
one item per warp slot).  items_timeline.py N [homologous|unrelated]"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from bench import synthetic_pair
from helpers import dna_scheme
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.engine import get_context
ctx = get_context(0)
sc = dna_scheme()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
hom = (sys.argv[2] != "unrelated") if len(sys.argv) > 2 else True
a, b = synthetic_pair(n, seed=1003 if hom else 1004, homologous=hom)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for _rep in range(reps):
  rep = {}
  swb.score_only(s1, s2, sc, report=rep)
  ms = ctx.last_kernel_ms
  t = ctx.debug_times().astype(np.float64)
  t0 = t[:, 0].min()
  st, en, wt = (t[:, 0] - t0) / 1e6, (t[:, 1] - t0) / 1e6, t[:, 2] / 1e6
  act = en - st
  slots = 148 * 8
  print(f"kernel {ms:.1f} ms items {len(t)} rpl {rep.get('rows_per_lane')} pruned {rep.get('pruned_fraction'):.3f} "
        f"busy-frac {(act - wt).sum() / (ms * slots):.3f} wait-frac {wt.sum() / (ms * slots):.3f} "
        f"idle-frac {1 - act.sum() / (ms * slots):.3f}")
  for k in range(0, len(t), slots):
      sl = slice(k, min(k + slots, len(t)))
      print(f" round {k // slots}: start {st[sl].min():7.1f}..{st[sl].max():7.1f} end {en[sl].min():7.1f}..{en[sl].max():7.1f} "
            f"active {act[sl].mean():7.1f} wait {wt[sl].mean():7.1f} ms")
