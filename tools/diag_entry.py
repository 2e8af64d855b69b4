"""Packed score pass on the C2 pair (or the C3 pair: diag_entry.py N): per
item, when it reaches its diagonal (proto 10 records the first block whose
columns pass the item's first row) and when it ends."""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synthetic_pair(n, seed=1002 if n == 1_000_000 else 1003)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
for prune in ((True, False, True) if n == 1_000_000 else (True,)):
    ctx.set_option("proto", 10)
    swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
    ctx.set_option("proto", 0)
    t = ctx.debug_times().astype(np.float64)
    t0 = t[:, 0].min()
    en, dg = (t[:, 1] - t0) / 1e6, (t[:, 2] - t0) / 1e6
    q = np.linspace(0, len(t) - 1, 33 if n > 1_000_000 else 17).astype(int)
    print(f"prune={prune} kernel {ctx.last_kernel_ms:.1f} ms")
    print("  item ", q.tolist())
    print("  diag ", np.round(dg[q], 1).tolist())
    print("  end  ", np.round(en[q], 1).tolist())
    d = np.diff(dg)
    print(f"  diag hop us: mean {d.mean()*1e3:.1f} by sixth {[round(float(x.mean())*1e3, 1) for x in np.array_split(d, 6)]}", flush=True)
