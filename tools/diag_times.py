"""Critical-path anatomy of the C2 pass: when does each item reach its diagonal?"""
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
a, b = synthetic_pair(1_000_000, seed=1002)
s1 = swb.Sequence.from_codes("a", a, sc.alphabet); s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
for prune in (True, False):
    ctx.set_option("proto", 10)
    r = swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
    ctx.set_option("proto", 2)
    t = ctx.debug_times().astype(np.float64)
    t0 = t[:, 0].min()
    st, en, dg = (t[:, 0] - t0) / 1e6, (t[:, 1] - t0) / 1e6, (t[:, 2] - t0) / 1e6
    print(f"prune={prune}: kernel {ctx.last_kernel_ms:.1f} ms items {len(t)}")
    q = np.linspace(0, len(t) - 1, 12).astype(int)
    print("  diag entry ms", np.round(dg[q], 1))
    print("  end ms       ", np.round(en[q], 1))
    d = np.diff(dg)
    print(f"  per-item diagonal advance: median {np.median(d) * 1000:.1f} us mean {np.mean(d) * 1000:.1f} us; "
          f"first/second half means {np.mean(d[:len(d)//2]) * 1000:.1f} / {np.mean(d[len(d)//2:]) * 1000:.1f} us", flush=True)
