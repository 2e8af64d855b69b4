"""Per-item timeline summary (start skew, active time, wait) for both kernels."""
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
for flag, R in ((1, 0), (1, 16)):
    for prune in (True, False):
        ctx.set_option("x2", flag); ctx.set_option("x2_R", R)
        swb.score_only(s1, s2, sc, swb.AlignConfig(prune=prune))
        ms = ctx.last_kernel_ms
        t = ctx.debug_times().astype(np.float64)
        t0 = t[:, 0].min()
        st, en, wt = (t[:, 0] - t0) / 1e6, (t[:, 1] - t0) / 1e6, t[:, 2] / 1e6
        act = en - st
        print(f"x2={flag} R={R} prune={prune}: kernel {ms:.1f} ms items={len(t)} span {en.max():.1f} "
              f"start[last]={st[-1]:.1f} start[mid]={st[len(t)//2]:.1f} active mean={act.mean():.1f} "
              f"max={act.max():.1f} wait mean={wt.mean():.1f} "
              f"busy-frac={(act - wt).sum() / (en.max() * len(t)):.3f}", flush=True)
        q = np.linspace(0, len(t) - 1, 9).astype(int)
        print("   start", np.round(st[q], 1), "end", np.round(en[q], 1), "wait", np.round(wt[q], 1))
