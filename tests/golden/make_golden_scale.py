"""Golden vectors at BASELINE scale, produced by running the REAL reference.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_scale.py [names...]

Inputs are the bench's own synthetic pairs (`bench.synthetic_pair`, seeds of
SURVEY.md §8(d)), regenerated bit-identically from the seed on any box, so only
the outputs are committed.  Each record runs the unmodified reference
(`/root/reference/pkg/src/wavealign`) with `AlignConfig(workers=8)`:

  C2        `align` on the full C2 pair (1 Mbp x 1 Mbp, seed 1002): phase 1 is
            exactly `score_only` (pipeline.py:74 vs :103-126), so score and end
            pin the headline pass; start and CIGAR pin phases 2-3.
  C3w       `align` on the first 200 kbp x 200 kbp of the C3 pair (seed 1003).
  C5w       `align` on the first 200 kbp x 200 kbp of the C5 pair (seed 1005).
  C4w       `score_only` on the first 1 Mbp x 1 Mbp of the C4 unrelated pair
            (seed 1004).
  C3w_split `align(split=2)` on the C3 window (split.py:84-182).

Each record is written to tests/golden/scale/<name>.json as it finishes, and
all finished records are gathered into tests/golden/golden_scale.json.gz.
"""
from __future__ import annotations

import gzip
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import wavealign as wa  # noqa: E402

from bench import synthetic_pair  # noqa: E402

WORKERS = 8
SYM = np.frombuffer(b"ACGT", dtype=np.uint8)

CASES = {
    # name: (pair n, seed, homologous, window (n1, n2) or None, op, split)
    "C3w": (5_000_000, 1003, True, (200_000, 200_000), "align", 1),
    "C5w": (32_000_000, 1005, True, (200_000, 200_000), "align", 1),
    "C3w_split": (5_000_000, 1003, True, (200_000, 200_000), "align", 2),
    "C4w": (10_000_000, 1004, False, (1_000_000, 1_000_000), "score_only", 1),
    "C2": (1_000_000, 1002, True, None, "align", 1),
}


def run(name: str) -> dict:
    n, seed, homologous, window, op, split = CASES[name]
    a, b = synthetic_pair(n, seed=seed, homologous=homologous)
    if window is not None:
        a, b = a[:window[0]], b[:window[1]]
    alpha = wa.Alphabet.dna()  # the bench's alphabet: ACGT + wildcard N
    scheme = wa.ScoringScheme.match_mismatch(alpha, 1, -3, 5, 2)
    s1 = wa.Sequence.make("target", SYM[a].tobytes().decode(), alpha)
    s2 = wa.Sequence.make("query", SYM[b].tobytes().decode(), alpha)
    cfg = wa.AlignConfig(workers=WORKERS, split=split)
    rec = {"name": name, "n": n, "seed": seed, "homologous": homologous,
           "window": list(window) if window else None, "op": op, "split": split,
           "n1": int(a.size), "n2": int(b.size), "workers": WORKERS,
           "scheme": "match_mismatch(Alphabet.dna(), 1, -3, 5, 2)"}
    rep: dict = {}
    t0 = time.perf_counter()
    if op == "score_only":
        sc = wa.score_only(s1, s2, scheme, cfg, report=rep)
        rec["score"], rec["end"] = sc.score, list(sc.end)
    else:
        summ, path = wa.align(s1, s2, scheme, cfg, report=rep)
        rec.update(score=summ.score, start=list(summ.start), end=list(summ.end),
                   cigar=wa.path_to_cigar(path))
    rec["ref_seconds"] = time.perf_counter() - t0
    rec["ref_report"] = {k: v for k, v in rep.items() if isinstance(v, (int, float, str))}
    return rec


def gather():
    recs = []
    for p in sorted((HERE / "scale").glob("*.json")):
        recs.append(json.loads(p.read_text()))
    with gzip.open(HERE / "golden_scale.json.gz", "wt") as fh:
        json.dump(recs, fh)
    print(f"golden_scale.json.gz: {[r['name'] for r in recs]}", flush=True)


def main(names):
    (HERE / "scale").mkdir(exist_ok=True)
    for name in names or list(CASES):
        out = HERE / "scale" / f"{name}.json"
        if out.exists():
            continue
        rec = run(name)
        out.write_text(json.dumps(rec))
        print(f"{name}: score {rec['score']} end {rec['end']} "
              f"({rec['ref_seconds']:.0f} s)", flush=True)
        gather()
    gather()


if __name__ == "__main__":
    main(sys.argv[1:])
