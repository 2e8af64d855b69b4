"""Generate golden vectors by running the REAL reference (`wavealign`) here.

Run in the build container (the reference is not available on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports /root/reference/pkg/src/wavealign unchanged, draws instances with the
reference test suite's own generators (pkg/tests/support.py:19-81) and records,
per instance: the two sequences, the scheme, and the outputs of
  * wavealign.score_only            (pipeline.py:103-126)
  * wavealign.align  split=1        (pipeline.py:46-100), default leaf_limit and
                                      a small leaf_limit (deep Myers-Miller)
  * wavealign.align  split=2        (split.py:84-182)
  * wavealign.oracle_local score/end (oracle.py:146-164)
as score / start / end / extended CIGAR.  The files are committed so the
parity tests never need the reference at run time.
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import wavealign as wa  # noqa: E402
from support import DNA, mutate, random_pair, random_scheme, random_text  # noqa: E402

OUT = Path(__file__).resolve().parent


def scheme_dict(s: wa.ScoringScheme) -> dict:
    return {
        "symbols": s.alphabet.symbols,
        "wildcard": s.alphabet.wildcard,
        "matrix": s.matrix.tolist(),
        "gap_open": s.gap_open,
        "gap_extend": s.gap_extend,
    }


def run_case(a: str, b: str, scheme: wa.ScoringScheme, alphabet, small_leaf: int,
             oracle: bool = True) -> dict:
    s1 = wa.Sequence.make("a", a, alphabet)
    s2 = wa.Sequence.make("b", b, alphabet)
    rec = {"seq1": a, "seq2": b, "scheme": scheme_dict(scheme)}
    rep: dict = {}
    sc = wa.score_only(s1, s2, scheme, wa.AlignConfig(), report=rep)
    rec["score_only"] = {"score": sc.score, "end": list(sc.end)}
    for tag, cfg in (("align", wa.AlignConfig()),
                     ("align_leaf", wa.AlignConfig(leaf_limit=small_leaf)),
                     ("align_split", wa.AlignConfig(split=2))):
        summ, path = wa.align(s1, s2, scheme, cfg)
        rec[tag] = {
            "score": summ.score,
            "start": list(summ.start),
            "end": list(summ.end),
            "cigar": wa.path_to_cigar(path),
        }
    rec["leaf_limit_small"] = small_leaf
    if oracle:
        osum, _ = wa.oracle_local(s1, s2, scheme, cell_budget=2 * 10 ** 8)
        rec["oracle_local"] = {"score": osum.score, "end": list(osum.end)}
    return rec


def small_cases(seed: int, n: int, max_len: int, alphabet, tag: str) -> list:
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        kind = t % 6
        a, b = random_pair(rng, kind, max_len, alphabet)
        scheme = random_scheme(rng, alphabet)
        small_leaf = int(rng.choice([4, 16, 64, 256]))
        rec = run_case(a, b, scheme, alphabet, small_leaf)
        rec["kind"] = kind
        rec["tag"] = tag
        out.append(rec)
    return out


def medium_cases(seed: int) -> list:
    """Homologous / unrelated / repetitive pairs of 1-6 kbp with the DNA
    benchmark scheme: several warp-strips deep on the GPU."""
    rng = np.random.default_rng(seed)
    scheme = wa.ScoringScheme.match_mismatch(DNA, 1, -3, 5, 2)
    out = []
    for t, (la, kind) in enumerate([(1500, "homologous"), (3000, "homologous"),
                                    (2500, "unrelated"), (4000, "homologous"),
                                    (1200, "repeat"), (6000, "homologous"),
                                    (2048, "homologous_indel"), (5000, "unrelated")]):
        a = random_text(rng, la, DNA)
        if kind.startswith("homologous"):
            b = mutate(a, 0.25 if kind.endswith("indel") else 0.10, rng, DNA)
            # embed in random flanks so start/end are interior
            b = random_text(rng, int(rng.integers(0, 300)), DNA) + b + \
                random_text(rng, int(rng.integers(0, 300)), DNA)
        elif kind == "repeat":
            unit = random_text(rng, 7, DNA)
            a = (unit * (la // 7 + 1))[:la]
            b = mutate(a, 0.05, rng, DNA)
        else:
            b = random_text(rng, int(la * 0.9), DNA)
        rec = run_case(a, b, scheme, DNA, 1024)
        rec["kind"] = kind
        rec["tag"] = "medium"
        out.append(rec)
    return out


def config1() -> dict:
    """BASELINE config 1: 10 kbp x ~10 kbp, mutate(a, 0.10), +1/-3, 5+2k.
    Seed 1001; first draw target, then query."""
    rng = np.random.default_rng(1001)
    a = random_text(rng, 10_000, DNA)
    b = mutate(a, 0.10, rng, DNA)
    scheme = wa.ScoringScheme.match_mismatch(DNA, 1, -3, 5, 2)
    rec = run_case(a, b, scheme, DNA, 4096)
    rec["tag"] = "config1"
    return rec


def main():
    cases = []
    cases += small_cases(20240811, 900, 300, DNA, "dna_small")
    cases += small_cases(7, 300, 60, DNA, "dna_tiny")
    cases += small_cases(99, 120, 200, wa.Alphabet.dna(wildcard=True), "dna_n")
    med = medium_cases(4242)
    c1 = config1()
    with gzip.open(OUT / "golden_small.json.gz", "wt") as fh:
        json.dump(cases, fh)
    with gzip.open(OUT / "golden_medium.json.gz", "wt") as fh:
        json.dump(med + [c1], fh)
    print(f"wrote {len(cases)} small and {len(med) + 1} medium cases")


if __name__ == "__main__":
    main()
