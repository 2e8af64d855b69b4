"""Shared test helpers: golden-record decoding and seeded generators.

The generators mirror the reference test suite's shapes (pkg/tests/support.py:
19-81) in vectorised numpy so genome-scale inputs build in milliseconds.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_1304_5966_b200 import Alphabet, ScoringScheme, Sequence


def golden_inputs(rec):
    sch = rec["scheme"]
    kind = "nucleotide" if len(sch["symbols"]) <= 5 else "protein"
    alpha = Alphabet(kind, sch["symbols"], sch["wildcard"])
    scheme = ScoringScheme(alpha, np.array(sch["matrix"], dtype=np.int64), sch["gap_open"],
                           sch["gap_extend"], int(np.max(sch["matrix"])))
    s1 = Sequence.make("a", rec["seq1"], alpha)
    s2 = Sequence.make("b", rec["seq2"], alpha)
    return s1, s2, scheme


def oracle_scheme(scheme: ScoringScheme) -> oracle.OracleScheme:
    return oracle.OracleScheme(np.asarray(scheme.matrix, dtype=np.int64), scheme.gap_open,
                               scheme.gap_extend)


def random_codes(rng, n, k=4):
    return rng.integers(0, k, size=n, dtype=np.uint8)


def mutate_codes(rng, a, rate, k=4):
    """Substitution / insertion / deletion each at rate/3 (support.py:37-53)."""
    n = a.size
    r = rng.random(n)
    sub = r < rate / 3
    ins = (r >= rate / 3) & (r < 2 * rate / 3)
    dele = (r >= 2 * rate / 3) & (r < rate)
    out = a.copy()
    out[sub] = rng.integers(0, k, size=int(sub.sum()), dtype=np.uint8)
    keep = ~dele
    reps = np.where(ins, 2, 1)[keep]
    base = np.repeat(out[keep], reps)
    # the inserted residue follows its anchor: overwrite every second copy
    pos = np.cumsum(reps) - 1
    ins_pos = pos[ins[keep]]
    base[ins_pos] = rng.integers(0, k, size=ins_pos.size, dtype=np.uint8)
    return base if base.size else a[:1].copy()


def dna_scheme(alpha=None, match=1, mismatch=-3, go=5, ge=2):
    alpha = alpha or Alphabet.dna(wildcard=False)
    return ScoringScheme.match_mismatch(alpha, match, mismatch, go, ge)
