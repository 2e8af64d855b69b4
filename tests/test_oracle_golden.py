"""Pin the CPU oracle to the real reference: every golden vector produced by
tests/golden/make_golden.py (wavealign run unchanged) must be reproduced by
oracle/ exactly — score, start, end and CIGAR for score_only, align at two
leaf limits, split=2 align, and oracle_local's (score, end)."""
import numpy as np
import pytest

import oracle
from helpers import golden_inputs, oracle_scheme
from paper_1304_5966_b200 import AlignmentPath, Coord, path_to_cigar


def _cigar(ops):
    return path_to_cigar(AlignmentPath(Coord(0, 0), ops))


def _check(rec, threads=1):
    s1, s2, scheme = golden_inputs(rec)
    osch = oracle_scheme(scheme)
    score, end, _ = oracle.score_only(s1.codes, s2.codes, osch, threads=threads)
    assert (score, list(end)) == (rec["score_only"]["score"], rec["score_only"]["end"])
    for tag, kw in (("align", {}), ("align_leaf", {"leaf_limit": rec["leaf_limit_small"]}),
                    ("align_split", {"split": 2})):
        sc, st, en, ops = oracle.align(s1.codes, s2.codes, osch, threads=threads, **kw)
        want = rec[tag]
        got = {"score": sc, "start": list(st), "end": list(en), "cigar": _cigar(ops)}
        assert got == want, (tag, got, want)
    if "oracle_local" in rec:
        sc, en = oracle.full_local_end(s1.codes, s2.codes, osch)
        assert (sc, list(en)) == (rec["oracle_local"]["score"], rec["oracle_local"]["end"])


def test_oracle_small_golden(golden_small):
    for rec in golden_small:
        _check(rec)


def test_oracle_protein_golden(golden_protein):
    # BLOSUM62, 24 symbols (tests/golden/make_golden_protein.py)
    for rec in golden_protein[:60]:
        _check(rec)


def test_oracle_medium_golden(golden_medium):
    for rec in golden_medium:
        _check(rec, threads=4)


def test_oracle_thread_invariance(golden_medium):
    rec = golden_medium[1]
    s1, s2, scheme = golden_inputs(rec)
    osch = oracle_scheme(scheme)
    a = oracle.align(s1.codes, s2.codes, osch, threads=1)
    b = oracle.align(s1.codes, s2.codes, osch, threads=4)
    assert a[:3] == b[:3] and np.array_equal(a[3], b[3])


def test_oracle_known_answers():
    # test_phase1.py:27-40 / test_oracle.py:26-50 known answers
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    acgt = np.array([0, 1, 2, 3], dtype=np.uint8)
    assert oracle.score_only(acgt, acgt, osch)[:2] == (4, (4, 4))
    g = np.array([2, 2, 2], dtype=np.uint8)
    c = np.array([1, 1, 1], dtype=np.uint8)
    assert oracle.score_only(g, c, osch)[:2] == (0, (0, 0))
    # endpoint tie-break lexicographic min: ATATATAT vs AT -> end (2, 2)
    at8 = np.array([0, 3] * 4, dtype=np.uint8)
    at = np.array([0, 3], dtype=np.uint8)
    assert oracle.full_local_end(at8, at, osch) == (2, (2, 2))
    assert oracle.score_only(at8, at, osch)[:2] == (2, (2, 2))


def test_oracle_prune_invariance(rng):
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    from helpers import mutate_codes, random_codes
    a = random_codes(rng, 3000)
    b = mutate_codes(rng, a, 0.1)
    p = oracle.score_only(a, b, osch, prune=True, block=(128, 128))
    q = oracle.score_only(a, b, osch, prune=False, block=(128, 128))
    assert p[:2] == q[:2]
    assert p[2].pruned > 0


def test_scale_goldens_self_consistent():
    """The BASELINE-scale reference records (tests/golden/make_golden_scale.py)
    are consistent with their own inputs: the CIGAR re-scores to the score and
    spans start..end (model.score_of_path, reference model.py:279-318)."""
    import gzip
    import json
    from pathlib import Path

    from bench import synthetic_pair
    from paper_1304_5966_b200 import Alphabet, ScoringScheme, Sequence, score_of_path
    from paper_1304_5966_b200.model import AlignmentPath, Coord, cigar_to_ops

    recs = json.load(gzip.open(Path(__file__).resolve().parent / "golden" / "golden_scale.json.gz", "rt"))
    assert {r["name"] for r in recs} >= {"C2", "C3w", "C5w", "C3w_split", "C4w"}
    scheme = ScoringScheme.match_mismatch(Alphabet.dna(), 1, -3, 5, 2)
    for r in recs:
        if "cigar" not in r:
            continue
        a, b = synthetic_pair(r["n"], seed=r["seed"], homologous=r["homologous"])
        if r["window"]:
            a, b = a[:r["window"][0]], b[:r["window"][1]]
        s1 = Sequence.from_codes("t", a, scheme.alphabet)
        s2 = Sequence.from_codes("q", b, scheme.alphabet)
        path = AlignmentPath(Coord(*r["start"]), cigar_to_ops(r["cigar"]))
        assert tuple(path.end) == tuple(r["end"]), r["name"]
        assert score_of_path(path, s1, s2, scheme) == r["score"], r["name"]
