"""Boundary types (model.py): same semantics as the reference model
(reference pkg/src/wavealign/model.py; tests modelled on test_model.py)."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from helpers import oracle_scheme
from paper_1304_5966_b200 import (
    AlignmentPath, AlignmentSummary, Alphabet, Coord, IllegalResidue, IncompleteMatrix,
    NonPositiveMaxScore, PathInconsistent, ScoringScheme, Sequence, cigar_to_ops, path_to_cigar,
    score_of_path, validate_scheme)
from paper_1304_5966_b200.errors import BUG_ERRORS, ScoreMismatch, StartNotFound

DNA = Alphabet.dna(wildcard=False)


def seq(t, a=DNA):
    return Sequence.make("s", t, a)


def test_alphabet_and_encoding():
    assert "N" in Alphabet.dna() and "N" not in DNA
    assert seq("acgt").codes.tolist() == [0, 1, 2, 3]
    with pytest.raises(IllegalResidue) as e:
        seq("AC*T")
    assert e.value.position == 2
    with pytest.raises(ValueError):
        Alphabet("nucleotide", "ACGA")


def test_scheme_validation():
    s = ScoringScheme.match_mismatch(DNA, 2, -1, 5, 2)
    assert validate_scheme(s).max_substitution_score == 2
    with pytest.raises(NonPositiveMaxScore):
        validate_scheme(ScoringScheme.match_mismatch(DNA, 0, 0, 5, 2))
    with pytest.raises(IncompleteMatrix):
        validate_scheme(ScoringScheme.from_table(DNA, {("A", "A"): 1}, 5, 2))
    stale = ScoringScheme(DNA, s.matrix, 5, 2, 1)
    assert validate_scheme(stale).max_substitution_score == 2
    w = ScoringScheme.match_mismatch(Alphabet.dna(), 2, -1, 5, 2)
    assert w.substitution("N", "A") == 0 and w.substitution("A", "A") == 2
    with pytest.raises(ValueError):
        ScoringScheme(DNA, s.matrix, -1, 2, 2)


def test_summary_invariants():
    AlignmentSummary(3, Coord(0, 0), Coord(2, 2))
    with pytest.raises(ValueError):
        AlignmentSummary(0, Coord(0, 0), Coord(1, 1))
    with pytest.raises(ValueError):
        AlignmentSummary(2, Coord(3, 0), Coord(1, 1))


def test_score_of_path_matches_oracle_rescore():
    rng = np.random.default_rng(4)
    s = ScoringScheme.match_mismatch(DNA, 2, -3, 4, 1)
    a = seq("ACGTTGCAACGT")
    b = seq("ACGTGCAACCGT")
    ops = cigar_to_ops("4=1D4=1I3=")
    p = AlignmentPath(Coord(0, 0), ops)
    assert score_of_path(p, a, b, s) == opl_rescore(p, a, b, s)
    with pytest.raises(PathInconsistent):
        score_of_path(AlignmentPath(Coord(0, 0), cigar_to_ops("2X")), a, b, s)
    with pytest.raises(PathInconsistent):
        score_of_path(AlignmentPath(Coord(10, 0), cigar_to_ops("5=")), a, b, s)


def opl_rescore(p, a, b, s):
    from oracle.pipeline import rescore
    return rescore(tuple(p.start), p.ops, a.codes, b.codes, oracle_scheme(s))


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(0, 3), max_size=60))
def test_cigar_round_trip(ops):
    arr = np.array(ops, dtype=np.uint8)
    p = AlignmentPath(Coord(0, 0), arr)
    assert np.array_equal(cigar_to_ops(path_to_cigar(p)), arr)


def test_path_end_and_errors():
    p = AlignmentPath(Coord(1, 2), cigar_to_ops("3=2I1D"))
    assert p.end == Coord(5, 7)
    assert AlignmentPath.empty().end == Coord(0, 0)
    with pytest.raises(ValueError):
        cigar_to_ops("3Q")
    assert set(BUG_ERRORS) == {ScoreMismatch, StartNotFound}


def test_plan_grid_matches_reference_tiling():
    from paper_1304_5966_b200 import plan_grid
    g = plan_grid(1000, 700, 512, 512)
    assert (g.grid_rows, g.grid_cols, g.anti_diagonals) == (2, 2, 3)
    assert g.row_span(1) == (512, 1000) and g.col_span(1) == (512, 700)
    assert plan_grid(10, 10, 512, 512).block_rows == 10
    import pytest
    with pytest.raises(ValueError):
        plan_grid(0, 5)
