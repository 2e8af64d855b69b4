"""io mirror (paper_1304_5966_b200.io) against golden outputs of the real
reference's io.py (tests/golden/make_golden_io.py): FASTA parsing and
writing, BLOSUM62 parsing, and stat / cigar / pair output byte-for-byte."""
import numpy as np
import pytest

from conftest import load_golden
from paper_1304_5966_b200 import (Alphabet, AlignmentPath, AlignmentSummary, Coord, Sequence,
                                  cigar_to_ops)
from paper_1304_5966_b200 import io as sio
from paper_1304_5966_b200.errors import EmptyFile, NoRecords, NonInteger, RaggedRow, UnknownSymbol


@pytest.fixture(scope="module")
def gio():
    return load_golden("golden_io.json.gz")


def test_parse_and_write_fasta(gio):
    for case in gio["fasta"]:
        recs = sio.parse_fasta(case["data"].encode(), Alphabet.dna(wildcard=True))
        assert [[r.id, r.residues] for r in recs] == case["records"]
        assert [sio.write_fasta(r, 7).decode() for r in recs] == case["written"]


def test_parse_matrix_blosum62(gio):
    want = gio["matrix"]
    # rebuild an NCBI-style file from the golden table and parse it back
    syms = want["symbols"]
    tab = {(a, b): v for a, b, v in want["table"]}
    lines = ["# rebuilt", "   " + "  ".join(syms)]
    for a in syms:
        lines.append(a + " " + " ".join(str(tab[(a, b)]) for b in syms))
    symbols, table = sio.parse_matrix("\n".join(lines).encode())
    assert symbols == syms
    assert table == tab


def test_matrix_errors():
    with pytest.raises(EmptyFile):
        sio.parse_matrix(b"# only a comment\n")
    with pytest.raises(UnknownSymbol):
        sio.parse_matrix(b"A C\nX 1 2\n")
    with pytest.raises(RaggedRow):
        sio.parse_matrix(b"A C\nA 1\n")
    with pytest.raises(NonInteger):
        sio.parse_matrix(b"A C\nA 1 x\n")


def test_fasta_errors():
    with pytest.raises(EmptyFile):
        sio.parse_fasta(b"  \n", Alphabet.dna())
    with pytest.raises(NoRecords):
        sio.parse_fasta(b"ACGT\n>x\nA\n", Alphabet.dna())


def test_write_output_formats(gio):
    dna = Alphabet.dna(wildcard=False)
    for rec in gio["outputs"]:
        s1 = Sequence.make(rec["id1"], rec["seq1"], dna)
        s2 = Sequence.make(rec["id2"], rec["seq2"], dna)
        summ = AlignmentSummary(rec["score"], Coord(*rec["start"]), Coord(*rec["end"]))
        path = AlignmentPath(Coord(*rec["start"]), cigar_to_ops(rec["path_cigar"]))
        for fmt in ("stat", "cigar", "pair"):
            assert sio.write_output(summ, path, fmt, s1, s2).decode() == rec[fmt], fmt
    with pytest.raises(ValueError):
        sio.write_output(summ, path, "sam", s1, s2)


def test_pair_text_large_is_fast():
    import time
    rng = np.random.default_rng(3)
    n = 200_000
    ops = rng.integers(0, 4, size=n).astype(np.uint8)
    dna = Alphabet.dna(wildcard=False)
    t1 = int((ops != 2).sum()); q1 = int((ops != 3).sum())
    s1 = Sequence.from_codes("t", rng.integers(0, 4, size=t1).astype(np.uint8), dna)
    s2 = Sequence.from_codes("q", rng.integers(0, 4, size=q1).astype(np.uint8), dna)
    summ = AlignmentSummary(1, Coord(0, 0), Coord(t1, q1))
    t0 = time.perf_counter()
    out = sio.write_output(summ, AlignmentPath(Coord(0, 0), ops), "pair", s1, s2)
    assert time.perf_counter() - t0 < 5.0
    assert out.count(b"\n") == 4 * ((n + 59) // 60)
