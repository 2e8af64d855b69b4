"""Golden vectors for the io module, from the REAL reference's io.py:
parse_fasta on odd inputs, parse_matrix on BLOSUM62, write_fasta, and
write_output in all three formats for golden alignments.  Run here:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_io.py
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import REF, wa  # noqa: E402
from support import DNA, mutate, random_text  # noqa: E402
from wavealign import io as wa_io  # noqa: E402

FASTAS = [
    b">seq1 first record\nACGT\nacgt\n\n>seq2\n  AC GT\tTT \n>empty_after\n\n>x y z\nNNACG\n",
    b">only\r\nACGTACGTAC\r\nGTT\r\n",
    b"\n\n>a\nA\n>b\nC\n>c\nG\n",
]


def main():
    out = {"fasta": [], "matrix": None, "outputs": []}
    for data in FASTAS:
        recs = wa_io.parse_fasta(data, wa.Alphabet.dna(wildcard=True))
        out["fasta"].append({"data": data.decode(), "records": [[r.id, r.residues] for r in recs],
                             "written": [wa_io.write_fasta(r, 7).decode() for r in recs]})
    mtext = (REF / "tests" / "data" / "BLOSUM62").read_bytes()
    symbols, table = wa_io.parse_matrix(mtext)
    out["matrix"] = {"symbols": symbols, "table": [[a, b, v] for (a, b), v in table.items()]}
    rng = np.random.default_rng(77)
    scheme = wa.ScoringScheme.match_mismatch(DNA, 1, -3, 5, 2)
    for t in range(24):
        a = random_text(rng, int(rng.integers(1, 400)), DNA)
        b = mutate(a, float(rng.choice([0.05, 0.2, 0.5])), rng, DNA) if t % 4 else random_text(rng, 50, DNA)
        if not b:
            b = "A"
        s1 = wa.Sequence.make("target_" + str(t), a, DNA)
        s2 = wa.Sequence.make("query_" + str(t), b, DNA)
        summ, path = wa.align(s1, s2, scheme)
        rec = {"seq1": a, "seq2": b, "id1": s1.id, "id2": s2.id,
               "score": summ.score, "start": list(summ.start), "end": list(summ.end),
               "path_cigar": wa.path_to_cigar(path)}
        for fmt in ("stat", "cigar", "pair"):
            rec[fmt] = wa_io.write_output(summ, path, fmt, s1, s2).decode()
        out["outputs"].append(rec)
    with gzip.open(HERE / "golden_io.json.gz", "wt") as fh:
        json.dump(out, fh)
    print("wrote io goldens:", len(out["fasta"]), "fasta,", len(out["outputs"]), "outputs")


if __name__ == "__main__":
    main()
