"""Golden command-line runs from the REAL reference's cli.run_cli: FASTA
inputs, argument lists, exit codes and the exact stdout bytes (stat, cigar,
pair; DNA with and without the N wildcard, protein with BLOSUM62, split=2,
unbanded/unpruned, usage and input errors).  Run here:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_cli.py
"""
from __future__ import annotations

import contextlib
import gzip
import io
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import REF, wa  # noqa: E402
from support import DNA, mutate, random_text  # noqa: E402
from wavealign import cli as wa_cli  # noqa: E402

PROTEIN = "ARNDCQEGHILKMFPSTWYV"
ACGT = wa.Alphabet.dna(wildcard=False)


def fasta(name, residues, width=60):
    lines = [f">{name} synthetic"] + [residues[k:k + width] for k in range(0, len(residues), width)]
    return "\n".join(lines) + "\n"


def main():
    rng = np.random.default_rng(4242)
    files = {}
    t = random_text(rng, 900, ACGT)
    q = mutate(t, 0.12, rng, ACGT)
    files["t.fa"] = fasta("target", t)
    files["q.fa"] = fasta("query", q)
    tn = list(random_text(rng, 700, ACGT))
    for k in rng.integers(0, 690, 12):
        tn[k] = "N"
    tn[300:310] = ["N"] * 10
    tn = "".join(tn)
    files["tn.fa"] = fasta("targetN", tn)
    files["qn.fa"] = fasta("queryN", mutate(tn.replace("N", "A"), 0.1, rng, ACGT))
    pt = "".join(rng.choice(list(PROTEIN), 400))
    pq = list(pt)
    for k in rng.integers(0, 400, 60):
        pq[k] = PROTEIN[int(rng.integers(0, 20))]
    files["pt.fa"] = fasta("prot_t", pt)
    files["pq.fa"] = fasta("prot_q", "".join(pq[20:380]))
    files["empty.fa"] = ""
    files["bad.fa"] = ">x\nACGTXQ\n"
    files["BLOSUM62"] = (REF / "tests" / "data" / "BLOSUM62").read_text()
    runs = []
    for fmt in ("stat", "cigar", "pair"):
        runs.append(["t.fa", "q.fa", "--out", fmt])
        runs.append(["tn.fa", "qn.fa", "--out", fmt])
        runs.append(["pt.fa", "pq.fa", "--matrix", "BLOSUM62", "--out", fmt])
    runs += [
        ["t.fa", "q.fa", "--split", "2", "--out", "cigar"],
        ["tn.fa", "qn.fa", "--split", "2", "--out", "pair"],
        ["t.fa", "q.fa", "--no-band", "--no-prune", "--leaf-limit", "100", "--out", "cigar"],
        ["t.fa", "q.fa", "--match", "2", "--mismatch", "-1", "--gap-open", "3", "--gap-extend", "1",
         "--out", "cigar"],
        ["pt.fa", "pq.fa", "--matrix", "BLOSUM62", "--gap-open", "11", "--gap-extend", "1",
         "--out", "cigar"],
        ["q.fa", "t.fa", "--workers", "3", "--block-rows", "64", "--block-cols", "100"],
        # errors (no alignment runs)
        ["tn.fa", "qn.fa", "--strict"],
        ["t.fa", "q.fa", "--matrix", "BLOSUM62", "--match", "2"],
        ["t.fa", "q.fa", "--workers", "0"],
        ["t.fa", "missing.fa"],
        ["empty.fa", "q.fa"],
        ["bad.fa", "q.fa"],
        ["t.fa", "q.fa", "--split", "3"],
    ]
    out = {"files": files, "runs": []}
    with tempfile.TemporaryDirectory() as d:
        for name, text in files.items():
            (Path(d) / name).write_text(text)
        for args in runs:
            argv = [str(Path(d) / a) if a in files or a.endswith(".fa") else a for a in args]
            so, se = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
                rc = wa_cli.run_cli(argv)
            out["runs"].append({"args": args, "rc": rc, "stdout": so.getvalue()})
            print(args, rc, len(so.getvalue()))
    with gzip.open(HERE / "golden_cli.json.gz", "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
