"""Protein golden vectors (BLOSUM62, 24-symbol alphabet) from the REAL
reference, for the shared-table kernels.  Run in the build
container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_protein.py

The matrix is parsed with the reference's own io.parse_matrix from
pkg/tests/data/BLOSUM62 and stored in every record (scheme.matrix), so the
parity tests do not need the reference at run time."""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import REF, run_case, wa  # noqa: E402
from support import PROTEIN, mutate, random_text  # noqa: E402
from wavealign import io as wa_io  # noqa: E402


def blosum62():
    symbols, table = wa_io.parse_matrix((REF / "tests" / "data" / "BLOSUM62").read_bytes())
    return wa.Alphabet.from_symbols("protein", symbols), table


def main():
    alphabet, table = blosum62()
    rng = np.random.default_rng(62)
    out = []
    gaps = [(10, 1), (11, 1), (5, 2), (0, 4)]
    for t in range(160):
        go, ge = gaps[t % len(gaps)]
        scheme = wa.ScoringScheme.from_table(alphabet, table, go, ge)
        n = int(rng.integers(1, 260 if t % 5 else 1200))
        a = random_text(rng, n, PROTEIN)
        kind = t % 3
        if kind == 0:
            b = mutate(a, float(rng.choice([0.1, 0.3, 0.5])), rng, PROTEIN)
        elif kind == 1:
            b = random_text(rng, int(rng.integers(1, 300)), PROTEIN)
        else:
            b = random_text(rng, int(rng.integers(0, 40)), PROTEIN) + mutate(a, 0.2, rng, PROTEIN) + \
                random_text(rng, int(rng.integers(0, 40)), PROTEIN)
        if not b:
            b = "A"
        rec = run_case(a, b, scheme, alphabet, int(rng.choice([16, 64, 256])), oracle=n < 300)
        rec["kind"] = kind
        rec["tag"] = "protein_blosum62"
        out.append(rec)
    with gzip.open(HERE / "golden_protein.json.gz", "wt") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} protein cases")


if __name__ == "__main__":
    main()
