"""The operator-level drop-in (paper_1304_5966_b200.operator) against the
reference package installed in baseline/_ref (pip install of /root/reference/pkg,
git-ignored, shipped to the GPU box).

CPU: the border family of every reference border builder (engine.py:340-401)
is recognised.  GPU: the reference's own pipeline.align / score_only run with
WavefrontEngine.run_wavefront and phase3.leaf_solve bound to the device
operators and reproduce the golden records."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def wavealign():
    if not (REF / "wavealign").is_dir():
        pytest.skip("baseline/_ref/wavealign is not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_swb")
    sys.path.insert(0, str(REF))
    try:
        import wavealign as wa
    except ImportError as exc:  # numba missing
        pytest.skip(f"reference not importable: {exc}")
    return wa


def _spec(wa, border, codes1, codes2, sub, go, ge):
    from wavealign.engine import PassSpec, global_borders, local_borders, restricted_borders
    n2 = codes2.size
    if border == "local":
        th, tf, left = local_borders(n2)
    elif border == "restricted":
        th, tf, left = restricted_borders(n2, ge)
    else:
        th, tf, left = global_borders(n2, go, ge, lead=border)
    return PassSpec(codes1=codes1, codes2=codes2, sub=sub, gap_open=go, gap_extend=ge,
                    clamp_zero=border == "local", track=0, top_h=th, top_f=tf, left_border=left)


def test_border_families_recognised(wavealign):
    from paper_1304_5966_b200.operator import infer_border
    sub = np.full((4, 4), -3, dtype=np.int64)
    np.fill_diagonal(sub, 1)
    c1 = np.zeros(10, dtype=np.uint8)
    c2 = np.zeros(7, dtype=np.uint8)
    for border in ("local", "restricted", "free", "continue", "charge"):
        assert infer_border(_spec(wavealign, border, c1, c2, sub, 5, 2)) == border
    bad = _spec(wavealign, "local", c1, c2, sub, 5, 2)
    bad.top_h[3] = 17
    with pytest.raises(ValueError):
        infer_border(bad)


@pytest.mark.gpu
def test_reference_pipeline_over_device_operators(wavealign, golden_small, golden_medium,
                                                  golden_protein):
    from helpers import golden_inputs  # noqa: F401  (conftest path)
    from paper_1304_5966_b200 import operator
    from paper_1304_5966_b200.engine import get_context
    wa = wavealign
    ctx = get_context(0)
    l0 = ctx.launch_count
    operator.bind(wa)
    try:
        for rec in golden_small[::12] + golden_medium + golden_protein[::16]:
            sch = rec["scheme"]
            kind = "nucleotide" if len(sch["symbols"]) <= 5 else "protein"
            alpha = wa.Alphabet(kind, sch["symbols"], sch["wildcard"])
            matrix = np.array(sch["matrix"], dtype=np.int64)
            scheme = wa.ScoringScheme(alpha, matrix, sch["gap_open"], sch["gap_extend"],
                                      int(matrix.max()))
            s1 = wa.Sequence.make("a", rec["seq1"], alpha)
            s2 = wa.Sequence.make("b", rec["seq2"], alpha)
            sc = wa.score_only(s1, s2, scheme)
            assert {"score": sc.score, "end": list(sc.end)} == rec["score_only"]
            for tag, cfg in (("align", wa.AlignConfig()),
                             ("align_leaf", wa.AlignConfig(leaf_limit=rec["leaf_limit_small"])),
                             ("align_split", wa.AlignConfig(split=2))):
                summ, path = wa.align(s1, s2, scheme, cfg)
                got = {"score": summ.score, "start": list(summ.start), "end": list(summ.end),
                       "cigar": wa.path_to_cigar(path)}
                assert got == rec[tag], (tag, rec.get("tag"))
    finally:
        operator.unbind(wa)
    assert ctx.launch_count > l0  # the device carried the passes
