"""Parity of the CUDA path (through libswb.so) with the reference.

Small/medium cases compare against golden vectors recorded from the real
reference; larger seeded cases compare against the pinned CPU oracle; the
full-size properties (prune/split invariance, re-scoring) run in
test_gpu_scale.py.  Bar: bit-exact score, start, end and CIGAR.
"""
import numpy as np
import pytest

import oracle
from helpers import dna_scheme, golden_inputs, mutate_codes, oracle_scheme, random_codes
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200 import AlignConfig, Alphabet, Sequence, path_to_cigar

pytestmark = pytest.mark.gpu


def _summ(summary, path):
    return {"score": summary.score, "start": list(summary.start), "end": list(summary.end),
            "cigar": path_to_cigar(path)}


def _check_rec(rec):
    s1, s2, scheme = golden_inputs(rec)
    sc = swb.score_only(s1, s2, scheme)
    assert {"score": sc.score, "end": list(sc.end)} == rec["score_only"]
    for tag, cfg in (("align", AlignConfig()),
                     ("align_leaf", AlignConfig(leaf_limit=rec["leaf_limit_small"])),
                     ("align_split", AlignConfig(split=2))):
        got = _summ(*swb.align(s1, s2, scheme, cfg))
        assert got == rec[tag], (tag, rec.get("tag"), got, rec[tag])


def test_golden_small(golden_small):
    for rec in golden_small:
        _check_rec(rec)


def test_golden_medium_and_config1(golden_medium):
    for rec in golden_medium:
        _check_rec(rec)


@pytest.mark.parametrize("world", [2, 4])
def test_golden_split_gpu_groups(golden_medium, golden_protein, world):
    """align_split goldens through the Figure-1 split across GPU groups
    (multigpu.run_split_slabs_concurrent: the multi-GPU schedule emulated in
    one launch; medium inputs leave every group one slab)."""
    from paper_1304_5966_b200.engine import Session, get_context
    from paper_1304_5966_b200.multigpu import run_split_slabs_concurrent
    for rec in golden_medium + golden_protein[::8]:
        s1, s2, scheme = golden_inputs(rec)
        with Session(get_context(0), s1.codes, s2.codes, scheme) as S:
            got = _summ(*run_split_slabs_concurrent(S, world))
        assert got == rec["align_split"], (rec.get("tag"), got, rec["align_split"])


def test_score_only_prune_report(golden_medium):
    rec = [r for r in golden_medium if r["tag"] == "config1"][0]
    s1, s2, scheme = golden_inputs(rec)
    rep_on, rep_off = {}, {}
    a = swb.score_only(s1, s2, scheme, AlignConfig(prune=True), report=rep_on)
    b = swb.score_only(s1, s2, scheme, AlignConfig(prune=False), report=rep_off)
    assert (a.score, a.end) == (b.score, b.end)
    assert rep_off["pruned_blocks"] == 0
    for key in ("score", "total_blocks", "pruned_blocks", "pruned_fraction", "cells_executed"):
        assert key in rep_on


@pytest.mark.parametrize("seed,n,kind", [(1, 20000, "hom"), (2, 33000, "hom"), (3, 25000, "unrel"),
                                         (4, 40000, "hom_indel")])
def test_vs_oracle_seeded(seed, n, kind):
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n)
    if kind == "unrel":
        b = random_codes(rng, int(n * 0.93))
    else:
        b = mutate_codes(rng, a, 0.25 if kind == "hom_indel" else 0.10)
        b = np.concatenate([random_codes(rng, 777), b, random_codes(rng, 333)])
    scheme = dna_scheme()
    alpha = scheme.alphabet
    s1, s2 = Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha)
    osch = oracle_scheme(scheme)
    want = oracle.align(a, b, osch)
    summary, path = swb.align(s1, s2, scheme)
    assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3]
    assert np.array_equal(path.ops, want[3])


@pytest.mark.parametrize("scheme_args", [(2, -1, 0, 1), (5, -5, 10, 5), (1, -1, 3, 1), (3, -2, 0, 4)])
def test_random_schemes_vs_oracle(scheme_args):
    rng = np.random.default_rng(sum(scheme_args) + 100)
    a = random_codes(rng, 5000)
    b = mutate_codes(rng, a, 0.2)
    scheme = dna_scheme(None, *scheme_args)
    s1 = Sequence.from_codes("a", a, scheme.alphabet)
    s2 = Sequence.from_codes("b", b, scheme.alphabet)
    osch = oracle_scheme(scheme)
    for cfg_kw in ({}, {"split": 2}, {"leaf_limit": 300}):
        want = oracle.align(a, b, osch, **cfg_kw)
        summary, path = swb.align(s1, s2, scheme, AlignConfig(**cfg_kw))
        assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3], cfg_kw
        assert np.array_equal(path.ops, want[3]), cfg_kw


def test_edge_shapes():
    scheme = dna_scheme()
    alpha = scheme.alphabet
    osch = oracle_scheme(scheme)
    rng = np.random.default_rng(5)
    shapes = [(1, 1), (1, 500), (500, 1), (2, 3000), (3000, 2), (31, 33), (1024, 1024),
              (1025, 100), (4095, 4097), (2048, 5)]
    for n1, n2 in shapes:
        a = random_codes(rng, n1)
        b = random_codes(rng, n2)
        if n1 == n2:
            b = a.copy()
        want = oracle.align(a, b, osch)
        summary, path = swb.align(Sequence.from_codes("a", a, alpha),
                                  Sequence.from_codes("b", b, alpha), scheme)
        assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3], (n1, n2)
        assert np.array_equal(path.ops, want[3]), (n1, n2)


def test_wildcard_alphabet():
    alpha = Alphabet.dna(wildcard=True)
    scheme = swb.ScoringScheme.match_mismatch(alpha, 2, -3, 4, 1)
    rng = np.random.default_rng(11)
    a = rng.integers(0, 5, size=3000, dtype=np.uint8)
    b = mutate_codes(rng, a, 0.15, k=5)
    osch = oracle_scheme(scheme)
    want = oracle.align(a, b, osch)
    summary, path = swb.align(Sequence.from_codes("a", a, alpha), Sequence.from_codes("b", b, alpha),
                              scheme)
    assert (summary.score, tuple(summary.start), tuple(summary.end)) == want[:3]
    assert np.array_equal(path.ops, want[3])


def test_engine_facade_final_rows():
    """WavefrontEngine.run_wavefront vs the oracle engine, all border modes,
    including final rows (engine.py:264-276)."""
    scheme = dna_scheme()
    osch = oracle_scheme(scheme)
    rng = np.random.default_rng(3)
    a = random_codes(rng, 1500)
    b = mutate_codes(rng, a, 0.1)[:1400]
    eng = swb.WavefrontEngine()
    # unbanded: every cell is computed by both, so final rows are comparable
    band = None
    for border, clamp, track in (("local", True, 1), ("restricted", False, 2), ("free", False, 0),
                                 ("continue", False, 0), ("charge", False, 1), ("free", False, 2)):
        spec = swb.PassSpec(a, b, scheme, border=border, clamp_zero=clamp, track=track, band=band)
        got = eng.run_wavefront(spec)
        want = oracle.run_wavefront(a, b, osch, border, clamp, track, band=band)
        assert (got.best_score, got.best_i, got.best_j) == (want.best, want.bi, want.bj), border
        fin = want.final_h > -(2 ** 40)
        assert np.array_equal(got.final_row_h[fin], want.final_h[fin]), border
        assert np.array_equal(got.final_row_h > -(2 ** 40), fin), border
        fin_f = want.final_f > -(2 ** 40)
        assert np.array_equal(got.final_row_f[fin_f], want.final_f[fin_f]), border


def test_golden_protein_blosum62(golden_protein):
    """24-symbol BLOSUM62 scheme: the shared-table kernels
    reproduce the reference's score, start, end and CIGAR."""
    for rec in golden_protein:
        _check_rec(rec)


@pytest.mark.parametrize("seed,n", [(1, 3000), (2, 12_000)])
def test_protein_vs_oracle(seed, n, golden_protein):
    s1g, _, scheme = golden_inputs(golden_protein[0])
    k = len(scheme.alphabet)
    rng = np.random.default_rng(seed)
    a = random_codes(rng, n, 20)
    b = mutate_codes(rng, a, 0.3, 20)
    osch = oracle_scheme(scheme)
    want = oracle.align(a, b, osch)
    s1 = Sequence.from_codes("a", a, scheme.alphabet)
    s2 = Sequence.from_codes("b", b, scheme.alphabet)
    summ, path = swb.align(s1, s2, scheme)
    assert (summ.score, tuple(summ.start), tuple(summ.end)) == (want[0], tuple(want[1]),
                                                              tuple(want[2]))
    assert np.array_equal(path.ops, want[3])
    assert k == 24


def test_allocation_meter_linear():
    """engine.AllocationMeter parity (test_engine.py:132-146): the device state
    a pass reports grows linearly with the sequence lengths."""
    from paper_1304_5966_b200 import AllocationMeter
    rng = np.random.default_rng(5)
    sc = dna_scheme()
    peaks = {}
    for n in (2000, 8000, 32000):
        c = random_codes(rng, n)
        meter = AllocationMeter()
        s = Sequence.from_codes("a", c, sc.alphabet)
        swb.align(s, s, sc, AlignConfig(meter=meter))
        peaks[n] = meter.peak
        assert meter.current == 0
    ratios = [peaks[n] / (2 * n) for n in peaks]
    assert max(ratios) / min(ratios) < 1.1
    assert max(ratios) < 16
