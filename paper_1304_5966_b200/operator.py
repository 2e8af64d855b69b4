"""Operator-level drop-in for the reference's wavefront engine and leaf kernel.

The reference's phases submit every DP pass to
``WavefrontEngine.run_wavefront(PassSpec) -> PassResult`` (engine.py:188-282)
and every Myers-Miller leaf to ``kernels.leaf_solve`` (kernels.py:91-185).
This module serves those two calls, with the reference's own argument and
result types, from the B200 kernels behind libswb.so:

* ``run_wavefront(spec)`` takes a reference ``PassSpec`` unchanged.  Its border
  arrays and ``left_border`` callable are recognised as one of the reference's
  border families (engine.py:340-401: local, restricted, global free /
  continue / charge) and become the C ABI's border enum; ``prune`` (the
  phase-1 hook, phase1.py:55-59) becomes the device's running-best pruning;
  ``band`` is passed as is.  As the reference engine does, the final DP row is
  written INTO ``spec.top_h`` / ``spec.top_f`` and returned as
  ``final_row_h`` / ``final_row_f`` (engine.py:97-99, :264-276).
* ``leaf_solve(...)`` has kernels.leaf_solve's signature and writes the ops to
  the front of ``ops_out``.
* ``bind(wavealign)`` installs both into an imported reference package (the
  swap INTEGRATION.md shows), ``unbind`` restores it.

A PassSpec whose borders are not one of the families raises ValueError:
there is no CPU fallback.
"""
from __future__ import annotations

import numpy as np

from .engine import TRACK_MIN, Session, get_context
from .model import Alphabet, ScoringScheme

NEG_INF = -(2 ** 61)
_SYMBOLS = "ABCDEFGHIJKLMNOPQRSTUVWXYZ012345"


def _scheme(sub: np.ndarray, go: int, ge: int) -> ScoringScheme:
    sub = np.asarray(sub, dtype=np.int64)
    k = int(sub.shape[0])
    if k > len(_SYMBOLS):
        raise ValueError(f"alphabets of {k} symbols are not supported on the device (max 32)")
    return ScoringScheme(Alphabet("custom", _SYMBOLS[:k]), sub, int(go), int(ge), int(sub.max()))


def infer_border(spec) -> str:
    """The reference border family that produced spec.top_h / top_f /
    left_border (engine.py:340-401)."""
    th = np.asarray(spec.top_h)
    tf = np.asarray(spec.top_f)
    go, ge = int(spec.gap_open), int(spec.gap_extend)
    cols = th.size - 1
    if not (tf == NEG_INF).all():
        raise ValueError("top F border is not minus infinity: not a reference border family")
    if (th == 0).all():
        return "local"
    if th[0] == 0 and (th[1:] == NEG_INF).all():
        return "restricted"
    ramp = -go - np.arange(cols + 1, dtype=np.int64) * ge
    ramp[0] = 0
    if np.array_equal(th, ramp):
        return "free"
    if (th == NEG_INF).all():
        _, _, f = spec.left_border(0, 1)
        if int(f[0]) == 0:
            return "continue"
        if int(f[0]) == -go:
            return "charge"
    raise ValueError("PassSpec borders are not one of the reference's border families")


def run_wavefront(spec, device: int = 0):
    """WavefrontEngine.run_wavefront(spec) on the device (engine.py:188-282);
    returns the reference's PassResult type when wavealign is importable."""
    border = infer_border(spec)
    c1 = np.ascontiguousarray(spec.codes1, dtype=np.uint8)
    c2 = np.ascontiguousarray(spec.codes2, dtype=np.uint8)
    if c1.size < 1 or c2.size < 1:
        raise ValueError("cannot tile an empty matrix")
    if spec.top_h.shape != (c2.size + 1,) or spec.top_f.shape != (c2.size + 1,):
        raise ValueError("top border arrays must have length cols+1")
    scheme = _scheme(spec.sub, spec.gap_open, spec.gap_extend)
    clamp = bool(spec.clamp_zero)
    if clamp and border != "local":
        raise ValueError("clamped passes use local borders")
    prune = spec.prune is not None and clamp and int(spec.track) == TRACK_MIN
    with Session(get_context(device), c1, c2, scheme) as S:
        r = S.run([dict(rows=(0, c1.size, 0), cols=(0, c2.size, 0), border=border, clamp=clamp,
                        track=int(spec.track), band=spec.band, prune=prune, want_final=True)])[0]
    # the engine owns top_h / top_f and returns them overwritten (engine.py:97-99)
    spec.top_h[:] = r.final_row_h
    spec.top_f[:] = r.final_row_f
    fields = dict(best_score=int(r.best_score), best_i=int(r.best_i), best_j=int(r.best_j),
                  final_row_h=spec.top_h, final_row_f=spec.top_f,
                  total_blocks=int(r.total_blocks), executed_blocks=int(r.executed_blocks),
                  pruned_blocks=int(r.pruned_blocks), banded_out_blocks=int(r.banded_out_blocks),
                  cells_executed=int(r.cells_executed))
    cls = getattr(type(spec), "_swb_result_type", None)
    if cls is None:
        import sys
        eng = sys.modules.get(type(spec).__module__)
        cls = getattr(eng, "PassResult", None)
    if cls is None:
        from types import SimpleNamespace
        return SimpleNamespace(**fields)
    return cls(**fields)


def leaf_solve(c1, c2, sub, go, ge, start_vgap, end_vgap, lo, hi, ops_out, device: int = 0):
    """kernels.leaf_solve (kernels.py:91-185) on the device: banded affine
    global alignment with traceback; ops in forward order at the front of
    ops_out; returns (score, count), (NEG_INF, -1) on a dead end."""
    from .engine import SUBPROBLEM_DTYPE
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    n, m = int(c1.size), int(c2.size)
    if n < 1 or m < 1:
        raise ValueError("leaf_solve needs a non-empty rectangle")
    scheme = _scheme(sub, go, ge)
    with Session(get_context(device), c1, c2, scheme) as S:
        leaf = np.zeros(1, dtype=SUBPROBLEM_DTYPE)
        leaf[0] = (0, 0, n, m, 0, int(bool(start_vgap)), int(bool(end_vgap)), 0, 0, int(lo), int(hi))
        ops, offsets, counts, scores = S.ctx.leaves(S.cs, S.s1, S.s2, leaf, 2)
    count = int(counts[0])
    if count < 0:
        return NEG_INF, -1
    ops_out[:count] = ops[int(offsets[0]):int(offsets[0]) + count]
    return int(scores[0]), count


_saved: dict = {}


def bind(wavealign, device: int = 0) -> None:
    """Install the device operators into an imported reference package: every
    WavefrontEngine.run_wavefront and every phase-3 leaf_solve call of its
    phases then runs on the B200."""
    eng = wavealign.engine
    ph3 = wavealign.phase3
    if not _saved:
        _saved["run_wavefront"] = eng.WavefrontEngine.run_wavefront
        _saved["leaf_solve"] = ph3.leaf_solve
    eng.WavefrontEngine.run_wavefront = lambda self, spec: run_wavefront(spec, device)
    ph3.leaf_solve = lambda *a: leaf_solve(*a, device=device)


def unbind(wavealign) -> None:
    if _saved:
        wavealign.engine.WavefrontEngine.run_wavefront = _saved.pop("run_wavefront")
        wavealign.phase3.leaf_solve = _saved.pop("leaf_solve")
