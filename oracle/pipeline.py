"""CPU restatement of the wavealign phases on top of the C oracle kernels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function cites the
reference code it restates; the arithmetic lives in swb_oracle.c.

Sequences are uint8 code arrays; a scheme is OracleScheme(sub (K x K int64),
gap_open, gap_extend).  Results are plain tuples:
  score_only -> (score, (end_i, end_j))
  align      -> (score, (start_i, start_j), (end_i, end_j), ops uint8)
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

NEG_INF = -(2 ** 61)  # kernels.py:14
_HERE = Path(__file__).resolve().parent
_LIB = None

BORDER = {"local": 0, "restricted": 1, "free": 2, "continue": 3, "charge": 4}
TRACK_NONE, TRACK_MIN, TRACK_MAX = 0, 1, 2  # kernels.py:16-18


class _Pass(ctypes.Structure):
    _fields_ = [
        ("c1", ctypes.c_void_p), ("n1", ctypes.c_int64),
        ("c2", ctypes.c_void_p), ("n2", ctypes.c_int64),
        ("sub", ctypes.c_void_p), ("k", ctypes.c_int32), ("border", ctypes.c_int32),
        ("go", ctypes.c_int64), ("ge", ctypes.c_int64),
        ("clamp0", ctypes.c_int32), ("track", ctypes.c_int32),
        ("has_band", ctypes.c_int32), ("band_lo", ctypes.c_int64), ("band_hi", ctypes.c_int64),
        ("prune", ctypes.c_int32), ("max_sub", ctypes.c_int64), ("fill_h", ctypes.c_int64),
        ("block_rows", ctypes.c_int64), ("block_cols", ctypes.c_int64),
        ("threads", ctypes.c_int32),
        ("top_h", ctypes.c_void_p), ("top_f", ctypes.c_void_p),
        ("row_offset", ctypes.c_int64),
    ]


class _Result(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("best", "bi", "bj", "total_blocks", "executed", "pruned", "banded", "cells")]


def _lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "libswb_oracle.so"
        if not so.exists():
            subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
        lib = ctypes.CDLL(str(so))
        lib.orc_run_wavefront.argtypes = [ctypes.POINTER(_Pass), ctypes.POINTER(_Result)]
        lib.orc_run_wavefront.restype = ctypes.c_int
        lib.orc_top_border.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.orc_local_end.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64)]
        lib.orc_local_end.restype = ctypes.c_int64
        lib.orc_leaf_solve.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64)]
        lib.orc_leaf_solve.restype = ctypes.c_int64
        lib.orc_fill_full.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]
        lib.orc_max_threads.restype = ctypes.c_int
        _LIB = lib
    return _LIB


@dataclass(frozen=True)
class OracleScheme:
    sub: np.ndarray  # (K, K) int64
    gap_open: int
    gap_extend: int

    @property
    def max_sub(self) -> int:
        return int(self.sub.max())

    @classmethod
    def match_mismatch(cls, k, match, mismatch, go, ge):
        m = np.full((k, k), mismatch, dtype=np.int64)
        np.fill_diagonal(m, match)
        return cls(m, int(go), int(ge))


def max_threads() -> int:
    return int(_lib().orc_max_threads())


def _c(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# -- engine --------------------------------------------------------------------

@dataclass
class PassOut:
    best: int
    bi: int
    bj: int
    final_h: np.ndarray
    final_f: np.ndarray
    total_blocks: int
    executed: int
    pruned: int
    banded: int
    cells: int


def run_wavefront(c1, c2, scheme: OracleScheme, border: str, clamp0: bool, track: int,
                  band=None, prune=False, fill_h=None, block=(512, 512), threads=None,
                  top=None, row_offset=0) -> PassOut:
    """engine.WavefrontEngine.run_wavefront (engine.py:188-282) with the border
    family of engine.py:340-401 and, when prune, the phase-1 hook
    (phase1.py:55-59).  `top` = (top_h, top_f) replaces the family's top
    border and `row_offset` shifts the left border (a row slab of a larger
    pass whose rows above produced `top`)."""
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    sub = np.ascontiguousarray(scheme.sub, dtype=np.int64)
    n2 = int(c2.size)
    top_h = np.empty(n2 + 1, dtype=np.int64)
    top_f = np.empty(n2 + 1, dtype=np.int64)
    lib = _lib()
    if top is None:
        lib.orc_top_border(BORDER[border], n2, scheme.gap_open, scheme.gap_extend, _c(top_h),
                           _c(top_f))
    else:
        top_h[:] = top[0]
        top_f[:] = top[1]
    p = _Pass()
    p.c1, p.n1, p.c2, p.n2 = _c(c1), c1.size, _c(c2), n2
    p.sub, p.k, p.border = _c(sub), sub.shape[0], BORDER[border]
    p.go, p.ge = scheme.gap_open, scheme.gap_extend
    p.clamp0, p.track = int(clamp0), int(track)
    if band is not None:
        p.has_band, p.band_lo, p.band_hi = 1, int(band[0]), int(band[1])
    p.prune, p.max_sub = int(prune), scheme.max_sub
    p.fill_h = (0 if clamp0 else NEG_INF) if fill_h is None else int(fill_h)
    p.block_rows, p.block_cols = block
    p.threads = int(threads or max_threads())
    p.top_h, p.top_f = _c(top_h), _c(top_f)
    p.row_offset = int(row_offset)
    r = _Result()
    rc = lib.orc_run_wavefront(ctypes.byref(p), ctypes.byref(r))
    if rc != 0:
        raise ValueError("cannot tile an empty matrix")
    return PassOut(r.best, r.bi, r.bj, top_h, top_f, r.total_blocks, r.executed, r.pruned,
                   r.banded, r.cells)


def full_local_end(c1, c2, scheme: OracleScheme):
    """oracle_local's score and end (oracle.py:146-164), linear memory."""
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    sub = np.ascontiguousarray(scheme.sub, dtype=np.int64)
    ei, ej = ctypes.c_int64(), ctypes.c_int64()
    s = _lib().orc_local_end(_c(c1), c1.size, _c(c2), c2.size, _c(sub), sub.shape[0],
                             scheme.gap_open, scheme.gap_extend, ctypes.byref(ei), ctypes.byref(ej))
    if s <= 0:
        return 0, (0, 0)
    return int(s), (int(ei.value), int(ej.value))


def full_matrices(c1, c2, scheme: OracleScheme, mode="affine", start_vgap=False):
    """oracle._matrices + _fill (oracle.py:38-109)."""
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    sub = np.ascontiguousarray(scheme.sub, dtype=np.int64)
    shape = (c1.size + 1, c2.size + 1)
    H, E, F = (np.empty(shape, dtype=np.int64) for _ in range(3))
    _lib().orc_fill_full(_c(c1), c1.size, _c(c2), c2.size, _c(sub), sub.shape[0],
                         scheme.gap_open, scheme.gap_extend,
                         {"local": 0, "affine": 1, "pinned": 2}[mode], int(start_vgap),
                         _c(H), _c(E), _c(F))
    return H, E, F


def leaf_solve(c1, c2, scheme: OracleScheme, start_vgap, end_vgap, lo, hi):
    """kernels.leaf_solve (kernels.py:91-185): (score, ops) or (NEG_INF, None)."""
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    sub = np.ascontiguousarray(scheme.sub, dtype=np.int64)
    cap = c1.size + c2.size
    ops = np.empty(max(cap, 1), dtype=np.uint8)
    cnt = ctypes.c_int64()
    s = _lib().orc_leaf_solve(_c(c1), c1.size, _c(c2), c2.size, _c(sub), sub.shape[0],
                              scheme.gap_open, scheme.gap_extend, int(start_vgap), int(end_vgap),
                              int(lo), int(hi), _c(ops), cap, ctypes.byref(cnt))
    if cnt.value < 0:
        return NEG_INF, None
    return int(s), ops[:cnt.value].copy()


# -- helpers -------------------------------------------------------------------

_C1 = np.array([1, 1, 0, 1], dtype=np.int64)  # model.py:236-237
_C2 = np.array([1, 1, 1, 0], dtype=np.int64)


class OracleMismatch(AssertionError):
    pass


def rescore(start, ops, c1, c2, scheme: OracleScheme) -> int:
    """Single-pass re-score (oracle.rescore_path, oracle.py:204-226)."""
    i, j = start
    total, prev = 0, -1
    for op in ops.tolist():
        if op <= 1:
            total += int(scheme.sub[c1[i], c2[j]])
            i += 1
            j += 1
        elif op == 2:
            total -= scheme.gap_extend + (scheme.gap_open if prev != 2 else 0)
            j += 1
        else:
            total -= scheme.gap_extend + (scheme.gap_open if prev != 3 else 0)
            i += 1
        prev = op
    return total


def _band_corridor(score, n_short, m_long, scheme):
    """phase2.compute_band + applied_interval (phase2.py:45-79), in
    longer-minus-shorter units."""
    ms, ge = scheme.max_sub, scheme.gap_extend
    t = min(score // ms, n_short)
    m_prime = min(n_short + (n_short - t) // ge, m_long)
    p = max(0, math.ceil(0.5 * (2 * n_short - t - m_prime)))
    lo, hi = -p, p + (m_long - n_short)
    g = max(0, (ms * n_short - score) // ge)
    return min(lo, -g), max(hi, g)


def _oriented(score, rows, cols, scheme):
    """Engine-unit (row - col) corridor for a restricted search
    (phase2.py:155-163, split._search_interval split.py:185-192)."""
    lo, hi = _band_corridor(score, min(rows, cols), max(rows, cols), scheme)
    return (lo, hi) if rows >= cols else (-hi, -lo)


def _restricted(rc1, rc2, scheme, target, band, track=TRACK_MAX, lead=None, threads=None):
    """phase2.restricted_search (phase2.py:82-138)."""
    border = "restricted" if lead is None else lead
    out = run_wavefront(rc1, rc2, scheme, border, False, track, band=band, threads=threads)
    if out.bi < 0 or out.best != target:
        raise OracleMismatch(f"no cell attains {target} (best {out.best})")
    return out.bi, out.bj


def _mm_band(rows, cols, score, scheme):
    """phase3.band_interval (phase3.py:83-98)."""
    d = rows - cols
    g = (scheme.max_sub * (rows + cols) - 2 * score) // (scheme.max_sub + 2 * scheme.gap_extend)
    g = min(max(g, abs(d)), rows + cols)
    pad = (g - abs(d)) // 2
    return min(0, d) - pad, max(0, d) + pad


def _crossing(sub, c1, c2, scheme, band, threads):
    """phase3.find_crossing + _pick_crossing (phase3.py:123-190)."""
    (si, sj), (ei, ej), exp, svg, evg = sub
    rows, cols = ei - si, ej - sj
    midr = rows // 2
    iv = _mm_band(rows, cols, exp, scheme) if band else None
    up = run_wavefront(c1[si:si + midr], c2[sj:ej], scheme, "continue" if svg else "free",
                       False, TRACK_NONE, band=iv, threads=threads)
    riv = None if iv is None else (rows - cols - iv[1], rows - cols - iv[0])
    dn = run_wavefront(c1[si + midr:ei][::-1], c2[sj:ej][::-1], scheme,
                       "charge" if evg else "free", False, TRACK_NONE, band=riv, threads=threads)
    hh = up.final_h + dn.final_h[::-1]
    ff = up.final_f + dn.final_f[::-1] + scheme.gap_open
    best = max(int(hh.max()), int(ff.max()))
    jh = int(np.flatnonzero(hh == best)[0]) if (hh == best).any() else 1 << 62
    jf = int(np.flatnonzero(ff == best)[0]) if (ff == best).any() else 1 << 62
    gap = jf < jh
    j = jf if gap else jh
    if best != exp:
        raise OracleMismatch(f"crossing {best} != expected {exp}")
    if gap:
        upper, lower = int(up.final_f[j]), int(dn.final_f[cols - j])
    else:
        upper, lower = int(up.final_h[j]), int(dn.final_h[cols - j])
    return (si + midr, sj + j), upper, lower, gap


def _leaf(sub, c1, c2, scheme, band):
    """phase3._solve_leaf (phase3.py:200-247)."""
    (si, sj), (ei, ej), exp, svg, evg = sub
    rows, cols = ei - si, ej - sj
    go, ge = scheme.gap_open, scheme.gap_extend
    if rows == 0 and cols == 0:
        if exp != 0:
            raise OracleMismatch("empty rectangle with nonzero score")
        return np.empty(0, dtype=np.uint8)
    if rows == 0:
        if svg or evg or exp != -(go + cols * ge):
            raise OracleMismatch("bad insert run")
        return np.full(cols, 2, dtype=np.uint8)
    if cols == 0:
        want = -((0 if svg else go) + rows * ge)
        if exp != want:
            raise OracleMismatch("bad delete run")
        return np.full(rows, 3, dtype=np.uint8)
    lo, hi = _mm_band(rows, cols, exp, scheme) if band else (-(rows + cols), rows + cols)
    s, ops = leaf_solve(c1[si:ei], c2[sj:ej], scheme, svg, evg, lo, hi)
    if ops is None or s != exp:
        raise OracleMismatch(f"leaf reached {s}, expected {exp}")
    return ops


def _solve_rect(root, c1, c2, scheme, leaf_limit, band, threads):
    """phase3.solve_rect (phase3.py:250-286): DFS, leaves in path order."""
    leaves = []
    stack = [root]
    while stack:
        s = stack.pop()
        (si, sj), (ei, ej) = s[0], s[1]
        rows, cols = ei - si, ej - sj
        if rows * cols <= leaf_limit or rows <= 1 or cols <= 1:
            leaves.append(s)
            continue
        mid, upper, lower, gap = _crossing(s, c1, c2, scheme, band, threads)
        lower_exp = lower + (scheme.gap_open if gap else 0)
        # push the lower child first so the upper child is expanded first
        stack.append((mid, s[1], lower_exp, gap, s[4]))
        stack.append((s[0], mid, upper, s[3], gap))
    parts = [_leaf(s, c1, c2, scheme, band) for s in leaves]
    return np.concatenate(parts) if parts else np.empty(0, dtype=np.uint8)


# -- public entry points -------------------------------------------------------

def score_only(c1, c2, scheme: OracleScheme, prune=True, block=(512, 512), threads=None):
    """pipeline.score_only -> phase1.best_local (pipeline.py:103-126,
    phase1.py:44-85)."""
    out = run_wavefront(c1, c2, scheme, "local", True, TRACK_MIN, prune=prune, fill_h=0,
                        block=block, threads=threads)
    if out.best <= 0:
        return 0, (0, 0), out
    return int(out.best), (out.bi + 1, out.bj + 1), out


def _phase23(c1, c2, scheme, score, end, leaf_limit, band, threads):
    """phase2.locate_start + phase3.reconstruct (phase2.py:141-165,
    phase3.py:289-312)."""
    ei, ej = end
    iv = None
    if band:
        lo, hi = _band_corridor(score, min(ei, ej), max(ei, ej), scheme)
        iv = (lo, hi) if ei >= ej else (-hi, -lo)
    ri, rj = _restricted(c1[:ei][::-1], c2[:ej][::-1], scheme, score, iv, threads=threads)
    start = (ei - ri - 1, ej - rj - 1)
    ops = _solve_rect((start, end, score, False, False), c1, c2, scheme, leaf_limit, band, threads)
    if rescore(start, ops, c1, c2, scheme) != score:
        raise OracleMismatch("reconstructed path does not re-score")
    return start, ops


def align(c1, c2, scheme: OracleScheme, leaf_limit=128 * 128, band=True, prune=True, split=1,
          threads=None):
    """pipeline.align (pipeline.py:46-100) and split.split_align (split.py:84-182)."""
    c1 = np.ascontiguousarray(c1, dtype=np.uint8)
    c2 = np.ascontiguousarray(c2, dtype=np.uint8)
    if split == 2:
        return _split_align(c1, c2, scheme, leaf_limit, band, threads)
    score, end, _ = score_only(c1, c2, scheme, prune=prune, threads=threads)
    if score == 0:
        return 0, (0, 0), (0, 0), np.empty(0, dtype=np.uint8)
    start, ops = _phase23(c1, c2, scheme, score, end, leaf_limit, band, threads)
    return score, start, end, ops


def _split_align(c1, c2, scheme, leaf_limit, band, threads):
    n1, n2 = c1.size, c2.size
    mid = n1 // 2
    go = scheme.gap_open
    dn = run_wavefront(c1[mid:][::-1], c2[::-1], scheme, "local", True, TRACK_MIN,
                       threads=threads)
    if mid >= 1:
        up = run_wavefront(c1[:mid], c2, scheme, "local", True, TRACK_MIN, threads=threads)
        u_score = max(0, up.best)
        u_end = (up.bi + 1, up.bj + 1) if u_score > 0 else (0, 0)
        hh = up.final_h + dn.final_h[::-1]
        ff = up.final_f + dn.final_f[::-1] + go
        m_score = max(int(hh.max()), int(ff.max()))
        jh = int(np.flatnonzero(hh == m_score)[0]) if (hh == m_score).any() else 1 << 62
        jf = int(np.flatnonzero(ff == m_score)[0]) if (ff == m_score).any() else 1 << 62
        gap = jf < jh
        jc = jf if gap else jh
        u_seg = int(up.final_f[jc]) if gap else int(up.final_h[jc])
        l_seg = int(dn.final_f[n2 - jc]) if gap else int(dn.final_h[n2 - jc])
    else:
        u_score, u_end, m_score, jc, gap, u_seg, l_seg = 0, (0, 0), 0, 0, False, 0, 0
    l_score = max(0, dn.best)
    l_start = (n1 - (dn.bi + 1), n2 - (dn.bj + 1)) if l_score > 0 else (0, 0)
    # classify_midcase (split.py:55-61): ties upper > midpoint > lower
    if u_score >= m_score and u_score >= l_score:
        if u_score == 0:
            return 0, (0, 0), (0, 0), np.empty(0, dtype=np.uint8)
        start, ops = _phase23(c1, c2, scheme, u_score, u_end, leaf_limit, band, threads)
        return u_score, start, u_end, ops
    if m_score < l_score:
        # _finish_lower (split.py:208-221)
        si, sj = l_start
        iv = _oriented(l_score, n1 - si, n2 - sj, scheme) if band else None
        ci, cj = _restricted(c1[si:], c2[sj:], scheme, l_score, iv, track=TRACK_MIN,
                             threads=threads)
        end = (si + ci + 1, sj + cj + 1)
        ops = _solve_rect((l_start, end, l_score, False, False), c1, c2, scheme, leaf_limit,
                          band, threads)
        return l_score, l_start, end, ops
    # _finish_midpoint (split.py:224-298)
    cross = (mid, jc)
    u_target = u_seg + (go if gap else 0)
    l_exp = l_seg + (go if gap else 0)
    if not gap and u_seg == 0:
        ustart, ops_up = cross, np.empty(0, dtype=np.uint8)
    else:
        iv = _oriented(u_target, mid, jc, scheme) if (band and u_target >= 1) else None
        lead = "continue" if gap else "free"
        ri, rj = _restricted(c1[:mid][::-1], c2[:jc][::-1], scheme, u_target, iv,
                             track=TRACK_MAX, lead=lead, threads=threads)
        ustart = (mid - ri - 1, jc - rj - 1)
        ops_up = _solve_rect((ustart, cross, u_seg, False, gap), c1, c2, scheme, leaf_limit,
                             band, threads)
    iv = _oriented(l_exp, n1 - mid, n2 - jc, scheme) if (band and l_exp >= 1) else None
    ci, cj = _restricted(c1[mid:], c2[jc:], scheme, l_exp, iv, track=TRACK_MIN,
                         lead="continue" if gap else "free", threads=threads)
    lend = (mid + ci + 1, jc + cj + 1)
    ops_dn = _solve_rect((cross, lend, l_exp, gap, False), c1, c2, scheme, leaf_limit, band,
                         threads)
    ops = np.concatenate([ops_up, ops_dn])
    if rescore(ustart, ops, c1, c2, scheme) != m_score:
        raise OracleMismatch("joined midpoint path does not re-score")
    return m_score, ustart, lend, ops


if os.environ.get("SWB_ORACLE_SELFTEST"):
    _lib()
