"""Device context and the pass operator API (replaces engine.py).

`DeviceContext` owns one libswb context (stream, scratch, uploaded
sequences) per device.  `Session` holds the two uploaded sequences of one
align()/score_only() call so every pass of every phase addresses slices of
the same device-resident forward/reversed copies (no per-pass H2D).

`WavefrontEngine.run_wavefront(PassSpec) -> PassResult` is the operator-level
drop-in for the reference engine (engine.py:143-282): same result fields, with
the PassSpec callables replaced by the border family / prune flag enums the
C ABI takes (include/swb.h).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import DeviceUnavailable
from .model import ScoringScheme

NEG_INF = _lib.NEG_INF_REF
TRACK_NONE, TRACK_MIN, TRACK_MAX = _lib.TRACK_NONE, _lib.TRACK_MIN, _lib.TRACK_MAX
BORDERS = {
    "local": _lib.BORDER_LOCAL,
    "restricted": _lib.BORDER_RESTRICTED,
    "free": _lib.BORDER_FREE,
    "continue": _lib.BORDER_CONTINUE,
    "charge": _lib.BORDER_CHARGE,
}
# Reference block dims (engine.py:30-31); accepted for API parity, the device
# tiling is fixed by the kernel (32 lanes x R rows per warp-strip).
DEFAULT_BLOCK_ROWS = 512
DEFAULT_BLOCK_COLS = 512

_contexts: dict[int, "DeviceContext"] = {}
_ctx_lock = threading.Lock()


def scheme_struct(scheme: ScoringScheme) -> _lib.Scheme:
    k = len(scheme.alphabet)
    if k > 32:
        raise ValueError(f"alphabets of {k} symbols are not supported on the device (max 32)")
    s = _lib.Scheme()
    s.k = k
    flat = np.asarray(scheme.matrix, dtype=np.int64).reshape(-1)
    if flat.size and (flat.max() > 2 ** 20 or flat.min() < -(2 ** 20)):
        raise ValueError("substitution scores out of the supported range")
    for x, v in enumerate(flat.tolist()):
        s.sub[x] = int(v)
    s.gap_open = int(scheme.gap_open)
    s.gap_extend = int(scheme.gap_extend)
    s.max_sub = int(flat.max())
    return s


class DeviceContext:
    def __init__(self, device: int = 0):
        lib = _lib.load()
        ptr = lib.swb_ctx_create(int(device))
        if not ptr:
            raise DeviceUnavailable(f"cannot create a B200 context on device {device}: "
                                    f"{_lib.last_error()}")
        self.lib = lib
        self.ptr = ptr
        self.device = int(device)
        self.lock = threading.Lock()

    # -- sequences -----------------------------------------------------------
    def upload(self, codes: np.ndarray) -> int:
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        sid = ctypes.c_int32()
        _lib.check(self.lib.swb_seq_upload(self.ptr, codes.ctypes.data_as(ctypes.c_void_p),
                                           codes.size, ctypes.byref(sid)), "swb_seq_upload")
        return int(sid.value)

    def release(self, sid: int) -> None:
        _lib.check(self.lib.swb_seq_release(self.ptr, int(sid)), "swb_seq_release")

    # -- operators -----------------------------------------------------------
    def passes(self, scheme: _lib.Scheme, descs: list[_lib.PassDesc]) -> list[_lib.PassOut]:
        n = len(descs)
        arr = (_lib.PassDesc * n)(*descs)
        outs = (_lib.PassOut * n)()
        _lib.check(self.lib.swb_pass(self.ptr, ctypes.byref(scheme), arr, n, outs), "swb_pass")
        return list(outs)

    def crossings(self, scheme, s1: int, s2: int, subs: np.ndarray, band: bool):
        """subs: structured array with _lib.Subproblem layout."""
        n = int(subs.shape[0])
        out = (_lib.Crossing * n)()
        cells = ctypes.c_int64()
        sub_ptr = subs.ctypes.data_as(ctypes.POINTER(_lib.Subproblem))
        _lib.check(self.lib.swb_crossings(self.ptr, ctypes.byref(scheme), s1, s2, sub_ptr, n,
                                          int(band), out, ctypes.byref(cells)), "swb_crossings")
        res = np.frombuffer(out, dtype=CROSSING_DTYPE, count=n).copy()
        return res, int(cells.value)

    def leaves(self, scheme, s1: int, s2: int, subs: np.ndarray, band: bool):
        n = int(subs.shape[0])
        rows = (subs["ei"] - subs["si"]).astype(np.int64)
        cols = (subs["ej"] - subs["sj"]).astype(np.int64)
        cap = rows + cols
        offsets = np.zeros(n, dtype=np.int64)
        if n > 1:
            offsets[1:] = np.cumsum(cap)[:-1]
        ops = np.empty(int(cap.sum()) + 1, dtype=np.uint8)
        counts = np.empty(n, dtype=np.int64)
        scores = np.empty(n, dtype=np.int64)
        vp = ctypes.c_void_p
        _lib.check(self.lib.swb_leaves(self.ptr, ctypes.byref(scheme), s1, s2,
                                       subs.ctypes.data_as(ctypes.POINTER(_lib.Subproblem)), n,
                                       int(band), ops.ctypes.data_as(vp),
                                       offsets.ctypes.data_as(vp), counts.ctypes.data_as(vp),
                                       scores.ctypes.data_as(vp)), "swb_leaves")
        return ops, offsets, counts, scores

    def measure_int_peak(self) -> dict:
        p = _lib.IntPeak()
        _lib.check(self.lib.swb_measure_int_peak(self.ptr, ctypes.byref(p)), "swb_measure_int_peak")
        return {name: getattr(p, name) for name, _ in _lib.IntPeak._fields_}

    def set_option(self, name: str, value: int) -> None:
        _lib.check(self.lib.swb_set_option(self.ptr, name.encode(), int(value)), "swb_set_option")

    def bounds_map(self, which: int) -> np.ndarray:
        """Raw tile bound map (1 forward, 2 reverse) of the current pair."""
        n = int(self.lib.swb_bounds_read(self.ptr, which, None, 0))
        out = np.zeros(max(n, 0), dtype=np.int32)
        if n > 0:
            self.lib.swb_bounds_read(self.ptr, which, out.ctypes.data, n)
        return out

    def bounds_device(self, which: int) -> tuple[int, int, int]:
        """(device address, nr * nc, nc) of the forward (1) / reverse (2) map."""
        p, n, nc = ctypes.c_uint64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(self.lib.swb_bounds_device(self.ptr, which, ctypes.byref(p), ctypes.byref(n),
                                              ctypes.byref(nc)), "swb_bounds_device")
        return int(p.value), int(n.value), int(nc.value)

    def get_option(self, name: str) -> int:
        return int(self.lib.swb_get_option(self.ptr, name.encode()))

    def timer_start(self) -> None:
        _lib.check(self.lib.swb_timer_start(self.ptr), "swb_timer_start")

    def timer_stop(self) -> float:
        ms = ctypes.c_double()
        _lib.check(self.lib.swb_timer_stop(self.ptr, ctypes.byref(ms)), "swb_timer_stop")
        return float(ms.value)

    def flush_l2(self, nbytes: int = 0) -> None:
        _lib.check(self.lib.swb_flush_l2(self.ptr, int(nbytes)), "swb_flush_l2")

    def debug_stats(self) -> dict:
        out = (ctypes.c_int64 * 2)()
        _lib.check(self.lib.swb_debug_stats(self.ptr, out, 2), "swb_debug_stats")
        return {"wait_cycles": int(out[0]), "strip_cycles": int(out[1])}

    def debug_times(self) -> np.ndarray:
        n = int(self.lib.swb_debug_times(self.ptr, None, 0)) if False else 1 << 20
        out = np.zeros(n, dtype=np.int64)
        m = self.lib.swb_debug_times(self.ptr, out.ctypes.data, n)
        return out[:max(0, min(m, n))].reshape(-1, 3)

    def debug_strips(self) -> np.ndarray:
        """Per-strip record of the last pass launch (include/swb.h
        swb_debug_strips): columns cb_static, cb_start, ce, exit_col, executed,
        skipped, live_lo, live_hi, launch, sm, cta, warp, start_ns, end_ns, key, i, j, has."""
        m = int(self.lib.swb_debug_strips(self.ptr, None, 0))
        raw = np.zeros(max(m, 0), dtype=np.int64)
        if m > 0:
            self.lib.swb_debug_strips(self.ptr, raw.ctypes.data, m)
        raw = raw.reshape(-1, 12)
        hi = (raw[:, :4] >> 32).astype(np.int32).astype(np.int64)
        lo = (raw[:, :4] & 0xffffffff).astype(np.uint32).view(np.int32).astype(np.int64)
        out = np.empty((raw.shape[0], 18), dtype=np.int64)
        out[:, 0:8:2] = hi
        out[:, 1:8:2] = lo
        out[:, 8] = raw[:, 4]
        out[:, 9] = raw[:, 5] >> 32
        out[:, 10] = (raw[:, 5] >> 8) & 0xffffff
        out[:, 11] = raw[:, 5] & 0xff
        out[:, 12] = raw[:, 6]
        out[:, 13] = raw[:, 7]
        out[:, 14:] = raw[:, 8:]
        return out

    def debug_claims(self, launch: int | None = None) -> np.ndarray:
        """Claim log entries (launch, kind, sm, cta, warp, value, ns), oldest
        first, optionally of one launch (include/swb.h swb_debug_claims)."""
        m = int(self.lib.swb_debug_claims(self.ptr, None, 0))
        if m <= 0:
            return np.zeros((0, 7), dtype=np.int64)
        raw = np.zeros(m, dtype=np.int64)
        self.lib.swb_debug_claims(self.ptr, raw.ctypes.data, m)
        total = int(raw[0])
        ent = raw[8:].reshape(-1, 4)
        idx = np.arange(max(0, total - 4096), total) % 4096
        ent = ent[idx]
        w = ent[:, 1].view(np.uint64)
        out = np.stack([ent[:, 0], (w >> 56).astype(np.int64), ((w >> 40) & 0xffff).astype(np.int64),
                        ((w >> 8) & 0xffffffff).astype(np.int64), (w & 0xff).astype(np.int64),
                        ent[:, 2], ent[:, 3]], axis=1)
        if launch is not None:
            out = out[out[:, 0] == launch]
        return out

    @property
    def launch_count(self) -> int:
        return int(self.lib.swb_launch_count(self.ptr))

    @property
    def last_kernel_ms(self) -> float:
        return float(self.lib.swb_last_kernel_ms(self.ptr))


@dataclass(frozen=True)
class BlockGrid:
    """engine.BlockGrid (engine.py:34-55): the reference's CPU tiling plan,
    kept for API parity (the device decomposes into warp strips instead;
    results do not depend on the tiling, SURVEY.md §0 finding 1)."""

    rows: int
    cols: int
    block_rows: int
    block_cols: int
    grid_rows: int
    grid_cols: int

    @property
    def anti_diagonals(self) -> int:
        return self.grid_rows + self.grid_cols - 1

    def row_span(self, bi: int) -> tuple[int, int]:
        r0 = bi * self.block_rows
        return r0, min(r0 + self.block_rows, self.rows)

    def col_span(self, bj: int) -> tuple[int, int]:
        c0 = bj * self.block_cols
        return c0, min(c0 + self.block_cols, self.cols)


def plan_grid(len1: int, len2: int, block_rows: int = DEFAULT_BLOCK_ROWS,
              block_cols: int = DEFAULT_BLOCK_COLS) -> BlockGrid:
    """engine.plan_grid (engine.py:58-71)."""
    if len1 < 1 or len2 < 1:
        raise ValueError("cannot tile an empty matrix")
    block_rows = max(1, min(block_rows, len1))
    block_cols = max(1, min(block_cols, len2))
    return BlockGrid(len1, len2, block_rows, block_cols, -(-len1 // block_rows),
                     -(-len2 // block_cols))


class AllocationMeter:
    """engine.AllocationMeter (engine.py:74-90): counts live DP-state elements.
    The device path reports, per launch, its row buffers and the lane state of
    its strips (Session.run), so the linear-memory property can be checked the
    same way as on the reference."""

    def __init__(self):
        self._lock = threading.Lock()
        self.current = 0
        self.peak = 0

    def add(self, n: int):
        with self._lock:
            self.current += n
            if self.current > self.peak:
                self.peak = self.current

    def release(self, n: int):
        with self._lock:
            self.current -= n


def bound_slack(scheme: ScoringScheme) -> int:
    """Slack of the tile-bound tests (same formula as swb_crossings): junction
    gaps and the cell counted by both halves of a split path."""
    min_sub = min(0, int(np.asarray(scheme.matrix).min()))
    return 4 * (scheme.gap_open + scheme.gap_extend) + 2 * (max(scheme.max_substitution_score, 0)
                                                           - min_sub)


SUBPROBLEM_DTYPE = np.dtype([("si", "<i8"), ("sj", "<i8"), ("ei", "<i8"), ("ej", "<i8"),
                             ("expected", "<i8"), ("start_vgap", "<i4"), ("end_vgap", "<i4"),
                             ("use_bounds", "<i4"), ("pad", "<i4"), ("prefix", "<i8"),
                             ("suffix", "<i8")])
CROSSING_DTYPE = np.dtype([("mid_i", "<i8"), ("mid_j", "<i8"), ("upper", "<i8"),
                           ("lower", "<i8"), ("gap_join", "<i4"), ("status", "<i4")])
assert SUBPROBLEM_DTYPE.itemsize == ctypes.sizeof(_lib.Subproblem)
assert CROSSING_DTYPE.itemsize == ctypes.sizeof(_lib.Crossing)


def get_context(device: int = 0) -> DeviceContext:
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = DeviceContext(device)
            _contexts[device] = ctx
        return ctx


# swb_pass_out.kernel: which device kernel carried the pass
KERNEL_NAMES = {0: "lane32", 1: "packed16x2", 2: "wide64"}


@dataclass
class PassResult:
    """engine.PassResult (engine.py:120-131); tiles replace 512x512 blocks."""

    best_score: int
    best_i: int
    best_j: int
    final_row_h: Optional[np.ndarray]
    final_row_f: Optional[np.ndarray]
    total_blocks: int
    executed_blocks: int
    pruned_blocks: int
    banded_out_blocks: int
    cells_executed: int
    kernel_ms: float = 0.0
    kernel: str = "lane32"     # "lane32", "packed16x2" or "wide64" (KERNEL_NAMES)
    rows_per_lane: int = 0


class Session:
    """The two sequences of one alignment, resident on one device."""

    def __init__(self, ctx: DeviceContext, codes1: np.ndarray, codes2: np.ndarray,
                 scheme: ScoringScheme):
        self.ctx = ctx
        self.n1 = int(codes1.size)
        self.n2 = int(codes2.size)
        self.codes1 = codes1
        self.codes2 = codes2
        self.scheme = scheme
        self.cs = scheme_struct(scheme)
        self.s1 = ctx.upload(codes1)
        self.s2 = ctx.upload(codes2)
        self.kernel_ms = 0.0
        self.cells = 0
        self.target_prune = True  # phase-2 restricted searches skip hopeless blocks
        self.bounds = False       # tile bound maps filled for this pair (reset_bounds)
        self.meter = None         # engine.AllocationMeter analogue (state_cells per pass)

    def reset_bounds(self) -> None:
        """Clear the pair's tile bound maps; phases 1 and 2 of
        an align() fill them, phases 2 and 3 prune with them."""
        _lib.check(self.ctx.lib.swb_bounds_reset(self.ctx.ptr, self.s1, self.s2),
                   "swb_bounds_reset")
        self.bounds = True

    def close(self):
        if self.s1 is not None:
            self.ctx.release(self.s1)
            self.ctx.release(self.s2)
            self.s1 = self.s2 = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def desc(self, rows: tuple, cols: tuple, border: str, clamp: bool, track: int,
             band=None, prune=False, final=None, row_offset=0, ext_in=None,
             ext_out=None, prune_target=0, corner=None, rows_after=0, bound_write=0,
             bound_read=0, bound_offset=0, shared_best=0) -> _lib.PassDesc:
        """rows/cols = (offset, length, reversed) slices of seq1/seq2;
        row_offset/ext_in/ext_out describe a row slab of a multi-GPU pass
        (multigpu.py, include/swb.h)."""
        d = _lib.PassDesc()
        d.seq1, d.seq2 = self.s1, self.s2
        d.off1, d.len1, d.rev1 = int(rows[0]), int(rows[1]), int(rows[2])
        d.off2, d.len2, d.rev2 = int(cols[0]), int(cols[1]), int(cols[2])
        d.border = BORDERS[border]
        d.clamp_zero = int(clamp)
        d.track = int(track)
        if band is not None:
            d.has_band, d.band_lo, d.band_hi = 1, int(band[0]), int(band[1])
        d.prune = int(prune)  # True -> 1 (running best); 2 / 3 target kinds
        d.prune_target = int(prune_target)
        if corner is not None:
            d.corner_i, d.corner_j = int(corner[0]), int(corner[1])
        if final is not None:
            d.want_final_rows = 1
            d.final_row_h = final[0].ctypes.data
            d.final_row_f = final[1].ctypes.data
        d.row_offset = int(row_offset)
        d.rows_after = int(rows_after)
        d.bound_write, d.bound_read = int(bound_write), int(bound_read)
        d.bound_offset = int(bound_offset)
        d.shared_best = int(shared_best or 0)
        if ext_in is not None:
            d.ext_in_buf, d.ext_in_progress = int(ext_in[0]), int(ext_in[1])
        if ext_out is not None:
            d.ext_out_buf, d.ext_out_progress = int(ext_out[0]), int(ext_out[1])
        return d

    def run(self, specs: list[dict]) -> list[PassResult]:
        """Run several passes in one device launch; each spec holds the
        keyword arguments of desc() plus want_final (bool)."""
        descs, finals = [], []
        for sp in specs:
            sp = dict(sp)
            want = sp.pop("want_final", False)
            fin = None
            if want:
                n2 = int(sp["cols"][1])
                fin = (np.empty(n2 + 1, dtype=np.int64), np.empty(n2 + 1, dtype=np.int64))
            finals.append(fin)
            descs.append(self.desc(final=fin, **sp))
        # device DP state of the launch, in array elements like the reference's
        # AllocationMeter (engine.py:197-205): two (H, F) row buffers per pass
        # plus the per-row lane state (H, E) of the strips in flight
        cells = sum(4 * (int(d.len2) + 1) + 2 * int(d.len1) for d in descs)
        if self.meter is not None:
            self.meter.add(cells)
        try:
            outs = self.ctx.passes(self.cs, descs)
        finally:
            if self.meter is not None:
                self.meter.release(cells)
        res = []
        for o, fin in zip(outs, finals):
            self.kernel_ms += o.kernel_ms
            self.cells += o.cells_executed
            res.append(PassResult(
                int(o.best_score), int(o.best_i), int(o.best_j),
                fin[0] if fin else None, fin[1] if fin else None,
                int(o.tiles_total), int(o.tiles_executed), int(o.tiles_pruned),
                int(o.tiles_banded_out), int(o.cells_executed), float(o.kernel_ms),
                KERNEL_NAMES.get(int(o.kernel), "lane32"), int(o.rows_per_lane)))
        # one launch carries all specs: count its time once
        if len(outs) > 1:
            self.kernel_ms -= sum(o.kernel_ms for o in outs[1:])
        return res


@dataclass
class PassSpec:
    """Device form of engine.PassSpec (engine.py:93-117): the left_border
    callable becomes `border`, the prune callable the phase-1 `prune` flag."""

    codes1: np.ndarray
    codes2: np.ndarray
    scheme: ScoringScheme
    border: str = "local"
    clamp_zero: bool = True
    track: int = TRACK_MIN
    band: Optional[tuple[int, int]] = None
    prune: bool = False
    want_final_rows: bool = True


class WavefrontEngine:
    """Reference-compatible engine facade (engine.py:143-185).  `workers`,
    block dims, `meter` and `trace` are accepted for signature parity; the
    device decomposition is fixed by the kernel."""

    def __init__(self, workers: int = 1, block_rows: int = DEFAULT_BLOCK_ROWS,
                 block_cols: int = DEFAULT_BLOCK_COLS, meter=None, trace=None, device: int = 0):
        if workers < 1:
            raise ValueError("workers must be >= 1")
        self.workers = workers
        self.block_rows = block_rows
        self.block_cols = block_cols
        self.meter = meter
        self.trace = trace
        self.device = device

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def run_wavefront(self, spec: PassSpec) -> PassResult:
        c1 = np.ascontiguousarray(spec.codes1, dtype=np.uint8)
        c2 = np.ascontiguousarray(spec.codes2, dtype=np.uint8)
        if c1.size < 1 or c2.size < 1:
            raise ValueError("cannot tile an empty matrix")
        with Session(get_context(self.device), c1, c2, spec.scheme) as S:
            S.meter = self.meter
            return S.run([dict(rows=(0, c1.size, 0), cols=(0, c2.size, 0), border=spec.border,
                               clamp=spec.clamp_zero, track=spec.track, band=spec.band,
                               prune=spec.prune, want_final=spec.want_final_rows)])[0]
