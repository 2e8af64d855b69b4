"""Multi-GPU decomposition of a wavefront pass.

A pass is one chain of warp-strips; across GPUs the chain simply continues:
GPU g owns a contiguous *row slab* of strips, and the bottom DP row of slab g
(H and F for every column, index 0 = left border) is the top border of slab
g+1.  On NVLink the device kernels stream that row through peer-mapped memory
strip block by strip block (publication protocol of DESIGN.md §3.2); the host
logic here — partitioning, the row handed over, the final merge of per-slab
bests with the reference's tie rules (engine.py:247-259) — is shared by the
device path and by the world-size-2 gloo test (tests/test_multigpu_gloo.py),
which checks that a slab-split pass reproduces the single pass exactly.
"""
from __future__ import annotations

from dataclasses import dataclass

TRACK_NONE, TRACK_MIN, TRACK_MAX = 0, 1, 2
SLAB_ROWS_PER_LANE = 32  # every rank uses the same strip height: 32 lanes x 32 rows
SLAB_STRIP_ROWS = 32 * SLAB_ROWS_PER_LANE


@dataclass(frozen=True)
class Slab:
    rank: int
    row0: int  # first DP row owned (cell row index)
    row1: int  # one past the last

    @property
    def rows(self) -> int:
        return self.row1 - self.row0


def slab_partition(n1: int, world: int, strip_rows: int = 1024) -> list[Slab]:
    """Split n1 rows into `world` contiguous slabs of whole strips, as even as
    possible (the last non-empty slab takes the ragged remainder).  With fewer
    strips than ranks the first `strips` ranks get one strip each and the rest
    an empty slab (rows == 0, always at the end): a slab that feeds another
    must end on a strip boundary, so rows are never split below a strip."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if n1 < 1:
        raise ValueError("cannot partition an empty pass")
    strips = -(-n1 // strip_rows)
    used = min(world, strips)
    bounds = [min(n1, ((strips * g) // used) * strip_rows) for g in range(used + 1)]
    bounds += [n1] * (world - used)
    return [Slab(g, bounds[g], bounds[g + 1]) for g in range(world)]


def merge_best(results: list[tuple[int, int, int]], track: int) -> tuple[int, int, int]:
    """Combine per-slab (score, i, j) with absolute rows; i < 0 means none.
    TRACK_MIN: max score, ties to the smallest (i, j), only positive scores;
    TRACK_MAX: max score, ties to the largest (i, j)."""
    best = None
    for s, i, j in results:
        if i < 0:
            continue
        if track == TRACK_MIN and s <= 0:
            continue
        if best is None:
            best = (s, i, j)
            continue
        bs, bi, bj = best
        if track == TRACK_MIN:
            take = s > bs or (s == bs and (i, j) < (bi, bj))
        else:
            take = s > bs or (s == bs and (i, j) > (bi, bj))
        if take:
            best = (s, i, j)
    if best is None:
        return (0, -1, -1) if track == TRACK_MIN else (-(2 ** 61), -1, -1)
    return best


def handoff_bytes(n2: int) -> int:
    """Bytes one slab boundary moves over NVLink: (H, F) int32 per column."""
    return 8 * n2


# -- device path ------------------------------------------------------------------

class Boundary:
    """Incoming boundary row of one GPU: int2[n2] + progress counter in its own
    device memory (written by the GPU above through a peer mapping)."""

    def __init__(self, ctx, n2: int):
        import ctypes
        from . import _lib
        self.ctx = ctx
        b, p = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(ctx.lib.swb_boundary_alloc(ctx.ptr, int(n2), ctypes.byref(b), ctypes.byref(p)),
                   "swb_boundary_alloc")
        self.buf, self.progress = int(b.value), int(p.value)

    def reset(self):
        from . import _lib
        _lib.check(self.ctx.lib.swb_boundary_reset(self.ctx.ptr, self.progress),
                   "swb_boundary_reset")

    def export(self) -> tuple[bytes, bytes]:
        return ipc_export(self.ctx, self.buf), ipc_export(self.ctx, self.progress)

    def free(self):
        from . import _lib
        _lib.check(self.ctx.lib.swb_boundary_free(self.ctx.ptr, self.buf, self.progress),
                   "swb_boundary_free")
        self.buf = self.progress = 0


def ipc_export(ctx, ptr: int) -> bytes:
    import ctypes
    from . import _lib
    h = (ctypes.c_uint8 * 64)()
    _lib.check(ctx.lib.swb_ipc_export(ctx.ptr, int(ptr), h), "swb_ipc_export")
    return bytes(h)


def ipc_import(ctx, handle: bytes) -> int:
    import ctypes
    from . import _lib
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = ctypes.c_uint64()
    _lib.check(ctx.lib.swb_ipc_import(ctx.ptr, h, ctypes.byref(p)), "swb_ipc_import")
    return int(p.value)


def slab_spec(slab: Slab, n1: int, n2: int, ext_in: tuple[int, int] | None,
              ext_out: tuple[int, int] | None, prune: bool = True, shared_best: int = 0) -> dict:
    """Session.run() spec of one slab of a local score pass (phase1.py:44-85).
    rows_after (the pass's rows below the slab) keeps the pruning bound of
    phase1.py:55-59 sound for paths that continue on the GPUs below;
    shared_best (a device word every slab reads and raises) gives every slab
    the running best of the whole pass, as the reference's barrier-refreshed
    best does for its blocks (engine.py:260-261)."""
    return dict(rows=(slab.row0, slab.rows, 0), cols=(0, n2, 0), border="local", clamp=True,
                track=TRACK_MIN, prune=prune, row_offset=slab.row0,
                ext_in=ext_in, ext_out=ext_out, rows_after=n1 - slab.row1,
                shared_best=shared_best if prune else 0)


def run_slabs_sequential(S, slabs: list[Slab], prune: bool = True):
    """One-GPU validation of the slab handoff: run the slabs of a score pass one
    after another on the same device, each consuming the previous slab's
    boundary row through the ext_in/ext_out path (no concurrent waiting).
    Returns the merged (score, i, j) and the per-slab results."""
    slabs = [sl for sl in slabs if sl.rows > 0]
    bounds = [Boundary(S.ctx, S.n2) for _ in slabs[1:]]
    S.ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
    try:
        results = []
        for g, slab in enumerate(slabs):
            ext_in = (bounds[g - 1].buf, bounds[g - 1].progress) if g > 0 else None
            ext_out = (bounds[g].buf, bounds[g].progress) if g + 1 < len(slabs) else None
            r = S.run([slab_spec(slab, S.n1, S.n2, ext_in, ext_out, prune)])[0]
            results.append(r)
        merged = merge_best([(r.best_score, r.best_i, r.best_j) for r in results], TRACK_MIN)
        return merged, results
    finally:
        S.ctx.set_option("rows_per_lane", 0)
        for b in bounds:
            b.free()


def run_slabs_concurrent(S, slabs: list[Slab], prune: bool = True, share_best: bool = True):
    """One-GPU emulation of N ranks running AT THE SAME TIME: every slab is a
    job of ONE persistent launch, and slab g+1's first strip consumes slab g's
    last strip through the same ext_in / ext_out boundary path (sys-scope
    release / acquire, __threadfence_system) the NVLink peer stores use.  Jobs
    are claimed job-major, so a strip only waits on an item claimed before it
    and the launch stays deadlock-free (separate waiting launches on one GPU
    are not: B200_PROFILING.md).  With share_best every slab prunes with the
    running best of the whole pass (swb_pass_desc.shared_best).  Returns the
    merged (score, i, j) and the per-slab results."""
    slabs = [sl for sl in slabs if sl.rows > 0]
    bounds = [Boundary(S.ctx, S.n2) for _ in slabs[1:]]
    best = Boundary(S.ctx, 1) if share_best else None  # its progress word: the shared best
    old_jm = S.ctx.get_option("job_major")
    S.ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
    S.ctx.set_option("job_major", 1)
    try:
        specs = []
        for g, slab in enumerate(slabs):
            ext_in = (bounds[g - 1].buf, bounds[g - 1].progress) if g > 0 else None
            ext_out = (bounds[g].buf, bounds[g].progress) if g + 1 < len(slabs) else None
            specs.append(slab_spec(slab, S.n1, S.n2, ext_in, ext_out, prune,
                                   best.progress if best else 0))
        results = S.run(specs)
        merged = merge_best([(r.best_score, r.best_i, r.best_j) for r in results], TRACK_MIN)
        return merged, results
    finally:
        S.ctx.set_option("rows_per_lane", 0)
        S.ctx.set_option("job_major", old_jm)
        for b in bounds + ([best] if best else []):
            b.free()


# -- Figure-1 split (split=2) across two GPU groups -------------------------------
#
# split.split_align's two local passes (upper rows [0, mid) forward, lower
# rows [mid, n1) reversed; reference split.py:84-122) each become a row-slab
# chain on their own GPU group: ranks [0, G/2) the upper half, [G/2, G) the
# lower half.  Every slab prunes against one running best shared by all G
# ranks; the last slab of each group holds its half's final row; rank 0
# gathers the two final rows ("one peer copy of the middle row", PAPER.md
# Figure 1), the per-slab bests and the tile maps, and finishes
# (split.combine_and_finish) exactly as on one GPU.

@dataclass(frozen=True)
class HalfSlab:
    half: str      # "up" (forward) or "dn" (reversed lower half)
    slab: Slab     # rows in the half's own pass coordinates
    index: int     # position in the group's chain
    last: bool     # holds the half's final row


def split_groups(world: int) -> tuple[list[int], list[int]]:
    """Ranks of the upper and lower groups (one each when world == 2)."""
    if world < 2:
        raise ValueError("a split across GPU groups needs at least 2 ranks")
    up = world // 2
    return list(range(up)), list(range(up, world))


def split_plan(n1: int, world: int, strip_rows: int = SLAB_STRIP_ROWS) -> list[HalfSlab]:
    """Per-rank slab of the Figure-1 split; mid = n1 // 2 (split.py:103)."""
    mid = n1 // 2
    ups, dns = split_groups(world)
    plan = []
    for half, ranks, rows in (("up", ups, mid), ("dn", dns, n1 - mid)):
        slabs = slab_partition(max(rows, 1), len(ranks), strip_rows) if rows else \
            [Slab(g, 0, 0) for g in range(len(ranks))]
        nonempty = [q for q, sl in enumerate(slabs) if sl.rows > 0]
        lastq = nonempty[-1] if nonempty else -1
        for q, sl in enumerate(slabs):
            plan.append(HalfSlab(half, sl, q, q == lastq))
    return plan


def half_slab_spec(hs: HalfSlab, n1: int, n2: int, ext_in, ext_out, shared_best: int) -> dict:
    """Session.run() spec of one slab of a split half (split.half_specs, cut
    into row slabs): the upper half reads rows forward, the lower half the
    reversed rows of [mid, n1) against the reversed columns; rows_after counts
    the rest of the half below the slab plus the other half."""
    mid = n1 // 2
    sl = hs.slab
    if hs.half == "up":
        rows, cols, rows_after, write = (sl.row0, sl.rows, 0), (0, n2, 0), n1 - sl.row1, 1
    else:
        nl = n1 - mid
        rows, cols = (n1 - sl.row1, sl.rows, 1), (0, n2, 1)
        rows_after, write = (nl - sl.row1) + mid, 2
    return dict(rows=rows, cols=cols, border="local", clamp=True, track=TRACK_MIN, prune=True,
                row_offset=sl.row0, ext_in=ext_in, ext_out=ext_out, rows_after=rows_after,
                shared_best=shared_best, want_final=hs.last, bound_write=write)


@dataclass
class HalfResult:
    """What split.combine_and_finish reads of a half's pass (PassResult subset)."""
    best_score: int
    best_i: int
    best_j: int
    final_row_h: object
    final_row_f: object
    cells_executed: int
    kernel_ms: float = 0.0


def merge_half(parts: list, final) -> HalfResult:
    """Merge the slab results of one half: best with the TRACK_MIN rule over
    the half's pass coordinates, final row from its last slab."""
    score, i, j = merge_best([(p[0], p[1], p[2]) for p in parts], TRACK_MIN)
    cells = sum(int(p[3]) for p in parts)
    return HalfResult(int(score), int(i), int(j), final[0], final[1], cells)


def run_split_slabs_concurrent(S, world: int, leaf_limit: int | None = None, band: bool = True,
                               report: dict | None = None):
    """One-GPU emulation of the Figure-1 split on `world` ranks: every slab of
    both halves is a job of ONE launch (job-major claiming keeps it deadlock
    free), each group's slabs chained through the ext boundary path, one
    shared running best; then the combine and finish of split.split_align.
    Returns (summary, path)."""
    from . import phase3
    from .split import combine_and_finish
    plan = split_plan(S.n1, world)
    S.reset_bounds()
    best = Boundary(S.ctx, 1)
    bounds = {}
    specs = []
    try:
        for g, hs in enumerate(plan):
            if hs.slab.rows == 0:
                continue
            nxt = plan[g + 1] if g + 1 < len(plan) else None
            feeds = nxt is not None and nxt.half == hs.half and nxt.slab.rows > 0
            if feeds:
                bounds[g] = Boundary(S.ctx, S.n2)
            ext_in = (bounds[g - 1].buf, bounds[g - 1].progress) if g - 1 in bounds else None
            ext_out = (bounds[g].buf, bounds[g].progress) if feeds else None
            specs.append((hs, half_slab_spec(hs, S.n1, S.n2, ext_in, ext_out, best.progress)))
        old_jm = S.ctx.get_option("job_major")
        S.ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
        S.ctx.set_option("job_major", 1)
        try:
            res = S.run([sp for _, sp in specs])
        finally:
            S.ctx.set_option("rows_per_lane", 0)
            S.ctx.set_option("job_major", old_jm)
    finally:
        best.free()
        for b in bounds.values():
            b.free()
    halves = {}
    for half in ("up", "dn"):
        sel = [(hs, r) for (hs, _), r in zip(specs, res) if hs.half == half]
        if not sel:
            halves[half] = None
            continue
        fin = [(r.final_row_h, r.final_row_f) for hs, r in sel if hs.last][0]
        halves[half] = merge_half([(r.best_score, r.best_i, r.best_j, r.cells_executed)
                                   for _, r in sel], fin)
    mid = S.n1 // 2
    return combine_and_finish(S, halves["up"] if mid >= 1 else None, halves["dn"], mid,
                              leaf_limit or phase3.DEFAULT_LEAF_LIMIT, band, report)


def split_align_distributed(seq1, seq2, scheme, config=None, report: dict | None = None,
                            group=None):
    """AlignConfig(split=2) on all GPUs of a torch.distributed job (NCCL, one
    process per GPU): the paper's Figure-1 schedule.  Ranks [0, G/2) run the
    upper half as row slabs, ranks [G/2, G) the reversed lower half, all at
    the same time, the slab boundary rows streamed over NVLink peer memory
    and the running best shared through a system-scope word in rank 0's
    memory.  Rank 0 receives the lower half's final row (the middle row) and
    the upper one over NCCL, merges the per-slab bests, max-reduces the tile
    maps, and finishes; every rank returns the same (summary, path), equal to
    split_align on one GPU (reference split.py:84-182).  `group` (a
    torch.distributed process group, default all ranks) lets several
    alignments share one job (align_both_strands_distributed)."""
    import os
    import time

    import numpy as np
    import torch
    import torch.distributed as dist

    from .engine import Session, get_context
    from .model import AlignmentPath, AlignmentSummary, Coord, validate_scheme
    from .pipeline import AlignConfig
    from .split import combine_and_finish

    cfg = config or AlignConfig(split=2)
    if len(seq1) < 1 or len(seq2) < 1:
        raise ValueError("alignment inputs must be non-empty")
    scheme = validate_scheme(scheme)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    local = int(os.environ.get("LOCAL_RANK", cfg.device))
    torch.cuda.set_device(local)
    ctx = get_context(local)
    if world < 2:
        from .split import split_align
        with Session(ctx, seq1.codes, seq2.codes, scheme) as S:
            return split_align(S, cfg.leaf_limit, cfg.band, report)
    t0 = time.perf_counter()
    plan = split_plan(len(seq1), world)
    me = plan[rank]
    with Session(ctx, seq1.codes, seq2.codes, scheme) as S:
        S.reset_bounds()
        n2 = S.n2
        feeds = (rank + 1 < world and plan[rank + 1].half == me.half and
                 plan[rank + 1].slab.rows > 0 and me.slab.rows > 0)
        fed = rank > 0 and plan[rank - 1].half == me.half and plan[rank - 1].slab.rows > 0 and \
            me.slab.rows > 0
        inbound = Boundary(ctx, n2) if fed else None
        best = Boundary(ctx, 1) if rank == 0 else None
        handles = [None] * world
        dist.all_gather_object(handles, (inbound.export() if inbound else None,
                                         ipc_export(ctx, best.progress) if best else None),
                              group=group)
        ext_out = None
        if feeds:
            hb, hp = handles[rank + 1][0]
            ext_out = (ipc_import(ctx, hb), ipc_import(ctx, hp))
        ext_in = (inbound.buf, inbound.progress) if inbound else None
        shared_best = best.progress if best else ipc_import(ctx, handles[0][1])
        try:
            dist.barrier(group=group)
            res = None
            if me.slab.rows > 0:
                ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
                try:
                    res = S.run([half_slab_spec(me, S.n1, n2, ext_in, ext_out, shared_best)])[0]
                finally:
                    ctx.set_option("rows_per_lane", 0)
            mine = (me.half, (res.best_score, res.best_i, res.best_j, res.cells_executed)
                    if res is not None else None)
            parts = [None] * world
            dist.all_gather_object(parts, mine, group=group)
            # the two final rows (int64 [n2 + 1] x 2 each) to rank 0 over NCCL
            finals = {}
            for half in ("up", "dn"):
                owner = next((g for g, hs in enumerate(plan) if hs.half == half and hs.last), None)
                if owner is None:
                    continue
                buf = torch.empty((2, n2 + 1), dtype=torch.int64, device=f"cuda:{local}")
                if rank == owner:
                    buf.copy_(torch.from_numpy(np.stack([res.final_row_h, res.final_row_f])))
                if owner != 0:
                    if rank == owner:
                        dist.send(buf, dst=glob(0), group=group)
                    elif rank == 0:
                        dist.recv(buf, src=glob(owner), group=group)
                if rank == 0:
                    h = buf.cpu().numpy()
                    finals[half] = (h[0].copy(), h[1].copy())
            # tile maps: every rank wrote its slab's tiles; max-reduce into rank 0
            for which in (1, 2):
                ptr, n, _ = ctx.bounds_device(which)
                full = torch.as_tensor(_DeviceRows(ptr, n), device=f"cuda:{local}")
                dist.reduce(full, dst=glob(0), op=dist.ReduceOp.MAX, group=group)
            torch.cuda.synchronize()
            out = [None]
            if rank == 0:
                halves = {}
                for half in ("up", "dn"):
                    ps = [p[1] for p in parts if p[0] == half and p[1] is not None]
                    halves[half] = merge_half(ps, finals[half]) if ps else None
                mid = S.n1 // 2
                summary, path = combine_and_finish(S, halves["up"] if mid >= 1 else None,
                                                   halves["dn"], mid, cfg.leaf_limit, cfg.band,
                                                   report)
                if report is not None:
                    report.update(split_seconds=time.perf_counter() - t0, split_ranks=world)
                out[0] = (summary.score, tuple(summary.start), tuple(summary.end),
                          tuple(path.start), path.ops.tobytes())
            dist.broadcast_object_list(out, src=glob(0), group=group)
        finally:
            dist.barrier(group=group)
            if ext_out:
                ctx.lib.swb_ipc_close(ctx.ptr, ext_out[0])
                ctx.lib.swb_ipc_close(ctx.ptr, ext_out[1])
            if not best:
                ctx.lib.swb_ipc_close(ctx.ptr, shared_best)
            dist.barrier(group=group)
            if inbound:
                inbound.free()
            if best:
                best.free()
    sc, st, en, pst, ops = out[0]
    if sc == 0:
        return AlignmentSummary.empty(), AlignmentPath.empty()
    return (AlignmentSummary(sc, Coord(*st), Coord(*en)),
            AlignmentPath(Coord(*pst), np.frombuffer(ops, dtype=np.uint8).copy()))


# -- both strands (§3: "four GPU cards in the case of aligning both
#    strands") ------------------------------------------------------------------

def reverse_complement_codes(codes, alphabet):
    """Reverse complement of DNA codes over "ACGT" (+ the wildcard 'N', which
    is its own complement)."""
    import numpy as np
    if alphabet.symbols[:4] != "ACGT" or len(alphabet) > 5:
        raise ValueError("both-strand alignment needs a DNA alphabet (ACGT, optionally N)")
    comp = np.array([3, 2, 1, 0, 4], dtype=np.uint8)
    return comp[np.asarray(codes, dtype=np.uint8)[::-1]]


def strand_groups(world: int) -> tuple[list[int], list[int]]:
    """Ranks aligning the forward and the reverse-complement strand."""
    if world < 2:
        raise ValueError("both strands across GPUs need at least 2 ranks")
    half = world // 2
    return list(range(half)), list(range(half, world))


def align_both_strands(seq1, seq2, scheme, config=None):
    """seq1 against seq2 and against the reverse complement of seq2 (one GPU,
    one after the other).  Returns {"+": (summary, path), "-": (summary,
    path)}; the "-" coordinates index the reverse-complemented seq2."""
    from .model import Sequence
    from .pipeline import align
    rc = Sequence.from_codes(seq2.id + "_rc", reverse_complement_codes(seq2.codes, scheme.alphabet),
                             scheme.alphabet)
    return {"+": align(seq1, seq2, scheme, config), "-": align(seq1, rc, scheme, config)}


def align_both_strands_distributed(seq1, seq2, scheme, config=None):
    """Both strands on all GPUs of a torch.distributed job: ranks [0, G/2)
    align the forward strand, [G/2, G) the reverse complement, each half with
    the Figure-1 split across its own two GPU groups when it has >= 2 ranks
    (split_align_distributed on a sub-group; 4 GPUs = the paper's four-card
    case), else on its one GPU.  Every rank returns the same
    {"+": (summary, path), "-": (summary, path)}."""
    import os

    import torch.distributed as dist

    from .engine import get_context
    from .model import Sequence
    from .pipeline import AlignConfig, align

    cfg = config or AlignConfig(split=2)
    rank, world = dist.get_rank(), dist.get_world_size()
    if world < 2:
        return align_both_strands(seq1, seq2, scheme, cfg)
    fwd, rev = strand_groups(world)
    groups = [dist.new_group(fwd), dist.new_group(rev)]  # every rank creates both
    mine = 0 if rank in fwd else 1
    ranks = fwd if mine == 0 else rev
    s2 = seq2 if mine == 0 else Sequence.from_codes(
        seq2.id + "_rc", reverse_complement_codes(seq2.codes, scheme.alphabet), scheme.alphabet)
    local = int(os.environ.get("LOCAL_RANK", cfg.device))
    get_context(local)
    if len(ranks) >= 2:
        res = split_align_distributed(seq1, s2, scheme, AlignConfig(
            leaf_limit=cfg.leaf_limit, band=cfg.band, split=2, device=local), group=groups[mine])
    else:
        res = align(seq1, s2, scheme, AlignConfig(leaf_limit=cfg.leaf_limit, band=cfg.band,
                                                  split=cfg.split, device=local))
    out = [None] * world
    dist.all_gather_object(out, (mine, (res[0].score, tuple(res[0].start), tuple(res[0].end),
                                        tuple(res[1].start), res[1].ops.tobytes())))
    return {("+" if m == 0 else "-"): _unpack(r) for m, r in (out[fwd[0]], out[rev[0]])}


def _unpack(r):
    import numpy as np
    from .model import AlignmentPath, AlignmentSummary, Coord
    sc, st, en, pst, ops = r
    if sc == 0:
        return AlignmentSummary.empty(), AlignmentPath.empty()
    return (AlignmentSummary(sc, Coord(*st), Coord(*en)),
            AlignmentPath(Coord(*pst), np.frombuffer(ops, dtype=np.uint8).copy()))


class _DeviceRows:
    """__cuda_array_interface__ view of int32 device memory (a tile-map slice)
    so that torch / NCCL can move it without a copy."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i4",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def map_row_tiles(slab: Slab, tile_rows: int = 1024) -> tuple[int, int]:
    # tile_rows: 2 ** ctx.get_option("map_tile_log2") of the maps in use
    """Forward-map row tiles [lo, hi) a slab's pass writes (slabs are cut in
    multiples of 1024 rows, so neighbouring slabs never share a tile row)."""
    return slab.row0 // tile_rows, -(-slab.row1 // tile_rows)


def align_distributed(seq1, seq2, scheme, config=None, report: dict | None = None):
    """Full alignment on all GPUs of a torch.distributed job (one process per
    GPU, NCCL): the phase-1 score pass runs as row slabs with the boundary rows
    streamed over NVLink peer memory; the per-slab bests merge
    with the reference's tie rule; each GPU's slab of the forward tile map
    (§3.6) is gathered into rank 0 over NCCL, and rank 0 runs phases 2 and 3
    (chains along the path, §7) with the whole map.  Every rank returns the
    same (summary, path), identical to pipeline.align() on one GPU."""
    import os

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import phase1
    from .engine import Session, get_context
    from .model import AlignmentPath, AlignmentSummary, Coord, validate_scheme
    from .pipeline import AlignConfig, finish
    import time

    cfg = config or AlignConfig()
    if cfg.split != 1:
        raise ValueError("align_distributed runs split=1 (the slab pipeline replaces split=2)")
    if len(seq1) < 1 or len(seq2) < 1:
        raise ValueError("alignment inputs must be non-empty")
    scheme = validate_scheme(scheme)
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", cfg.device))
    torch.cuda.set_device(local)
    ctx = get_context(local)
    t0 = time.perf_counter()
    with Session(ctx, seq1.codes, seq2.codes, scheme) as S:
        S.reset_bounds()
        slabs = slab_partition(S.n1, world, SLAB_STRIP_ROWS)
        me = slabs[rank]
        # a small pass leaves trailing ranks with an empty slab: they idle
        inbound = Boundary(ctx, S.n2) if rank > 0 and me.rows > 0 else None
        best = Boundary(ctx, 1) if rank == 0 else None  # shared running best (rank 0's memory)
        handles = [None] * world
        dist.all_gather_object(handles, (inbound.export() if inbound else None,
                                         ipc_export(ctx, best.progress) if best else None))
        ext_out = None
        if rank + 1 < world and slabs[rank + 1].rows > 0:
            hb, hp = handles[rank + 1][0]
            ext_out = (ipc_import(ctx, hb), ipc_import(ctx, hp))
        ext_in = (inbound.buf, inbound.progress) if inbound else None
        shared_best = best.progress if best else ipc_import(ctx, handles[0][1])
        try:
            dist.barrier()
            mine = (0, -1, -1)
            if me.rows > 0:
                if world > 1:
                    ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
                try:
                    spec = slab_spec(me, S.n1, S.n2, ext_in, ext_out, cfg.prune, shared_best)
                    spec["bound_write"] = 1 if S.bounds else 0
                    res = S.run([spec])[0]
                    mine = (res.best_score, res.best_i, res.best_j)
                finally:
                    ctx.set_option("rows_per_lane", 0)
            bests = [None] * world
            dist.all_gather_object(bests, mine)
            score, bi, bj = merge_best([tuple(b) for b in bests], TRACK_MIN)
            scored = (phase1.ScoredEndpoint(score, Coord(bi + 1, bj + 1)) if score > 0
                      else phase1.ScoredEndpoint(0, Coord(0, 0)))
            # assemble the forward tile map on rank 0 (row tiles are disjoint)
            if S.bounds and world > 1:
                ptr, n, nc = ctx.bounds_device(1)
                full = torch.as_tensor(_DeviceRows(ptr, n), device=f"cuda:{local}")
                tile_rows = 1 << ctx.get_option("map_tile_log2")
                for g in range(1, world):
                    lo, hi = map_row_tiles(slabs[g], tile_rows)
                    if hi <= lo or slabs[g].rows == 0:
                        continue
                    part = full[lo * nc:hi * nc]
                    if rank == g:
                        dist.send(part, dst=0)
                    elif rank == 0:
                        dist.recv(part, src=g)
                torch.cuda.synchronize()
            out = [None]
            if rank == 0:
                summary, path = finish(S, scored, cfg, report, t0)
                out[0] = (summary.score, tuple(summary.start), tuple(summary.end),
                          tuple(path.start), path.ops.tobytes())
            dist.broadcast_object_list(out, src=0)
        finally:
            dist.barrier()
            if ext_out:
                ctx.lib.swb_ipc_close(ctx.ptr, ext_out[0])
                ctx.lib.swb_ipc_close(ctx.ptr, ext_out[1])
            if not best:
                ctx.lib.swb_ipc_close(ctx.ptr, shared_best)
            dist.barrier()
            if inbound:
                inbound.free()
            if best:
                best.free()
    sc, st, en, pst, ops = out[0]
    if sc == 0:
        return AlignmentSummary.empty(), AlignmentPath.empty()
    return (AlignmentSummary(sc, Coord(*st), Coord(*en)),
            AlignmentPath(Coord(*pst), np.frombuffer(ops, dtype=np.uint8).copy()))
