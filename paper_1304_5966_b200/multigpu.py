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
    possible (the last slab takes the ragged remainder).  Every rank gets at
    least one row when n1 >= world."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if n1 < 1:
        raise ValueError("cannot partition an empty pass")
    strips = -(-n1 // strip_rows)
    bounds = []
    for g in range(world + 1):
        k = (strips * g) // world
        bounds.append(min(n1, k * strip_rows))
    if strips < world:  # fewer strips than ranks: split rows directly
        bounds = [(n1 * g) // world for g in range(world + 1)]
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


class _DeviceRows:
    """__cuda_array_interface__ view of int32 device memory (a tile-map slice)
    so that torch / NCCL can move it without a copy."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i4",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def map_row_tiles(slab: Slab, tile_rows: int = 1024) -> tuple[int, int]:
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
        inbound = Boundary(ctx, S.n2) if rank > 0 else None
        best = Boundary(ctx, 1) if rank == 0 else None  # shared running best (rank 0's memory)
        handles = [None] * world
        dist.all_gather_object(handles, (inbound.export() if inbound else None,
                                         ipc_export(ctx, best.progress) if best else None))
        ext_out = None
        if rank + 1 < world:
            hb, hp = handles[rank + 1][0]
            ext_out = (ipc_import(ctx, hb), ipc_import(ctx, hp))
        ext_in = (inbound.buf, inbound.progress) if inbound else None
        shared_best = best.progress if best else ipc_import(ctx, handles[0][1])
        try:
            dist.barrier()
            if world > 1:
                ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
            try:
                spec = slab_spec(me, S.n1, S.n2, ext_in, ext_out, cfg.prune, shared_best)
                spec["bound_write"] = 1 if S.bounds else 0
                res = S.run([spec])[0]
            finally:
                ctx.set_option("rows_per_lane", 0)
            bests = [None] * world
            dist.all_gather_object(bests, (res.best_score, res.best_i, res.best_j))
            score, bi, bj = merge_best([tuple(b) for b in bests], TRACK_MIN)
            scored = (phase1.ScoredEndpoint(score, Coord(bi + 1, bj + 1)) if score > 0
                      else phase1.ScoredEndpoint(0, Coord(0, 0)))
            # assemble the forward tile map on rank 0 (row tiles are disjoint)
            if S.bounds and world > 1:
                ptr, n, nc = ctx.bounds_device(1)
                full = torch.as_tensor(_DeviceRows(ptr, n), device=f"cuda:{local}")
                for g in range(1, world):
                    lo, hi = map_row_tiles(slabs[g])
                    if hi <= lo:
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
