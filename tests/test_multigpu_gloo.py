"""World-size-2 gloo test of the multi-GPU row-slab decomposition (CPU).

Each rank runs its row slab of a pass with the CPU oracle engine; rank g
receives the bottom DP row (H, F) of slab g-1 as its top border (the NVLink
handoff of DESIGN.md §6), then the per-slab bests are gathered and merged with
multigpu.merge_best.  The result must equal the single pass exactly, for
every border family and tracking mode the path uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1304_5966_b200.multigpu import merge_best, slab_partition

CASES = [("local", True, 1), ("restricted", False, 2), ("free", False, 0), ("continue", False, 1),
         ("charge", False, 2)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(seed=9):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from helpers import mutate_codes, random_codes
    rng = np.random.default_rng(seed)
    a = random_codes(rng, 2600)
    b = mutate_codes(rng, a, 0.12)[:2300]
    return a, b


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    a, b = _inputs()
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    slabs = slab_partition(a.size, world, strip_rows=512)
    me = slabs[rank]
    results = {}
    for border, clamp, track in CASES:
        top = None
        if rank > 0:
            buf = torch.empty(2, b.size + 1, dtype=torch.int64)
            dist.recv(buf, src=rank - 1)
            top = (buf[0].numpy(), buf[1].numpy())
        out = oracle.run_wavefront(a[me.row0:me.row1], b, osch, border, clamp, track, top=top,
                                   row_offset=me.row0, threads=1)
        if rank + 1 < world:
            dist.send(torch.from_numpy(np.stack([out.final_h, out.final_f])), dst=rank + 1)
        bi = out.bi + me.row0 if out.bi >= 0 else -1
        mine = torch.tensor([out.best, bi, out.bj], dtype=torch.int64)
        gathered = [torch.empty(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, mine)
        merged = merge_best([tuple(int(x) for x in t.tolist()) for t in gathered], track)
        if rank == world - 1:
            results[border] = (merged, out.final_h.copy(), out.final_f.copy())
    if rank == world - 1:
        out_q.put(results)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_slab_split_matches_single_pass(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = _inputs()
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    for border, clamp, track in CASES:
        full = oracle.run_wavefront(a, b, osch, border, clamp, track, threads=1)
        merged, fh, ff = results[border]
        if track != 0:
            assert merged == (full.best, full.bi, full.bj), border
        assert np.array_equal(fh, full.final_h), border
        assert np.array_equal(ff, full.final_f), border


def test_slab_partition_shapes():
    s = slab_partition(10_000, 4, 1024)
    assert s[0].row0 == 0 and s[-1].row1 == 10_000
    assert all(x.row1 == y.row0 for x, y in zip(s, s[1:]))
    assert all(x.row0 % 1024 == 0 for x in s)
    s2 = slab_partition(3, 8, 1024)
    assert sum(x.rows for x in s2) == 3


def test_merge_best_tie_rules():
    assert merge_best([(5, 10, 3), (5, 2, 9), (4, 0, 0)], 1) == (5, 2, 9)
    assert merge_best([(5, 10, 3), (5, 2, 9)], 2) == (5, 10, 3)
    assert merge_best([(0, 1, 1), (-3, 2, 2)], 1) == (0, -1, -1)


def _split_worker(rank, world, port, out_q):
    """One rank of the Figure-1 split (multigpu.split_plan / half_slab_spec)
    on the CPU oracle: its slab of its half, the top border from the previous
    slab of its group, then rank 0 gathers the per-slab bests and the two
    final rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1304_5966_b200.multigpu import half_slab_spec, merge_half, split_plan
    a, b = _inputs(seed=21)
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    plan = split_plan(a.size, world, strip_rows=256)
    me = plan[rank]
    spec = half_slab_spec(me, a.size, b.size, None, None, 0)
    off, ln, rev = spec["rows"]
    c1 = a[off:off + ln][::-1] if rev else a[off:off + ln]
    c2 = b[::-1] if spec["cols"][2] else b
    fed = rank > 0 and plan[rank - 1].half == me.half
    feeds = rank + 1 < world and plan[rank + 1].half == me.half
    top = None
    if fed:
        buf = torch.empty(2, b.size + 1, dtype=torch.int64)
        dist.recv(buf, src=rank - 1)
        top = (buf[0].numpy(), buf[1].numpy())
    out = oracle.run_wavefront(c1, c2, osch, "local", True, 1, top=top,
                               row_offset=me.slab.row0, threads=1)
    if feeds:
        dist.send(torch.from_numpy(np.stack([out.final_h, out.final_f])), dst=rank + 1)
    bi = out.bi + me.slab.row0 if out.bi >= 0 else -1
    parts = [None] * world
    dist.all_gather_object(parts, (me.half, (out.best, bi, out.bj, out.cells),
                                   (out.final_h.copy(), out.final_f.copy()) if me.last else None))
    if rank == 0:
        res = {}
        for half in ("up", "dn"):
            ps = [p[1] for p in parts if p[0] == half]
            fin = [p[2] for p in parts if p[0] == half and p[2] is not None][0]
            h = merge_half(ps, fin)
            res[half] = ((h.best_score, h.best_i, h.best_j), h.final_row_h, h.final_row_f)
        out_q.put(res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_figure1_split_groups_match_single_halves(world):
    """The Figure-1 split across GPU groups reproduces split.split_align's two
    half passes (reference split.py:103-122): same bests, same final rows."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = _inputs(seed=21)
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    mid = a.size // 2
    up = oracle.run_wavefront(a[:mid], b, osch, "local", True, 1, threads=1)
    dn = oracle.run_wavefront(a[mid:][::-1], b[::-1], osch, "local", True, 1, threads=1)
    for half, ref in (("up", up), ("dn", dn)):
        best, fh, ff = got[half]
        assert best == (ref.best, ref.bi, ref.bj), half
        assert np.array_equal(fh, ref.final_h) and np.array_equal(ff, ref.final_f), half


def test_split_plan_shapes():
    from paper_1304_5966_b200.multigpu import split_groups, split_plan
    assert split_groups(2) == ([0], [1]) and split_groups(8) == ([0, 1, 2, 3], [4, 5, 6, 7])
    plan = split_plan(10_000, 4, strip_rows=1024)
    assert [hs.half for hs in plan] == ["up", "up", "dn", "dn"]
    assert plan[0].slab.row0 == 0 and plan[1].slab.row1 == 5_000
    assert plan[2].slab.row0 == 0 and plan[3].slab.row1 == 5_000
    assert [hs.last for hs in plan] == [False, True, False, True]
    small = split_plan(900, 8, strip_rows=1024)  # fewer strips than ranks: trailing ranks idle
    assert [hs.slab.rows for hs in small] == [450, 0, 0, 0, 450, 0, 0, 0]
    assert [hs.last for hs in small] == [True, False, False, False, True, False, False, False]


def test_reverse_complement_and_strand_groups():
    from paper_1304_5966_b200 import Alphabet
    from paper_1304_5966_b200.multigpu import reverse_complement_codes, strand_groups
    codes = np.array([0, 1, 2, 3, 4, 0], dtype=np.uint8)  # A C G T N A
    assert reverse_complement_codes(codes, Alphabet.dna()).tolist() == [3, 4, 0, 1, 2, 3]
    assert strand_groups(4) == ([0, 1], [2, 3]) and strand_groups(2) == ([0], [1])
    with pytest.raises(ValueError):
        reverse_complement_codes(codes, Alphabet.protein())
