"""CUDA-IPC boundary handoff between two processes on one GPU.

Rank 1 allocates its inbound boundary row and exports it; rank 0 imports the
peer pointers and runs the upper row slab, publishing its bottom row through
them; only after rank 0's kernel has finished (gloo barrier) does rank 1 run the
lower slab consuming it.  The kernels never wait on each other concurrently
(one GPU), but the full cross-process path — IPC handles, sys-scope release /
acquire, peer stores — is exercised, and the merged result must equal the
single pass."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    sys.path.insert(0, str(here))
    sys.path.insert(0, str(here.parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from helpers import dna_scheme, mutate_codes, random_codes
    from paper_1304_5966_b200.engine import Session, get_context
    from paper_1304_5966_b200.multigpu import (SLAB_ROWS_PER_LANE, SLAB_STRIP_ROWS, Boundary,
                                              ipc_import, merge_best, slab_partition, slab_spec)
    rng = np.random.default_rng(31)
    a = random_codes(rng, 40_000)
    b = mutate_codes(rng, a, 0.1)[:35_000]
    scheme = dna_scheme()
    ctx = get_context(0)
    ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
    slabs = slab_partition(a.size, 2, SLAB_STRIP_ROWS)
    inbound = Boundary(ctx, b.size) if rank == 1 else None
    handles = [None, None]
    dist.all_gather_object(handles, inbound.export() if inbound else None)
    with Session(ctx, a, b, scheme) as S:
        if rank == 0:
            hb, hp = handles[1]
            ext_out = (ipc_import(ctx, hb), ipc_import(ctx, hp))
            r = S.run([slab_spec(slabs[0], S.n1, S.n2, None, ext_out)])[0]
            dist.barrier()  # slab 0 complete before slab 1 starts
            ctx.set_option("rows_per_lane", 0)
            single = S.run([dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local",
                                 clamp=True, track=1, prune=True)])[0]
        else:
            dist.barrier()
            r = S.run([slab_spec(slabs[1], S.n1, S.n2, (inbound.buf, inbound.progress), None)])[0]
            single = None
    got = [None, None]
    dist.all_gather_object(got, (r.best_score, r.best_i, r.best_j))
    if rank == 0:
        q.put((merge_best([tuple(x) for x in got], 1),
               (single.best_score, single.best_i, single.best_j)))
        ctx.lib.swb_ipc_close(ctx.ptr, ext_out[0])
        ctx.lib.swb_ipc_close(ctx.ptr, ext_out[1])
    dist.barrier()
    if inbound:
        inbound.free()
    dist.destroy_process_group()


def test_ipc_slab_handoff_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    merged, single = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert merged == single
