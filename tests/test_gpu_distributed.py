"""multigpu.align_distributed (slab phase 1 + tile-map gather + phases 2-3 on
rank 0) under torchrun equals pipeline.align.  One GPU here: world size 1
covers the code path end to end; the N > 1 handoff semantics are covered by
test_gpu_multigpu.py (sequential slabs), test_gpu_ipc.py and the concurrent
one-launch emulation of test_gpu_scale_golden.py.  On a box with two or more
GPUs the world-size-2 tests run the real cross-GPU handoff concurrently,
repeated to catch ordering races."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _torchrun(nproc, *args, timeout=600):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           "--nproc-per-node", str(nproc), "--master-addr", "127.0.0.1",
                           "--master-port", str(port), *args],
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.gpu
def test_align_distributed_world1():
    out = _torchrun(1, str(ROOT / "tools" / "dist_align_check.py"), "3000,40000,300000")
    assert out.returncode == 0, out.stderr[-2000:]
    assert "DIST OK" in out.stdout, out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("rep", range(3))
def test_align_distributed_world2(rep):
    """Both ranks' slabs run at once, the boundary row crossing GPUs through
    peer memory; sizes include n1 < 2 x 1024 (a trailing empty slab)."""
    out = _torchrun(2, str(ROOT / "tools" / "dist_align_check.py"), "1500,40000,300000")
    assert out.returncode == 0, out.stderr[-2000:]
    assert "DIST OK" in out.stdout, out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
def test_bench_two_gpus():
    """bench.py under torchrun at N = 2: the C4 strong-scaling pass with the
    shared running best; rank 0 prints one JSON line with parity."""
    import json
    out = _torchrun(2, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
                    "--no-cpu", "--no-align", timeout=1200)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
