"""multigpu.align_distributed (slab phase 1 + tile-map gather + phases 2-3 on
rank 0) under torchrun equals pipeline.align.  One GPU here: world size 1
covers the code path end to end; the N > 1 handoff semantics are covered by
test_gpu_multigpu.py (sequential slabs) and test_gpu_ipc.py."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_align_distributed_world1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), str(ROOT / "tools" / "dist_align_check.py"),
                          "3000,40000,300000"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "DIST OK" in out.stdout, out.stdout
