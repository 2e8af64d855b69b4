"""CPU oracle for the SW# hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference `wavealign` algorithm
(/root/reference/pkg/src/wavealign) on the CPU: C kernels in swb_oracle.c
(affine_block, run_wavefront, leaf_solve, the full-matrix oracle) and the
phase orchestration in pipeline.py.  It is the parity checker for the CUDA
path and the CPU baseline timed by bench.py.

Parity is pinned: tests/test_oracle_golden.py checks this oracle against
golden vectors produced by the real reference (tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py (CPU-baseline leg and
`--impl reference`) may import it.  The product package
paper_1304_5966_b200 never does.
"""
from .pipeline import (  # noqa: F401
    NEG_INF,
    OracleScheme,
    align,
    full_local_end,
    leaf_solve,
    run_wavefront,
    score_only,
)
