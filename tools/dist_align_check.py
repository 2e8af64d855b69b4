"""Run under torchrun: multigpu.align_distributed against pipeline.align,
multigpu.split_align_distributed against align(split=2) and
align_both_strands_distributed against align_both_strands on the same pairs;
prints one line per check and "DIST OK" when all match.
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P tools/dist_align_check.py [SIZES]"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch.distributed as dist
from bench import synthetic_pair
import paper_1304_5966_b200 as swb
from paper_1304_5966_b200.multigpu import (align_both_strands, align_both_strands_distributed,
                                          align_distributed, split_align_distributed)

dist.init_process_group("nccl")
rank = dist.get_rank()
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3000, 40000, 300000]
sc = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
ok = True
for n in sizes:
    a, b = synthetic_pair(n, seed=n)
    s1 = swb.Sequence.from_codes("a", a, sc.alphabet)
    s2 = swb.Sequence.from_codes("b", b, sc.alphabet)
    summ, path = align_distributed(s1, s2, sc)
    if rank == 0:
        ref, rpath = swb.align(s1, s2, sc)
        same = (summ == ref) and path.start == rpath.start and np.array_equal(path.ops, rpath.ops)
        ok &= bool(same)
        print(f"n={n} score={summ.score} start={tuple(summ.start)} end={tuple(summ.end)} same={same}", flush=True)
    summ2, path2 = split_align_distributed(s1, s2, sc)
    both = align_both_strands_distributed(s1, s2, sc)
    if rank == 0:
        ref2, rpath2 = swb.align(s1, s2, sc, swb.AlignConfig(split=2))
        same2 = (summ2 == ref2) and np.array_equal(path2.ops, rpath2.ops)
        want = align_both_strands(s1, s2, sc, swb.AlignConfig(split=2))
        same3 = all(both[k][0] == want[k][0] and np.array_equal(both[k][1].ops, want[k][1].ops)
                    for k in "+-")
        ok &= bool(same2 and same3)
        print(f"n={n} split2 same={same2} both-strands same={same3} "
              f"(+ {both['+'][0].score}, - {both['-'][0].score})", flush=True)
if rank == 0:
    print("DIST OK" if ok else "DIST MISMATCH", flush=True)
dist.destroy_process_group()
