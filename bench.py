"""Benchmark of the SW# hot path on B200 (contract: one JSON line on rank 0).

Default (N=1): BASELINE config C2 — synthetic 1 Mbp x 1 Mbp homologous DNA pair
(mutate 10 %, seed 1002), match +1 / mismatch -3 / gap 5 + 2k, forward local
score pass with endpoint (score_only).  A step is one full score pass.

  value     GCUPS = n1*n2 / device time, inputs resident in HBM, CUDA events on
            the launching stream around each step, L2 flushed (512 MiB write)
            between steps outside the timed region.
  e2e       the same metric through the public API score_only(Sequence, ...)
            with host buffers: H2D of both sequences, device reverse copies,
            the pass and the D2H of the result inside the timed region.
  roofline  integer/DPX issue roofline of the pass kernel: ALU-pipe instructions
            per executed cell (packed 16x2 kernel: 5 per cell pair = 2.5; 32-bit
            kernel: 6) against the chip DPX issue rate measured
            live by swb_measure_int_peak.
  cpu_baseline  the CPU oracle port (oracle/, C + OpenMP block wavefront, a
            restatement of the reference engine) on a bounded window of the
            same pair, all host threads.

  align_e2e  end-to-end full alignments through `align` (host buffers, phases
            1-3): C1 10 kbp on the GPU and on the CPU port with a byte-equality
            check, C3 5 Mbp on the GPU (CPU time extrapolated, lower bound).

`--impl reference` times that CPU port alone on the same metric (rank 0 only).
Multi-GPU (torchrun, N>1): ONE alignment of an (N x 1 Mbp) x 1 Mbp pair split
into row slabs, one per GPU, the slab boundary rows streamed GPU to GPU over
NVLink through CUDA-IPC peer memory (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT = 1_000_000
# ALU-pipe instructions per cell of the recurrence:
#   lane32     PRMT + 4 VIADDMNMX + running max                       = 6
#   packed16x2 PRMT + VIMNMX3 + 3 VIADDMNMX per two cells (S16x2)   = 2.5
OPS_PER_CELL = {"lane32": 6.0, "packed16x2": 2.5}
DTYPE = {"lane32": "int32", "packed16x2": "int16x2"}
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}


def synthetic_pair(n: int, seed: int = 1002, homologous: bool = True):
    """Uniform ACGT target; query = mutate(target, 0.10) (subst/ins/del each
    at rate/3) or an independent draw."""
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 4, size=n, dtype=np.uint8)
    if not homologous:
        return a, rng.integers(0, 4, size=n, dtype=np.uint8)
    r = rng.random(n)
    rate = 0.10
    sub = r < rate / 3
    ins = (r >= rate / 3) & (r < 2 * rate / 3)
    dele = (r >= 2 * rate / 3) & (r < rate)
    out = a.copy()
    out[sub] = rng.integers(0, 4, size=int(sub.sum()), dtype=np.uint8)
    keep = ~dele
    reps = np.where(ins, 2, 1)[keep]
    b = np.repeat(out[keep], reps)
    pos = np.cumsum(reps) - 1
    ip = pos[ins[keep]]
    b[ip] = rng.integers(0, 4, size=ip.size, dtype=np.uint8)
    return a, b


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
               "utilization.gpu,clocks_event_reasons.active", "--format=csv,noheader,nounits",
               "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 4:
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]), float(parts[2]),
                                             int(parts[3], 16)))
                    except ValueError:
                        pass

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        load = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for s in load:
            for bit, name in THROTTLE_BITS.items():
                if s[3] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in load),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons),
                "samples": len(load)}


def cpu_window(a, b, target_s: float = 15.0):
    """Time the oracle score pass (reference engine restated in C, OpenMP over
    the blocks of each anti-diagonal, 512x512 blocks, pruning on) on a square
    window of the same pair sized for ~target_s seconds."""
    import oracle
    from oracle.pipeline import max_threads
    osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
    threads = max_threads()
    probe = min(20_000, a.size)
    t0 = time.perf_counter()
    oracle.score_only(a[:probe], b[:probe], osch, threads=threads)
    rate = probe * probe / max(time.perf_counter() - t0, 1e-3)
    w = int(min(a.size, b.size, max(probe, (rate * target_s) ** 0.5)))
    t0 = time.perf_counter()
    score, end, _ = oracle.score_only(a[:w], b[:w], osch, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": w * w / dt / 1e9, "unit": "GCUPS", "cores": threads, "kind": "port",
            "sample": f"score pass on the first {w} x {w} residues of the same pair "
                      f"({dt:.1f} s, score {score})"}, w, dt


def align_e2e(swb, scheme, cpu_gcups, with_cpu: bool):
    """End-to-end alignment time through the public API (`align`, host
    buffers, phases 1-3), BASELINE configs C1 and C3.  C1 is also run on the
    CPU port of the reference (oracle/, all host threads) and compared
    byte-for-byte; C3 on the CPU is extrapolated from the measured CPU score-pass
    rate (a lower bound: phase 1 alone)."""
    out = {}
    a, b = synthetic_pair(10_000, seed=1001)
    s1 = swb.Sequence.from_codes("target", a, scheme.alphabet)
    s2 = swb.Sequence.from_codes("query", b, scheme.alphabet)
    swb.align(s1, s2, scheme)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        summ, path = swb.align(s1, s2, scheme)
        ts.append(time.perf_counter() - t0)
    c1 = {"pair": "10 kbp x 10 kbp, mutate 10%, seed 1001", "gpu_s": min(ts), "score": summ.score,
          "start": list(summ.start), "end": list(summ.end)}
    if with_cpu:
        import oracle
        from oracle.pipeline import max_threads
        osch = oracle.OracleScheme.match_mismatch(4, 1, -3, 5, 2)
        t0 = time.perf_counter()
        ref = oracle.align(a, b, osch, threads=max_threads())
        c1.update(cpu_s=time.perf_counter() - t0, cpu_cores=max_threads(), cpu_kind="port",
                  identical=bool(ref[0] == summ.score and tuple(ref[1]) == tuple(summ.start)
                                 and tuple(ref[2]) == tuple(summ.end)
                                 and np.array_equal(ref[3], path.ops)))
    out["C1"] = c1
    a, b = synthetic_pair(5_000_000, seed=1003)
    s1 = swb.Sequence.from_codes("target", a, scheme.alphabet)
    s2 = swb.Sequence.from_codes("query", b, scheme.alphabet)
    t0 = time.perf_counter()
    swb.align(s1, s2, scheme)
    first = time.perf_counter() - t0  # includes lazy loading of the phase-2/3 kernels
    rep = {}
    t0 = time.perf_counter()
    summ, path = swb.align(s1, s2, scheme, report=rep)
    dt = time.perf_counter() - t0
    c3 = {"pair": "5 Mbp x 5 Mbp, mutate 10%, seed 1003", "gpu_s": dt, "gpu_s_first_call": first,
          "phase_s": [round(x, 3) for x in rep.get("phase_seconds", [])], "score": summ.score,
          "start": list(summ.start), "end": list(summ.end), "path_ops": int(path.ops.size)}
    if cpu_gcups:
        c3["cpu_s_extrapolated_lower_bound"] = a.size * b.size / (cpu_gcups * 1e9)
    out["C3"] = c3
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU port of the reference path (oracle/)."""
    if rank != 0:
        return 0
    a, b = synthetic_pair(args.n, homologous=not args.unrelated)
    vals, secs = [], []
    base = None
    for it in range(args.warmup + args.steps):
        cb, w, dt = cpu_window(a, b, target_s=args.cpu_seconds)
        if it >= args.warmup:
            vals.append(cb["value"])
            secs.append(dt)
            base = cb
    value = statistics.mean(vals)
    line = {
        "metric": "GCUPS (score pass, full-matrix cells / time)", "value": value, "unit": "GCUPS",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"C2 window: score pass on a square window of the "
                               f"{args.n} x {args.n} homologous pair", "n1": args.n, "n2": args.n,
                   "scheme": "match +1 / mismatch -3 / gap 5+2k"},
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": base["cores"], "kind": "port",
                         "sample": base["sample"]},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_multi(args, rank, world, local, dist):
    """N GPUs, one alignment: the target is N x n residues (weak scaling, n x n
    cells per GPU), split into row slabs; GPU g streams the bottom DP row of its
    slab into GPU g+1's boundary buffer through CUDA-IPC peer memory over
    NVLink.  Time = max over ranks of the CUDA-event time."""
    import torch
    import paper_1304_5966_b200 as swb
    from paper_1304_5966_b200.engine import Session, get_context
    from paper_1304_5966_b200.multigpu import (SLAB_ROWS_PER_LANE, SLAB_STRIP_ROWS, Boundary,
                                              ipc_import, merge_best, slab_partition, slab_spec)
    a, b = synthetic_pair(args.n * world, seed=1002, homologous=not args.unrelated)
    b = b[:args.n]
    scheme = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
    ctx = get_context(local)
    peak = ctx.measure_int_peak()
    ctx.set_option("rows_per_lane", SLAB_ROWS_PER_LANE)
    slabs = slab_partition(a.size, world, SLAB_STRIP_ROWS)
    me = slabs[rank]
    inbound = Boundary(ctx, b.size) if rank > 0 else None
    handles = [None] * world
    dist.all_gather_object(handles, inbound.export() if inbound else None)
    ext_out = None
    if rank + 1 < world:
        hb, hp = handles[rank + 1]
        ext_out = (ipc_import(ctx, hb), ipc_import(ctx, hp))
    ext_in = (inbound.buf, inbound.progress) if inbound else None

    def step(S):
        if inbound:
            inbound.reset()
        torch.cuda.synchronize()
        dist.barrier()
        ctx.timer_start()
        r = S.run([slab_spec(me, S.n1, S.n2, ext_in, ext_out)])[0]
        return r, ctx.timer_stop()

    with Session(ctx, a, b, scheme) as S:
        for _ in range(args.warmup):
            step(S)
        times, res = [], None
        with ClockSampler(local) as clocks:
            l0 = ctx.launch_count
            for _ in range(args.steps):
                res, ms = step(S)
                times.append(ms)
            launches = ctx.launch_count - l0
        # end to end: host codes -> device (Session upload) + pass + result D2H
        e2e_ms = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            with Session(ctx, a, b, scheme) as S2:
                step(S2)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    t = torch.tensor([sum(times), sum(e2e_ms)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t[0].item())
    e2e_total = float(t[1].item())
    bests = [None] * world
    dist.all_gather_object(bests, (res.best_score, res.best_i, res.best_j))
    cells_all = [None] * world
    dist.all_gather_object(cells_all, res.cells_executed)
    merged = merge_best([tuple(x) for x in bests], 1)
    cells = a.size * b.size
    value = cells * args.steps / (total_ms * 1e-3) / 1e9
    if rank == 0:
        exec_cells = sum(cells_all)
        achieved = exec_cells * OPS_PER_CELL[res.kernel] / (total_ms / args.steps * 1e-3) / 1e12
        line = {
            "metric": "GCUPS (score pass, full-matrix cells / time)", "value": value,
            "unit": "GCUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE[res.kernel], "data": "synthetic",
            "config": {"workload": f"one alignment: {a.size} x {b.size} homologous pair "
                                   f"({args.n} x {args.n} cells per GPU), score + endpoint pass",
                       "n1": int(a.size), "n2": int(b.size), "prune": True,
                       "parallelism": f"{world} GPUs, row slabs, boundary rows streamed over "
                                      "NVLink (CUDA IPC peer stores)",
                       "l2": "inputs resident; boundary rows live in L2 (see DESIGN.md §6)",
                       "score": merged[0], "end": [merged[1] + 1, merged[2] + 1]},
            "e2e": {"value": cells * args.steps / (e2e_total * 1e-3) / 1e9, "unit": "GCUPS",
                    "h2d_bytes_per_step": int(a.size + b.size),
                    "d2h_bytes_per_step": int(16 * (me.rows // SLAB_STRIP_ROWS + 1) + 40)},
            "gpu_launches": launches, "clocks": clocks.summary(),
            "roofline": {"bound": "int", "achieved": achieved,
                         "peak": world * peak["viaddmnmx"] / 1e12, "unit": "Tops/s",
                         "frac": achieved / (world * peak["viaddmnmx"] / 1e12), "traffic": None},
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if ext_out:
        ctx.lib.swb_ipc_close(ctx.ptr, ext_out[0])
        ctx.lib.swb_ipc_close(ctx.ptr, ext_out[1])
    dist.barrier()
    if inbound:
        inbound.free()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--unrelated", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-align", action="store_true",
                    help="skip the end-to-end alignment section (C1 vs CPU port, C3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "native" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl" if args.impl == "native" else "gloo")
        dist = tdist
    if args.impl == "reference":
        rc = run_reference(args, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return rc
    if world > 1:
        rc = run_multi(args, rank, world, local, dist)
        dist.destroy_process_group()
        return rc

    import paper_1304_5966_b200 as swb
    from paper_1304_5966_b200.engine import TRACK_MIN, Session, get_context

    a, b = synthetic_pair(args.n, seed=1002 + rank, homologous=not args.unrelated)
    scheme = swb.ScoringScheme.match_mismatch(swb.Alphabet.dna(), 1, -3, 5, 2)
    ctx = get_context(0 if world == 1 else local)
    peak = ctx.measure_int_peak()
    cells = a.size * b.size

    def barrier():
        if dist is not None:
            import torch
            torch.cuda.synchronize()
            dist.barrier()

    # -- device-resident value -------------------------------------------------
    step_ms, res = [], None
    launches = 0
    with Session(ctx, a, b, scheme) as S:
        spec = [dict(rows=(0, S.n1, 0), cols=(0, S.n2, 0), border="local", clamp=True,
                     track=TRACK_MIN, prune=True)]
        for _ in range(args.warmup):
            S.run(spec)
        barrier()
        with ClockSampler(local) as clocks:
            l0 = ctx.launch_count
            for _ in range(args.steps):
                ctx.flush_l2()
                ctx.timer_start()
                res = S.run(spec)[0]
                step_ms.append(ctx.timer_stop())
            launches = ctx.launch_count - l0
        barrier()
    kernel_ms = res.kernel_ms
    total_ms = sum(step_ms)
    if dist is not None:
        import torch
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * cells * args.steps / (total_ms * 1e-3) / 1e9

    # -- end to end through the public API ----------------------------------------
    s1 = swb.Sequence.from_codes("target", a, scheme.alphabet)
    s2 = swb.Sequence.from_codes("query", b, scheme.alphabet)
    swb.score_only(s1, s2, scheme)
    barrier()
    e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r2 = swb.score_only(s1, s2, scheme)
        e_ms.append((time.perf_counter() - t0) * 1e3)
    barrier()
    e_total = sum(e_ms)
    if dist is not None:
        import torch
        t = torch.tensor([e_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_total = float(t.item())
    e2e = world * cells * args.steps / (e_total * 1e-3) / 1e9
    assert (r2.score, r2.end) == (res.best_score, (res.best_i + 1, res.best_j + 1))

    # -- roofline -------------------------------------------------------------------
    exec_cells = res.cells_executed
    opc = OPS_PER_CELL[res.kernel]
    achieved = exec_cells * opc / (kernel_ms * 1e-3) / 1e12
    peak_t = peak["viaddmnmx"] / 1e12
    strips = (a.size + 1023) // 1024
    roofline = {"bound": "int", "achieved": achieved, "peak": peak_t, "unit": "Tops/s",
                "frac": achieved / peak_t, "traffic": None,
                "peak_source": "live swb_measure_int_peak (VIADDMNMX issue rate, all SMs)",
                "ops_per_cell": opc, "kernel": res.kernel, "rows_per_lane": res.rows_per_lane,
                "cells_executed": exec_cells,
                "gcups_executed": exec_cells / (kernel_ms * 1e-3) / 1e9,
                "kernel_ms": kernel_ms, "pruned_fraction": res.pruned_blocks / max(1, res.total_blocks)}
    prof = ROOT / "profiles" / "r01_traffic.json"
    if prof.exists():
        try:
            roofline["traffic"] = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _, _ = cpu_window(a, b, target_s=args.cpu_seconds)
    align = None
    if rank == 0 and world == 1 and not args.no_align:
        align = align_e2e(swb, scheme, cpu["value"] if cpu else None, not args.no_cpu)

    if rank == 0:
        line = {
            "metric": "GCUPS (score pass, full-matrix cells / time)", "value": value,
            "unit": "GCUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE[res.kernel], "data": "synthetic",
            "config": {"workload": "C2: 1 Mbp x 1 Mbp homologous DNA pair (mutate 10%, seed 1002), "
                                   "score + endpoint forward pass" if args.n == N_DEFAULT and
                                   not args.unrelated else
                                   f"{a.size} x {b.size} {'unrelated' if args.unrelated else 'homologous'} pair, score pass",
                       "n1": int(a.size), "n2": int(b.size),
                       "scheme": "match +1 / mismatch -3 / gap 5+2k, default ACGT+N alphabet",
                       "prune": True, "l2": "flushed (512 MiB write) between timed steps",
                       "parallelism": "1 GPU" if world == 1 else f"{world} replicas (one pair per GPU)",
                       "score": res.best_score, "end": [res.best_i + 1, res.best_j + 1]},
            "e2e": {"value": e2e, "unit": "GCUPS", "h2d_bytes_per_step": int(a.size + b.size),
                    "d2h_bytes_per_step": int(16 * strips + 40)},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "align_e2e": align,
            "int_peak": {k: v for k, v in peak.items() if k != "ms_last"},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
