#!/usr/bin/env python
"""bench.py — block-MINRES iterations/s on B200 (driver contract).

A "step" is one bminres_solve call on the workload with a fixed iteration budget
(--iters, default 2000 banded iterations = 250 block steps at p = 8): the start block
(a0), then every row a1..a5 of the hot path once per block step.  The workload is
BASELINE.json configs[1] (config 2: 3-D 7-point Laplacian 64^3 shifted by -3, p = 8,
Gaussian B from seed 0), synthetic, fp64.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

`value`   = banded iterations of the solve / max-over-ranks device time (CUDA events).
`e2e`     = the same metric through the C ABI with HOST buffers (A, B in; X out).
`roofline`= the dominant kernel's algorithmic bytes per launch / its mean launch time
            (CUDA events around every launch inside the timed region) vs MEASURED_PEAKS.
`cpu_baseline` = the C oracle (tests' reference implementation) on a bounded sample.
With N > 1 (torchrun) the ranks run ONE solve of the workload with the rows partitioned over
them (halo exchange + allreduces over NCCL; strong scaling).  Testing
aids: BENCH_BACKEND=gloo + BENCH_COMM=gloo run the same path with the host-callback transport
(e.g. two ranks sharing one GPU).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic panel transfers per launch; K1 also streams CSR A
# algorithmic panel transfers per launch.  The fused M/X update moves 5 panels on average: it
# reads V_k, M_{k-2}, M_{k-1} and writes M_k every block, and reads + writes X every other block
# (X updates deferred in pairs); the standalone K4b moves 6.
# BASELINE.json's metric (the value is iterations/s; the achieved HBM GB/s against the roofline is
# reported in "roofline" / "step_roofline")
METRIC = "block-MINRES iterations/s and achieved HBM GB/s (fp64) vs roofline, 1/2/4/8 B200"
PHASE_BYTES_PANELS = {"spmm": 3, "spmm_fused": 8, "orth": 3, "update": 6,
                      # split mode (large panels): K1a reads V_k once (gathers) and writes AV; K1 then
                      # streams AV, V_k, V_{k-1} and writes W (+ the fused update)
                      "spmm_av": 2, "epilogue": 4, "epilogue_fused": 9}
PHASE_READS_A = {"spmm", "spmm_fused", "spmm_av"}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def problem(cfg):
    import synth
    key = cfg if cfg == "1c" else int(cfg)
    return synth.config(key)


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if os.environ.get("BENCH_BACKEND", "nccl") == "nccl" else "gloo")
    return world, rank, local


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_sample_iters(P, budget_s: float = 15.0) -> int:
    """Iterations of the bounded oracle sample: ~budget_s of one-thread CPU work, from the oracle's
    measured cost on config 2 (~0.8 ns per unit of nnz + 8 n p per iteration), 2 .. 400 (configs 4/5: the
    oracle's start block alone is tens of seconds)."""
    units = float(P.A.nnz) + 8.0 * P.n * P.p
    est = budget_s / (0.82e-9 * units)
    return int(max(2, min(400, est)))


def cpu_baseline(P, iters: int):
    """The oracle as it stands, one thread, on the first `iters` iterations of the workload."""
    import oracle
    oracle.lib()
    t0 = time.perf_counter()
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=iters, tau=P.tau, pool_size=1)
    dt = time.perf_counter() - t0
    return {"value": r.iterations / dt, "unit": "iterations/s", "cores": 1, "kind": "oracle",
            "sample": f"{P.name}: one oracle solve of {r.iterations} iterations (start block included), "
                      f"{dt:.1f} s, 1 thread"}


def run_reference(args):
    world, rank, local = dist_init()
    if rank != 0:
        return 0
    P = problem(args.config)
    import oracle
    oracle.lib()
    iters = args.ref_iters
    for _ in range(args.warmup):
        oracle.solve(P.A, P.B, tol=P.tol, maxit=max(2, iters // 8), tau=P.tau)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        r = oracle.solve(P.A, P.B, tol=P.tol, maxit=iters, tau=P.tau, pool_size=1)
        total += r.iterations
    dt = time.perf_counter() - t0
    value = total / dt
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": P.name, "n": P.n, "p": P.p, "iters_per_step": iters},
            "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} oracle solves of {iters} iterations of {P.name}"},
            "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    world, rank, local = dist_init()
    local = local % max(1, torch.cuda.device_count())   # (ranks may share a GPU when testing)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1301_2102_b200 import DeviceCsr, Solver

    P = problem(args.config)
    n, p = P.n, P.p
    # N > 1: one solve of the workload, rows partitioned over the ranks (halo exchange and
    # allreduces over NCCL) -- strong scaling
    off = [n * q // world for q in range(world + 1)]
    r0, r1 = off[rank], off[rank + 1]
    A = DeviceCsr.from_host(P.A, dev) if world == 1 else DeviceCsr.rows_from_host(P.A, r0, r1, dev)
    Bh_full = np.ascontiguousarray(P.B[r0:r1])
    B = torch.from_numpy(Bh_full).to(dev)
    X = torch.zeros_like(B)
    comm = None
    if world > 1:
        from paper_1301_2102_b200 import TorchComm
        comm = TorchComm() if os.environ.get("BENCH_COMM", "nccl") == "gloo" else "nccl"
    n_loc = r1 - r0
    stream = torch.cuda.Stream(device=dev)
    iters = args.iters
    peak, peak_kind = load_peaks()
    nnz_loc = int(P.A.indptr[r1]) - int(P.A.indptr[r0])
    abytes = 12.0 * nnz_loc + 4.0 * (n_loc + 1)   # this rank's CSR rows
    panel = 8.0 * n_loc * p

    # ---- timed region: the product's launch mode (CUDA graphs, main/side branches overlapped)
    solver = Solver(local, pool_size=1, use_graphs=not args.no_graphs, timing=False, record_history=False,
                    stream=stream.cuda_stream, rank=rank, world=world, comm=comm)

    def step(s):
        return s.solve(A, B, X, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)

    for _ in range(args.warmup):
        step(solver)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    total_iters, launches, slow = 0, 0, 0
    for _ in range(args.steps):
        r = step(solver)
        total_iters += r.iterations
        launches += r.stats["gpu_launches"]
        slow += r.stats["slow_blocks"]
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world, dev)
    value = total_iters / (ms_max / 1e3)   # iterations of the (one, partitioned) solve per second
    solver.close()

    # ---- kernel-timing region: the same steps with a CUDA event pair around every kernel
    # launch (explicit launches, kernels serialised on one stream), for the roofline
    roof = None
    if not args.no_kernel_timing:
        st_t = Solver(local, pool_size=1, use_graphs=False, timing=True, record_history=False,
                      stream=stream.cuda_stream, rank=rank, world=world, comm=comm)
        step(st_t)
        phase_ms, phase_n = {}, {}
        for _ in range(args.steps):
            r = step(st_t)
            for k, v in r.stats["phase_ms"].items():
                phase_ms[k] = phase_ms.get(k, 0.0) + v
                phase_n[k] = phase_n.get(k, 0) + r.stats["phase_launches"][k]
        st_t.close()
        cand = {k: phase_ms[k] for k in PHASE_BYTES_PANELS if phase_n.get(k)}
        dom = max(cand, key=cand.get)
        per_launch_ms = phase_ms[dom] / phase_n[dom]
        bytes_launch = PHASE_BYTES_PANELS[dom] * panel + (abytes if dom in PHASE_READS_A else 0.0)
        achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(f"{P.name}:{dom}")
            except Exception:
                traffic = None
        step_ms = sum(phase_ms[k] for k in ("spmm", "spmm_fused", "orth", "smallqr", "update", "reduce", "spmm_av",
                                            "epilogue", "epilogue_fused") if k in phase_ms)
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "bytes_per_launch": bytes_launch, "mean_launch_us": per_launch_ms * 1e3,
                "share_of_step": phase_ms[dom] / step_ms if step_ms else None,
                "timing": "CUDA events around every launch on the solver stream, the graph's kernels issued "
                          "explicitly in the graph's order and serialised (timing mode)",
                "phase_us_per_block_step": {k: 1e3 * phase_ms[k] / max(1, phase_n[k]) for k in phase_ms if phase_n[k]}}
    # whole-step algorithmic roofline (CSR A + 10 panels per block step)
    blk_bytes = abytes + 10 * panel
    blocks = total_iters / p
    step_roof = {"bytes_per_block_step": blk_bytes,
                 "achieved_GBps": blk_bytes * blocks / (ms / 1e3) / 1e9}
    step_roof["frac_of_measured"] = step_roof["achieved_GBps"] / peak

    # end to end through the C ABI with host buffers (pinned A arrays, B and X)
    e2e = None
    if not args.no_e2e:
        from paper_1301_2102_b200 import HostCsrRows
        Ah = HostCsrRows.from_host(P.A, 0, P.A.n) if world == 1 else HostCsrRows.from_host(P.A, r0, r1)

        def pinned(a):   # numpy view of a pinned copy (the library's H2D copies then run at DMA speed)
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        Ahost = HostCsrRows(Ah.n, pinned(Ah.indptr), pinned(Ah.indices), pinned(Ah.data), Ah.row_begin, Ah.n_global)
        Bh = torch.from_numpy(Bh_full).pin_memory()
        Xh = torch.zeros_like(Bh).pin_memory()
        s2 = Solver(local, pool_size=1, use_graphs=True, timing=False, record_history=False,
                    stream=stream.cuda_stream, rank=rank, world=world, comm=comm)
        s2.solve(Ahost, Bh, Xh, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        e_iters = 0
        for _ in range(args.steps):
            r = s2.solve(Ahost, Bh, Xh, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)
            e_iters += r.iterations
        dt = time.perf_counter() - t0
        dt = max_over_ranks(dt, world, dev)
        s2.close()
        e2e = {"value": e_iters / dt, "unit": "iterations/s",
               "h2d_bytes_per_step": int(abytes + panel), "d2h_bytes_per_step": int(panel)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(P, args.cpu_iters if args.cpu_iters > 0 else cpu_sample_iters(P))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iterations/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": P.name, "n": n, "p": p, "nnz": P.A.nnz, "iters_per_step": iters,
                           "tol": P.tol, "deflation_tol": P.tau, "pool_size": 1,
                           "l2": "inputs larger than L2 (working set per block step "
                                 f"{blk_bytes / 1e6:.0f} MB > 126 MB L2); no flush",
                           "parallelism": (f"row-partitioned x{world} (halo + allreduce over "
                                           f"{'NCCL' if comm == 'nccl' else 'host callbacks, testing'})")
                           if world > 1 else "single GPU",
                           "launch_mode": "plain launches" if (args.no_graphs or (world > 1 and comm != "nccl"))
                           else "CUDA graphs (main/side branches)"},
                "gpu_launches": launches, "slow_blocks": slow,
                "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "hbm_peak_GBps": peak}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="2")
    ap.add_argument("--iters", type=int, default=2000, help="banded iterations per step (maxit of one solve)")
    ap.add_argument("--no-graphs", action="store_true", help="plain launches instead of CUDA graphs")
    ap.add_argument("--no-kernel-timing", action="store_true", help="skip the per-kernel event region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=0, help="oracle iterations of cpu_baseline (0: ~15 s sample)")
    ap.add_argument("--ref-iters", type=int, default=40)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
