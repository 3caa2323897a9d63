#!/usr/bin/env python
"""bench.py — block-MINRES iterations/s on B200 (driver contract).

Workload (default): BASELINE.json configs[3] -- config 4, the 3-D 7-point Laplacian on a 256^3
grid shifted by -3 (n = 16.8M, nnz = 117M), p = 32 Gaussian right-hand sides from seed 0, fp64:
the configuration BASELINE.json's metric ("... 1/2/4/8 B200") and the north star's targets are
quoted on, and the largest one that fits one GPU.  A "step" is one bminres_solve call with a fixed
budget of --iters banded iterations (default 6400 = 200 block steps at p = 32, SURVEY §8(d)'s
window): the start block (row a0), then every row a1..a5 of the hot path once per block step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

`value`      = banded iterations / max-over-ranks device time (CUDA events on the solver stream).
`e2e`        = the same metric through the C ABI with HOST buffers (A, B in; X out per step).
`roofline`   = the dominant kernel's algorithmic bytes per launch / its mean launch time (CUDA
               events around every launch, timing mode) vs MEASURED_PEAKS.json.
`step_roofline` = (CSR A + 10 panels) per block step / graph-mode time per block step.
`cpu_baseline`  = the C oracle (the tests' reference implementation), one thread, on a bounded
               sample of the same workload, run in a subprocess beside the GPU measurements.
`secondary`  = config 2 (3-D 64^3, p = 8: BASELINE configs[1]) measured the same way (no e2e).
`time_to_tol`= config 2 solved to tol 1e-8 (the north star's convergence gate at scale): iterations,
               device time with and without one-time setup, true residuals, against the oracle's
               count from tests/golden when present.
With --gpus N > 1 the script re-executes itself under torch.distributed.run (one rank per GPU over
NCCL) unless WORLD_SIZE is already set; the ranks run ONE solve with the rows partitioned (halo
exchange + allreduces; strong scaling).  Testing aids: BENCH_BACKEND=gloo +
BENCH_COMM=gloo run the same path with the host-callback transport (e.g. two ranks on one GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json's metric (the value is iterations/s; the achieved HBM GB/s against the roofline is
# reported in "roofline" / "step_roofline")
METRIC = "block-MINRES iterations/s and achieved HBM GB/s (fp64) vs roofline, 1/2/4/8 B200"
# algorithmic panel transfers per launch; K1 also streams CSR A.  The fused M/X
# update moves 5 panels on average: it reads V_k, M_{k-2}, M_{k-1} and writes M_k every block, and
# reads + writes X every other block (X updates deferred in pairs); the standalone K4b moves 6.
PHASE_BYTES_PANELS = {"spmm": 3, "spmm_fused": 8, "orth": 3, "update": 6,
                      # split mode (large panels): K1a reads V_k once (gathers) and writes AV; K1 then
                      # streams AV, V_k, V_{k-1} and writes W (+ the fused update)
                      "spmm_av": 2, "epilogue": 4, "epilogue_fused": 9,
                      # split mode, p >= 16: the update as its own kernel (V_{k-2}, M_{k-4}, M_{k-3} read,
                      # M_{k-2} written, X read + written every other block: 5 on average)
                      "update_main": 5}
PHASE_READS_A = {"spmm", "spmm_fused", "spmm_av"}


def phase_flops_per_row(k: str, p: int) -> float:
    """Algorithmic fp64 flops per row and launch of the DMMA kernels (DESIGN.md §6 "fp64 tensor
    roofline"): an upper-triangular p x p factor costs p(p+1), a full one 2p^2, a symmetric Gram
    p(p+1); X += M Z (2p^2) runs every other block in pairs, so 2p^2 on average.  The pool's
    4Qp and the norms' 2p are left out (< 1%)."""
    tri, full = p * (p + 1), 2.0 * p * p
    epi = tri + 2 * full              # (A V_k) Tr_k, V_{k-1} D, V_k^T W
    upd = tri + 2 * full + full       # V_k (Tr_k R^-1), M_{k-2} B2, M_{k-1} B1; X += M Z (average)
    orth = full + tri                 # V_k (Tr_k G_s), W'^T W'
    return {"epilogue": epi, "update_main": upd, "orth": orth, "epilogue_fused": epi + upd,
            "spmm_fused": epi + upd, "update": upd}.get(k, 0.0)


def load_fp64_peak():
    """fp64 tensor-core (DMMA m8n8k4) peak measured on this pool's B200 by scripts/micro/fp64_mix.cu
    (profiles/r02_fp64_peaks.json); NVIDIA's nominal B200 fp64 tensor figure is 40 TF/s."""
    path = os.path.join(ROOT, "profiles", "r02_fp64_peaks.json")
    try:
        with open(path) as f:
            return float(json.load(f)["dmma_tflops"]), "measured (profiles/r02_fp64_peaks.json, scripts/micro/fp64_mix.cu)"
    except Exception:
        return 37.1, "measured (DESIGN.md §6, scripts/micro/spmm_lab.cu)"
# (configs 4 and 5: a window of 200 block steps per solve, SURVEY §8(d)'s timing protocol)
DEFAULT_ITERS = {"1": 2000, "1c": 2000, "2": 2000, "3": 2000, "4": 6400, "5": 3200}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_info() -> dict:
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


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
    t = torch.tensor([x], dtype=torch.float64, device=device if os.environ.get("BENCH_BACKEND", "nccl") == "nccl"
                     else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------------- the oracle (CPU baseline)

ORACLE_SAMPLE = r"""
import json, sys, time
sys.path.insert(0, {root!r})
import oracle, synth
cfg = {cfg!r}
P = synth.config(cfg if cfg == "1c" else int(cfg))
oracle.lib()
r = oracle.solve(P.A, P.B, tol=P.tol, maxit={iters}, tau=P.tau, pool_size=1, history=False)
print(json.dumps({{"iterations": r.iterations, "start_s": r.start_s, "loop_s": r.loop_s, "name": P.name}}))
"""


def oracle_sample_iters(P, budget_s: float = 20.0) -> int:
    """Iterations of the bounded oracle sample: ~budget_s of one-thread loop time, from the oracle's
    measured cost on config 2 (26 ms per iteration: ~0.8 ns per unit of nnz/p + 8 n (2p+1) per
    iteration), 2 .. 400."""
    units = float(P.A.nnz) + 8.0 * P.n * P.p
    est = budget_s / (0.82e-9 * units)
    return int(max(2, min(400, est)))


def start_oracle_sample(cfg: str, iters: int):
    """The oracle as it stands, one thread, in a subprocess (it runs beside the GPU measurements on
    another host core): one solve of `iters` iterations of the workload.  Its loop time (the start
    block and the pool are timed separately) gives the per-iteration rate."""
    code = ORACLE_SAMPLE.format(root=ROOT, cfg=cfg, iters=iters)
    return subprocess.Popen([sys.executable, "-c", code], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def finish_oracle_sample(proc, kind="oracle"):
    out, err = proc.communicate()
    if proc.returncode != 0:
        return {"value": None, "unit": "iterations/s", "cores": 1, "kind": kind,
                "sample": f"oracle sample failed: {err.strip().splitlines()[-1:] if err else proc.returncode}"}
    d = json.loads(out.strip().splitlines()[-1])
    value = d["iterations"] / d["loop_s"] if d["loop_s"] > 0 else None
    return {"value": value, "unit": "iterations/s", "cores": 1, "kind": kind,
            "sample": (f"{d['name']}: one oracle solve of {d['iterations']} banded iterations, one thread; value = "
                       f"iterations / loop time ({d['loop_s']:.1f} s); its start block + pool took "
                       f"{d['start_s']:.1f} s (not in the value)"),
            "start_block_s": d["start_s"], "loop_s": d["loop_s"], "iterations": d["iterations"], **host_info()}


def run_reference(args):
    """The reference arm: the oracle (this tier has no reference code) on the same workload.  One
    bounded sample: a solve of W + K banded iterations; value = iterations / loop time."""
    world, rank, local = dist_init()
    if rank != 0:
        return 0
    cfg = args.config
    P = problem(cfg)
    iters = max(2, args.warmup + args.steps) if args.ref_iters <= 0 else args.ref_iters
    del P
    t0 = time.perf_counter()
    cpu = finish_oracle_sample(start_oracle_sample(cfg, iters))
    wall = time.perf_counter() - t0
    value = cpu["value"]
    P = problem(cfg)
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * cpu["loop_s"] / max(1, cpu["iterations"]) if value else None,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": P.name, "n": P.n, "p": P.p, "nnz": P.A.nnz,
                       "step": "one banded iteration of one oracle solve (W + K iterations in total)"},
            "cpu_baseline": cpu, "wall_s": wall,
            "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm


def measure(P, args, iters, world, rank, local, dev, *, e2e: bool, kernel_timing: bool):
    """Device-timed solves of the workload (graphs, the product's launch mode), the per-kernel
    roofline in timing mode, and optionally the end-to-end host-buffer solves."""
    import torch
    from paper_1301_2102_b200 import DeviceCsr, HostCsrRows, Solver
    n, p = P.n, P.p
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
    peak, peak_kind = load_peaks()
    nnz_loc = int(P.A.indptr[r1]) - int(P.A.indptr[r0])
    abytes = 12.0 * nnz_loc + 4.0 * (n_loc + 1)   # this rank's CSR rows
    panel = 8.0 * n_loc * p
    kw = dict(pool_size=1, record_history=False, stream=stream.cuda_stream, rank=rank, world=world, comm=comm,
              plan_reuse=True)

    # ---- timed region: the product's launch mode (CUDA graphs, main/side branches overlapped)
    solver = Solver(local, use_graphs=not args.no_graphs, timing=False, **kw)

    def step(s, Ain=A, Bin=B, Xin=X):
        return s.solve(Ain, Bin, Xin, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)

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

    # ---- kernel-timing region: the same steps with a CUDA event pair around every kernel launch
    # (explicit launches in the graph's order, serialised on the solver stream), for the roofline
    roof = None
    if kernel_timing:
        st_t = Solver(local, use_graphs=False, timing=True, **kw)
        step(st_t)
        phase_ms, phase_n = {}, {}
        for _ in range(max(1, min(args.steps, 3))):
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
                                            "epilogue", "epilogue_fused", "update_main") if k in phase_ms)
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "bytes_per_launch": bytes_launch, "mean_launch_us": per_launch_ms * 1e3,
                "share_of_step": phase_ms[dom] / step_ms if step_ms else None,
                "timing": "CUDA events around every launch on the solver stream, the graph's kernels issued "
                          "explicitly in the graph's order and serialised (timing mode)",
                "phase_us_per_block_step": {k: 1e3 * phase_ms[k] / max(1, phase_n[k]) for k in phase_ms if phase_n[k]}}
        # the same kernel against the fp64 tensor-core (DMMA) peak: at p = 32 the DMMA kernels are
        # bound by both (ncu: DMMA pipe 68-76% busy beside 58-61% of DRAM peak)
        fl = phase_flops_per_row(dom, p) * n_loc
        if fl > 0:
            tpk, tkind = load_fp64_peak()
            t_ach = fl / (per_launch_ms / 1e3) / 1e12
            roof["tensor"] = {"achieved": t_ach, "peak": tpk, "peak_kind": tkind, "unit": "TFLOP/s",
                              "frac": t_ach / tpk, "flops_per_launch": fl}
            roof["tensor_by_kernel"] = {
                k: (phase_flops_per_row(k, p) * n_loc) / (phase_ms[k] / phase_n[k] / 1e3) / 1e12 / tpk
                for k in phase_ms if phase_n.get(k) and phase_flops_per_row(k, p) > 0}
            if t_ach / tpk > roof["frac"]:
                # the binding resource is the fp64 tensor pipe: report it as the primary bound
                hb = {kk: roof[kk] for kk in ("achieved", "peak", "peak_kind", "unit", "frac")}
                roof.update({"bound": "tensor", "achieved": t_ach, "peak": tpk, "peak_kind": tkind,
                             "unit": "TFLOP/s", "frac": t_ach / tpk, "hbm": hb})
    # whole-step algorithmic roofline (CSR A + 10 panels per block step)
    blk_bytes = abytes + 10 * panel
    blocks = total_iters / p
    step_roof = {"bytes_per_block_step": blk_bytes, "ms_per_block_step": ms_max / max(blocks, 1),
                 "achieved_GBps": blk_bytes * blocks / (ms_max / 1e3) / 1e9,
                 "note": "graph-mode device time of the whole solve (start block included) per block step"}
    step_roof["frac_of_measured"] = step_roof["achieved_GBps"] / peak
    # the whole step against the fp64 tensor peak: the DMMA kernels' algorithmic flops per block step
    dm_flops = sum(phase_flops_per_row(k, p) for k in ("epilogue", "update_main", "orth")) * n_loc if p >= 16 else 0.0
    if dm_flops > 0:
        tpk, _ = load_fp64_peak()
        step_roof["dmma_flops_per_block_step"] = dm_flops
        step_roof["tensor_TFps"] = dm_flops * blocks / (ms_max / 1e3) / 1e12
        step_roof["tensor_frac_of_measured"] = step_roof["tensor_TFps"] / tpk
        step_roof["tensor_floor_ms_per_block_step"] = dm_flops / (tpk * 1e12) * 1e3

    # ---- end to end through the C ABI with host buffers (pinned A arrays, B and X)
    e2e_d = None
    if e2e:
        Ah = HostCsrRows.from_host(P.A, 0, P.A.n) if world == 1 else HostCsrRows.from_host(P.A, r0, r1)

        def pinned(a):   # numpy view of a pinned copy (the library's H2D copies then run at DMA speed)
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        Ahost = HostCsrRows(Ah.n, pinned(Ah.indptr), pinned(Ah.indices), pinned(Ah.data), Ah.row_begin, Ah.n_global)
        del Ah
        Bh = torch.from_numpy(Bh_full).pin_memory()
        Xh = torch.zeros_like(Bh).pin_memory()
        del A, B, X, step   # (the device copies are not needed by the host-buffer solves)
        torch.cuda.empty_cache()
        s2 = Solver(local, use_graphs=True, timing=False, **kw)
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
        e2e_d = {"value": e_iters / dt, "unit": "iterations/s",
                 "h2d_bytes_per_step": int(abytes + panel), "d2h_bytes_per_step": int(panel),
                 "timing": "host wall clock around bminres_solve with pinned host A, B, X (copies inside)"}
    torch.cuda.empty_cache()
    return {"value": value, "ms": ms_max, "total_iters": total_iters, "launches": launches, "slow_blocks": slow,
            "clocks": clk, "roofline": roof, "step_roofline": step_roof, "e2e": e2e_d, "peak": peak,
            "abytes": abytes, "panel": panel, "n_loc": n_loc}


def time_to_tol(cfg, local, dev):
    """One solve of the config to its tol (maxit = the config's), cold (first call on a fresh handle:
    workspace, graph capture) and warm (second call).  Device times from the library's CUDA events;
    the cold call's host wall time includes the one-time setup."""
    import torch
    from paper_1301_2102_b200 import DeviceCsr, Solver
    P = problem(cfg)
    A = DeviceCsr.from_host(P.A, dev)
    B = torch.from_numpy(P.B).to(dev)
    out = {"workload": P.name, "tol": P.tol, "maxit": P.maxit}
    with Solver(local, pool_size=1, record_history=False) as s:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = s.solve(A, B, tol=P.tol, maxit=P.maxit, deflation_tol=P.tau, history=False, raise_on_error=False)
        cold = time.perf_counter() - t0
        t0 = time.perf_counter()
        r2 = s.solve(A, B, tol=P.tol, maxit=P.maxit, deflation_tol=P.tau, history=False, raise_on_error=False)
        warm = time.perf_counter() - t0
    out.update({"status": r2.status_name, "iterations": r2.iterations, "block_steps": r2.stats["block_steps"],
                "slow_blocks": r2.stats["slow_blocks"], "events": len(r2.events),
                "device_ms": r2.stats["solve_ms"], "loop_ms": r2.stats["loop_ms"],
                "wall_s_cold_with_setup": cold, "wall_s_warm": warm,
                "iterations_per_s": r2.iterations / (r2.stats["solve_ms"] / 1e3),
                "max_true_res": max(r2.stats["true_res"]), "max_comp_res": max(r2.stats["comp_res"]),
                "true_res_le_tol": bool(max(r2.stats["true_res"]) <= P.tol),
                "cold_equals_warm_iterations": r.iterations == r2.iterations})
    gpath = os.path.join(ROOT, "tests", "golden", f"{P.name}_tol.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        out["oracle_iterations"] = g["iterations"]
        out["oracle_status"] = g["status"]
        out["count_rel_diff"] = (r2.iterations - g["iterations"]) / max(1, g["iterations"])
        out["oracle_ms_per_iteration"] = g.get("ms_per_iteration")
    return out


def precond_block(which, args, local, dev):
    """f3: IC(0) split-preconditioned solves (reading R8).
    model200: the paper's own preconditioned experiment (A = -L - 200 I on 200 x 200, h = 1/199,
    IC(0) of -L, tol 1e-8) at p = 8, solved to tol (the paper's p = 10 is not a compiled
    block size); cfg4: config 4's operator with IC(0) of the unshifted Laplacian, iterations/s over a
    fixed window.  The triangular kernels are latency-bound by the dependency depth (levels): their
    line reports achieved GB/s on their algorithmic bytes and the time per level."""
    import torch
    import synth
    from synth.studies import model_matrix
    from paper_1301_2102_b200 import DeviceCsr, Solver
    peak, _ = load_peaks()
    out = {}
    for w in which.split(","):
        if w == "model200":
            N = 200
            A = model_matrix(N)
            s_ = float((N - 1) ** 2)
            M = synth.stencil_csr((N, N), 4.0 * s_, -s_)
            B = np.random.default_rng(0).standard_normal((A.n, 8))
            tol, maxit, name = 1e-8, 20000, "paper_model_200_ic0_p8"
        elif w == "cfg4":
            P = problem("4")
            A, B, tol, name = P.A, P.B, P.tol, "cfg4_lap3d_256_shift3_ic0"
            M = synth.laplacian_3d(256)
            maxit = 256   # (8 block steps: the triangular pair dominates; a window for iterations/s)
            del P
        else:
            continue
        dA, dM = DeviceCsr.from_host(A, dev), DeviceCsr.from_host(M, dev)
        dB = torch.from_numpy(np.ascontiguousarray(B)).to(dev)
        n, p = A.n, B.shape[1]
        with Solver(local, pool_size=1, record_history=False) as s:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.set_preconditioner(dM)
            torch.cuda.synchronize()
            setup_s = time.perf_counter() - t0
            s.solve(dA, dB, tol=tol, maxit=maxit, history=False, raise_on_error=False)   # warm-up
            ms, its = [], 0
            for _ in range(max(1, min(3, args.steps))):
                r = s.solve(dA, dB, tol=tol, maxit=maxit, history=False, raise_on_error=False)
                ms.append(r.stats["solve_ms"])
                its = r.iterations
            st = r.stats
        with Solver(local, pool_size=1, record_history=False, use_graphs=False, timing=True) as s:
            s.set_preconditioner(dM)
            r2 = s.solve(dA, dB, tol=tol, maxit=min(maxit, 64 * p), history=False, raise_on_error=False)
            ph, pn = r2.stats["phase_ms"], r2.stats["phase_launches"]
        nnzl = (M.nnz + n) // 2
        tri_bytes = 2 * (12.0 * nnzl + 4.0 * (n + 1)) + 12.0 * A.nnz + 4.0 * (n + 1) + 4 * 8.0 * n * p
        prec_ms = ph["prec"] / max(1, pn["prec"])
        d = {"n": n, "p": p, "tol": tol, "maxit": maxit, "status": r.status_name, "iterations": its,
             "device_ms": statistics.median(ms), "iterations_per_s": its / (statistics.median(ms) / 1e3),
             "ic0_setup_s": setup_s, "levels": st["prec_levels"],
             "max_true_res_unpreconditioned": max(st["true_res"]), "max_comp_res": max(st["comp_res"]),
             "slow_blocks": st["slow_blocks"],
             "prec_op_us_per_block_step": prec_ms * 1e3,
             "prec_op": {"bound": "latency (dependency depth) and hbm", "bytes_per_launch_pair": tri_bytes,
                         "achieved_GBps": tri_bytes / (prec_ms / 1e3) / 1e9,
                         "frac_of_hbm": tri_bytes / (prec_ms / 1e3) / 1e9 / peak,
                         "us_per_level": prec_ms * 1e3 / (2.0 * st["prec_levels"]),
                         "note": "Z = L^-T V_k then AV = L^-1 (A Z): 2 sync-free level-scheduled launches per block "
                                 "step, timed with CUDA events (timing mode)"},
             "phase_us_per_block_step": {k: 1e3 * ph[k] / max(1, pn[k]) for k in ph if pn[k]}}
        if w == "model200":
            d["paper_context"] = {"block_minres_iterations_p10": 1048, "sequential_minres_iterations": 3787,
                                  "source": "P:1034-1035 (Matlab R2011b, 2.3 GHz Core i5; ten Matlab rand() "
                                            "right-hand sides): context only"}
        out[name] = d
        del dA, dM, dB
        torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_init()
    local = local % max(1, torch.cuda.device_count())   # (ranks may share a GPU when testing)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    cfg = args.config
    iters = args.iters if args.iters > 0 else DEFAULT_ITERS[cfg]
    P = problem(cfg)
    # the CPU baseline runs in its own process on another host core while the GPU is measured
    cpu_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_proc = start_oracle_sample(cfg, args.cpu_iters if args.cpu_iters > 0 else oracle_sample_iters(P))
    main = measure(P, args, iters, world, rank, local, dev, e2e=not args.no_e2e,
                   kernel_timing=not args.no_kernel_timing)
    n, p, name, nnz, tol, tau = P.n, P.p, P.name, P.A.nnz, P.tol, P.tau
    del P

    secondary = {}
    if world == 1 and args.secondary and args.secondary != "none":
        for c in args.secondary.split(","):
            if c and c != cfg:
                Q = problem(c)
                m = measure(Q, args, DEFAULT_ITERS[c], 1, 0, local, dev, e2e=False, kernel_timing=True)
                secondary[Q.name] = {"value": m["value"], "unit": "iterations/s", "iters_per_step": DEFAULT_ITERS[c],
                                     "n": Q.n, "p": Q.p, "ms_per_step": m["ms"] / args.steps,
                                     "roofline": m["roofline"], "step_roofline": m["step_roofline"],
                                     "gpu_launches": m["launches"], "clocks": m["clocks"]}
                del Q
    ttt = None
    if world == 1 and args.time_to_tol and args.time_to_tol != "none":
        ttt = time_to_tol(args.time_to_tol, local, dev)

    prec = None
    if world == 1 and args.precond and args.precond != "none":
        prec = precond_block(args.precond, args, local, dev)

    cpu = finish_oracle_sample(cpu_proc) if cpu_proc else None

    if rank == 0:
        blk_bytes = main["abytes"] + 10 * main["panel"]
        line = {"metric": METRIC, "value": main["value"], "unit": "iterations/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms"] / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": name, "n": n, "p": p, "nnz": nnz, "iters_per_step": iters,
                           "tol": tol, "deflation_tol": tau, "pool_size": 1,
                           "l2": "inputs larger than L2 (working set per block step "
                                 f"{blk_bytes / 1e6:.0f} MB > 126 MB L2); no flush",
                           "parallelism": (f"row-partitioned x{world} (halo + allreduce over "
                                           f"{'NCCL' if os.environ.get('BENCH_COMM', 'nccl') == 'nccl' else 'host callbacks, testing'})")
                           if world > 1 else "single GPU",
                           "launch_mode": "plain launches" if (args.no_graphs or (world > 1 and os.environ.get(
                               "BENCH_COMM", "nccl") != "nccl")) else "CUDA graphs (main/side branches)"},
                "gpu_launches": main["launches"], "slow_blocks": main["slow_blocks"],
                "roofline": main["roofline"], "step_roofline": main["step_roofline"], "cpu_baseline": cpu,
                "e2e": main["e2e"], "clocks": main["clocks"], "hbm_peak_GBps": main["peak"],
                "secondary": secondary or None, "time_to_tol": ttt, "preconditioned": prec}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="4")
    ap.add_argument("--iters", type=int, default=0, help="banded iterations per step (0: 6400 / 3200 for configs 4 / 5, "
                                                          "2000 otherwise)")
    ap.add_argument("--secondary", default="2,5", help="comma-separated configs measured after the main one (N = 1; 'none' to skip)")
    ap.add_argument("--time-to-tol", default="2", help="config solved to tol at N = 1 ('none' to skip)")
    ap.add_argument("--precond", default="model200,cfg4",
                    help="f3 IC(0)-preconditioned measurements at N = 1 ('none' to skip)")
    ap.add_argument("--no-graphs", action="store_true", help="plain launches instead of CUDA graphs")
    ap.add_argument("--no-kernel-timing", action="store_true", help="skip the per-kernel event region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=0, help="oracle iterations of cpu_baseline (0: ~20 s sample)")
    ap.add_argument("--ref-iters", type=int, default=0, help="oracle iterations of --impl reference (0: W + K)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU: re-execute under torch.distributed.run (the driver's launch, made here)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
