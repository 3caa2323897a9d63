#!/usr/bin/env python
"""Write oracle-only golden files under tests/golden/ (test infrastructure).

Every value written here comes from ``oracle.solve`` (plain C, one thread, the paper's
per-iteration algorithm) on the seeded ``synth`` inputs -- never from the CUDA path.

  python scripts/make_golden.py first50 4      # config 4: first 50 iterations (history, events)
  python scripts/make_golden.py first50 5      # config 5
  python scripts/make_golden.py first 4 160    # config 4: first 160 iterations (5 block steps at p = 32)
  python scripts/make_golden.py tol 2          # config 2 run to tol 1e-8 (hours, one thread)
  python scripts/make_golden.py tol 3 600000 1e-6   # config 3 at eps = 1e-6

Files: tests/golden/<workload>_first50.json and <workload>_tol.json, each naming the oracle
call that produced it, the host (nproc, CPU model) and the wall time.
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth   # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def host() -> dict:
    return {"nproc": os.cpu_count(), "cpu": cpu_model(), "threads_used": 1}


def write(name: str, d: dict) -> None:
    os.makedirs(GOLD, exist_ok=True)
    path = os.path.join(GOLD, name)
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print("wrote", path, flush=True)


def first50(cfg, N: int = 50) -> None:
    P = synth.config(cfg)
    t0 = time.perf_counter()
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=N, tau=P.tau, pool_size=1)
    dt = time.perf_counter() - t0
    write(f"{P.name}_first{N}.json", {
        "source": f"oracle.solve(synth.config({cfg!r}), tol={P.tol}, maxit={N}, tau={P.tau}, pool_size=1, seed=0)",
        "workload": P.name, "n": P.n, "p": P.p, "nnz": P.A.nnz,
        "status": r.status, "iterations": r.iterations,
        "history": r.history.tolist(), "events": r.events,
        "true_res": r.true_res.tolist(), "comp_res": r.comp_res.tolist(),
        "wall_s": dt, "host": host()})


def to_tol(cfg, maxit: int, eps: float | None = None) -> None:
    P = synth.config(cfg) if eps is None else synth.config(cfg, eps=eps)
    t0 = time.perf_counter()
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=maxit, tau=P.tau, pool_size=1)
    dt = time.perf_counter() - t0
    h = r.history
    every = 1000
    write(f"{P.name}_tol.json", {
        "source": (f"oracle.solve(synth.config({cfg!r}" + ("" if eps is None else f", eps={eps!r}")
                   + f"), tol={P.tol}, maxit={maxit}, tau={P.tau}, pool_size=1, seed=0)"),
        "workload": P.name, "n": P.n, "p": P.p, "nnz": P.A.nnz,
        "status": r.status, "iterations": r.iterations,
        "history_first50": h[:51].tolist(),
        "history_every": every, "history_sampled": h[::every].tolist(), "history_last": h[-1].tolist(),
        "events": r.events, "true_res": r.true_res.tolist(), "comp_res": r.comp_res.tolist(),
        "wall_s": dt, "ms_per_iteration": 1e3 * dt / max(1, r.iterations), "host": host()})


if __name__ == "__main__":
    mode, cfg = sys.argv[1], sys.argv[2]
    cfg = cfg if cfg == "1c" else int(cfg)
    if mode == "first50":
        first50(cfg)
    elif mode == "first":
        first50(cfg, int(sys.argv[3]))
    elif mode == "tol":
        to_tol(cfg, int(sys.argv[3]) if len(sys.argv) > 3 else 600_000,
               float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        raise SystemExit(__doc__)
