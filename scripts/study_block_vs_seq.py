#!/usr/bin/env python
"""Block-vs-sequential studies on the GPU (the paper's §8 experiments).

Every solve runs through the product (libbminres.so, C ABI): the block solve with p right-hand
sides and the "sequential MINRES" comparison as p independent p = 1 solves (block MINRES with
p = 1 is MINRES, P:48-49 -- pinned against SciPy's MINRES in tests/test_oracle_pins.py).
Independent solves run concurrently: a pool of host threads, each with its own handle and CUDA
stream (the C call releases the GIL), batches many small systems onto the one GPU.

Studies (inputs: synth/studies.py, unpreconditioned -- the paper's ichol preconditioner is row f3):
  fig2   ratio block / sequential iterations for B = [ones, e_1 .. e_{p-1}], p = 1..8, 16
  fig4   the pairs (e_1, ones) and (e_1, e_2)
  fig5   eqn.smalleigsRHS pairs, averaged over R random pairs per m
  fig6   eqn.largeeigsRHS pairs

  python scripts/study_block_vs_seq.py [--N 200] [--pairs 10] [--out profiles/r02_study_block_vs_seq.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import studies  # noqa: E402


class Runner:
    """A pool of solver handles, one per host thread (each on its own CUDA stream)."""

    def __init__(self, A, threads: int = 4, tol: float = 1e-8, maxit: int = 200_000):
        import torch
        from paper_1301_2102_b200 import DeviceCsr
        self.torch = torch
        self.A = DeviceCsr.from_host(A, "cuda:0")
        self.tol, self.maxit = tol, maxit
        self.local = threading.local()
        self.pool = ThreadPoolExecutor(max_workers=threads)
        self.handles = []

    def _solver(self):
        s = getattr(self.local, "s", None)
        if s is None:
            from paper_1301_2102_b200 import Solver
            stream = self.torch.cuda.Stream(device="cuda:0")
            s = Solver(0, pool_size=1, record_history=False, stream=stream.cuda_stream)
            self.local.s, self.local.stream = s, stream
            self.handles.append(s)
        return s

    def _solve(self, B):
        s = self._solver()
        with self.torch.cuda.stream(self.local.stream):
            dB = self.torch.from_numpy(np.ascontiguousarray(B)).to("cuda:0", non_blocking=False)
        self.local.stream.synchronize()
        r = s.solve(self.A, dB, tol=self.tol, maxit=self.maxit, history=False, raise_on_error=False)
        return {"iterations": r.iterations, "status": r.status_name, "max_true_res": max(r.stats["true_res"]),
                "ms": r.stats["solve_ms"]}

    def block_and_sequential(self, B):
        """The block solve of B and the p sequential p = 1 solves, concurrently."""
        futs = [self.pool.submit(self._solve, B)] + [self.pool.submit(self._solve, B[:, c:c + 1])
                                                    for c in range(B.shape[1])]
        res = [f.result() for f in futs]
        return res[0], res[1:]

    def close(self):
        self.pool.shutdown()
        for s in self.handles:
            s.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=200)
    ap.add_argument("--pairs", type=int, default=10, help="random pairs per m (the paper: 100)")
    ap.add_argument("--threads", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_study_block_vs_seq.json"))
    args = ap.parse_args()
    N = args.N
    band = max(1, N // 2) if N < 200 else 100
    A = studies.model_matrix(N)
    n = A.n
    run = Runner(A, threads=args.threads)
    out = {"problem": f"A = -L - 200 I on the {N}x{N} grid, h = 1/{N - 1}, unpreconditioned (P:1020-1025)",
           "n": n, "tol": run.tol, "note": "sequential = p independent p = 1 solves (MINRES) of the columns; "
                                          "iterations are banded iterations j / MINRES iterations"}
    t0 = time.perf_counter()
    # Fig. 2
    fig2 = []
    for p in (1, 2, 3, 4, 5, 6, 7, 8, 16):
        blk, seq = run.block_and_sequential(studies.fig2_rhs(n, p))
        tot = sum(s["iterations"] for s in seq)
        fig2.append({"p": p, "block": blk["iterations"], "sequential": tot, "ratio": blk["iterations"] / tot,
                     "block_status": blk["status"], "block_max_true_res": blk["max_true_res"]})
        print("fig2", fig2[-1], flush=True)
    out["fig2"] = fig2
    # Fig. 4
    fig4 = []
    for name, B in zip(("(e1, ones)", "(e1, e2)"), studies.fig4_pairs(n)):
        blk, seq = run.block_and_sequential(B)
        fig4.append({"pair": name, "block": blk["iterations"], "sequential": [s["iterations"] for s in seq],
                     "ratio": blk["iterations"] / sum(s["iterations"] for s in seq)})
        print("fig4", fig4[-1], flush=True)
    out["fig4"] = fig4
    # Figs. 5, 6
    for fig, kind, ms in (("fig5", "small", (0, 1, 5, 10, 25, 50, 75, 99, band)),
                          ("fig6", "large", (0, 1, 10, 25, 50, 100, 150, 2 * band))):
        rows = []
        for m in ms:
            if kind == "small" and m > band or kind == "large" and m > 2 * band:
                continue
            b_it, s_it = [], []
            for r in range(args.pairs):
                blk, seq = run.block_and_sequential(studies.eigmix_pair(N, m, kind, seed=1000 * m + r, band=band))
                b_it.append(blk["iterations"])
                s_it.append(sum(s["iterations"] for s in seq))
            rows.append({"m": m, "pairs": args.pairs, "block_mean": float(np.mean(b_it)),
                         "sequential_mean": float(np.mean(s_it)), "ratio": float(np.mean(b_it) / np.mean(s_it))})
            print(fig, rows[-1], flush=True)
        out[fig] = rows
    out["wall_s"] = time.perf_counter() - t0
    run.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
