"""Diagnostic (GPU): dense small systems whose block Krylov space is exhausted mid-solve, every
compiled p, several n and maxit, graphs on / off -- GPU against the oracle (status, counts, events,
history, X).  Usage: python scripts/diag_sweep.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from test_gpu_parity import gpu_solve  # noqa: E402

for p in [1, 2, 3, 4, 5, 6, 7, 8, 16, 32]:
    for n in (3 * p + 1, 3 * p + 2, 4 * p - 1) if p > 1 else (3, 5):
        rng = np.random.default_rng(n * 1000 + p)
        D = rng.standard_normal((n, n))
        A = synth.dense_to_csr(D + D.T)
        B = rng.standard_normal((n, p))
        for maxit in (n - p + 1, n - p + 2, 4 * n):
            ref = oracle.solve(A, B, tol=1e-10, maxit=maxit)
            ratios = [f"{e['ratio']:.0e}" for e in ref.events]
            for g in (True, False):
                r = gpu_solve(A, B, tol=1e-10, maxit=maxit, use_graphs=g)
                same_ev = [(e["j"], e["kind"], e["action"]) for e in r.events] == \
                          [(e["j"], e["kind"], e["action"]) for e in ref.events]
                sc = max(np.abs(ref.X).max(), 1.0)
                ex = np.abs(r.X - ref.X).max() / sc
                k = min(len(r.history), len(ref.history))
                eh = np.max(np.abs(r.history[:k] - ref.history[:k]) / np.maximum(np.abs(ref.history[:k]), 1e-300)) \
                    if k else 0.0
                ok = r.status_name == ref.status_name and r.iterations == ref.iterations and same_ev
                flag = "OK " if ok and ex < 1e-7 and eh < 1e-9 else "BAD"
                print(f"{flag} p={p:2d} n={n:3d} maxit={maxit:4d} g={int(g)} st={r.status_name}/{ref.status_name} "
                      f"it={r.iterations}/{ref.iterations} ev_same={int(same_ev)} nev={len(ref.events)} "
                      f"ratios={ratios[:4]} errX={ex:.1e} errH={eh:.1e}", flush=True)
