"""Diagnostic (GPU): X after a solve that ends inside a column-path block, against the oracle's
X at the same and nearby maxit.  Usage: python scripts/diag_tiny.py [p ...]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from test_gpu_parity import gpu_solve  # noqa: E402

ps = [int(a) for a in sys.argv[1:]] or [4, 7, 8]
for p in ps:
    n = 3 * p
    rng = np.random.default_rng(n * 100 + p)
    D = rng.standard_normal((n, n))
    A = synth.dense_to_csr(D + D.T)
    B = rng.standard_normal((n, p))
    refs = {m: oracle.solve(A, B, tol=1e-10, maxit=m) for m in range(1, 4 * p)}
    for m in range(2 * p - 1, 4 * p - 1):
        for g in (True, False):
            r = gpu_solve(A, B, tol=1e-10, maxit=m, use_graphs=g)
            ref = refs[m]
            sc = max(np.abs(ref.X).max(), 1.0)
            e = np.abs(r.X - ref.X).max() / sc
            near = {mm: np.abs(r.X - refs[mm].X).max() / sc for mm in range(max(1, m - p), min(4 * p - 1, m + 2))}
            best = min(near, key=near.get)
            colerr = np.abs(r.X - ref.X).max(axis=0) / sc
            Ad = A.to_dense() if hasattr(A, "to_dense") else None
            if Ad is None:
                Ad = np.zeros((n, n))
                for i in range(n):
                    Ad[i, A.indices[A.indptr[i]:A.indptr[i + 1]]] = A.data[A.indptr[i]:A.indptr[i + 1]]
            tr_g = np.linalg.norm(B - Ad @ r.X, axis=0) / np.linalg.norm(B, axis=0)
            tr_o = np.linalg.norm(B - Ad @ ref.X, axis=0) / np.linalg.norm(B, axis=0)
            print(f"   true_res gpu {np.array2string(tr_g, precision=3)}\n   true_res ora {np.array2string(tr_o, precision=3)}"
                  f"\n   hist gpu {np.array2string(r.history[-1], precision=3)}\n   hist ora {np.array2string(ref.history[-1], precision=3)}")
            print(f"p={p} maxit={m:3d} graphs={int(g)} st={r.status_name}/{ref.status_name} it={r.iterations}/{ref.iterations} "
                  f"ev={[(ev['j'], ev['action']) for ev in r.events]} err={e:.2e} best_match=maxit{best}:{near[best]:.1e} "
                  f"cols={np.array2string(colerr, precision=1, max_line_width=200)}", flush=True)
