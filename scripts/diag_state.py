"""Diagnostic (GPU): side-branch state at exit (BMINRES_DEBUG_STATE=1) against the oracle's
\\bar H blocks.  Usage: BMINRES_DEBUG_STATE=1 python scripts/diag_state.py p maxit graphs"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from test_gpu_parity import gpu_solve  # noqa: E402

p, m, g = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n = 3 * p
rng = np.random.default_rng(n * 100 + p)
D = rng.standard_normal((n, n))
A = synth.dense_to_csr(D + D.T)
B = rng.standard_normal((n, p))
ref = oracle.solve(A, B, tol=1e-10, maxit=m, debug_iters=m)
H = ref.dbg["H"]   # H[r-1, j-1] = h_{r,j}
np.set_printoptions(precision=6, linewidth=250)
k = (m - 1) // p + 1
print("block", k)
for name, r0, c0 in (("diag A_k", (k - 1) * p, (k - 1) * p), ("C_{k-1}", (k - 1) * p, (k - 2) * p), ("C_k", k * p, (k - 1) * p)):
    blk = np.zeros((p, p))
    for a in range(p):
        for c in range(p):
            j = c0 + c + 1
            if j <= m and r0 + a < H.shape[0]:
                blk[a, c] = H[r0 + a, j - 1]
    print(name, "(rows: u index, cols: iteration)")
    print(blk)
sys.stdout.flush()
r = gpu_solve(A, B, tol=1e-10, maxit=m, use_graphs=bool(g))
print("hist gpu", r.history[-1], "\nhist ora", ref.history[-1], flush=True)
