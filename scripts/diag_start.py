"""Diagnostic (GPU): one short solve of a config (the start block dominates), for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import synth  # noqa: E402
from paper_1301_2102_b200 import DeviceCsr, Solver  # noqa: E402

P = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
dA = DeviceCsr.from_host(P.A, "cuda:0")
dB = torch.from_numpy(P.B).cuda()
X = torch.zeros_like(dB)
with Solver(0, pool_size=1, record_history=False, use_graphs=False) as s:
    r = s.solve(dA, dB, X, tol=P.tol, maxit=int(sys.argv[2]) if len(sys.argv) > 2 else 1, deflation_tol=P.tau,
                history=False)
torch.cuda.synchronize()
print("events", len(r.events), "it", r.iterations)
