"""Diagnostic (GPU): solve vs block-loop device time and host wall time per solve (config 2)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import synth  # noqa: E402
from paper_1301_2102_b200 import DeviceCsr, Solver  # noqa: E402

P = synth.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dA = DeviceCsr.from_host(P.A, "cuda:0")
dB = torch.from_numpy(P.B).cuda()
X = torch.zeros_like(dB)
with Solver(0, pool_size=1, record_history=False) as s:
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = s.solve(dA, dB, X, tol=P.tol, maxit=2000, deflation_tol=P.tau, history=False)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        st = r.stats
        print(f"solve {i}: wall {wall:.3f} ms  solve_ms {st['solve_ms']:.3f}  loop_ms {st['loop_ms']:.3f}  "
              f"outside loop {st['solve_ms'] - st['loop_ms']:.3f} ms  it {r.iterations}", flush=True)
