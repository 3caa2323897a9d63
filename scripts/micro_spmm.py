"""Microbenchmark: plain SpMM (bminres_spmm) on a config's matrix vs a torch copy of equal bytes.
Run under ncu for per-kernel device times (python scripts/micro_spmm.py [cfg] [p] [reps])."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1301_2102_b200 import DeviceCsr, Solver

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
P = synth.config(int(cfg) if cfg != "1c" else cfg)
A = DeviceCsr.from_host(P.A, "cuda:0")
n = P.n
X = torch.randn(n, p, dtype=torch.float64, device="cuda:0")
Y = torch.empty_like(X)
big = torch.empty(int(12 * P.A.nnz / 8 + 3 * n * p) // 2, dtype=torch.float64, device="cuda:0")
big2 = torch.empty_like(big)
with Solver(0) as s:
    for _ in range(reps):
        s.spmm(A, X, Y)
        big2.copy_(big)
    torch.cuda.synchronize()
print("ok", n, p, P.A.nnz)
