"""K3b (small banded QR) phase times from the device tracer: prologue (factor), the serial chain
(warp 0: phase A reflectors + phase B), the stores.  usage: python scripts/trace_k3b.py P [launch]"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
p = int(sys.argv[1]) if len(sys.argv) > 1 else 32
launch = sys.argv[2] if len(sys.argv) > 2 else "20"
f = os.path.join(tempfile.gettempdir(), "bmr_trace_k3b.bin")
os.environ["BMINRES_TRACE"] = launch
os.environ["BMINRES_TRACE_FILE"] = f
import torch, synth
from paper_1301_2102_b200 import DeviceCsr, Solver
if os.environ.get("K3B_CFG3"):   # config 3's problem (2-D 512^2, dependent right-hand sides, eps = 0)
    pr = synth.config(3)
    A, B = pr.A, pr.B
else:
    A = synth.laplacian_3d(40, shift=3.0)
    B = synth.gaussian_rhs(A.n, p, seed=1)
dA, dB = DeviceCsr.from_host(A, "cuda:0"), torch.from_numpy(B).to("cuda:0")
res = []
for graphs in (False, True):
    with Solver(0, pool_size=1, record_history=False, use_graphs=graphs) as s:
        s.solve(dA, dB, tol=0.0, maxit=40 * p, history=False)
    t = np.fromfile(f, dtype=np.uint64).reshape(7, 1024, -1).astype(np.int64)
    x = t[4, 0]
    # points: 0 begin, 2 prologue (factor) done, 4 phase A done, 3 phase B + R^-1 done, 6 stores +
    # update factors done, 7 Q_k accumulated, 5 end
    seq = [(0, "begin"), (2, "prologue+factor"), (4, "load+H+phaseA"), (3, "phaseB+Rinv"), (6, "stores+uf"),
           (7, "Qacc"), (5, "tail")]
    parts = []
    for (a, _), (b, name) in zip(seq, seq[1:]):
        parts.append(f"{name} {(x[b] - x[a]) / 1e3:.1f}")
    print(f"p={p} graphs={graphs}: " + ", ".join(parts) + f" us; total {(x[5] - x[0]) / 1e3:.1f} us")
    if os.environ.get("K3B_PROF"):   # (library built with -DK3B_PROF: phase-B cycle sums in CTA 1's slot)
        c = t[4, 1][:6]
        print("   phase B cycles: (loop tail)+x2+sum %d, dlarfg %d, vj+sH %d, cols+T+max %d, tail-of-loop %d, Rinv %d" % tuple(c))
