"""Timeline of one block step in graph mode from the device tracer (BMINRES_TRACE).
usage: python scripts/trace_timeline.py [cfg] [launch] [iters]"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
launch = sys.argv[2] if len(sys.argv) > 2 else "40"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 800
f = os.path.join(tempfile.gettempdir(), "bmr_trace.bin")
os.environ["BMINRES_TRACE"] = launch
os.environ["BMINRES_TRACE_FILE"] = f
import torch, synth
from paper_1301_2102_b200 import DeviceCsr, Solver
P = synth.config(int(cfg))
A = DeviceCsr.from_host(P.A, "cuda:0")
B = torch.from_numpy(P.B).to("cuda:0")
X = torch.zeros_like(B)
with Solver(0, pool_size=1, record_history=False) as s:
    s.solve(A, B, X, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)
    s.solve(A, B, X, tol=P.tol, maxit=iters, deflation_tol=P.tau, history=False)
t = np.fromfile(f, dtype=np.uint64).reshape(7, 1024, -1).astype(np.int64)
names = ["K1", "red1", "K2", "red2", "K3b", "K4b", "K1a"]
pts = ["start", "pt1", "pt2", "pt3", "pt4", "end", "cpart", "tail0", "t_sum", "t_ld", "t_mm", "t_end", "x12", "x13", "x14", "x15"]
t0 = None
rows = []
for k in range(7):
    x = t[k]
    live = x[:, 0] > 0
    if not live.any():
        continue
    x = x[live]
    if t0 is None or x[:, 0].min() < t0:
        t0 = x[:, 0].min()
    rows.append((k, x))
print(f"launch {launch} of each kernel kind (us, relative to the earliest start); per point: min / median / max over CTAs")
for k, x in sorted(rows, key=lambda r: r[1][:, 0].min()):
    cols = []
    for p in range(8):  # (tail-only points printed below)
        v = x[:, p]
        v = v[v > 0]
        if len(v):
            cols.append(f"{pts[p]} {((v.min() - t0) / 1e3):7.2f}/{((np.median(v) - t0) / 1e3):7.2f}/{((v.max() - t0) / 1e3):7.2f}")
    print(f"{names[k]:5s} ctas {len(x):4d} | " + " | ".join(cols))

for k, x in rows:
    tl = x[x[:, 7] > 0]
    for r in tl:
        print(f"{names[k]} tail CTA:", " ".join(f"{pts[p]} {(r[p] - t0) / 1e3:.2f}" for p in range(x.shape[1]) if r[p] > 0))
