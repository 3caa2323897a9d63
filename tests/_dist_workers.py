"""Worker processes of the row-partition tests (spawned; gloo on 127.0.0.1).

Each worker writes its result as a .npz into the given directory.  Kept importable without a
GPU: the CPU worker only uses the host-only halo planner and the host-callback transport.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port):
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    return dist


def _split(n, world):
    return [n * q // world for q in range(world + 1)]


def _as_ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def plan_worker(rank, world, port, outdir, kind):
    """CPU: the halo plan of this rank's rows + the callback transport (TorchComm over gloo):
    exchange the halo requests and rows, check the local SpMM against the global product, and
    the allreduce against the rank-order sum."""
    dist = _init(rank, world, port)
    import synth
    from paper_1301_2102_b200 import TorchComm, halo_plan
    A = synth.laplacian_3d(7, 6, 5, shift=1.3) if kind == "lap3d" else synth.random_sym_sparse(57, 0.08, seed=3)
    off = _split(A.n, world)
    ip = np.asarray(A.indptr, dtype=np.int64)
    k0, k1 = int(ip[off[rank]]), int(ip[off[rank + 1]])
    cols = np.asarray(A.indices[k0:k1], dtype=np.int32)
    local, halo_rows, cnt = halo_plan(world, rank, off, cols)
    comm = TorchComm()
    # halo requests: how many rows this rank reads from each rank, then which
    one = np.ones(world, dtype=np.int64)
    scnt = np.ascontiguousarray(cnt, dtype=np.int64)
    rcnt = np.zeros(world, dtype=np.int64)
    assert comm.cb.alltoallv(None, _as_ptr(scnt, C.c_int64), _as_ptr(one, C.c_int64), _as_ptr(rcnt, C.c_int64),
                             _as_ptr(one, C.c_int64)) == 0
    req = np.zeros(max(int(rcnt.sum()), 1), dtype=np.int64)
    hr = np.ascontiguousarray(halo_rows, dtype=np.int64)
    if hr.size == 0:
        hr = np.zeros(1, dtype=np.int64)
    assert comm.cb.alltoallv(None, _as_ptr(hr, C.c_int64), _as_ptr(scnt, C.c_int64), _as_ptr(req, C.c_int64),
                             _as_ptr(rcnt, C.c_int64)) == 0
    req = req[:int(rcnt.sum())]
    # the rows of X this rank sends (panel p = 3), exchanged into the halo region
    p = 3
    X = np.random.default_rng(7).standard_normal((A.n, p))
    mine = X[off[rank]:off[rank + 1]]
    send = np.ascontiguousarray(mine[req - off[rank]].reshape(-1)) if len(req) else np.zeros(1)
    recv = np.zeros(max(len(halo_rows) * p, 1))
    sc_d, rc_d = rcnt * p, scnt * p
    assert comm.cb.exchange(None, _as_ptr(send, C.c_double), _as_ptr(np.ascontiguousarray(sc_d), C.c_int64),
                            _as_ptr(recv, C.c_double), _as_ptr(np.ascontiguousarray(rc_d), C.c_int64)) == 0
    Xext = np.vstack([mine, recv[:len(halo_rows) * p].reshape(-1, p)])
    rp = ip[off[rank]:off[rank + 1] + 1] - k0
    Y = np.zeros((off[rank + 1] - off[rank], p))
    vals = np.asarray(A.data[k0:k1])
    for i in range(len(Y)):
        for e in range(rp[i], rp[i + 1]):
            Y[i] += vals[e] * Xext[local[e]]
    dense = synth.csr_to_dense(A)
    ref = (dense @ X)[off[rank]:off[rank + 1]]
    # allreduce: all-gather summed in rank order, identical on every rank
    v = np.random.default_rng(100 + rank).standard_normal(5)
    red = v.copy()
    assert comm.cb.allreduce(None, _as_ptr(red, C.c_double), 5) == 0
    np.savez(os.path.join(outdir, f"plan{rank}.npz"), Y=Y, ref=ref, red=red, v=v, n_halo=len(halo_rows),
             req=req, halo_rows=halo_rows)
    dist.barrier()
    dist.destroy_process_group()


def problem(name):
    """The partition-test problems: BASELINE config 1' (p = 4) and a 3-D Laplacian with p = 8."""
    import synth
    if name == "1c":
        return synth.config("1c")
    if name == "lap3d12p8":
        A = synth.laplacian_3d(12, shift=2.5)
        return synth.Problem("lap3d12p8", A, synth.gaussian_rhs(A.n, 8, seed=1), 1e-10, 4000)
    if name == "slab16":   # z-slabs of a 3-D Laplacian with p = 16, solved in split mode (halo overlap)
        A = synth.laplacian_3d(12, 12, 16, shift=2.5)
        return synth.Problem("slab16", A, synth.gaussian_rhs(A.n, 16, seed=3), 1e-10, 4000)
    if name == "dep2d":   # config 3's recipe (B = [G, G C + eps N], eps = 0) on a small grid: step-0 events
        A = synth.laplacian_2d(20, shift=2.5)
        return synth.Problem("dep2d", A, synth.dependent_rhs(A.n, 4, 0.0, seed=0), 1e-10, 4000)
    if name in ("irr8", "irr16s", "irr32s"):
        # irregular symmetric indefinite matrices (random columns everywhere: every rank reads rows of
        # every other rank, and no run of rows is interior -- config 5's situation on a partition);
        # the "s" problems are solved in split mode (the overlap path with an empty interior)
        p = {"irr8": 8, "irr16s": 16, "irr32s": 32}[name]
        rng = np.random.default_rng(4000 + p)
        A = synth.irregular_sym_csr(1500 + 37 * p, rng, hubs=2, empty_rows=0)
        return synth.Problem(name, A, np.ascontiguousarray(rng.standard_normal((A.n, p))), 0.0, 4000)
    raise ValueError(name)


def solve_worker(rank, world, port, outdir, name, maxit):
    """GPU: a row-partitioned solve of this rank's rows on cuda:0 (host-callback transport)."""
    dist = _init(rank, world, port)
    import torch
    from paper_1301_2102_b200 import DeviceCsr, Solver, TorchComm
    P = problem(name)
    off = _split(P.n, world)
    A = DeviceCsr.rows_from_host(P.A, off[rank], off[rank + 1], "cuda:0")
    B = torch.from_numpy(np.ascontiguousarray(P.B[off[rank]:off[rank + 1]])).to("cuda:0")
    # slab16: split mode (K1a alone, its interior rows overlapping the halo exchange; the update kernel)
    with Solver(0, rank=rank, world=world, comm=TorchComm(),
                split_spmm=1 if name in ("slab16", "irr16s", "irr32s") else 0) as s:
        r = s.solve(A, B, tol=P.tol, maxit=maxit, deflation_tol=P.tau)
        X = r.X.cpu().numpy()
    ev = np.array([[e["j"], e["col"], e["kind"], e["action"]] for e in r.events], dtype=np.int64).reshape(-1, 4)
    np.savez(os.path.join(outdir, f"solve{rank}.npz"), X=X, hist=r.history, it=r.iterations, status=r.status,
             true_res=np.array(r.stats["true_res"]), events=ev)
    dist.barrier()
    dist.destroy_process_group()
