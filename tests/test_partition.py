"""Row-partitioned solves (world > 1).

CPU (`-m "not gpu"`): the host-only halo planner (bminres_halo_plan through the C ABI) against
the global product on 1..4-way partitions, and the same planner plus the host-callback
transport (TorchComm) across two gloo processes: halo requests and rows exchanged, local SpMM
rows equal to the global A X rows, allreduce identical on both ranks.
GPU (`-m gpu`): a two-rank solve on one B200 (two processes sharing cuda:0, gloo callbacks --
the exchange is host-mediated, so no kernel waits on another process's kernel) matches the
single-rank solve to the parity bar; the NCCL transport at world = 1 (graphs with the
allreduce captured) is bitwise identical to the plain solve.
"""
import os
import socket

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp
    mp.start_processes(fn, args=(world, _free_port()) + args, nprocs=world, join=True, start_method="spawn")


def _local_spmm(A, off, rank, local, halo_rows, X):
    ip = np.asarray(A.indptr, dtype=np.int64)
    k0 = ip[off[rank]]
    Xext = np.vstack([X[off[rank]:off[rank + 1]], X[halo_rows]])
    Y = np.zeros((off[rank + 1] - off[rank], X.shape[1]))
    for i in range(len(Y)):
        for e in range(ip[off[rank] + i] - k0, ip[off[rank] + i + 1] - k0):
            Y[i] += A.data[k0 + e] * Xext[local[e]]
    return Y


@pytest.mark.parametrize("world", [2, 4])
def test_interior_rows_of_z_slabs(world):
    """The overlap's interior (bminres_interior_rows): for z-slabs of a 3-D 7-point stencil
    (nx x ny planes, lexicographic, z slowest) a rank's interior is its slab minus its first plane
    (unless it is rank 0) and its last plane (unless it is the last rank) -- the closed form of the
    rows with no neighbour in another slab; a random matrix has (almost) none."""
    from paper_1301_2102_b200 import halo_plan, interior_rows
    nx, ny, nz = 6, 5, 4 * world
    A = synth.laplacian_3d(nx, ny, nz, shift=1.3)
    plane = nx * ny
    off = [plane * (nz * q // world) for q in range(world + 1)]
    ip = np.asarray(A.indptr, dtype=np.int64)
    for r in range(world):
        k0, k1 = ip[off[r]], ip[off[r + 1]]
        local, _, _ = halo_plan(world, r, off, A.indices[k0:k1])
        lo, hi = interior_rows((ip[off[r]:off[r + 1] + 1] - k0).astype(np.int32), local)
        n_loc = off[r + 1] - off[r]
        assert (lo, hi) == ((plane if r > 0 else 0), (n_loc - plane if r < world - 1 else n_loc))
    B = synth.random_sym_sparse(60, 0.3, seed=2)
    off = [0, 30, 60]
    ip = np.asarray(B.indptr, dtype=np.int64)
    local, _, _ = halo_plan(2, 0, off, B.indices[:ip[30]])
    lo, hi = interior_rows(ip[:31].astype(np.int32), local)
    rows_ok = [all(local[e] < 30 for e in range(ip[i], ip[i + 1])) for i in range(30)]
    assert hi - lo == max((len(run) for run in "".join("1" if x else "0" for x in rows_ok).split("0")), default=0)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["lap3d", "random"])
def test_halo_plan_reproduces_global_product(world, kind):
    from paper_1301_2102_b200 import halo_plan
    A = synth.laplacian_3d(7, 6, 5, shift=1.3) if kind == "lap3d" else synth.random_sym_sparse(57, 0.08, seed=3)
    off = [A.n * q // world for q in range(world + 1)]
    X = np.random.default_rng(1).standard_normal((A.n, 3))
    ref = synth.csr_to_dense(A) @ X
    total_halo = 0
    for r in range(world):
        ip = np.asarray(A.indptr, dtype=np.int64)
        cols = A.indices[ip[off[r]]:ip[off[r + 1]]]
        local, halo_rows, cnt = halo_plan(world, r, off, cols)
        assert np.all(np.diff(halo_rows) > 0), "halo rows ascending (grouped by owner)"
        assert not np.any((halo_rows >= off[r]) & (halo_rows < off[r + 1])), "own rows are not halo"
        assert cnt[r] == 0 and cnt.sum() == len(halo_rows)
        for q in range(world):   # counts per owner
            assert cnt[q] == np.count_nonzero((halo_rows >= off[q]) & (halo_rows < off[q + 1]))
        assert np.array_equal(np.unique(cols[(cols < off[r]) | (cols >= off[r + 1])]), halo_rows)
        np.testing.assert_allclose(_local_spmm(A, off, r, local, halo_rows, X), ref[off[r]:off[r + 1]],
                                   rtol=1e-13, atol=1e-13)
        total_halo += len(halo_rows)
    if world == 1:
        assert total_halo == 0


def test_halo_plan_rejects_bad_columns():
    from paper_1301_2102_b200 import BminresError, halo_plan
    with pytest.raises(BminresError):
        halo_plan(2, 0, [0, 3, 6], np.array([0, 7], dtype=np.int32))


@pytest.mark.parametrize("kind", ["lap3d", "random"])
def test_callback_transport_gloo_world2(tmp_path, kind):
    """Two gloo processes: halo requests / rows through TorchComm, local rows of A X, allreduce."""
    from tests._dist_workers import plan_worker
    _spawn(plan_worker, 2, str(tmp_path), kind)
    r0, r1 = (np.load(tmp_path / f"plan{r}.npz") for r in range(2))
    for r in (r0, r1):
        np.testing.assert_allclose(r["Y"], r["ref"], rtol=1e-13, atol=1e-13)
    assert np.array_equal(r0["red"], r1["red"]), "allreduce must be bitwise identical on every rank"
    np.testing.assert_allclose(r0["red"], r0["v"] + r1["v"], rtol=1e-15)
    # what rank 1 sends rank 0 is exactly what rank 0 reads from rank 1, and vice versa
    assert np.array_equal(np.sort(r1["req"]), r0["halo_rows"][r0["halo_rows"] >= 0])
    assert np.array_equal(np.sort(r0["req"]), r1["halo_rows"])


# ----------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name,maxit", [("1c", 120), ("lap3d12p8", 160)])
def test_two_rank_solve_matches_single_rank(tmp_path, name, maxit):
    import torch
    from tests._dist_workers import problem, solve_worker
    from paper_1301_2102_b200 import DeviceCsr, Solver
    _spawn(solve_worker, 2, str(tmp_path), name, maxit)
    parts = [np.load(tmp_path / f"solve{r}.npz") for r in range(2)]
    P = problem(name)
    with Solver(0) as s:
        ref = s.solve(DeviceCsr.from_host(P.A, "cuda:0"), torch.from_numpy(P.B).to("cuda:0"), tol=P.tol,
                      maxit=maxit, deflation_tol=P.tau)
    Xref = ref.X.cpu().numpy()
    for d in parts:
        assert int(d["it"]) == ref.iterations and int(d["status"]) == ref.status
        k = min(51, len(ref.history))
        h, hr = d["hist"][:k], ref.history[:k]
        assert np.all(np.abs(h - hr) <= 1e-9 * np.abs(hr) + 1e-14), np.max(np.abs(h - hr) / np.abs(hr))
        np.testing.assert_allclose(d["true_res"], ref.stats["true_res"], rtol=1e-6, atol=1e-13)
    assert np.array_equal(parts[0]["hist"], parts[1]["hist"]), "replicated QR: identical histories on all ranks"
    X = np.vstack([parts[0]["X"], parts[1]["X"]])
    np.testing.assert_allclose(X, Xref, rtol=1e-7, atol=1e-9 * np.abs(Xref).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name,maxit,world", [("1c", 120, 2), ("lap3d12p8", 160, 2), ("dep2d", 200, 2), ("slab16", 192, 2),
                                               ("irr8", 64, 2), ("irr16s", 96, 2), ("irr32s", 128, 2),
                                               ("slab16", 96, 3), ("irr16s", 64, 3)])
def test_two_rank_solve_matches_oracle(tmp_path, name, maxit, world):
    """(world = 3: uneven row blocks, a middle rank with two neighbours; irr*: irregular matrices whose
    rows read every other rank and leave no interior run.)
    Row a6 against the ORACLE (not the single-rank GPU solve): the 2-rank partitioned solve
    (halo exchange + allreduces, replicated small QR, the block factored once per rank after the
    allreduce) gives the oracle's residual history to 1e-9 over the first 50 iterations, its
    iteration count and status, its dependence events (dep2d: step-0 replacements of columns 5-8)
    and its X.  slab16: z-slabs in split mode -- K1a's interior rows run before the halo lands, the
    boundary rows after it."""
    import oracle
    from tests._dist_workers import problem, solve_worker
    _spawn(solve_worker, world, str(tmp_path), name, maxit)
    parts = [np.load(tmp_path / f"solve{r}.npz") for r in range(world)]
    P = problem(name)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=maxit, tau=P.tau, pool_size=1)
    ref_ev = [[e["j"], e["col"], e["kind"], e["action"]] for e in ref.events]
    if name == "dep2d":
        assert [e[:2] for e in ref_ev] == [[0, 5], [0, 6], [0, 7], [0, 8]]
    for d in parts:
        assert int(d["it"]) == ref.iterations and int(d["status"]) == ref.status
        k = min(51, len(ref.history))
        h, hr = d["hist"][:k], ref.history[:k]
        assert np.all(np.abs(h - hr) <= 1e-9 * np.abs(hr) + 1e-14), np.max(np.abs(h - hr) / np.abs(hr))
        assert d["events"].tolist() == ref_ev
        np.testing.assert_allclose(d["true_res"], ref.true_res, rtol=1e-6, atol=1e-13)
    X = np.vstack([d["X"] for d in parts])
    atol = 1e-9 * np.abs(ref.X).max()
    if name.startswith("irr"):   # (hub rows: see test_seeded_sweep_irregular_matrices)
        sens = oracle.solve(P.A, P.B * (1.0 + np.random.default_rng(0).integers(-1, 2, P.B.shape) * 2.0 ** -52),
                            tol=P.tol, maxit=maxit, tau=P.tau, pool_size=1)
        atol += 50.0 * np.abs(sens.X - ref.X).max()
    np.testing.assert_allclose(X, ref.X, rtol=1e-7, atol=atol)


@pytest.mark.gpu
@pytest.mark.parametrize("p,one_comm", [(4, False), (8, False), (8, True)])
def test_nccl_transport_world1_bitwise(p, one_comm, monkeypatch):
    """The partition path with the NCCL transport (allreduce / exchange captured in the graphs) at
    world = 1 gives bitwise the plain solve's results (a 1-rank sum is exact).  The halo exchange
    has a communicator of its own (ncclCommSplit); one_comm: shared."""
    import torch
    if one_comm:
        monkeypatch.setenv("BMINRES_NCCL_ONE_COMM", "1")
    from paper_1301_2102_b200 import DeviceCsr, Solver
    A = synth.laplacian_3d(14, shift=2.5)
    B = synth.gaussian_rhs(A.n, p, seed=2)
    dA, dB = DeviceCsr.from_host(A, "cuda:0"), torch.from_numpy(B).to("cuda:0")
    with Solver(0) as s:
        r0 = s.solve(dA, dB, tol=1e-10, maxit=300)
    with Solver(0, comm="nccl") as s:
        r1 = s.solve(dA, dB, tol=1e-10, maxit=300)
    assert r0.iterations == r1.iterations
    assert np.array_equal(r0.history, r1.history)
    assert torch.equal(r0.X, r1.X)
