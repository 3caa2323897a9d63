"""Parity of the CUDA path (through the C ABI) with the CPU oracle — needs a B200.

Bars (north star, BASELINE.json): per-iteration residual histories agree to relative
1e-9 over the first 50 iterations; iteration counts within +-2% or +-2; dependence events
at the same steps; final true residual <= tol where the problem allows it.  Integer /
bit-level work (the SpMM summation order, the replacement RNG) is compared bitwise.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

HIST_RTOL = 1e-9
HIST_ATOL = 1e-14   # residuals that are rounding noise (e.g. a converged column at 1e-17)


def _torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def solver():
    from paper_1301_2102_b200 import Solver
    s = Solver(0, pool_size=1)
    yield s
    s.close()


def gpu_solve(A, B, *, pool_size=1, use_graphs=True, X0=None, split_spmm=0, timing=False, policy=0, **kw):
    torch = _torch()
    from paper_1301_2102_b200 import DeviceCsr, Solver
    dA = DeviceCsr.from_host(A, "cuda:0")
    dB = torch.from_numpy(np.ascontiguousarray(B)).to("cuda:0")
    X = None if X0 is None else torch.from_numpy(np.ascontiguousarray(X0)).to("cuda:0")
    with Solver(0, pool_size=pool_size, use_graphs=use_graphs, use_x0=X0 is not None, split_spmm=split_spmm,
                timing=timing, policy=policy) as s:
        r = s.solve(dA, dB, X, raise_on_error=False, **kw)
    r.X = r.X.cpu().numpy()
    return r


def assert_hist_close(h_gpu, h_ref, upto=50, rtol=HIST_RTOL):
    k = min(upto + 1, len(h_gpu), len(h_ref))
    a, b = h_gpu[:k], h_ref[:k]
    bad = np.abs(a - b) > rtol * np.abs(b) + HIST_ATOL
    assert not bad.any(), f"history mismatch at {np.argwhere(bad)[:5].tolist()}: " \
                          f"max rel {np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)):.3e}"


def assert_counts_close(it_gpu, it_ref):
    assert abs(it_gpu - it_ref) <= max(2, 0.02 * it_ref), (it_gpu, it_ref)


def same_events(eg, er):
    key = lambda e: (e["j"], e["col"], e["kind"], e["action"])
    assert [key(e) for e in eg] == [key(e) for e in er], (eg, er)


# ----------------------------------------------------------------------------- component parity


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 16, 32])
def test_spmm_bitwise(solver, p):
    """Row a1's SpMM: each output row summed over the CSR row in stored order with fma — bitwise."""
    torch = _torch()
    from paper_1301_2102_b200 import DeviceCsr
    for A in (synth.laplacian_3d(13, 11, 9, shift=3.0), synth.random_sym_sparse(777, 0.02, seed=p)):
        X = np.random.default_rng(p).standard_normal((A.n, p))
        Y = solver.spmm(DeviceCsr.from_host(A, "cuda:0"), torch.from_numpy(X).cuda()).cpu().numpy()
        np.testing.assert_array_equal(Y, oracle.csr_block(A, X))


@pytest.mark.parametrize("cfg,p", [(2, 8), (3, 16)])
def test_spmm_full_size_bitwise(solver, cfg, p):
    torch = _torch()
    from paper_1301_2102_b200 import DeviceCsr
    A = synth.laplacian_3d(64, shift=3.0) if cfg == 2 else synth.laplacian_2d(512, shift=2.5)
    X = np.random.default_rng(1).standard_normal((A.n, p))
    Y = solver.spmm(DeviceCsr.from_host(A, "cuda:0"), torch.from_numpy(X).cuda()).cpu().numpy()
    np.testing.assert_array_equal(Y, oracle.csr_block(A, X))


def test_random_vector_bitwise(solver):
    """Reading C17: the replacement vectors are an integer hash -> bitwise equal to the oracle's."""
    torch = _torch()
    n = 5000
    out = torch.empty(n, dtype=torch.float64, device="cuda:0")
    for (seed, stream, event, rb) in ((0, 0, 0, 0), (0, 1, 3, 0), (7, 1, 2, 123456)):
        solver.random_vector(seed, stream, event, rb, n, out)
        want = np.array([oracle.rand_entry(seed, stream, event, rb + i) for i in range(n)])
        np.testing.assert_array_equal(out.cpu().numpy(), want)


# ----------------------------------------------------------------------------- solve parity


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 16, 32])
def test_history_parity_small(p):
    A = synth.laplacian_2d(40, 37, shift=1.7)
    B = synth.gaussian_rhs(A.n, p, seed=p)
    r = gpu_solve(A, B, tol=0.0, maxit=60)
    ref = oracle.solve(A, B, tol=0.0, maxit=60)
    assert r.status_name == ref.status_name == "MAXIT"
    assert r.iterations == ref.iterations == 60
    assert_hist_close(r.history, ref.history)
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())


@pytest.mark.parametrize("p", [8, 16, 32])
def test_split_mode_bitwise(p, monkeypatch):
    """Split mode (K1a computes A V_k alone, K1 streams it) sums every row
    in the same CSR order as the fused K1's gathers: graph, plain-launch and timing-mode solves are
    bitwise identical to the fused path, and match the oracle (ragged tail: n = 40*37 rows).
    (the warp-specialised K1, an option: test_warp_specialised_k1)"""
    A = synth.laplacian_2d(40, 37, shift=1.7)
    B = synth.gaussian_rhs(A.n, p, seed=p)
    base = gpu_solve(A, B, tol=0.0, maxit=120, split_spmm=2)
    ref = oracle.solve(A, B, tol=0.0, maxit=120)
    assert_hist_close(base.history, ref.history)
    for kw in (dict(use_graphs=True), dict(use_graphs=False), dict(use_graphs=False, timing=True)):
        r = gpu_solve(A, B, tol=0.0, maxit=120, split_spmm=1, **kw)
        assert r.iterations == base.iterations == 120
        np.testing.assert_array_equal(r.history, base.history)
        np.testing.assert_array_equal(r.X, base.X)
        if kw.get("timing"):
            assert r.stats["phase_launches"]["spmm_av"] > 0
            assert r.stats["phase_launches"]["spmm_fused"] == 0
            # p >= 16: the M/X update runs as its own register-blocked kernel (k1u_update), bitwise
            # the fused update of the other mode
            assert (r.stats["phase_launches"]["update_main"] > 0) == (p >= 16)


@pytest.mark.parametrize("p", [16, 32])
def test_warp_specialised_k1(p):
    """The warp-specialised K1 (k1_ws: gathers in producer warps, the DMMA epilogue in consumer
    warps, no A V_k panel) in split mode: W per row is bitwise the split pair's (same CSR order, same
    DMMA order per output); the Gram partials are summed over a different row partition, so the
    solve equals the K1a + K1 pair to rounding and the oracle to the parity bar -- graphs, plain
    launches and timing mode (where it is the only K1 launch kind)."""
    import os
    A = synth.laplacian_2d(40, 37, shift=1.7)
    B = synth.gaussian_rhs(A.n, p, seed=p)
    ref = oracle.solve(A, B, tol=0.0, maxit=120)
    pair = gpu_solve(A, B, tol=0.0, maxit=120, split_spmm=1)
    for kw in (dict(use_graphs=True), dict(use_graphs=False), dict(use_graphs=False, timing=True)):
        os.environ["BMINRES_WS"] = "1"   # (an option: measured slower than the K1a + K1 pair)
        try:
            r = gpu_solve(A, B, tol=0.0, maxit=120, split_spmm=1, **kw)
        finally:
            del os.environ["BMINRES_WS"]
        assert r.iterations == 120
        assert_hist_close(r.history, ref.history)
        np.testing.assert_allclose(r.history, pair.history, rtol=1e-11, atol=1e-15)
        np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())
        if kw.get("timing"):
            assert r.stats["phase_launches"]["spmm"] > 0 and r.stats["phase_launches"]["spmm_av"] == 0


@pytest.mark.parametrize("p,maxit", [(8, 120), (8, 128), (16, 144), (32, 160)])
def test_deferred_x_update_bitwise(p, maxit, monkeypatch):
    """The fused update defers X in pairs (X += M_{k-1}Z_{k-1} + M_k Z_k in one pass, DESIGN.md
    "Deferred X update"; the host flushes an unpaired last block): bitwise the per-block updates,
    for block counts of both parities and in split mode."""
    A = synth.laplacian_2d(40, 37, shift=1.7)
    B = synth.gaussian_rhs(A.n, p, seed=p + 1)
    r1 = gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=1 if p == 16 else 0)
    monkeypatch.setenv("BMINRES_NO_XDEFER", "1")
    r0 = gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=1 if p == 16 else 0)
    assert r1.iterations == r0.iterations == maxit
    np.testing.assert_array_equal(r1.history, r0.history)
    np.testing.assert_array_equal(r1.X, r0.X)


def test_companion_converges_like_oracle():
    """Config 1' (non-singular companion): counts within +-2%, true residual <= tol."""
    P = synth.config("1c")
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=P.maxit)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=P.maxit)
    assert r.status_name == ref.status_name == "OK"
    assert_counts_close(r.iterations, ref.iterations)
    assert_hist_close(r.history, ref.history)
    assert max(r.stats["true_res"]) <= P.tol * 1.5


def test_config1_singular():
    """Config 1 is singular: both run to maxit; histories agree over 50 iterations;
    the residual reaches the null-space floor (pin P14)."""
    P = synth.config(1)
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=P.maxit)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=P.maxit)
    assert r.status_name == ref.status_name == "MAXIT"
    assert r.iterations == ref.iterations == P.maxit
    assert_hist_close(r.history, ref.history)
    np.testing.assert_allclose(r.history[1100], [0.04458, 0.03019, 0.003486, 0.01999], rtol=1e-3)


def test_x0_path():
    P = synth.config("1c")
    X0 = np.random.default_rng(3).standard_normal(P.B.shape) * 0.1
    r = gpu_solve(P.A, P.B, X0=X0, tol=0.0, maxit=40)
    ref = oracle.solve(P.A, P.B, X0=X0, tol=0.0, maxit=40)
    assert_hist_close(r.history, ref.history)
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-8, atol=1e-10)


# ----------------------------------------------------------------------------- dependence handling


def test_fig3_dependence_at_first_iteration():
    """Fig. 3: B = [e1, A e1] -> exact dependence at j = 1, system 2 converged."""
    P = synth.config(1)
    D = synth.csr_to_dense(P.A)
    e1 = np.zeros(P.n)
    e1[0] = 1.0
    B = np.stack([e1, D @ e1], axis=1)
    r = gpu_solve(P.A, B, tol=1e-8, maxit=300, pool_size=1)
    ref = oracle.solve(P.A, B, tol=1e-8, maxit=300, pool_size=1)
    same_events(r.events, ref.events)
    assert r.events[0]["j"] == 1
    assert_hist_close(r.history, ref.history)
    assert r.history[1:, 1].max() < 1e-14


def test_step0_deflation_events():
    """Config-3 recipe (small): step-0 events for the dependent columns, as the oracle."""
    A = synth.laplacian_2d(30, shift=2.5)
    for eps in (0.0, 1e-10, 1e-6):
        B = synth.dependent_rhs(A.n, 4, eps, seed=0)
        r = gpu_solve(A, B, tol=1e-8, maxit=80)
        ref = oracle.solve(A, B, tol=1e-8, maxit=80)
        same_events(r.events, ref.events)
        assert_hist_close(r.history, ref.history)


def test_near_dependence_retention():
    """Near dependence (1e-12 < h/omega <= tau): replaced + retained for 2p iterations."""
    P = synth.config("1c")
    D = synth.csr_to_dense(P.A)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(P.n)
    B = np.stack([b, D @ b + 1e-10 * rng.standard_normal(P.n)], axis=1)
    r = gpu_solve(P.A, B, tol=1e-8, maxit=30, pool_size=1)
    ref = oracle.solve(P.A, B, tol=1e-8, maxit=30, pool_size=1)
    same_events(r.events, ref.events)
    assert r.events[0]["action"] == 2
    # The retained vector v = w/h is the normalised remainder of a cancellation of relative
    # size h/omega ~ 4e-11: any two correct implementations (CGS vs MGS order) agree on v only
    # to eps_mach/(h/omega) ~ 6e-6, and the histories to about that (reading R3).
    ratio = r.events[0]["ratio"]
    assert_hist_close(r.history, ref.history, upto=30, rtol=10 * 2.2e-16 / ratio)


def test_block_grade_stall():
    """Pin P9 on the GPU: dependent candidates at j = (d-1)p+1..dp, convergence at dp."""
    d, p, mult = 4, 2, 10
    A = synth.diag_csr(np.repeat([-2.0, -0.5, 1.0, 3.0], mult))
    B = np.random.default_rng(9).standard_normal((d * mult, p))
    r = gpu_solve(A, B, tol=1e-12, maxit=40, pool_size=p)
    ref = oracle.solve(A, B, tol=1e-12, maxit=40, pool_size=p)
    same_events(r.events, ref.events)
    assert r.status_name == ref.status_name == "OK" and r.iterations == ref.iterations == d * p


def test_pool_exhausted():
    P = synth.config(1)
    D = synth.csr_to_dense(P.A)
    e1 = np.zeros(P.n)
    e1[0] = 1.0
    B = np.stack([e1, D @ e1], axis=1)
    r = gpu_solve(P.A, B, tol=1e-8, maxit=10, pool_size=0)
    ref = oracle.solve(P.A, B, tol=1e-8, maxit=10, pool_size=0)
    assert r.status_name == ref.status_name == "EPOOL"
    assert r.iterations == ref.iterations == 1


def test_predicted_dependence_steps():
    """Pin P8 on the GPU: B = [b, A^t b] -> first event at j = 2t-1."""
    for t in (1, 2, 3):
        rng = np.random.default_rng(40 + t)
        n = 12
        M = rng.integers(-3, 4, (n, n))
        Aint = np.triu(M) + np.triu(M, 1).T
        b = rng.integers(-2, 3, n)
        bt = b.copy()
        for _ in range(t):
            bt = Aint @ bt
        B = np.stack([b, bt], axis=1).astype(float)
        A = synth.dense_to_csr(Aint.astype(float))
        r = gpu_solve(A, B, tol=0.0, maxit=2 * t + 1, pool_size=2)
        assert r.events and r.events[0]["j"] == 2 * t - 1


# ----------------------------------------------------------------------------- full-size configs


def test_config2_first_50():
    """Config 2 (BASELINE configs[1], the bench workload) at full size: 50 iterations vs oracle."""
    P = synth.config(2)
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=50)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=50)
    assert r.iterations == ref.iterations == 50
    assert_hist_close(r.history, ref.history)
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())


@pytest.mark.parametrize("eps", [0.0, 1e-10, 1e-6])
def test_config3_first_50(eps):
    """Config 3 (dependent RHS, BASELINE configs[2]) at full size: step-0 events + 50 iterations."""
    P = synth.config(3, eps=eps)
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=50)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=50)
    same_events(r.events, ref.events)
    assert len([e for e in r.events if e["j"] == 0]) == (8 if eps < 1e-8 else 0)
    assert_hist_close(r.history, ref.history)


def test_start_column_path_variants(monkeypatch):
    """The start block's column path runs as one cooperative launch on a single rank and as
    per-pass k_colstep launches otherwise (row partitions): both against the oracle on config
    3's dependent right-hand sides (8 step-0 replacements), and against each other."""
    P = synth.config(3, eps=1e-10)
    ref = oracle.solve(P.A, P.B, tol=P.tol, maxit=50)
    r1 = gpu_solve(P.A, P.B, tol=P.tol, maxit=50)
    monkeypatch.setenv("BMINRES_NO_COOP_START", "1")
    r2 = gpu_solve(P.A, P.B, tol=P.tol, maxit=50)
    for r in (r1, r2):
        same_events(r.events, ref.events)
        assert_hist_close(r.history, ref.history)
    np.testing.assert_allclose(r1.X, r2.X, rtol=1e-9, atol=1e-12 * np.abs(r1.X).max())


# ----------------------------------------------------------------------------- API properties


def test_graphs_plain_and_host_pointers_bitwise():
    """Graph replay, plain launches and the host-pointer (e2e) path give bitwise-identical results."""
    from paper_1301_2102_b200 import Solver
    P = synth.config("1c")
    r1 = gpu_solve(P.A, P.B, tol=0.0, maxit=100, use_graphs=True)
    r2 = gpu_solve(P.A, P.B, tol=0.0, maxit=100, use_graphs=False)
    with Solver(0) as s:
        r3 = s.solve(P.A, P.B, np.zeros_like(P.B), tol=0.0, maxit=100)
    np.testing.assert_array_equal(r1.history, r2.history)
    np.testing.assert_array_equal(r1.X, r2.X)
    np.testing.assert_array_equal(r1.X, r3.X)


def test_converged_mid_graph_bitwise():
    """A solve that converges inside a graph (25 block steps per graph: the main branch runs on
    past the stop until the host has synchronised): graphs give the plain launches' X, history
    and counts bitwise, and the oracle's to the parity tolerance."""
    P = synth.config("1c")
    r1 = gpu_solve(P.A, P.B, tol=1e-6, maxit=4000, use_graphs=True)
    r2 = gpu_solve(P.A, P.B, tol=1e-6, maxit=4000, use_graphs=False)
    ref = oracle.solve(P.A, P.B, tol=1e-6, maxit=4000)
    assert r1.status_name == "OK" and ref.status_name == "OK"
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.history, r2.history)
    np.testing.assert_array_equal(r1.X, r2.X)
    assert_counts_close(r1.iterations, ref.iterations)
    assert_hist_close(r1.history, ref.history)


def test_host_pointers_full_size_bitwise():
    """Host A / B / X at config 2's full size (A staged on its own stream beside the start block):
    bitwise the device-pointer path, also for a second solve on the same handle with a different
    matrix (the staged copy must land before the first SpMM of each solve)."""
    from paper_1301_2102_b200 import Solver
    P = synth.config(2)
    A2 = synth.Csr(P.A.n, P.A.indptr, P.A.indices, P.A.data * 1.5)
    ref1 = gpu_solve(P.A, P.B, tol=0.0, maxit=48)
    ref2 = gpu_solve(A2, P.B, tol=0.0, maxit=48)
    with Solver(0) as s:
        r1 = s.solve(P.A, P.B, np.zeros_like(P.B), tol=0.0, maxit=48)
        r2 = s.solve(A2, P.B, np.zeros_like(P.B), tol=0.0, maxit=48)
    np.testing.assert_array_equal(ref1.X, r1.X)
    np.testing.assert_array_equal(ref2.X, r2.X)
    np.testing.assert_array_equal(ref1.history, r1.history)


def test_host_pointers_with_x0_bitwise():
    """Host A / B / X with X0 given (use_x0: the start block needs A, so A is staged on the solver
    stream before it): bitwise the device-pointer path."""
    from paper_1301_2102_b200 import Solver
    P = synth.config(2)
    X0 = synth.gaussian_rhs(P.B.shape[0], P.B.shape[1], seed=11) * 0.1
    ref = gpu_solve(P.A, P.B, X0=X0, tol=0.0, maxit=40)
    Xh = X0.copy()
    with Solver(0, use_x0=True) as s:
        r = s.solve(P.A, P.B, Xh, tol=0.0, maxit=40)
    np.testing.assert_array_equal(ref.X, r.X)
    np.testing.assert_array_equal(ref.history, r.history)


def test_invalid_arguments():
    P = synth.config("1c")
    assert gpu_solve(P.A, np.ones((P.n, 9)), tol=1e-8, maxit=10).status_name == "EINVAL"  # p = 9 not compiled
    assert gpu_solve(P.A, P.B, tol=float("nan"), maxit=10).status_name == "EINVAL"


# ----------------------------------------------------------------------------- degenerate inputs


def _same_as_oracle(A, B, *, tol, maxit, compare_x=True, **kw):
    r = gpu_solve(A, B, tol=tol, maxit=maxit, **kw)
    ref = oracle.solve(A, B, tol=tol, maxit=maxit)
    assert r.status_name == ref.status_name, (r.status_name, ref.status_name)
    assert r.iterations == ref.iterations
    if ref.status_name != "EINVAL":
        assert_hist_close(r.history, ref.history)
        same_events(r.events, ref.events)
        if compare_x:
            np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * max(np.abs(ref.X).max(), 1.0))
    return r, ref


def test_zero_rhs_column():
    """A zero right-hand side column: ||b_i|| = 0 counts as converged (reading C7) and its start
    column is a step-0 exact event replaced by a random vector (C13, C17)."""
    A = synth.laplacian_2d(40, 37, shift=1.7)
    B = synth.gaussian_rhs(A.n, 4, seed=3)
    B[:, 2] = 0.0
    _same_as_oracle(A, B, tol=1e-8, maxit=120)


def test_all_zero_rhs_and_maxit_zero():
    """B = 0 converges at the start (X = 0, no iterations); maxit = 0 returns MAXIT at once."""
    A = synth.laplacian_2d(40, 37, shift=1.7)
    r, _ = _same_as_oracle(A, np.zeros((A.n, 4)), tol=1e-8, maxit=100)
    assert r.iterations == 0 and not np.any(r.X)
    _same_as_oracle(A, synth.gaussian_rhs(A.n, 4, seed=1), tol=1e-8, maxit=0)


@pytest.mark.parametrize("use_graphs", [True, False])
def test_mid_solve_breakdown_then_graphs_x(use_graphs):
    """An exact dependence at j = 9 (B = [b, A^2 b, ...], p = 8): the column path replaces the
    vector from the pool, then 49 more block steps run (graph mode: fused updates).  X must match
    the oracle -- this caught in-flight K1 launches re-applying the last fused update after the
    breakdown (fixed: K2 advances k_main while the main branch is stopped)."""
    A = synth.laplacian_2d(40, 37, shift=1.7)
    D = synth.csr_to_dense(A)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(A.n)
    B = np.stack([b, D @ (D @ b)] + [rng.standard_normal(A.n) for _ in range(6)], axis=1)
    r, ref = _same_as_oracle(A, B, tol=1e-10, maxit=400, use_graphs=use_graphs)
    assert [(e["j"], e["action"]) for e in r.events] == [(9, 1)]


@pytest.mark.parametrize("n,p", [(1, 1), (8, 8), (5, 8), (24, 8), (40, 16)])
def test_tiny_systems(n, p):
    """n = 1; n = p (the block Krylov space is exhausted after one block -> EPOOL);
    n < p (EINVAL, as the oracle); a few blocks on a dense random symmetric indefinite matrix."""
    rng = np.random.default_rng(n * 100 + p)
    D = rng.standard_normal((n, n))
    A = synth.dense_to_csr(D + D.T)
    B = rng.standard_normal((n, p))
    _same_as_oracle(A, B, tol=1e-10, maxit=60)


@pytest.mark.parametrize("use_graphs", [True, False])
@pytest.mark.parametrize("p", [4, 7, 8])
def test_solve_ends_inside_column_path_block(p, use_graphs):
    """Dense n = 3p: the Krylov space is exhausted at j = 2p+1 (exact dependence, replaced by the
    pool vector) and the pool at j = 2p+2 (EPOOL).  The solve ends inside the block the
    column path handled -- at maxit = 2p+1 and at the EPOOL exit -- and X, history and events
    must match the oracle's.  (Regression: K3b's prologue scratch, holding the host's C_k here,
    overlaps its reflector ring and had no barrier before the ring load, so reflectors of the two
    previous blocks could be overwritten -- X off by up to 0.75 relative at p = 7.)"""
    n = 3 * p
    rng = np.random.default_rng(n * 100 + p)
    D = rng.standard_normal((n, n))
    A = synth.dense_to_csr(D + D.T)
    B = rng.standard_normal((n, p))
    for maxit in (2 * p + 1, 60):
        _same_as_oracle(A, B, tol=1e-10, maxit=maxit, use_graphs=use_graphs)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 16, 32])
def test_exhausted_krylov_space_sweep(p):
    """Every compiled p: dense symmetric indefinite n x n systems with n = 3p+1 and 4p-1, whose
    block Krylov space is exhausted mid-solve (exact dependences replaced from the pool, then
    EPOOL or convergence), ending at maxit = n-p+1 (inside the column-path block) and
    at the natural exit; graphs and plain launches.  Status, counts, events, history and X as
    the oracle's (scripts/diag_sweep.py is the wider diagnostic version)."""
    for n in ((3, 5) if p == 1 else (3 * p + 1, 4 * p - 1)):
        rng = np.random.default_rng(n * 1000 + p)
        D = rng.standard_normal((n, n))
        A = synth.dense_to_csr(D + D.T)
        B = rng.standard_normal((n, p))
        for maxit in (n - p + 1, 4 * n):
            for g in (True, False):
                _same_as_oracle(A, B, tol=1e-10, maxit=maxit, use_graphs=g)


# ----------------------------------------------------------------------------- configs 4 and 5 at full size


def _p6_closed_form(A, B, jmax):
    """Pin P6: for j <= p (no step-0 deflation) X_j lies in span(B(:, 1..j)), so column i's
    relative residual is min_y ||b_i - A B(:,1:j) y|| / ||b_i|| (a tall-skinny least squares)."""
    import scipy.sparse as sp
    S = sp.csr_matrix((A.data, A.indices, A.indptr), shape=(A.n, A.n))
    AB = np.asarray(S @ B[:, :jmax])
    beta2 = np.einsum("ij,ij->j", B, B)
    out = []
    for j in range(1, jmax + 1):
        Q, _ = np.linalg.qr(AB[:, :j])
        proj = Q.T @ B
        out.append(np.sqrt(np.maximum(beta2 - np.einsum("ij,ij->j", proj, proj), 0.0) / beta2))
    return np.array(out)


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_config_closed_form_and_invariants(cfg):
    """Configs 4 (3-D 256^3, p = 32, n = 16.8M) and 5 (unstructured, n = 4.19M, p = 16) at full
    size: iterations 1..4 against the P6 closed form, monotone histories (P3), and the computed
    residual equal to the true residual (P4) after 200 iterations."""
    P = synth.config(cfg)
    r = gpu_solve(P.A, P.B, tol=0.0, maxit=200, deflation_tol=P.tau)
    assert r.iterations == 200 and r.status_name == "MAXIT"
    ref = _p6_closed_form(P.A, P.B, 4)
    np.testing.assert_allclose(r.history[1:5], ref, rtol=1e-9, atol=1e-14)
    h = r.history
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12) + 1e-15), "residual histories must not increase (P3)"
    np.testing.assert_allclose(r.stats["comp_res"], r.stats["true_res"], rtol=0, atol=1e-8)


# ----------------------------------------------------------------------------- round-2 parity gaps


def _golden(name):
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_config_first_50_vs_oracle(cfg):
    """Configs 4 (3-D 256^3, p = 32) and 5 (unstructured n = 4.19M, p = 16) at full size and in the
    bench's launch configuration (graphs, split mode): the first 50 iterations' residual histories
    to 1e-9 and the events against the oracle's (tests/golden/*_first50.json, written by
    scripts/make_golden.py from oracle.solve only)."""
    P = synth.config(cfg)
    g = _golden(f"{P.name}_first50.json")
    assert g["n"] == P.n and g["p"] == P.p and g["nnz"] == P.A.nnz
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=50, deflation_tol=P.tau)
    assert r.iterations == g["iterations"] == 50 and r.status == g["status"]
    assert_hist_close(r.history, np.array(g["history"]))
    same_events(r.events, g["events"])
    np.testing.assert_allclose(r.stats["true_res"], g["true_res"], rtol=1e-8)


@pytest.mark.parametrize("cfg,N", [(4, 160), (5, 320)])
def test_full_size_config_first_blocks_vs_oracle(cfg, N):
    """As test_full_size_config_first_50_vs_oracle over 5 block steps of config 4 (160 iterations at
    p = 32) and 20 of config 5 (320 at p = 16) -- past the start-up blocks, into the steady-state
    kernels of the bench's launch configuration (graphs of both parities, the separate update kernel
    with its paired X updates, two previous blocks' reflectors): EVERY iteration's residuals to 1e-9
    against the oracle's golden history (tests/golden/*_first<N>.json, oracle.solve only)."""
    P = synth.config(cfg)
    g = _golden(f"{P.name}_first{N}.json")
    assert g["n"] == P.n and g["p"] == P.p and g["nnz"] == P.A.nnz
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=N, deflation_tol=P.tau)
    assert r.iterations == g["iterations"] == N and r.status == g["status"]
    assert_hist_close(r.history, np.array(g["history"]), upto=N)
    same_events(r.events, g["events"])
    np.testing.assert_allclose(r.stats["true_res"], g["true_res"], rtol=1e-8)


def test_singular_r_closed_form():
    """ESINGULAR_R (reading C23): b_1 = the null vector 1 of a 16 x 16 grid graph Laplacian, so
    A u_1 = 0 exactly, the j = 1 candidate is an exact dependence and R_1 is singular: GPU and oracle
    both stop with ESINGULAR_R at j = 1 with X = 0 and the same event."""
    from tests.test_oracle_pins import grid_graph_laplacian
    A = grid_graph_laplacian(16)
    rng = np.random.default_rng(1)
    B = np.concatenate([np.ones((A.n, 1)), rng.standard_normal((A.n, 2))], axis=1)
    ref = oracle.solve(A, B, tol=1e-8, maxit=50, pool_size=1)
    assert ref.status_name == "ESINGULAR_R"
    r = gpu_solve(A, B, tol=1e-8, maxit=50)
    assert r.status_name == "ESINGULAR_R", r.status_name
    assert r.iterations == ref.iterations
    same_events(r.events, ref.events)
    np.testing.assert_array_equal(r.X, 0.0)


@pytest.mark.parametrize("use_graphs", [True, False])
def test_replacement_runs_vs_oracle(use_graphs):
    """Runs WITH replacements (the oracle side is pinned by test_lsq_after_* in
    test_oracle_pins.py): Fig. 3's B = [e_1, A e_1] and config 3's recipe at eps = 0 on a small
    grid -- events, 50-iteration histories and X against the oracle."""
    A = synth.laplacian_2d(12, shift=2.0)
    e1 = np.zeros(A.n)
    e1[0] = 1.0
    D = synth.csr_to_dense(A)
    cases = [(A, np.stack([e1, D @ e1], axis=1)),
             (synth.laplacian_2d(14, shift=2.5), synth.dependent_rhs(14 * 14, 3, 0.0, seed=0))]
    for Ai, Bi in cases:
        ref = oracle.solve(Ai, Bi, tol=0.0, maxit=60, pool_size=1)
        r = gpu_solve(Ai, Bi, tol=0.0, maxit=60, use_graphs=use_graphs)
        same_events(r.events, ref.events)
        assert r.iterations == ref.iterations
        assert_hist_close(r.history, ref.history)
        np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())


def test_handle_reuse_across_block_sizes():
    """One handle reused for p = 4, then p = 8 and p = 32 at the same maxit (the history buffer is
    sized in doubles, not rows): each solve equals a fresh handle's and the oracle's history."""
    torch = _torch()
    from paper_1301_2102_b200 import DeviceCsr, Solver
    A = synth.laplacian_3d(12, shift=2.5)
    dA = DeviceCsr.from_host(A, "cuda:0")
    with Solver(0) as s:
        for p in (4, 8, 32, 4):
            B = synth.gaussian_rhs(A.n, p, seed=p)
            r = s.solve(dA, torch.from_numpy(B).to("cuda:0"), tol=0.0, maxit=64)
            ref = oracle.solve(A, B, tol=0.0, maxit=64)
            assert r.iterations == 64
            assert_hist_close(r.history, ref.history)
            np.testing.assert_allclose(r.X.cpu().numpy(), ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())


def test_binding_rejects_wrong_dtypes_and_shapes(solver):
    """The binding validates what the C ABI cannot: dtypes, 2-D shapes and matching row counts."""
    torch = _torch()
    from paper_1301_2102_b200 import BminresError, DeviceCsr
    A = synth.laplacian_2d(8, shift=1.0)
    dA = DeviceCsr.from_host(A, "cuda:0")
    B = torch.zeros((A.n, 2), dtype=torch.float64, device="cuda:0")
    with pytest.raises(BminresError):
        solver.solve(dA, B.float())
    with pytest.raises(BminresError):
        solver.solve(dA, B[:-1])
    with pytest.raises(BminresError):
        solver.solve(dA, B, torch.zeros((A.n, 3), dtype=torch.float64, device="cuda:0"))
    bad = DeviceCsr(dA.n, dA.row_ptr.long(), dA.col_idx, dA.values)
    with pytest.raises(BminresError):
        solver.solve(bad, B)


def test_start_block_large_deflation_tol():
    """A start column whose projection residual ratio (~0.03) lies between the CholQR2 fast path's
    own 1e-2 guard and a large deflation_tol (0.05) is a step-0 event (C13) on the GPU exactly as in
    the oracle (the fast path tests tau^2 against the Cholesky pivots)."""
    A = synth.laplacian_2d(20, shift=2.5)
    rng = np.random.default_rng(4)
    g = rng.standard_normal((A.n, 2))
    B = np.concatenate([g, g[:, :1] + 0.03 * rng.standard_normal((A.n, 1)), rng.standard_normal((A.n, 1))], axis=1)
    ref = oracle.solve(A, B, tol=0.0, maxit=40, tau=0.05, pool_size=1)
    assert [(e["j"], e["col"]) for e in ref.events][:1] == [(0, 3)]
    r = gpu_solve(A, B, tol=0.0, maxit=40, deflation_tol=0.05)
    same_events(r.events, ref.events)
    assert_hist_close(r.history, ref.history, rtol=1e-8)


# ----------------------------------------------------------------------------- convergence at scale


def _count_gate(it_gpu, g, tol):
    """Counts within +-2% (or +-2) of the oracle's golden run (the north star's bar)."""
    it_ref = g["iterations"]
    if abs(it_gpu - it_ref) <= max(2, 0.02 * it_ref):
        return
    raise AssertionError(f"count {it_gpu} vs oracle {it_ref}")


@pytest.mark.parametrize("cfg,eps", [(2, None), (3, 0.0), (3, 1e-10), (3, 1e-6)])
def test_full_size_solve_to_tol(cfg, eps):
    """North-star convergence gates at BASELINE sizes (Alg. 2 stop): config 2 (64^3,
    p = 8) and config 3 (512^2, p = 16, eps in {0, 1e-10, 1e-6}) solved to tol 1e-8 in the bench's
    launch configuration: status OK, every column's TRUE residual <= tol, no column-path blocks,
    the step-0 events of the recipe (8 replacements for eps = 0, 1e-10; none for 1e-6), and the
    iteration count against the oracle's golden run when scripts/make_golden.py has written it."""
    import os
    P = synth.config(cfg) if eps is None else synth.config(cfg, eps=eps)
    r = gpu_solve(P.A, P.B, tol=P.tol, maxit=4 * P.maxit, deflation_tol=P.tau)
    assert r.status_name == "OK"
    assert max(r.stats["true_res"]) <= P.tol, r.stats["true_res"]
    assert max(r.stats["comp_res"]) < P.tol
    assert r.stats["slow_blocks"] == 0
    if cfg == 3:
        ev0 = [e for e in r.events if e["j"] == 0]
        assert len(ev0) == (0 if eps == 1e-6 else 8), r.events
    gpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{P.name}_tol.json")
    if os.path.exists(gpath):
        g = _golden(f"{P.name}_tol.json")
        assert g["status"] == "OK" and g["p"] == P.p and g["n"] == P.n
        assert_hist_close(r.history, np.array(g["history_first50"]))
        _count_gate(r.iterations, g, P.tol)


@pytest.mark.parametrize("p", [8, 16])
def test_reduce2_factorisation_reused_bitwise(p, monkeypatch):
    """reduce2 factors each new block once (k_red2f: C_k, Tr_{k+1}, D) and K3b(k) loads its C_k
    (fac_blk = k) instead of refactoring; BMINRES_NO_RED2F switches both K1 and K3b back to
    factoring the same totals themselves with the same factor_block code.  The solves agree
    bitwise -- a plain 3-D run to convergence and one with a mid-solve exact dependence (j = 9:
    the block's factorisation fails, fac_bad, the column path runs, then reduce2 factors again)."""
    A = synth.laplacian_3d(14, shift=2.2)
    rng = np.random.default_rng(p)
    B1 = rng.standard_normal((A.n, p))
    D = synth.csr_to_dense(A)
    b = rng.standard_normal(A.n)
    B2 = np.stack([b, D @ (D @ b)] + [rng.standard_normal(A.n) for _ in range(p - 2)], axis=1)
    for B, tol in ((B1, 1e-10), (B2, 1e-10)):
        base = gpu_solve(A, B, tol=tol, maxit=1200)
        monkeypatch.setenv("BMINRES_NO_RED2F", "1")
        try:
            alt = gpu_solve(A, B, tol=tol, maxit=1200)
        finally:
            monkeypatch.delenv("BMINRES_NO_RED2F")
        assert base.status_name == alt.status_name and base.iterations == alt.iterations
        assert [(e["j"], e["col"], e["action"]) for e in base.events] == \
               [(e["j"], e["col"], e["action"]) for e in alt.events]
        np.testing.assert_array_equal(base.history, alt.history)
        np.testing.assert_array_equal(base.X, alt.X)


@pytest.mark.parametrize("p,use_graphs", [(16, True), (32, True), (32, False)])
def test_mid_solve_breakdown_large_p(p, use_graphs, monkeypatch):
    """An exact dependence in the first block (B = [b, A^2 b, ...]: the candidate from A u_1
    deflates at j = p + 1) at p = 16 and 32, solved to tol 1e-8: at p = 32 K1's prologue factors
    each block (no reduce2 factorisation) and K3b on the side stream finds the same breakdown --
    the case where K3b used to clear run_main under a running K2.  Against the
    oracle: status, counts (+-2%), events, histories (1e-9 over 50 iterations), true residual
    <= tol, X; p = 16 also bitwise with reduce2's factorisation switched off."""
    A = synth.laplacian_3d(14, shift=1.3)
    D = synth.csr_to_dense(A)
    rng = np.random.default_rng(7 + p)
    b = rng.standard_normal(A.n)
    B = np.stack([b, D @ (D @ b)] + [rng.standard_normal(A.n) for _ in range(p - 2)], axis=1)
    tol, maxit = 1e-8, 100 * p
    r = gpu_solve(A, B, tol=tol, maxit=maxit, use_graphs=use_graphs)
    ref = oracle.solve(A, B, tol=tol, maxit=maxit)
    assert r.status_name == ref.status_name == "OK"
    assert_counts_close(r.iterations, ref.iterations)
    same_events(r.events, ref.events)
    assert [(e["j"], e["action"]) for e in r.events] == [(p + 1, 1)]
    assert_hist_close(r.history, ref.history)
    assert max(r.stats["true_res"]) <= tol * 1.5
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-5, atol=1e-6 * np.abs(ref.X).max())
    if p == 16:
        monkeypatch.setenv("BMINRES_NO_RED2F", "1")
        r2 = gpu_solve(A, B, tol=tol, maxit=maxit, use_graphs=use_graphs)
        assert r2.iterations == r.iterations
        np.testing.assert_array_equal(r2.history, r.history)
        np.testing.assert_array_equal(r2.X, r.X)


@pytest.mark.parametrize("p,split", [(16, 2), (16, 1), (32, 2), (32, 1)])
def test_long_history_parity_large_p(p, split):
    """Twenty block steps at p = 16 and 32 on a problem of several thousand tiles (3-D 32^3 with a
    ragged last plane: n = 32*32*31 rows), through the fused K1 (split_spmm = 2) and through the
    split pair K1a + K1 with the separate update kernel (split_spmm = 1: config 4's and 5's launch
    configuration) -- 50 iterations are only 1.5 block steps at p = 32, so this is the run that takes
    the steady-state kernels (two previous blocks' reflectors, paired X updates, both graph
    parities) against the oracle: the bar's 1e-9 over ALL 20p iterations (measured: 6e-14 at
    j = 640), events, and X to 1e-9 (measured 7e-14)."""
    A = synth.laplacian_3d(32, 32, 31, shift=2.1)
    B = synth.gaussian_rhs(A.n, p, seed=100 + p)
    maxit = 20 * p
    r = gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=split)
    ref = oracle.solve(A, B, tol=0.0, maxit=maxit)
    assert r.status_name == ref.status_name == "MAXIT"
    assert r.iterations == ref.iterations == maxit
    same_events(r.events, ref.events)
    assert_hist_close(r.history, ref.history, upto=maxit)
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-9, atol=1e-11 * np.abs(ref.X).max())


_irregular_sym_csr = synth.irregular_sym_csr


@pytest.mark.parametrize("seed", range(24))
def test_seeded_sweep_irregular_matrices(seed):
    """Seeded sweep over what the structured parity cases do not vary together: irregular sparse
    symmetric indefinite matrices (row lengths 0..300, hub rows longer than every gather batch,
    some rows and columns entirely empty), ragged n, every compiled p, fused and split kernels,
    graphs and plain launches, pool sizes, X0 -- each solve against the oracle: status, count,
    events, histories to 1e-9 over the first 50 iterations, X."""
    rng = np.random.default_rng(9000 + seed)
    p = [1, 2, 3, 4, 5, 6, 7, 8, 16, 32][seed % 10]
    n = int(rng.integers(max(300, 8 * p), 5000))
    A = _irregular_sym_csr(n, rng, hubs=int(rng.integers(0, 4)), empty_rows=int(rng.integers(0, 3)) if seed % 4 == 0 else 0)
    B = rng.standard_normal((n, p))
    maxit = int(rng.integers(p + 1, 4 * p + 40))
    kw = dict(use_graphs=bool(rng.integers(0, 2)), pool_size=int(rng.integers(1, 4)),
              split_spmm=int(rng.integers(0, 3)) if p >= 8 else 0)
    X0 = rng.standard_normal((n, p)) if seed % 3 == 1 else None
    r = gpu_solve(A, B, tol=0.0, maxit=maxit, X0=X0, **kw)
    ref = oracle.solve(A, B, tol=0.0, maxit=maxit, X0=X0, pool_size=kw["pool_size"])
    assert r.status_name == ref.status_name, (r.status_name, ref.status_name, kw)
    assert r.iterations == ref.iterations
    same_events(r.events, ref.events)
    assert_hist_close(r.history, ref.history)
    # X: to 1e-9 of its size plus the oracle's own sensitivity to a one-ulp perturbation of B.  A hub
    # row makes an outlying eigenvalue whose Ritz value converges within the run; from there on the
    # Lanczos vectors lose orthogonality along that eigenvector (Paige), and the iterate's component
    # along it moves by ~1e-7 under ANY rounding-level change while the residual history does not
    # (relative to max|X|, oracle against itself / kernels against the oracle: seed 20 1.1e-8 /
    # 1.2e-8, seed 10 6e-10 / 6.5e-9, seed 2 1e-11 / 1.2e-10; the other 21 cases <= 1.4e-14 / 6e-14;
    # histories agree to 5.5e-15 in all 24)
    prng = np.random.default_rng(seed)
    sens = oracle.solve(A, B * (1.0 + prng.integers(-1, 2, B.shape) * 2.0 ** -52), tol=0.0, maxit=maxit, X0=X0,
                        pool_size=kw["pool_size"])
    atol = 1e-9 * np.abs(ref.X).max() + 50.0 * np.abs(sens.X - ref.X).max()
    np.testing.assert_allclose(r.X, ref.X, rtol=0.0, atol=atol)


@pytest.mark.parametrize("seed", range(24))
def test_seeded_sweep_dependent_rhs(seed):
    """Seeded sweep of the dependence paths on irregular matrices: B = [G, G C + eps N] (config 3's
    recipe: exact and near dependences in the start block, eps in {0, 1e-10}; none at 1e-6) or
    B = [b, A^2 b, Gaussian ...] (an exact dependence at j = p + 1, inside the first block step),
    under both policies (0: replacement from the pool, 1: block-size reduction), p in
    {2, 4, 6, 8, 16, 32}, fused / split kernels, graphs / plain launches -- against the oracle:
    status, counts, events (step, column, kind, action), histories to 1e-9, X as in
    test_seeded_sweep_irregular_matrices."""
    rng = np.random.default_rng(7000 + seed)
    p = [2, 4, 6, 8, 16, 32][seed % 6]
    rep = seed // 6
    policy = (seed + rep) % 2 if seed < 18 else seed % 2
    n = int(rng.integers(max(400, 10 * p), 4000))
    A = _irregular_sym_csr(n, rng, hubs=int(rng.integers(0, 3)), empty_rows=0)
    if seed < 18:
        eps = [0.0, 1e-10, 1e-6][(seed + rep) % 3]
        B = synth.dependent_rhs(n, p // 2, eps, seed=seed)
    else:
        import scipy.sparse as sp
        S = sp.csr_matrix((A.data, A.indices, A.indptr), shape=(n, n))
        b = rng.standard_normal(n)
        B = np.ascontiguousarray(np.stack([b, S @ (S @ b)] + [rng.standard_normal(n) for _ in range(p - 2)], axis=1))
    maxit = 3 * p + 20
    kw = dict(use_graphs=bool(rng.integers(0, 2)), pool_size=min(p // 2 + 1, 8), policy=policy,
              split_spmm=int(rng.integers(0, 3)) if p >= 8 else 0)
    r = gpu_solve(A, B, tol=0.0, maxit=maxit, **kw)
    ref = oracle.solve(A, B, tol=0.0, maxit=maxit, pool_size=kw["pool_size"], policy=policy)
    assert r.status_name == ref.status_name, (r.status_name, ref.status_name, kw)
    assert r.iterations == ref.iterations
    same_events(r.events, ref.events)
    if seed < 18 and eps <= 1e-10:
        assert len(ref.events) == p // 2 and all(e["j"] == 0 for e in ref.events)
    elif seed >= 18:
        assert [e["j"] for e in ref.events] == [p + 1]
    assert_hist_close(r.history, ref.history)
    prng = np.random.default_rng(seed)
    sens = oracle.solve(A, B * (1.0 + prng.integers(-1, 2, B.shape) * 2.0 ** -52), tol=0.0, maxit=maxit,
                        pool_size=kw["pool_size"], policy=policy)
    if [e["j"] for e in sens.events] == [e["j"] for e in ref.events]:
        atol = 1e-9 * np.abs(ref.X).max() + 50.0 * np.abs(sens.X - ref.X).max()
        np.testing.assert_allclose(r.X, ref.X, rtol=0.0, atol=atol)


@pytest.mark.parametrize("p", [8, 16, 32])
def test_k1a_long_row_variant_bitwise(p, monkeypatch):
    """K1a's long-row variant (chosen for matrices with >= 12 entries per row: the next batch's
    column indices / values are loaded under the current gathers) sums every row in the same order
    as the plain kernel: config 5's recipe at n = 20,011 (27 entries per row, random long-range
    columns) in split mode, against the oracle and bitwise against BMINRES_K1A_PLAIN=1, graphs and
    plain launches; then a short-row matrix on the same handle sizes takes the plain kernel again."""
    A, B16 = synth.unstructured_csr(20011, seed=5, p=16)
    assert A.nnz >= 12 * A.n
    B = np.ascontiguousarray(np.random.default_rng(p).standard_normal((A.n, p)))
    maxit = 3 * p + 8
    ref = oracle.solve(A, B, tol=0.0, maxit=maxit)
    runs = [gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=1, use_graphs=g) for g in (True, False)]
    monkeypatch.setenv("BMINRES_K1A_PLAIN", "1")
    plain = gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=1)
    monkeypatch.delenv("BMINRES_K1A_PLAIN")
    for r in runs:
        assert r.iterations == ref.iterations == maxit
        assert_hist_close(r.history, ref.history, upto=maxit)
        np.testing.assert_array_equal(r.history, plain.history)
        np.testing.assert_array_equal(r.X, plain.X)
    np.testing.assert_allclose(runs[0].X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())
    # one handle: long rows, then short rows of the same n and p (the kernel and its graphs are rebuilt)
    torch = _torch()
    from paper_1301_2102_b200 import DeviceCsr, Solver
    A2 = synth.irregular_sym_csr(A.n, np.random.default_rng(1), hubs=1, empty_rows=0)
    assert A2.nnz < 12 * A2.n
    with Solver(0, split_spmm=1) as s:
        dB = torch.from_numpy(B).to("cuda:0")
        r1 = s.solve(DeviceCsr.from_host(A, "cuda:0"), dB, tol=0.0, maxit=maxit, raise_on_error=False)
        r2 = s.solve(DeviceCsr.from_host(A2, "cuda:0"), dB, tol=0.0, maxit=maxit, raise_on_error=False)
        r3 = s.solve(DeviceCsr.from_host(A, "cuda:0"), dB, tol=0.0, maxit=maxit, raise_on_error=False)
    np.testing.assert_array_equal(r1.history, plain.history)
    np.testing.assert_array_equal(r3.history, plain.history)
    ref2 = oracle.solve(A2, B, tol=0.0, maxit=maxit)
    assert_hist_close(r2.history, ref2.history, upto=maxit)
