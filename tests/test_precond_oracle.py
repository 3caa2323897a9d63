"""Pins of the oracle's f3 row -- IC(0) split preconditioning (reading R8) -- CPU only.

The oracle's factor, substitutions and preconditioned solve are checked against what the
mathematics fixes: IC(0) is the exact Cholesky factor when the pattern admits no fill (tridiagonal:
numpy's Cholesky, and the closed form of the 1-D Laplacian's factor), the identity for M = I, the
pattern residual (L L^T - M)_ik = 0 on the pattern, a pivot breakdown at the predicted row; the
substitutions against SciPy's dense triangular solves; the composed operator against dense
L^-1 A L^-T; the preconditioned iterate against brute-force least squares over the block Krylov
space of the transformed system; L = I reduces to the unpreconditioned oracle bitwise; an exact
factor (A = M tridiagonal) converges at j = p.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth

from tests.test_oracle_pins import banded_krylov_basis, lsq_residuals


def dense(A):
    return synth.csr_to_dense(A)


def tridiag_csr(d, e):
    n = len(d)
    M = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    return synth.dense_to_csr(M)


# ----------------------------------------------------------------------------- IC(0)


def test_ic0_identity():
    L = oracle.ic0(synth.diag_csr(np.ones(7)))
    np.testing.assert_array_equal(dense(L), np.eye(7))


def test_ic0_1d_laplacian_closed_form():
    """tridiag(-1, 2, -1): l_ii = sqrt((i+1)/i), l_{i+1,i} = -sqrt(i/(i+1)) (1-based), no fill."""
    n = 50
    L = dense(oracle.ic0(tridiag_csr(2.0 * np.ones(n), -np.ones(n - 1))))
    i = np.arange(1, n + 1, dtype=float)
    np.testing.assert_allclose(np.diag(L), np.sqrt((i + 1) / i), rtol=1e-14)
    np.testing.assert_allclose(np.diag(L, -1), -np.sqrt(i[:-1] / (i[:-1] + 1)), rtol=1e-14)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ic0_tridiagonal_is_cholesky(seed):
    """No fill is possible for a tridiagonal M, so IC(0) = the exact Cholesky factor."""
    rng = np.random.default_rng(seed)
    n = 40
    e = rng.standard_normal(n - 1)
    d = 2.5 + np.abs(e).sum() / n + rng.uniform(1, 2, n) + np.r_[np.abs(e), 0] + np.r_[0, np.abs(e)]
    M = tridiag_csr(d, e)
    np.testing.assert_allclose(dense(oracle.ic0(M)), np.linalg.cholesky(dense(M)), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("grid", [(20,), (7, 9)])
def test_ic0_pattern_residual(grid):
    """(L L^T)_ik = m_ik for every (i, k) in the pattern (the definition); fill outside it is nonzero."""
    M = synth.laplacian_2d(*grid) if len(grid) == 1 else synth.laplacian_3d(*grid, 5)
    L = oracle.ic0(M)
    Md, Ld = dense(M), dense(L)
    assert np.all(np.triu(Ld, 1) == 0)
    assert np.all((Ld != 0) <= (np.tril(Md) != 0))          # pattern of L within M's lower triangle
    R = Ld @ Ld.T - Md
    on = Md != 0
    assert np.abs(R[on]).max() <= 1e-13 * np.abs(Md).max()
    assert np.abs(R[~on]).max() > 1e-3                      # IC(0) is not the exact factor here
    # idempotence: the IC(0) of the pattern-projected L L^T is L again
    P = np.where(on, Ld @ Ld.T, 0.0)
    np.testing.assert_allclose(dense(oracle.ic0(synth.dense_to_csr(P))), Ld, rtol=1e-12, atol=1e-14)


def test_ic0_pivot_breakdown_row():
    """[[1,2],[2,1]]: l_21 = 2, pivot 1 - 4 < 0 at row 1 (0-based); a negative first pivot at row 0."""
    with pytest.raises(oracle.PivotBreakdown) as ei:
        oracle.ic0(synth.dense_to_csr(np.array([[1.0, 2.0], [2.0, 1.0]])))
    assert ei.value.row == 1
    with pytest.raises(oracle.PivotBreakdown) as ei:
        oracle.ic0(synth.diag_csr([-1.0, 1.0]))
    assert ei.value.row == 0


# ----------------------------------------------------------------------------- substitutions, operator


def test_trsv_against_dense_solves():
    rng = np.random.default_rng(3)
    n, p = 30, 4
    Ld = np.tril(rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.3), -1) + np.diag(rng.uniform(1, 2, n))
    L = synth.dense_to_csr(Ld)
    X = rng.standard_normal((n, p))
    np.testing.assert_allclose(oracle.trsv_lower(L, Ld @ X), X, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(oracle.trsv_upper(L, Ld.T @ X), X, rtol=1e-11, atol=1e-12)
    b = rng.standard_normal(n)
    np.testing.assert_allclose(oracle.trsv_lower(L, b), sla.solve_triangular(Ld, b, lower=True), rtol=1e-12)
    np.testing.assert_allclose(oracle.trsv_upper(L, b), sla.solve_triangular(Ld.T, b, lower=False), rtol=1e-12)


def test_prec_operator_dense_and_symmetric():
    A = synth.laplacian_2d(9, shift=2.0)
    L = oracle.ic0(synth.laplacian_2d(9))
    Ld, Ad = dense(L), dense(A)
    Ahat = sla.solve_triangular(Ld, sla.solve_triangular(Ld, Ad, lower=True).T, lower=True).T
    rng = np.random.default_rng(0)
    X = rng.standard_normal((A.n, 5))
    Y = oracle.prec_op_block(A, L, X)
    np.testing.assert_allclose(Y, Ahat @ X, rtol=1e-11, atol=1e-12 * np.abs(Y).max())
    Z = rng.standard_normal((A.n, 5))
    G = Z.T @ oracle.prec_op_block(A, L, X) - (X.T @ oracle.prec_op_block(A, L, Z)).T
    assert np.abs(G).max() <= 1e-10 * np.abs(Y).max() * np.abs(Z).max() * A.n


# ----------------------------------------------------------------------------- preconditioned solve


def test_identity_factor_is_the_plain_oracle_bitwise():
    A = synth.laplacian_2d(12, shift=2.0)
    B = synth.gaussian_rhs(A.n, 3, 0)
    I = synth.diag_csr(np.ones(A.n))
    r0 = oracle.solve(A, B, tol=1e-10, maxit=300)
    r1 = oracle.solve(A, B, tol=1e-10, maxit=300, prec=I)
    assert r0.iterations == r1.iterations and r0.status == r1.status
    np.testing.assert_array_equal(r0.history, r1.history)
    np.testing.assert_array_equal(r0.X, r1.X)
    np.testing.assert_allclose(r1.ptrue_res, r0.true_res, rtol=1e-12)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_prec_iterate_is_least_squares_of_the_transformed_system(p):
    """Every j: Yhat_j minimises ||Rhat_0 - Ahat Y|| over the block Krylov space of (Ahat, Rhat_0)
    (the method on the transformed system, reading R8), and X_j = L^-T Yhat_j."""
    A = synth.laplacian_2d(7, shift=1.0)          # indefinite
    M = synth.laplacian_2d(7)                      # -L: SPD
    L = oracle.ic0(M)
    Ld, Ad = dense(L), dense(A)
    Ahat = sla.solve_triangular(Ld, sla.solve_triangular(Ld, Ad, lower=True).T, lower=True).T
    B = np.random.default_rng(7 + p).standard_normal((A.n, p))
    Rh = sla.solve_triangular(Ld, B, lower=True)
    jmax = 18
    Q = banded_krylov_basis(Ahat, Rh, jmax)
    beta = np.linalg.norm(Rh, axis=0)
    for j in range(1, jmax + 1):
        r = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=0, prec=L)
        assert r.iterations == j and r.status_name == "MAXIT"
        res, Yls = lsq_residuals(Ahat, Rh, Q, j)
        big = res > 1e-12 * beta
        np.testing.assert_allclose((r.history[j] * beta)[big], res[big], rtol=1e-8, atol=1e-11 * beta.max())
        Xls = sla.solve_triangular(Ld.T, Yls, lower=False)
        np.testing.assert_allclose(r.X, Xls, rtol=1e-7, atol=1e-8 * np.abs(Xls).max())
        # computed (preconditioned) residual = true preconditioned residual; unpreconditioned reported
        np.testing.assert_allclose(r.comp_res, r.true_res, rtol=1e-6, atol=1e-13)
        np.testing.assert_allclose(r.ptrue_res, np.linalg.norm(B - Ad @ r.X, axis=0) / np.linalg.norm(B, axis=0),
                                   rtol=1e-9)


def test_prec_nonzero_initial_guess():
    A = synth.laplacian_2d(8, shift=1.0)
    L = oracle.ic0(synth.laplacian_2d(8))
    rng = np.random.default_rng(1)
    B = rng.standard_normal((A.n, 2))
    X0 = rng.standard_normal((A.n, 2))
    r = oracle.solve(A, B, tol=1e-11, maxit=400, X0=X0, prec=L)
    assert r.status_name == "OK"
    np.testing.assert_allclose(dense(A) @ r.X, B, atol=1e-8 * np.abs(B).max())
    # the residual norms are relative to ||L^-1 (b - A x0)||
    Ld = dense(L)
    rh0 = np.linalg.norm(sla.solve_triangular(Ld, B - dense(A) @ X0, lower=True), axis=0)
    rh = np.linalg.norm(sla.solve_triangular(Ld, B - dense(A) @ r.X, lower=True), axis=0)
    np.testing.assert_allclose(r.true_res, rh / rh0, rtol=1e-6, atol=1e-14)


def test_exact_factor_converges_at_j_equal_p():
    """A = M tridiagonal SPD: IC(0) is exact, Ahat = I, the block Krylov space of Rhat_0 holds the
    solution after the first p iterations (every candidate is then an exact dependence)."""
    n, p = 60, 4
    A = tridiag_csr(2.0 * np.ones(n), -np.ones(n - 1))
    L = oracle.ic0(A)
    B = np.random.default_rng(2).standard_normal((n, p))
    r = oracle.solve(A, B, tol=1e-12, maxit=50, pool_size=8, prec=L)
    assert r.status_name == "OK" and r.iterations == p
    assert r.ptrue_res.max() < 1e-12
    assert all(e["kind"] == 0 for e in r.events)


def test_prec_reduces_iterations_shifted_laplacian():
    """SPEC precond example: the 20x20 shifted Laplacian with IC(0) of -L needs fewer iterations."""
    A = synth.laplacian_2d(20, shift=1.5)
    L = oracle.ic0(synth.laplacian_2d(20))
    B = synth.gaussian_rhs(A.n, 2, 0)
    r0 = oracle.solve(A, B, tol=1e-8, maxit=4000)
    r1 = oracle.solve(A, B, tol=1e-8, maxit=4000, prec=L)
    assert r0.status_name == "OK" and r1.status_name == "OK"
    assert r1.iterations < r0.iterations
    assert r1.ptrue_res.max() < 1e-6


def test_paper_fig1_iteration_counts():
    """The paper's own preconditioned experiment: A = -L - 200 I on the 200 x 200 grid,
    h = 1/199, IC(0) of -L (ichol default), ten random right-hand sides, tol 1e-8.  Printed: block
    MINRES 1048 iterations, sequential MINRES 3787 (tests/golden/paper_fig1_counts.json).  The
    right-hand sides' generator differs (Matlab mt19937ar), so the counts are compared
    within 5%; a wrong operator transform, a missing preconditioner or a wrong stop test moves them
    by far more (unpreconditioned: ~3500 block iterations)."""
    import json
    import os
    from synth.studies import model_matrix
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fig1_counts.json")))
    N = 200
    A = model_matrix(N)
    s = float((N - 1) ** 2)
    L = oracle.ic0(synth.stencil_csr((N, N), 4.0 * s, -s))      # -L
    B = np.random.default_rng(0).standard_normal((A.n, gold["p"]))
    r = oracle.solve(A, B, tol=1e-8, maxit=20000, prec=L)
    assert r.status_name == "OK"
    assert abs(r.iterations / gold["block_iterations"] - 1) < 0.05
    seq = sum(oracle.solve(A, B[:, c:c + 1], tol=1e-8, maxit=20000, prec=L).iterations for c in range(gold["p"]))
    assert abs(seq / gold["sequential_iterations"] - 1) < 0.05
    assert r.ptrue_res.max() < 1e-6
