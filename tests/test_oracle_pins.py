"""Pins of the CPU oracle to things other than itself (CPU only, no GPU).

Every test here checks ``oracle/`` against what the paper or the mathematics
fixes: brute-force dense least squares over an explicitly built block Krylov
basis, SciPy's scalar MINRES, closed forms, exact rational arithmetic, the
paper's printed structures.  A plausible mistake in the oracle (a dropped
term, a wrong sign or index, a transposed operand) fails at least one of them.
"""
import numpy as np
import pytest

import oracle
import synth

# ----------------------------------------------------------------------------- helpers


def banded_krylov_basis(D, F0, jmax):
    """Orthonormal Q whose first j columns span R(U_j) (banded order).

    Built independently of the oracle: the sequence f_1..f_p, A q_1, A q_2, ... with
    CGS2 against *all* previous vectors (a stable explicit QR of the banded Krylov
    sequence [F0, A F0, A^2 F0, ...] taken column by column)."""
    n, p = F0.shape
    Q = []
    for i in range(p):
        v = F0[:, i].copy()
        for _ in range(2):
            for q in Q:
                v -= (q @ v) * q
        Q.append(v / np.linalg.norm(v))
    for ell in range(jmax):
        v = D @ Q[ell]
        for _ in range(2):
            for q in Q:
                v -= (q @ v) * q
        Q.append(v / np.linalg.norm(v))
    return np.array(Q).T


def lsq_residuals(D, B, Q, j):
    """min_y ||b_i - A Q_j y|| for every column i, and the minimisers X_j = Q_j y."""
    AQ = D @ Q[:, :j]
    Y, *_ = np.linalg.lstsq(AQ, B, rcond=None)
    R = B - AQ @ Y
    return np.linalg.norm(R, axis=0), Q[:, :j] @ Y


def dense(A):
    return synth.csr_to_dense(A)


# ----------------------------------------------------------------------------- P1 brute force


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("seed", [0, 1])
def test_dense_least_squares(p, seed):
    """P1: x_j^(i) minimises ||b_i - A x|| over R(U_j) (eqn.min-resid), every j, every i."""
    n = 48
    A = synth.random_sym_sparse(n, 0.2, seed=seed)
    D = dense(A)
    B = np.random.default_rng(100 + seed).standard_normal((n, p))
    jmax = 24
    Q = banded_krylov_basis(D, B, jmax)
    beta = np.linalg.norm(B, axis=0)
    for j in range(1, jmax + 1):
        r = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=0)
        assert r.iterations == j and r.status_name == "MAXIT"
        res, Xls = lsq_residuals(D, B, Q, j)
        got = r.history[j] * beta
        big = res > 1e-12 * beta
        np.testing.assert_allclose(got[big], res[big], rtol=1e-8)
        np.testing.assert_allclose(r.X, Xls, rtol=1e-7, atol=1e-8 * np.abs(Xls).max())


@pytest.mark.parametrize("p", [1, 3, 4])
def test_dense_least_squares_irregular_matrix(p):
    """P1 on the irregular recipe of the GPU sweeps (synth.irregular_sym_csr: a hub row, an empty
    row and column -- A singular, the component of b on the empty row is never reduced): the
    oracle's iterate is still the least-squares minimiser over R(U_j) at every j."""
    n = 60
    A = synth.irregular_sym_csr(n, np.random.default_rng(21), hubs=1, empty_rows=1)
    D = dense(A)
    assert (np.diff(A.indptr) == 0).sum() == 1
    B = np.random.default_rng(200 + p).standard_normal((n, p))
    jmax = 20
    Q = banded_krylov_basis(D, B, jmax)
    beta = np.linalg.norm(B, axis=0)
    for j in range(1, jmax + 1):
        r = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=0)
        assert r.iterations == j and r.status_name == "MAXIT"
        res, Xls = lsq_residuals(D, B, Q, j)
        np.testing.assert_allclose(r.history[j] * beta, res, rtol=1e-8)
        np.testing.assert_allclose(r.X, Xls, rtol=1e-7, atol=1e-8 * np.abs(Xls).max())
    e = int(np.where(np.diff(A.indptr) == 0)[0][0])
    assert np.all(r.history[jmax] * beta >= np.abs(B[e]) * (1 - 1e-12))   # the empty row's residual stays b_e


def test_nonzero_initial_guess():
    """X0 != 0: F0 = B - A X0 generates the space and x_j - x_0 in R(U_j)."""
    n, p = 40, 3
    A = synth.random_sym_sparse(n, 0.25, seed=5)
    D = dense(A)
    rng = np.random.default_rng(7)
    B = rng.standard_normal((n, p))
    X0 = rng.standard_normal((n, p))
    F0 = B - D @ X0
    Q = banded_krylov_basis(D, F0, 12)
    for j in (1, 5, 12):
        r = oracle.solve(A, B, tol=0.0, maxit=j, X0=X0, pool_size=0)
        res, Y = lsq_residuals(D, F0, Q, j)
        np.testing.assert_allclose(np.linalg.norm(B - D @ r.X, axis=0), res, rtol=1e-8)
        np.testing.assert_allclose(r.X, X0 + Y, rtol=1e-7, atol=1e-9)


# ----------------------------------------------------------------------------- P2 p = 1 is MINRES


def test_p1_is_scalar_minres():
    """P2: with p = 1 the method is MINRES: iterates equal SciPy's."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.linalg import minres

    A = synth.laplacian_2d(12, shift=1.3)
    D = csr_matrix((A.data, A.indices, A.indptr), shape=(A.n, A.n))
    b = np.random.default_rng(3).standard_normal(A.n)
    xs = []
    minres(D, b, rtol=1e-15, maxiter=40, callback=lambda xk: xs.append(xk.copy()))
    bn = np.linalg.norm(b)
    for k in (1, 2, 5, 10, 20, 30, 40):
        r = oracle.solve(A, b[:, None], tol=0.0, maxit=k, pool_size=0)
        ref = np.linalg.norm(b - D @ xs[k - 1]) / bn
        assert abs(r.history[k, 0] - ref) <= 1e-10 * max(ref, 1e-3), (k, r.history[k, 0], ref)
        np.testing.assert_allclose(r.X[:, 0], xs[k - 1], rtol=1e-8, atol=1e-10)


# ----------------------------------------------------------------------------- P3/P4


@pytest.mark.parametrize("cfg", ["1c", 1])
def test_monotone_and_computed_equals_true(cfg):
    """P3: residuals never increase (nested spaces).  P4: computed residual
    (eqn.comp-resid) equals the true residual while above 1e-12, before the
    singular config's orthogonality loss (C23)."""
    P = synth.config(cfg)
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=300)
    h = r.history
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12) + 1e-300)
    for k in (10, 50, 300):
        rk = oracle.solve(P.A, P.B, tol=0.0, maxit=k)
        assert np.all(np.abs(rk.comp_res - rk.true_res) <= 1e-8)


def test_companion_converges_to_tol():
    """Config 1' (non-singular companion): all columns reach tol; true residual <= tol."""
    P = synth.config("1c")
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=P.maxit)
    assert r.status_name == "OK"
    assert r.history[-1].max() < P.tol
    assert r.true_res.max() <= P.tol * 1.5
    assert r.history[-2].max() >= P.tol


# ----------------------------------------------------------------------------- P5/P11 structure


def _debug_run(n=36, p=3, iters=15, seed=2):
    A = synth.random_sym_sparse(n, 0.25, seed=seed)
    B = np.random.default_rng(seed).standard_normal((n, p))
    r = oracle.solve(A, B, tol=0.0, maxit=iters, pool_size=0, debug_iters=iters)
    return A, dense(A), B, r


def test_lanczos_relation_and_band():
    """P5: A U_j = U_{j+p} \\bar H_j (eqn.Ruhe-bl-Arnoldi-rel), H_j = U_j^T A U_j symmetric
    (P:225-227), band +-p in H, <= 2p superdiagonals in R."""
    p, j = 3, 15
    A, D, B, r = _debug_run(p=p, iters=j)
    U, H, R = r.dbg["U"], r.dbg["H"], r.dbg["R"]
    Uj, Ujp = U[:, :j], U[:, : j + p]
    assert np.linalg.norm(D @ Uj - Ujp @ H[: j + p, :j]) <= 1e-12 * np.linalg.norm(D) * np.sqrt(j)
    np.testing.assert_allclose(Ujp.T @ Ujp, np.eye(j + p), atol=1e-12)
    np.testing.assert_allclose(H[:j, :j], Uj.T @ D @ Uj, atol=1e-12)
    np.testing.assert_allclose(H[:j, :j], H[:j, :j].T, atol=0)
    for c in range(j):
        for rr in range(j + p):
            if abs(rr - c) > p:
                assert H[rr, c] == 0.0
            if rr > c or rr < c - 2 * p:
                if rr < j:
                    assert R[rr, c] == 0.0


def test_R_is_qr_of_H_and_invariants():
    """P11: the assembled R is the R of a dense QR of \\bar H_j up to row signs;
    M_j R_j = U_j; ||S||_F^2 = sum ||z_l||^2 + ||T||_F^2 (orthogonal Q_j)."""
    p, j = 3, 15
    A, D, B, r = _debug_run(p=p, iters=j)
    H, R, M, U, Z, S = (r.dbg[k] for k in "HRMUZS")
    Rd = np.linalg.qr(H[: j + p, :j], mode="r")
    np.testing.assert_allclose(np.abs(R), np.abs(Rd[:j]), atol=1e-12 * np.abs(Rd).max())
    np.testing.assert_allclose(M[:, :j] @ R, U[:, :j], atol=1e-10)
    beta = np.linalg.norm(B, axis=0)
    T2 = np.sum((r.history[j] * beta) ** 2)
    np.testing.assert_allclose(np.sum(Z**2) + T2, np.sum(S**2), rtol=1e-12)
    # S from the thin QR: F0 = U_p S (eqn.init-QR), diag >= 0
    np.testing.assert_allclose(U[:, :p] @ S, B, atol=1e-12 * np.abs(B).max())
    assert np.all(np.diag(S) >= 0) and np.allclose(np.tril(S, -1), 0)
    # X_j = M_j Z_j (eqn.minres-approx)
    np.testing.assert_allclose(M[:, :j] @ Z, r.X, atol=1e-10)


def test_C_antidiagonal_paper_example():
    """P15: p = 5, j = 7 (eqn.anti-diag-symmetry): the superdiagonal h_{2..6,7} of the
    current column equals the antidiagonal of C_{pxp} (columns = Hessenberg columns 2..6), and
    equals the inner products u_i^T A u_7 it stands in for."""
    n, p, j = 40, 5, 7
    A = synth.random_sym_sparse(n, 0.3, seed=11)
    D = dense(A)
    B = np.random.default_rng(11).standard_normal((n, p))
    r = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=0, debug_iters=j)
    H, U = r.dbg["H"], r.dbg["U"]
    h = lambda a, b: H[a - 1, b - 1]  # 1-based, paper notation
    Cpp = np.array([[h(c + 1 + rr, c + 1) for c in range(1, p + 1)] for rr in range(1, p + 1)])
    assert Cpp[0, 0] == h(3, 2) and Cpp[p - 1, 0] == h(7, 2) and Cpp[0, p - 1] == h(7, 6)
    anti = np.array([Cpp[p - c, c - 1] for c in range(1, p + 1)])    # h_{7,2} .. h_{7,6}
    sup = np.array([h(i, 7) for i in range(2, 7)])
    np.testing.assert_array_equal(sup, anti)
    assert h(1, 7) == 0.0                                             # first entry of \bar H_7(:,7) is 0
    ip = np.array([U[:, i - 1] @ D @ U[:, 6] for i in range(2, 7)])
    np.testing.assert_allclose(sup, ip, atol=1e-12)


# ----------------------------------------------------------------------------- P6 closed forms


def test_first_iteration_closed_form_config1():
    """P6: at j = 1, x^(i) in span(b_1): res_i^2 = ||b_i||^2 - (b_i^T A b_1)^2/||A b_1||^2.
    Config 1 with default_rng(0): 0.6936, 0.99984, 0.99997, 0.99945."""
    P = synth.config(1)
    D = dense(P.A)
    B = P.B
    Ab1 = D @ B[:, 0]
    want = np.sqrt(np.sum(B**2, 0) - (B.T @ Ab1) ** 2 / (Ab1 @ Ab1)) / np.linalg.norm(B, axis=0)
    r = oracle.solve(P.A, P.B, tol=0.0, maxit=4)
    np.testing.assert_allclose(r.history[1], want, rtol=1e-12)
    np.testing.assert_allclose(want, [0.6936, 0.99984, 0.99997, 0.99945], atol=5e-5)
    # j <= p: X_j in span(b_1..b_j) -> tall-skinny least squares
    for j in range(2, 5):
        AB = D @ B[:, :j]
        Y, *_ = np.linalg.lstsq(AB, B, rcond=None)
        np.testing.assert_allclose(r.history[j] if j < len(r.history) else None,
                                   np.linalg.norm(B - AB @ Y, axis=0) / np.linalg.norm(B, axis=0), rtol=1e-10)


# ----------------------------------------------------------------------------- P7 Fig. 3


def test_fig3_dependent_rhs():
    """P7 / Fig. 3: B = [e_1, A e_1] -> dependence at iteration 1; system 2
    converges immediately (x_2 = e_1); system 1 continues after the random replacement."""
    P = synth.config(1)
    D = dense(P.A)
    n = P.n
    e1 = np.zeros(n)
    e1[0] = 1.0
    B = np.stack([e1, D @ e1], axis=1)
    r = oracle.solve(P.A, B, tol=1e-8, maxit=1, pool_size=1)
    assert r.events and r.events[0]["j"] == 1 and r.events[0]["col"] == 1
    assert r.events[0]["kind"] == 0 and r.events[0]["ratio"] < 1e-14 and r.events[0]["action"] == 1
    # closed form after j = 1: x_1 = e_1 (e_1^T A e_1)/||A e_1||^2 = e_1/3, x_2 = e_1
    np.testing.assert_allclose(r.X[:, 0], e1 / 3, atol=1e-15)
    np.testing.assert_allclose(r.X[:, 1], e1, atol=1e-15)
    np.testing.assert_allclose(r.history[1], [np.sqrt(1 / 3), 0.0], atol=1e-15)
    r = oracle.solve(P.A, B, tol=1e-8, maxit=3000, pool_size=1)
    assert r.status_name in ("OK", "MAXIT")
    assert r.history[1:, 1].max() < 1e-14            # system 2 stays converged
    assert r.history[-1, 0] < r.history[1, 0] * 0.5  # system 1 keeps converging


def test_pool_exhausted_is_reported():
    """C18: a breakdown with an empty pool and no convergence -> EPOOL."""
    P = synth.config(1)
    D = dense(P.A)
    e1 = np.zeros(P.n)
    e1[0] = 1.0
    B = np.stack([e1, D @ e1], axis=1)
    r = oracle.solve(P.A, B, tol=1e-8, maxit=10, pool_size=0)
    assert r.status_name == "EPOOL" and r.iterations == 1 and r.events[0]["action"] == 3


def test_happy_breakdown_p1_is_ok():
    """C18: p = 1 'happy breakdown' has converged: OK, not EPOOL."""
    A = synth.diag_csr([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    b = np.array([[1.0, 1.0, 1.0, 0.0, 0.0, 0.0]])
    r = oracle.solve(A, b.T, tol=1e-10, maxit=10, pool_size=0)
    assert r.status_name == "OK" and r.iterations == 3
    np.testing.assert_allclose(r.X[:, 0], [1, 0.5, 1 / 3, 0, 0, 0], atol=1e-14)


# ----------------------------------------------------------------------------- P8 exact dependence steps


def _first_dependent_iteration_exact(Aint, Bint):
    """Exact rational arithmetic: banded Krylov sequence s_1..s_p = B cols, s_{p+l} = A s_l
    (without replacement); return the first iteration j whose candidate A u_j lies in the
    span of the previous j+p-1 sequence vectors."""
    import sympy as sp

    A = sp.Matrix(Aint)
    n, p = Bint.shape
    seq = [sp.Matrix(Bint[:, i]) for i in range(p)]
    for j in range(1, n + 1):
        seq.append(A * seq[j - 1])
        M = sp.Matrix.hstack(*seq)
        if M.rank() < len(seq):
            return j
    return None


@pytest.mark.parametrize("t", [1, 2, 3])
def test_predicted_dependence_step(t):
    """P8: B = [b, A^t b] (p = 2): the first dependent candidate is at j = 2t-1 (exact
    SymPy ranks), and the oracle records its first breakdown exactly there."""
    rng = np.random.default_rng(40 + t)
    n = 12
    M = rng.integers(-3, 4, (n, n))
    Aint = np.triu(M) + np.triu(M, 1).T
    b = rng.integers(-2, 3, n)
    bt = b.copy()
    for _ in range(t):
        bt = Aint @ bt
    Bint = np.stack([b, bt], axis=1)
    jx = _first_dependent_iteration_exact(Aint, Bint)
    assert jx == 2 * t - 1
    A = synth.dense_to_csr(Aint.astype(float))
    r = oracle.solve(A, Bint.astype(float), tol=0.0, maxit=2 * t + 1, pool_size=2)
    assert r.events, "no breakdown recorded"
    assert r.events[0]["j"] == jx and r.events[0]["kind"] == 0


def test_step0_dependent_columns():
    """Config-3 recipe at small size: B = [G, G C + eps N] -> step-0 events for columns
    p/2+1..p when eps*||N||/||GC|| << tau; none when it is >> tau (C13; BASELINE configs[2])."""
    A = synth.laplacian_2d(20, shift=2.5)
    for eps, n_ev in ((0.0, 4), (1e-10, 4), (1e-6, 0)):
        B = synth.dependent_rhs(A.n, 4, eps, seed=0)
        r = oracle.solve(A, B, tol=1e-8, maxit=60, pool_size=1)
        ev0 = [e for e in r.events if e["j"] == 0]
        assert len(ev0) == n_ev, (eps, r.events)
        assert [e["col"] for e in ev0] == list(range(5, 5 + n_ev))
        if eps == 0.0:
            assert all(e["kind"] == 0 for e in ev0)
        # the replaced start block is still orthonormal and the history monotone
        h = r.history
        assert np.all(h[1:] <= h[:-1] * (1 + 1e-12) + 1e-300)


# ----------------------------------------------------------------------------- P9 block grade


def test_block_grade_stall():
    """P9 / Prop. prop.block-grade-ident: A = diag with d distinct eigenvalues of
    multiplicity >= p: candidates are dependent at j = (d-1)p+1 .. dp; all columns converge at dp."""
    d, p, mult = 4, 2, 10
    A = synth.diag_csr(np.repeat([-2.0, -0.5, 1.0, 3.0], mult))
    B = np.random.default_rng(9).standard_normal((d * mult, p))
    r = oracle.solve(A, B, tol=1e-12, maxit=40, pool_size=p)
    js = [e["j"] for e in r.events]
    assert js == list(range((d - 1) * p + 1, d * p + 1)), r.events
    assert r.status_name == "OK" and r.iterations == d * p
    assert r.true_res.max() < 1e-12


# ----------------------------------------------------------------------------- P10 §6 bound


def test_section6_bound_vs_minres():
    """P10 (§6, reading C10): ||f_j^(i)|| <= ||r^MINRES_J(b_i)|| with J = floor((j-i)/p)+1."""
    n, p = 40, 3
    A = synth.random_sym_sparse(n, 0.25, seed=4)
    D = dense(A)
    B = np.random.default_rng(4).standard_normal((n, p))
    r = oracle.solve(A, B, tol=0.0, maxit=24, pool_size=0)
    for i in range(1, p + 1):
        b = B[:, i - 1]
        for j in range(i, 25):
            J = (j - i) // p + 1
            K = np.stack([np.linalg.matrix_power(D, k) @ b for k in range(J)], axis=1)
            Qk, _ = np.linalg.qr(K)
            y, *_ = np.linalg.lstsq(D @ Qk, b, rcond=None)
            ref = np.linalg.norm(b - D @ Qk @ y)
            assert r.history[j, i - 1] * np.linalg.norm(b) <= ref * (1 + 1e-8)


# ----------------------------------------------------------------------------- P13 patterns after replacement


def test_replacement_zero_pattern_paper_example():
    """P13: p = 2, dependence at column 5: \\hat H has zeros at (7,5), (5,7);
    \\hat R has zeros at r_{3,7} and r_{5,9}; band and symmetry are unchanged."""
    rng = np.random.default_rng(5)
    n = 30
    M = rng.integers(-3, 4, (n, n))
    Aint = np.triu(M) + np.triu(M, 1).T
    b = rng.integers(-2, 3, n)
    b3 = Aint @ (Aint @ (Aint @ b))
    B = np.stack([b, b3], axis=1).astype(float)
    A = synth.dense_to_csr(Aint.astype(float))
    r = oracle.solve(A, B, tol=0.0, maxit=10, pool_size=1, debug_iters=10)
    assert r.events[0]["j"] == 5
    H, R = r.dbg["H"], r.dbg["R"]
    assert H[6, 4] == 0.0 and H[4, 6] == 0.0
    assert R[2, 6] == 0.0 and R[4, 8] == 0.0
    assert R[3, 6] != 0.0 and R[5, 8] != 0.0 and H[5, 4] != 0.0
    np.testing.assert_allclose(H[:10, :10], H[:10, :10].T, atol=0)


def test_near_dependence_retained():
    """C15/C16 + P:797-805: a near-dependent candidate (1e-12 < h/omega <= tau) is replaced and
    retained; later vectors are orthogonal to it while it lives."""
    P = synth.config("1c")
    D = dense(P.A)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(P.n)
    B = np.stack([b, D @ b + 1e-10 * rng.standard_normal(P.n)], axis=1)
    r = oracle.solve(P.A, B, tol=1e-8, maxit=12, pool_size=1, debug_iters=12)
    e = r.events[0]
    assert e["j"] == 1 and e["kind"] == 1 and e["action"] == 2 and 1e-12 < e["ratio"] <= 1e-8
    U = r.dbg["U"]
    # the replacement u_3 is a unit vector orthogonal to u_1, u_2
    np.testing.assert_allclose(U[:, :3].T @ U[:, :3], np.eye(3), atol=1e-12)
    # vectors made while v is retained (iterations 2..1+2p -> u_4..u_7) are orthogonal to v,
    # the normalised rejected candidate; v is recovered from the Lanczos relation at j = 1:
    # A u_1 - sum_i h_{i,1} u_i = h v
    D1 = D @ U[:, 0] - U[:, :3] @ r.dbg["H"][:3, 0]
    v = D1 / np.linalg.norm(D1)
    assert np.abs(v @ U[:, 3:7]).max() < 1e-6
    # retention "no longer follows the mathematical derivation": the relation
    # A U_j = U_{j+p} H_j is perturbed, so only monotonicity (a property of the QR) is pinned
    h = r.history
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))
    assert h[1, 1] < 1e-9   # system 2 (= A b + tiny) converges at j = 1, as in Fig. 3


# ----------------------------------------------------------------------------- P12 / RNG / SpMM


def test_householder_invariants():
    """P12: reflector maps x to beta e_1; involution; norm preservation."""
    rng = np.random.default_rng(0)
    v, tau, beta = oracle.house_gen(np.array([3.0, 4.0]))
    assert abs(abs(beta) - 5.0) < 1e-15
    np.testing.assert_allclose(oracle.house_apply(v, tau, [3.0, 4.0]), [beta, 0.0], atol=1e-15)
    v, tau, beta = oracle.house_gen(np.array([2.0, 0.0, 0.0]))
    assert tau == 0.0 and beta == 2.0
    for _ in range(200):
        L = int(rng.integers(2, 34))
        x = rng.standard_normal(L)
        v, tau, beta = oracle.house_gen(x)
        y = oracle.house_apply(v, tau, x)
        assert abs(y[0] - beta) <= 1e-14 * abs(beta) and np.abs(y[1:]).max() <= 1e-14 * abs(beta)
        z = rng.standard_normal(L)
        zz = oracle.house_apply(v, tau, oracle.house_apply(v, tau, z))
        np.testing.assert_allclose(zz, z, atol=1e-14 * np.linalg.norm(z))
        assert abs(np.linalg.norm(oracle.house_apply(v, tau, z)) - np.linalg.norm(z)) <= 1e-14 * np.linalg.norm(z)


def test_splitmix64_reference_value():
    """C17's generator is SplitMix64: its published first output for state 0 is 0xE220A8397B1DCDAF."""
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF
    x = oracle.splitmix64(oracle.splitmix64(0) ^ 5)
    want = 2.0 * ((x >> 11) * 2.0**-53) - 1.0
    assert oracle.rand_entry(0, 0, 0, 5) == want
    vals = np.array([oracle.rand_entry(0, 1, 0, i) for i in range(4000)])
    assert vals.min() >= -1 and vals.max() < 1 and abs(vals.mean()) < 0.05


def test_csr_block_matches_dense():
    """The SpMM oracle: Y = A X equals the dense product; columns independent."""
    A = synth.laplacian_3d(6, shift=3.0)
    X = np.random.default_rng(0).standard_normal((A.n, 5))
    Y = oracle.csr_block(A, X)
    np.testing.assert_allclose(Y, dense(A) @ X, rtol=1e-14, atol=1e-14)
    Y1 = oracle.csr_block(A, X[:, 2:3].copy())
    np.testing.assert_array_equal(Y1[:, 0], Y[:, 2])


# ----------------------------------------------------------------------------- P14 singular config 1


def test_config1_singular_floor():
    """P14 (C23): config 1 is exactly singular (eigenvalue 2-2cos(11pi/33)*2 = 0); each column's
    residual plateaus at |v^T b_i|/||b_i||, v = sin(11 pi x/33) sin(11 pi y/33) normalised."""
    P = synth.config(1)
    x = np.arange(1, 33)
    s = np.sin(11 * np.pi * x / 33)
    v = np.outer(s, s).ravel()
    v /= np.linalg.norm(v)
    assert np.linalg.norm(dense(P.A) @ v) < 1e-13
    floor = np.abs(v @ P.B) / np.linalg.norm(P.B, axis=0)
    np.testing.assert_allclose(floor, [0.04458, 0.03019, 0.003486, 0.01999], rtol=1e-3)
    r = oracle.solve(P.A, P.B, tol=P.tol, maxit=1100)
    assert r.status_name == "MAXIT"
    assert np.all(r.history >= floor * (1 - 1e-6))
    np.testing.assert_allclose(r.history[1100], floor, rtol=1e-4)


# ----------------------------------------------------------------------------- P1 / P4 after replacements


def _lsq_over_own_basis(A, B, maxit, *, pool_size=1):
    """P1 on runs WITH replacement events: the replaced basis still satisfies the Lanczos relation
    (h_{j+p,j} := 0, exact dependence), so x_j must still minimise ||b_i - A x|| over
    R(U_j) -- here U_j is the oracle's own basis (dbg_U), the minimiser found by dense least squares."""
    D = dense(A)
    r = oracle.solve(A, B, tol=0.0, maxit=maxit, pool_size=pool_size, debug_iters=maxit)
    U = r.dbg["U"]
    beta = np.linalg.norm(B, axis=0)
    for j in range(1, maxit + 1):
        rj = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=pool_size)
        res, Xls = lsq_residuals(D, B, U, j)
        big = res > 1e-12 * beta
        np.testing.assert_allclose(rj.history[j][big] * beta[big], res[big], rtol=1e-8)
        # P4: the computed residual is the true residual
        assert np.all(np.abs(rj.comp_res - rj.true_res) <= 1e-9 * np.maximum(1.0, rj.true_res))
        if j in (1, maxit // 2, maxit):
            np.testing.assert_allclose(rj.X, Xls, rtol=1e-7, atol=1e-8 * max(1.0, np.abs(Xls).max()))
    return r


def test_lsq_after_replacement_fig3():
    """Fig. 3's B = [e_1, A e_1]: column 1's candidate at j = 1 is exactly dependent
    and replaced by a random vector; every later iterate is still the least-squares minimiser over
    the (replaced) basis, and computed = true residual."""
    A = synth.laplacian_2d(12, shift=2.0)
    D = dense(A)
    e1 = np.zeros(A.n)
    e1[0] = 1.0
    B = np.stack([e1, D @ e1], axis=1)
    r = _lsq_over_own_basis(A, B, 30)
    assert [(e["j"], e["col"], e["action"]) for e in r.events] == [(1, 1, 1)]


def test_lsq_after_step0_replacement_config3_recipe():
    """Config 3's recipe B = [G, G C + eps N] at eps = 0 on a small grid: the last p/2 start columns
    deflate at step 0 (eqn.init-QR, reading C13) and are replaced; the iterates remain the
    least-squares minimisers over the oracle's basis at every j."""
    A = synth.laplacian_2d(14, shift=2.5)
    B = synth.dependent_rhs(A.n, 3, 0.0, seed=0)
    r = _lsq_over_own_basis(A, B, 36)
    assert [(e["j"], e["col"]) for e in r.events] == [(0, 4), (0, 5), (0, 6)]


# ----------------------------------------------------------------------------- ESINGULAR_R closed form


def grid_graph_laplacian(m):
    """Neumann graph Laplacian of an m x m grid: integer entries, A 1 = 0 exactly in fp64."""
    n = m * m
    D = np.zeros((n, n))
    for y in range(m):
        for x in range(m):
            i = y * m + x
            for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                if 0 <= x + dx < m and 0 <= y + dy < m:
                    D[i, (y + dy) * m + x + dx] = -1.0
                    D[i, i] += 1.0
    return synth.dense_to_csr(D)


def test_singular_r_closed_form():
    """r_11 = 0 exactly: b_1 = the null vector 1 of a graph Laplacian (m = 16, so u_1 = 1/16 and
    A u_1 = 0 in exact fp64).  The candidate of j = 1 is w = 0 (omega = 0: an exact dependence,
    replaced), the Hessenberg column h_1 is zero, so R_1 is singular and the solve stops with
    ESINGULAR_R at j = 1 (reading C23; x cannot be updated)."""
    A = grid_graph_laplacian(16)
    D = dense(A)
    assert np.all(D @ np.full(A.n, 1 / 16) == 0.0)
    rng = np.random.default_rng(1)
    B = np.concatenate([np.ones((A.n, 1)), rng.standard_normal((A.n, 2))], axis=1)
    r = oracle.solve(A, B, tol=1e-8, maxit=50, pool_size=1)
    assert r.status_name == "ESINGULAR_R"
    assert r.events and r.events[0]["j"] == 1 and r.events[0]["col"] == 1 and r.events[0]["kind"] == 0
    assert r.iterations == 0
    np.testing.assert_array_equal(r.X, 0.0)


# ----------------------------------------------------------------------------- f1: block-size reduction ("shrink")


def _shrink_example():
    """p = 2, B = [b, A^3 b] on a random integer symmetric matrix: A u_5 is exactly dependent (the
    first dependent candidate of B = [b, A^t b] is at j = 2t - 1, P8) -- the paper's example of
    P:601-611 (dependence at column 5, p = 2)."""
    rng = np.random.default_rng(7)
    n = 12
    M = rng.integers(-3, 4, (n, n))
    M = np.triu(M, 1)
    M = M + M.T
    M[np.diag_indices(n)] = rng.integers(-4, 5, n)
    b = rng.integers(-2, 3, n).astype(float)
    B = np.stack([b, M @ M @ M @ b], axis=1).astype(float)
    return synth.dense_to_csr(M.astype(float)), M.astype(float), B


def test_shrink_patterns_of_the_paper():
    """Shrink policy: u_7 = 0 is removed, hence u_9 = u_11 = 0; columns 7, 9
    and rows 7, 9, 11 of H_10 vanish and the compacted H~_10 has exactly the printed pattern
    (eqn.H10-dep); A U~_10 = U~_12 H~_10; R~_10 is the QR factor of H~_10 (dense
    brute force), with the bold zero r_{5,10} of eqn.R10-dep.  Reading C25: the printed
    bold zero r_{2,6} is not a structural zero (reflector 2 spans rows 2..4 and h_{4,6} = h_{6,4} > 0);
    brute force gives a nonzero entry, which the oracle reproduces."""
    A, M, B = _shrink_example()
    r = oracle.solve(A, B, tol=0.0, maxit=10, pool_size=1, policy=1, debug_iters=10)
    assert [(e["j"], e["col"], e["kind"], e["action"]) for e in r.events] == [(5, 1, 0, 4)]
    H, R, U = r.dbg["H"], r.dbg["R"], r.dbg["U"]
    assert np.all(H[[6, 8, 10], :] == 0) and np.all(H[:, [6, 8]] == 0)
    assert np.all(U[:, [6, 8, 10]] == 0)
    rows = [0, 1, 2, 3, 4, 5, 7, 9, 11]      # u_1..u_6, u_8, u_10, u_12
    cols = [0, 1, 2, 3, 4, 5, 7, 9]           # columns 1..6, 8, 10
    Ht = H[np.ix_(rows, cols)]
    printed = np.array([  # eqn.H10-dep, nonzero pattern
        [1, 1, 1, 0, 0, 0, 0, 0],
        [1, 1, 1, 1, 0, 0, 0, 0],
        [1, 1, 1, 1, 1, 0, 0, 0],
        [0, 1, 1, 1, 1, 1, 0, 0],
        [0, 0, 1, 1, 1, 1, 0, 0],
        [0, 0, 0, 1, 1, 1, 1, 0],
        [0, 0, 0, 0, 0, 1, 1, 1],
        [0, 0, 0, 0, 0, 0, 1, 1],
        [0, 0, 0, 0, 0, 0, 0, 1]])
    np.testing.assert_array_equal(np.abs(Ht) > 1e-10, printed.astype(bool))
    np.testing.assert_allclose(M @ U[:, cols], U[:, rows] @ Ht, atol=1e-12 * np.abs(M).sum())
    Rt = R[np.ix_(cols, cols)]
    _, Rd = np.linalg.qr(Ht)
    np.testing.assert_allclose(np.abs(Rt), np.abs(Rd), rtol=1e-10, atol=1e-12)
    assert abs(Rt[4, 7]) < 1e-12                                  # bold zero r_{5,10}
    assert abs(Rt[1, 5]) > 1e-3                                   # r_{2,6}: reading C25
    assert np.all(R[:, [6, 8]] == 0) and np.all(R[[6, 8], :] == 0)


def test_shrink_bandwidth_drops_in_two_stages():
    """removing one dependent vector reduces the bandwidth of the compacted H~ by one at
    column i (= 5, the dependent candidate: h_{7,5} = 0) and by a second one at column i + p (= 7,
    u_7 removed: column deleted), two vectors fewer in the Lanczos window from then on."""
    A, M, B = _shrink_example()
    r = oracle.solve(A, B, tol=0.0, maxit=10, pool_size=1, policy=1, debug_iters=10)
    H = r.dbg["H"]
    present = [i for i in range(12) if i not in (6, 8, 10)]
    width = []
    for c in range(10):
        if c in (6, 8):
            continue
        nz = [present.index(i) for i in present if abs(H[i, c]) > 1e-10]
        width.append(max(nz) - min(nz))   # sub- plus superdiagonals of compact column c
    # compact columns 4, 5, 6, 8, 10: the full width 2p = 4 drops to 3 at column 5 (h_{7,5} = 0)
    # and to 2 at column 8 (u_7 removed: no h_{7,8}) -- two vectors fewer, in two stages
    assert width[3:] == [4, 3, 3, 2, 2], width


@pytest.mark.parametrize("case", ["fig3", "p2_dependent"])
def test_shrink_iterates_are_least_squares_over_the_compact_basis(case):
    """P1 for the shrink policy: x_j minimises ||b_i - A x|| over the span of the non-removed basis
    vectors among u_1..u_j (the compacted basis), every j; computed = true residual (P4)."""
    if case == "fig3":
        A = synth.laplacian_2d(10, shift=2.0)
        D = dense(A)
        e1 = np.zeros(A.n)
        e1[0] = 1.0
        B = np.stack([e1, D @ e1], axis=1)
    else:
        A, D, B = _shrink_example()
    jmax = 10 if case == "p2_dependent" else 30
    r = oracle.solve(A, B, tol=0.0, maxit=jmax, pool_size=1, policy=1, debug_iters=jmax)
    assert r.events and all(e["action"] == 4 for e in r.events)
    U = r.dbg["U"]
    beta = np.linalg.norm(B, axis=0)
    for j in range(1, r.iterations + 1):
        rj = oracle.solve(A, B, tol=0.0, maxit=j, pool_size=1, policy=1)
        Q = U[:, :j][:, np.linalg.norm(U[:, :j], axis=0) > 0]
        res, Xls = lsq_residuals(D, B, Q, Q.shape[1])
        big = res > 1e-10 * beta
        np.testing.assert_allclose(rj.history[j][big] * beta[big], res[big], rtol=1e-7)
        assert np.all(np.abs(rj.comp_res - rj.true_res) <= 1e-9 * np.maximum(1.0, rj.true_res))


def test_shrink_step0_removal():
    """Shrink at step 0 (reading C13 under P:582-636): a dependent start column is removed (u_i = 0,
    S_ii = 0), not replaced; the other columns converge as if the block were smaller."""
    A = synth.laplacian_2d(14, shift=2.5)
    B = synth.dependent_rhs(A.n, 3, 0.0, seed=0)
    r = oracle.solve(A, B, tol=1e-10, maxit=2000, pool_size=1, policy=1)
    assert [(e["j"], e["col"], e["action"]) for e in r.events][:3] == [(0, 4, 4), (0, 5, 4), (0, 6, 4)]
    assert r.status_name == "OK" and r.true_res.max() < 1e-9
