"""Row f1: the block-size reduction ("shrink") dependence policy on the
GPU, against the oracle (policy = 1).  The oracle side is pinned in test_oracle_pins.py
(test_shrink_*: the printed H~10 pattern, the compacted Lanczos relation, R~ = QR(H~), least squares
over the compacted basis).  Removed lanes stay zero columns of the p-wide panels: the block
factorisation takes a placeholder pivot for them, K3b deletes their Hessenberg columns.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def gpu_solve(A, B, *, policy=1, use_graphs=True, split_spmm=0, **kw):
    import torch
    from paper_1301_2102_b200 import DeviceCsr, Solver
    dA = DeviceCsr.from_host(A, "cuda:0")
    dB = torch.from_numpy(np.ascontiguousarray(B)).to("cuda:0")
    with Solver(0, pool_size=1, use_graphs=use_graphs, policy=policy, split_spmm=split_spmm) as s:
        r = s.solve(dA, dB, raise_on_error=False, **kw)
    r.X = r.X.cpu().numpy()
    return r


def key(evs):
    return [(e["j"], e["col"], e["kind"], e["action"]) for e in evs]


def check(r, ref, upto=50, rtol=1e-9):
    assert key(r.events) == key(ref.events)
    assert r.status_name == ref.status_name, (r.status_name, ref.status_name)
    assert abs(r.iterations - ref.iterations) <= max(2, 0.02 * ref.iterations), (r.iterations, ref.iterations)
    k = min(upto + 1, len(r.history), len(ref.history))
    a, b = r.history[:k], ref.history[:k]
    bad = np.abs(a - b) > rtol * np.abs(b) + 1e-14
    assert not bad.any(), np.argwhere(bad)[:5]


def test_paper_example_p2():
    """p = 2, B = [b, A^3 b]: A u_5 is dependent, u_7, u_9, ... are removed."""
    from tests.test_oracle_pins import _shrink_example
    A, _, B = _shrink_example()
    ref = oracle.solve(A, B, tol=0.0, maxit=10, pool_size=1, policy=1)
    r = gpu_solve(A, B, tol=0.0, maxit=10)
    check(r, ref, rtol=1e-8)
    assert key(r.events) == [(5, 1, 0, 4)]
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-7, atol=1e-9 * np.abs(ref.X).max())


def test_block_grade_stall_all_lanes_removed():
    """P9 under shrink: both lanes die at j = 7, 8 and the residual is exactly 0 at j = dp = 8."""
    A = synth.diag_csr(np.repeat([-2.0, -0.5, 1.0, 3.0], 10))
    B = np.random.default_rng(3).standard_normal((40, 2))
    ref = oracle.solve(A, B, tol=1e-10, maxit=20, pool_size=1, policy=1)
    r = gpu_solve(A, B, tol=1e-10, maxit=20)
    assert key(ref.events) == [(7, 1, 0, 4), (8, 2, 0, 4)]
    check(r, ref)
    assert r.status_name == "OK" and r.iterations == 8


@pytest.mark.parametrize("use_graphs", [True, False])
def test_step0_removal_converges(use_graphs):
    """Config 3's recipe (B = [G, G C]) on a small grid: the dependent start columns are removed at
    step 0 and the solve converges with the remaining lanes; counts, events, histories, X, true
    residual against the oracle."""
    A = synth.laplacian_2d(14, shift=2.5)
    B = synth.dependent_rhs(A.n, 3, 0.0, seed=0)
    ref = oracle.solve(A, B, tol=1e-10, maxit=2000, pool_size=1, policy=1)
    r = gpu_solve(A, B, tol=1e-10, maxit=2000, use_graphs=use_graphs)
    check(r, ref)
    assert r.status_name == "OK" and max(r.stats["true_res"]) <= 1e-9
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-6, atol=1e-8 * np.abs(ref.X).max())


@pytest.mark.parametrize("p,split", [(8, 0), (16, 1), (32, 1)])
def test_mid_solve_removal_block_kernels(p, split):
    """B = [G, A G] (p/2 Gaussian columns and their images): the candidates A u_1 .. A u_{p/2} lie in
    the start block's span, so p/2 lanes are removed in block 1 (the column path) and every later
    block runs the fast kernels with those lanes zero -- the DMMA K1 (fused at p = 8, split mode with
    the separate update at p = 16, 32), the factorisation's placeholder pivots and K3b's deleted
    columns -- against the oracle: events, 50-iteration histories, counts and X."""
    A = synth.laplacian_2d(20, 19, shift=1.7)
    G = np.random.default_rng(p).standard_normal((A.n, p // 2))
    D = synth.csr_to_dense(A)
    B = np.ascontiguousarray(np.concatenate([G, D @ G], axis=1))
    maxit = 12 * p
    ref = oracle.solve(A, B, tol=0.0, maxit=maxit, pool_size=1, policy=1)
    assert [e["j"] for e in ref.events] == list(range(1, p // 2 + 1))
    assert all(e["action"] in (4, 5) for e in ref.events)
    r = gpu_solve(A, B, tol=0.0, maxit=maxit, split_spmm=split)
    check(r, ref, rtol=1e-8)
    np.testing.assert_allclose(r.X, ref.X, rtol=1e-6, atol=1e-8 * np.abs(ref.X).max())
