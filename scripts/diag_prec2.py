"""Diagnostic: count sensitivity -- GPU vs oracle vs the oracle under 1-ulp perturbations of B."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle, synth
from synth.studies import model_matrix
from tests.test_gpu_precond import neg_laplacian, prec_solve
from tests.test_gpu_parity import gpu_solve


def counts(A, M, B, tol, maxit):
    L = oracle.ic0(M) if M is not None else None
    c0 = oracle.solve(A, B, tol=tol, maxit=maxit, prec=L, history=False).iterations
    cs = []
    for s in range(4):
        rng = np.random.default_rng(100 + s)
        Bp = B * (1 + np.ldexp(rng.choice([-1.0, 1.0], B.shape), -52))
        cs.append(oracle.solve(A, Bp, tol=tol, maxit=maxit, prec=L, history=False).iterations)
    g = (prec_solve(A, M, B, tol=tol, maxit=maxit) if M is not None else gpu_solve(A, B, tol=tol, maxit=maxit)).iterations
    return c0, cs, g


A = synth.laplacian_2d(40, shift=2.5)
Bd = synth.dependent_rhs(A.n, 4, 0.0, 0)
Bg = synth.gaussian_rhs(A.n, 8, 0)
print("dep plain", counts(A, None, Bd, 1e-8, 8000), flush=True)
print("dep prec", counts(A, synth.laplacian_2d(40), Bd, 1e-8, 8000), flush=True)
print("gauss8 plain", counts(A, None, Bg, 1e-8, 8000), flush=True)
print("gauss8 prec", counts(A, synth.laplacian_2d(40), Bg, 1e-8, 8000), flush=True)
Bd6 = synth.dependent_rhs(A.n, 4, 1e-6, 0)
print("dep1e-6 prec", counts(A, synth.laplacian_2d(40), Bd6, 1e-8, 8000), flush=True)
N = 48
for p in (1, 2, 4):
    B = synth.gaussian_rhs(N * N, p, 3)
    print("model plain p", p, counts(model_matrix(N), None, B, 1e-8, 8000), flush=True)
    print("model prec p", p, counts(model_matrix(N), neg_laplacian(N), B, 1e-8, 8000), flush=True)
