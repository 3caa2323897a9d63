"""Diagnostic: GPU vs oracle histories of preconditioned solves (where do they part?)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle, synth
from synth.studies import model_matrix
from tests.test_gpu_precond import neg_laplacian, prec_solve


def run(name, A, M, B, tol, maxit, **kw):
    ro = oracle.solve(A, B, tol=tol, maxit=maxit, prec=oracle.ic0(M), **kw)
    rg = prec_solve(A, M, B, tol=tol, maxit=maxit)
    k = min(len(ro.history), len(rg.history))
    rel = np.abs(rg.history[:k] - ro.history[:k]).max(1) / ro.history[:k].max(1)
    print(name, "its gpu", rg.iterations, "oracle", ro.iterations)
    for j in list(range(0, k, max(1, k // 40))) + [k - 1]:
        print(f"  j={j:5d} rel={rel[j]:.2e} o={ro.history[j].max():.3e} g={rg.history[j].max():.3e}")
    np.savez(f"gpurun_out/diag_{name}.npz", ho=ro.history, hg=rg.history)


N = 48
run("model_p1", model_matrix(N), neg_laplacian(N), synth.gaussian_rhs(N * N, 1, 3), 1e-8, 3000)
A = synth.laplacian_2d(40, shift=2.5)
run("dep", A, synth.laplacian_2d(40), synth.dependent_rhs(A.n, 4, 0.0, 0), 1e-8, 4000)
# unpreconditioned controls (the plain solver) on the same problems
from tests.test_gpu_parity import gpu_solve
for name, A, B in (("plain_model_p1", model_matrix(N), synth.gaussian_rhs(N * N, 1, 3)),):
    ro = oracle.solve(A, B, tol=1e-8, maxit=3000)
    rg = gpu_solve(A, B, tol=1e-8, maxit=3000)
    print(name, "its gpu", rg.iterations, "oracle", ro.iterations)
