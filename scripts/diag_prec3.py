"""Diagnostic: computed vs true residuals at the stop (GPU and oracle) on the 40 x 40 shifted problem."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle, synth
from tests.test_gpu_precond import prec_solve
from tests.test_gpu_parity import gpu_solve

np.set_printoptions(precision=3, linewidth=200)
A = synth.laplacian_2d(40, shift=2.5)
M = synth.laplacian_2d(40)
for name, B in (("dep", synth.dependent_rhs(A.n, 4, 0.0, 0)), ("gauss8", synth.gaussian_rhs(A.n, 8, 0))):
    for prec in (False, True):
        L = oracle.ic0(M) if prec else None
        ro = oracle.solve(A, B, tol=1e-8, maxit=8000, prec=L)
        rg = prec_solve(A, M, B, tol=1e-8, maxit=8000) if prec else gpu_solve(A, B, tol=1e-8, maxit=8000)
        st = rg.stats
        print(name, "prec" if prec else "plain", "its o/g", ro.iterations, rg.iterations)
        print("  oracle comp", ro.comp_res, "true", ro.true_res)
        print("  gpu    comp", np.array(st["comp_res"]), "true", np.array(st["prec_true_res"] if prec else st["true_res"]))
        # the oracle's history at the GPU's stop, and the GPU's true residual trajectory proxy
        print("  oracle hist at gpu stop", ro.history[rg.iterations])
        print("  slow_blocks", st["slow_blocks"], "events", len(rg.events), len(ro.events))
