"""Seeded inputs of the paper's block-vs-sequential studies -- generators only.

The paper's model problem (§8 Numerical Results): L = h^-2 (I (+) T + T (+) I) on an
N x N grid, T = tridiag(1, -2, 1), h = 1/199 for N = 200 as printed (the survey's erratum:
h only rescales A), A = -L - 200 I (indefinite).  The paper preconditions with ichol(-L)
(P:1026-1027); these studies are UNPRECONDITIONED (preconditioning is row f3, not built), so the
absolute iteration counts are not the paper's -- only the block/sequential comparisons are studied.

Right-hand sides:
  * Fig. 2: b_1 = ones, b_2..b_p = e_1 .. e_{p-1}.
  * Fig. 4: (e_1, ones) and (e_1, e_2).
  * Figs. 5-6: pairs built from the orthonormal eigenvectors q_1, q_2, ... of A ordered
    by |eigenvalue| (analytic here: q_{kl}(x, y) = (2/(N+1)) sin(k pi (x+1)/(N+1)) sin(l pi (y+1)/(N+1)),
    eigenvalue h^-2 (4 sin^2(k pi/(2(N+1))) + 4 sin^2(l pi/(2(N+1)))) - 200), coefficients uniform on
    [0, 1) (Matlab rand(); numpy default_rng(seed) here):
      eqn.smalleigsRHS: b_1 = sum_{i=1}^{100+m} alpha_i q_i, b_2 = sum_{i=100-m+1}^{200} beta_i q_i;
      eqn.largeeigsRHS: b_1 = sum_{i=1}^{200} alpha_i q_i + sum_{i=n-199}^{n-200+m} alpha_i q_i,
                        b_2 = sum_{i=201-m}^{200} beta_i q_i + sum_{i=n-199}^{n} beta_i q_i
    (the printed "beta{i}" is beta_i).  For a smaller grid the index bands scale with
    `band` (100 for N = 200).
No method arithmetic lives here (the sines are the closed-form eigenvectors of the stencil).
"""
from __future__ import annotations

import numpy as np

from .problems import Csr, stencil_csr


def model_matrix(N: int = 200, shift: float = 200.0, h: float | None = None) -> Csr:
    """A = -L - shift I, L = h^-2 (I (+) T + T (+) I) on the N x N grid."""
    h = 1.0 / (N - 1) if h is None else h
    s = 1.0 / (h * h)
    return stencil_csr((N, N), 4.0 * s - shift, -s)


def eigenpairs(N: int = 200, shift: float = 200.0, h: float | None = None):
    """Eigenvalues of model_matrix (analytic) and the (k, l) mode indices, ordered by |eigenvalue|
    ascending (ties: by k, then l).  Returns (lam, k, l), each of length N*N."""
    h = 1.0 / (N - 1) if h is None else h
    s1 = 4.0 * np.sin(np.arange(1, N + 1) * np.pi / (2 * (N + 1))) ** 2 / (h * h)
    K, L_ = np.meshgrid(np.arange(1, N + 1), np.arange(1, N + 1), indexing="ij")
    lam = (s1[K - 1] + s1[L_ - 1] - shift).ravel()
    kk, ll = K.ravel(), L_.ravel()
    order = np.lexsort((ll, kk, np.abs(lam)))
    return lam[order], kk[order], ll[order]


def eigvec_combination(N: int, k: np.ndarray, l: np.ndarray, coef: np.ndarray) -> np.ndarray:
    """sum_i coef_i q_{k_i l_i} as an N*N vector (lexicographic, x fastest)."""
    x = np.arange(1, N + 1)
    Sx = np.sin(np.outer(x, np.arange(1, N + 1)) * np.pi / (N + 1)) * np.sqrt(2.0 / (N + 1))   # Sx[x-1, k-1]
    C = np.zeros((N, N))
    np.add.at(C, (np.asarray(k) - 1, np.asarray(l) - 1), coef)
    # v[y, x] = sum_{k,l} C[k, l] sin(k x) sin(l y)  ->  (Sy C^T Sx^T)
    V = Sx @ C.T @ Sx.T
    return np.ascontiguousarray(V.ravel())


def fig2_rhs(n: int, p: int) -> np.ndarray:
    """[ones, e_1, ..., e_{p-1}]."""
    B = np.zeros((n, p))
    B[:, 0] = 1.0
    for c in range(1, p):
        B[c - 1, c] = 1.0
    return B


def fig4_pairs(n: int):
    """(e_1, ones) and (e_1, e_2)."""
    e1, e2, one = np.zeros(n), np.zeros(n), np.ones(n)
    e1[0] = 1.0
    e2[1] = 1.0
    return np.stack([e1, one], axis=1), np.stack([e1, e2], axis=1)


def eigmix_pair(N: int, m: int, kind: str, seed: int, band: int = 100, shift: float = 200.0,
                h: float | None = None) -> np.ndarray:
    """One pair of eqn.smalleigsRHS (kind 'small', 0 <= m <= band) or eqn.largeeigsRHS (kind 'large',
    0 <= m <= 2 band) right-hand sides as an n x 2 array; coefficients from default_rng(seed)."""
    lam, k, l = eigenpairs(N, shift, h)
    n = N * N
    rng = np.random.default_rng(seed)
    if kind == "small":
        i1 = np.arange(0, band + m)                     # q_1 .. q_{100+m}
        i2 = np.arange(band - m, 2 * band)              # q_{100-m+1} .. q_200
    elif kind == "large":
        i1 = np.concatenate([np.arange(0, 2 * band), np.arange(n - 2 * band, n - 2 * band + m)])
        i2 = np.concatenate([np.arange(2 * band - m, 2 * band), np.arange(n - 2 * band, n)])
    else:
        raise ValueError(kind)
    alpha = rng.random(len(i1))
    beta = rng.random(len(i2))
    b1 = eigvec_combination(N, k[i1], l[i1], alpha)
    b2 = eigvec_combination(N, k[i2], l[i2], beta)
    return np.ascontiguousarray(np.stack([b1, b2], axis=1))
