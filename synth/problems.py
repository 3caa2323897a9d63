"""Seeded generators for the test matrices and right-hand sides.

Recipes (DESIGN.md "Input recipe" restates them):

* Shifted Laplacians, the paper's model problem family (§8, P:1020-1025:
  L = I⊗T + T⊗I with T = tridiag(1,-2,1)).  BASELINE.json's configs use the
  unscaled stencil "diag d - shift, off-diagonal -1" with Dirichlet boundaries
  (neighbours outside the grid are dropped); lexicographic ordering, x fastest,
  z slowest.  Column indices inside a row are strictly increasing.
* Right-hand sides: ``numpy.random.default_rng(seed).standard_normal((n, p))`` as
  a C-order (row-major n×p) array — the panel layout of the GPU path.
* Config 3's dependent block B = [G, G·C + eps·N] (BASELINE.json configs[2]).
* Config 5's unstructured band + long-range matrix (BASELINE.json configs[4]),
  drawn in the order SURVEY.md §8(d) fixes.

CSR arrays are (indptr int32, indices int32, data float64); nnz < 2**31.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Csr", "Problem", "stencil_csr", "laplacian_2d", "laplacian_3d", "gaussian_rhs",
    "dependent_rhs", "unstructured_csr", "random_sym_sparse", "irregular_sym_csr", "diag_csr", "dense_to_csr",
    "csr_to_dense", "config", "CONFIGS",
]


@dataclass
class Csr:
    n: int
    indptr: np.ndarray   # int32, n+1
    indices: np.ndarray  # int32, nnz
    data: np.ndarray     # float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def bytes_model(self) -> int:
        """Bytes the CSR arrays occupy (fp64 values + int32 cols + int32 row_ptr)."""
        return 12 * self.nnz + 4 * (self.n + 1)


@dataclass
class Problem:
    name: str
    A: Csr
    B: np.ndarray            # row-major n×p float64
    tol: float
    maxit: int
    tau: float = 1e-8        # deflation_tol (the paper's gamma)
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.A.n

    @property
    def p(self) -> int:
        return self.B.shape[1]


def stencil_csr(dims, diag: float, off: float = -1.0) -> Csr:
    """(2·len(dims)+1)-point stencil on a Dirichlet grid; dims = (nx,) , (nx, ny) or (nx, ny, nz)."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    r = np.arange(n, dtype=np.int64)
    coords = []
    stride = 1
    strides = []
    for d in dims:
        coords.append((r // stride) % d)
        strides.append(stride)
        stride *= d
    # neighbour offsets in increasing column order: slowest axis first, negative side
    cand_cols = []
    cand_vals = []
    for ax in reversed(range(len(dims))):
        ok = coords[ax] > 0
        cand_cols.append(np.where(ok, r - strides[ax], -1))
        cand_vals.append(off)
    cand_cols.append(r)
    cand_vals.append(diag)
    for ax in range(len(dims)):
        ok = coords[ax] < dims[ax] - 1
        cand_cols.append(np.where(ok, r + strides[ax], -1))
        cand_vals.append(off)
    cols = np.stack(cand_cols, axis=1)                 # n × K, row-major → row order kept
    vals = np.broadcast_to(np.asarray(cand_vals, dtype=np.float64), cols.shape)
    mask = cols >= 0
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    assert indptr[-1] < 2**31
    indices = cols[mask].astype(np.int32)
    data = np.ascontiguousarray(vals[mask], dtype=np.float64)
    return Csr(n, indptr.astype(np.int32), indices, data)


def laplacian_2d(nx: int, ny: int | None = None, shift: float = 0.0) -> Csr:
    """2-D 5-point Laplacian (diag 4, off -1) minus shift·I."""
    return stencil_csr((nx, ny or nx), 4.0 - shift)


def laplacian_3d(nx: int, ny: int | None = None, nz: int | None = None, shift: float = 0.0) -> Csr:
    """3-D 7-point Laplacian (diag 6, off -1) minus shift·I."""
    return stencil_csr((nx, ny or nx, nz or nx), 6.0 - shift)


def gaussian_rhs(n: int, p: int, seed: int = 0) -> np.ndarray:
    return np.ascontiguousarray(np.random.default_rng(seed).standard_normal((n, p)))


def dependent_rhs(n: int, half: int, eps: float, seed: int = 0) -> np.ndarray:
    """B = [G, G·C + eps·N], drawn G (n×half), then C (half×half), then N (n×half)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, half))
    C = rng.standard_normal((half, half))
    N = rng.standard_normal((n, half))
    return np.ascontiguousarray(np.concatenate([G, G @ C + eps * N], axis=1))


def _coo_to_csr(n, rows, cols, vals) -> Csr:
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    # sum duplicates
    key = rows.astype(np.int64) * n + cols
    uniq, start = np.unique(key, return_index=True)
    sums = np.add.reduceat(vals, start) if len(vals) else vals
    urows = (uniq // n).astype(np.int64)
    ucols = (uniq % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, urows + 1, 1)
    np.cumsum(indptr, out=indptr)
    assert indptr[-1] < 2**31
    return Csr(n, indptr.astype(np.int32), ucols, np.ascontiguousarray(sums, dtype=np.float64))


def unstructured_csr(n: int, half_width: int = 13, seed: int = 0, p: int = 16):
    """BASELINE.json configs[4]: band of half-width 13 + long-range pairs, symmetrised.

    Draw order (SURVEY.md §8(d) cfg 5): band values k=1..13, long-range i then j
    (2n each, kept if |i-j| > half_width), their values, the diagonal U[-2,2], then B.
    Returns (Csr, B).
    """
    rng = np.random.default_rng(seed)
    s = 1.0 / np.sqrt(27.0)
    rows, cols, vals = [], [], []
    for k in range(1, half_width + 1):
        v = rng.standard_normal(n - k) * s
        i = np.arange(n - k, dtype=np.int64)
        rows += [i, i + k]
        cols += [i + k, i]
        vals += [v, v]
    li = rng.integers(0, n, 2 * n)
    lj = rng.integers(0, n, 2 * n)
    keep = np.abs(li - lj) > half_width
    li, lj = li[keep], lj[keep]
    lv = rng.standard_normal(len(li)) * s
    rows += [li, lj]
    cols += [lj, li]
    vals += [lv, lv]
    d = rng.uniform(-2.0, 2.0, n)
    rows.append(np.arange(n, dtype=np.int64))
    cols.append(np.arange(n, dtype=np.int64))
    vals.append(d)
    B = np.ascontiguousarray(rng.standard_normal((n, p)))
    A = _coo_to_csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    return A, B


def dense_to_csr(M: np.ndarray) -> Csr:
    M = np.asarray(M, dtype=np.float64)
    n = M.shape[0]
    r, c = np.nonzero(M)
    return _coo_to_csr(n, r.astype(np.int64), c.astype(np.int64), M[r, c])


def csr_to_dense(A: Csr) -> np.ndarray:
    D = np.zeros((A.n, A.n))
    for i in range(A.n):
        for k in range(A.indptr[i], A.indptr[i + 1]):
            D[i, A.indices[k]] += A.data[k]
    return D


def random_sym_sparse(n: int, density: float = 0.15, seed: int = 0, shift: float | None = None) -> Csr:
    """Small random sparse symmetric indefinite matrix for the brute-force pins."""
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
    M = np.triu(M, 1)
    M = M + M.T
    d = rng.uniform(-2.0, 2.0, n) if shift is None else np.full(n, shift)
    M[np.diag_indices(n)] = d
    return dense_to_csr(M)


def irregular_sym_csr(n: int, rng, hubs: int = 0, empty_rows: int = 0) -> Csr:
    """Random sparse symmetric indefinite CSR with an irregular row-length mix (test input only):
    degrees 0..12 drawn per row, `hubs` rows with up to 300 entries (rows longer than every gather
    batch), `empty_rows` rows with no entry at all (zero row and column), a diagonal U[-2, 2]."""
    import scipy.sparse as sp
    deg = rng.integers(0, 13, n)
    for h in rng.choice(n, hubs, replace=False):
        hi = min(300, n - 1)
        deg[h] = rng.integers(60 if hi > 60 else max(1, hi // 2), hi)   # (small n: a proportionally long row)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size) / 3.0
    S = sp.triu(sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr(), 1)
    S = (S + S.T + sp.diags(rng.uniform(-2.0, 2.0, n))).tolil()
    for e in rng.choice(n, empty_rows, replace=False):
        S[e, :] = 0.0
        S[:, e] = 0.0
    S = S.tocsr()
    S.eliminate_zeros()
    S.sort_indices()
    return Csr(n, S.indptr.astype(np.int32), S.indices.astype(np.int32), S.data.astype(np.float64))


def diag_csr(d) -> Csr:
    d = np.asarray(d, dtype=np.float64)
    n = len(d)
    return Csr(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), d.copy())


def config(idx, eps: float = 0.0, seed: int = 0) -> Problem:
    """BASELINE.json configs by 1-based index; "1c" is the non-singular companion."""
    if idx == 1:
        A = laplacian_2d(32, shift=2.0)
        return Problem("cfg1_lap2d_32_shift2", A, gaussian_rhs(A.n, 4, seed), 1e-8, 2000)
    if idx == "1c":
        A = laplacian_2d(31, shift=2.0)
        return Problem("cfg1c_lap2d_31_shift2", A, gaussian_rhs(A.n, 4, seed), 1e-8, 2000)
    if idx == 2:
        A = laplacian_3d(64, shift=3.0)
        return Problem("cfg2_lap3d_64_shift3", A, gaussian_rhs(A.n, 8, seed), 1e-8, 500_000)
    if idx == 3:
        A = laplacian_2d(512, shift=2.5)
        return Problem(f"cfg3_lap2d_512_shift2.5_eps{eps:g}", A, dependent_rhs(A.n, 8, eps, seed),
                       1e-8, 1_000_000, meta={"eps": eps})
    if idx == 4:
        A = laplacian_3d(256, shift=3.0)
        return Problem("cfg4_lap3d_256_shift3", A, gaussian_rhs(A.n, 32, seed), 1e-6, 2_000_000)
    if idx == 5:
        A, B = unstructured_csr(4_194_304, seed=seed)
        return Problem("cfg5_unstructured_4M", A, B, 1e-6, 2_000_000)
    raise ValueError(idx)


CONFIGS = [1, "1c", 2, 3, 4, 5]
