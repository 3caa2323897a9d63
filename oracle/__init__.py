"""CPU oracle for banded-Lanczos block MINRES — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product
(``paper_1301_2102_b200``) never imports it and has no CPU fallback.

The arithmetic lives in ``bminres_oracle.c`` (plain C, one thread, fp64),
written from PAPER.md in the paper's per-iteration order (Alg. 1 inside Alg. 2,
with the index corrections of DESIGN.md "Readings of the paper").  This module
only compiles it with gcc and marshals arguments through ctypes.

Pins: see tests/test_oracle_pins.py.  "parity unpinned": the replacement
vectors' values (reading C17 — the paper's own generator, Matlab mt19937ar,
P:1017-1019, is not reproducible here).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bminres_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MAX_P = 64
STATUS = {0: "OK", 1: "MAXIT", -1: "EINVAL", -4: "ENOMEM", -5: "EPOOL", -6: "ESINGULAR_R"}


class Event(C.Structure):
    _fields_ = [("j", C.c_int64), ("col", C.c_int32), ("kind", C.c_int32), ("action", C.c_int32),
                ("pad", C.c_int32), ("ratio", C.c_double)]


class Config(C.Structure):
    _fields_ = [("p", C.c_int32), ("pool_size", C.c_int32), ("use_x0", C.c_int32), ("policy", C.c_int32),
                ("tol", C.c_double), ("tau", C.c_double), ("maxit", C.c_int64), ("seed", C.c_uint64),
                ("history", C.c_void_p), ("history_cap", C.c_int64),
                ("events", C.c_void_p), ("events_cap", C.c_int64),
                ("dbg_cap", C.c_int64), ("dbg_U", C.c_void_p), ("dbg_H", C.c_void_p),
                ("dbg_R", C.c_void_p), ("dbg_M", C.c_void_p), ("dbg_Z", C.c_void_p),
                ("dbg_S", C.c_void_p)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_int32), ("iterations", C.c_int64),
                ("n_events", C.c_int64), ("true_res", C.c_double * MAX_P),
                ("comp_res", C.c_double * MAX_P), ("start_s", C.c_double), ("loop_s", C.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_solve.restype = C.c_int
        _lib.orc_solve.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.POINTER(Config), C.POINTER(Result)]
        _lib.orc_csr_block.restype = None
        _lib.orc_csr_block.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                       C.c_void_p, C.c_void_p]
        _lib.orc_rand_entry.restype = C.c_double
        _lib.orc_rand_entry.argtypes = [C.c_uint64] * 4
        _lib.orc_splitmix64.restype = C.c_uint64
        _lib.orc_splitmix64.argtypes = [C.c_uint64]
        _lib.orc_house_gen.restype = None
        _lib.orc_house_gen.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_house_apply.restype = None
        _lib.orc_house_apply.argtypes = [C.c_int32, C.c_void_p, C.c_double, C.c_void_p]
        _lib.orc_ic0.restype = C.c_int
        _lib.orc_ic0.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_int64)]
        _lib.orc_trsv_lower.restype = None
        _lib.orc_trsv_lower.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_trsv_upper.restype = None
        _lib.orc_trsv_upper.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_prec_op_block.restype = None
        _lib.orc_prec_op_block.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        _lib.orc_solve_prec.restype = C.c_int
        _lib.orc_solve_prec.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Config), C.POINTER(Result),
                                        C.c_void_p]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class OracleResult:
    status: int
    iterations: int
    history: np.ndarray            # (iterations+1) × p computed relative residuals
    events: list                   # list of dicts
    X: np.ndarray
    true_res: np.ndarray
    comp_res: np.ndarray
    dbg: dict = field(default_factory=dict)
    start_s: float = 0.0           # wall time of the start block + pool (instrumentation)
    loop_s: float = 0.0            # wall time of the iteration loop (instrumentation)
    ptrue_res: np.ndarray | None = None   # preconditioned solves: unpreconditioned ||b - A x|| / ||b||

    @property
    def status_name(self) -> str:
        return STATUS.get(self.status, str(self.status))


def solve(A, B, *, tol=1e-8, maxit=100, tau=1e-8, seed=0, pool_size=1, X0=None,
          history=True, events_cap=4096, debug_iters=0, policy=0, prec=None) -> OracleResult:
    """Run the oracle.  A: synth.Csr; B: n×p float64 (row-major).  policy: 0 replacement
    (P:690-729), 1 block-size reduction "shrink".  prec: an IC(0) factor L (from
    ``ic0``) -- the split-preconditioned solve of reading R8 (f3): the method on
    L^-1 A L^-T with Rhat_0 = L^-1 (B - A X0), X = X0 + L^-T Yhat; history / comp_res / true_res are
    the preconditioned residuals (relative to ||Rhat_0||), ptrue_res the unpreconditioned one."""
    B = np.ascontiguousarray(B, dtype=np.float64)
    n, p = B.shape
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int32)
    indices = np.ascontiguousarray(A.indices, dtype=np.int32)
    data = np.ascontiguousarray(A.data, dtype=np.float64)
    X = np.zeros((n, p)) if X0 is None else np.array(X0, dtype=np.float64, order="C", copy=True)
    cfg = Config()
    cfg.p, cfg.pool_size, cfg.use_x0, cfg.policy = p, pool_size, int(X0 is not None), int(policy)
    cfg.tol, cfg.tau, cfg.maxit, cfg.seed = tol, tau, maxit, seed
    hist = np.zeros((maxit + 1, p)) if history else None
    if hist is not None:
        cfg.history, cfg.history_cap = _ptr(hist).value, maxit + 1
    ev = (Event * max(events_cap, 1))()
    cfg.events, cfg.events_cap = C.addressof(ev), events_cap
    dbg = {}
    if debug_iters:
        d = debug_iters
        dbg = dict(U=np.zeros((d + p, n)), H=np.zeros((d, d + p)), R=np.zeros((d, d)),
                   M=np.zeros((d, n)), Z=np.zeros((d, p)), S=np.zeros((p, p)))
        cfg.dbg_cap = d
        cfg.dbg_U, cfg.dbg_H, cfg.dbg_R = _ptr(dbg["U"]).value, _ptr(dbg["H"]).value, _ptr(dbg["R"]).value
        cfg.dbg_M, cfg.dbg_Z, cfg.dbg_S = _ptr(dbg["M"]).value, _ptr(dbg["Z"]).value, _ptr(dbg["S"]).value
    res = Result()
    ptrue = None
    if prec is None:
        lib().orc_solve(n, _ptr(indptr), _ptr(indices), _ptr(data), _ptr(B), _ptr(X), C.byref(cfg), C.byref(res))
    else:
        if debug_iters:
            raise ValueError("debug dumps are not kept for preconditioned solves")
        Lp, Li, Lx = _csr_arrays(prec)
        ptrue = np.zeros(p)
        lib().orc_solve_prec(n, _ptr(indptr), _ptr(indices), _ptr(data), _ptr(Lp), _ptr(Li), _ptr(Lx), _ptr(B),
                             _ptr(X), C.byref(cfg), C.byref(res), _ptr(ptrue))
    it = int(res.iterations)
    events = [dict(j=int(e.j), col=int(e.col), kind=int(e.kind), action=int(e.action), ratio=float(e.ratio))
              for e in ev[: min(res.n_events, events_cap)]]
    if debug_iters:
        # stored transposed (column-major in C) → give natural orientation
        dbg = dict(U=dbg["U"].T.copy(), H=dbg["H"].T.copy(), R=dbg["R"].T.copy(), M=dbg["M"].T.copy(),
                   Z=dbg["Z"], S=dbg["S"])
    return OracleResult(int(res.status), it, hist[: it + 1].copy() if hist is not None else None, events, X,
                        np.array(res.true_res[:p]), np.array(res.comp_res[:p]), dbg, float(res.start_s),
                        float(res.loop_s), ptrue)


def csr_block(A, X: np.ndarray) -> np.ndarray:
    """Y = A X, each row summed in CSR order with fma (oracle of the SpMM)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, p = X.shape
    Y = np.empty_like(X)
    lib().orc_csr_block(n, _ptr(np.ascontiguousarray(A.indptr, dtype=np.int32)),
                        _ptr(np.ascontiguousarray(A.indices, dtype=np.int32)),
                        _ptr(np.ascontiguousarray(A.data, dtype=np.float64)), p, _ptr(X), _ptr(Y))
    return Y


def rand_entry(seed: int, stream: int, event: int, row: int) -> float:
    return lib().orc_rand_entry(seed, stream, event, row)


def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def house_gen(x: np.ndarray):
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = np.empty_like(x)
    tau, beta = C.c_double(), C.c_double()
    lib().orc_house_gen(len(x), _ptr(x), _ptr(v), C.byref(tau), C.byref(beta))
    return v, tau.value, beta.value


def house_apply(v: np.ndarray, tau: float, y: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    y = np.array(y, dtype=np.float64, copy=True)
    lib().orc_house_apply(len(v), _ptr(v), tau, _ptr(y))
    return y


# ---- f3: IC(0) split preconditioning (reading R8) ----

def _csr_arrays(A):
    return (np.ascontiguousarray(A.indptr, dtype=np.int32), np.ascontiguousarray(A.indices, dtype=np.int32),
            np.ascontiguousarray(A.data, dtype=np.float64))


class PivotBreakdown(ValueError):
    def __init__(self, row):
        super().__init__(f"IC(0) pivot <= 0 at row {row}")
        self.row = row


def ic0(M):
    """Zero-fill incomplete Cholesky L of the symmetric CSR M (both triangles, columns ascending):
    L has the pattern of M's lower triangle, the diagonal last per row, and (L L^T)_ik = m_ik on it.
    Returns a synth-style Csr (same class as M).  Raises PivotBreakdown on a pivot <= 0."""
    ip, ix, dx = _csr_arrays(M)
    n = len(ip) - 1
    nzl = int(np.count_nonzero(ix <= np.repeat(np.arange(n), np.diff(ip))))
    Lp = np.zeros(n + 1, dtype=np.int32)
    Li = np.zeros(max(nzl, 1), dtype=np.int32)
    Lx = np.zeros(max(nzl, 1))
    bad = C.c_int64(-1)
    st = lib().orc_ic0(n, _ptr(ip), _ptr(ix), _ptr(dx), _ptr(Lp), _ptr(Li), _ptr(Lx), C.byref(bad))
    if st == -7:
        raise PivotBreakdown(int(bad.value))
    if st != 0:
        raise ValueError(f"orc_ic0: status {st} (row {bad.value}: missing diagonal?)")
    return type(M)(n, Lp, Li[:nzl].copy(), Lx[:nzl].copy())


def trsv_lower(L, b: np.ndarray) -> np.ndarray:
    """y = L^-1 b (forward substitution); b a vector or a row-major n x p block (column by column)."""
    return _trsv(L, b, lib().orc_trsv_lower, transpose=False)


def trsv_upper(L, v: np.ndarray) -> np.ndarray:
    """z = L^-T v (backward substitution on L^T)."""
    return _trsv(L, v, lib().orc_trsv_upper, transpose=True)


def _transpose(L):
    n = len(L.indptr) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(L.indptr))
    order = np.lexsort((rows, L.indices))      # by column, then row
    Up = np.zeros(n + 1, dtype=np.int32)
    np.add.at(Up, L.indices.astype(np.int64) + 1, 1)
    return np.cumsum(Up).astype(np.int32), rows[order].astype(np.int32), np.ascontiguousarray(L.data[order])


def _trsv(L, b, fn, transpose):
    b = np.asarray(b, dtype=np.float64)
    vec = b.ndim == 1
    Bm = b.reshape(len(b), -1)
    if transpose:
        ip, ix, dx = _transpose(L)
    else:
        ip, ix, dx = _csr_arrays(L)
    n = len(ip) - 1
    out = np.empty_like(Bm)
    for c in range(Bm.shape[1]):
        x = np.ascontiguousarray(Bm[:, c])
        y = np.empty(n)
        fn(n, _ptr(ip), _ptr(ix), _ptr(dx), _ptr(x), _ptr(y))
        out[:, c] = y
    return out[:, 0].copy() if vec else out


def prec_op_block(A, L, X: np.ndarray) -> np.ndarray:
    """Y = L^-1 A L^-T X for a row-major n x p block (the operator of the preconditioned solve)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, p = X.shape
    Y = np.empty_like(X)
    ip, ix, dx = _csr_arrays(A)
    Lp, Li, Lx = _csr_arrays(L)
    lib().orc_prec_op_block(n, _ptr(ip), _ptr(ix), _ptr(dx), _ptr(Lp), _ptr(Li), _ptr(Lx), p, _ptr(X), _ptr(Y))
    return Y
