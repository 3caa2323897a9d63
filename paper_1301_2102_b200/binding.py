"""Thin ctypes binding of include/bminres.h — argument marshalling only.

Every step of the method runs in ``libbminres.so`` (CUDA, sm_100a).  There is no
CPU fallback: if the library or a CUDA device is missing, these calls raise.
PyTorch is used only to hold device memory and to hand raw pointers over.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _build

MAX_P = 32
NPHASE = 15
PHASES = ["spmm", "orth", "smallqr", "update", "slowpath", "start", "resid", "other", "reduce", "spmm_fused",
          "spmm_av", "epilogue", "epilogue_fused", "update_main", "prec"]
STATUS = {0: "OK", 1: "MAXIT", -1: "EINVAL", -2: "ECUDA", -3: "ENCCL", -4: "ENOMEM", -5: "EPOOL",
          -6: "ESINGULAR_R", -7: "EPIVOT"}
SUPPORTED_P = (1, 2, 3, 4, 5, 6, 7, 8, 16, 32)


class BminresError(RuntimeError):
    pass


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("stream", C.c_void_p),
                ("seed", C.c_uint64), ("pool_size", C.c_int32), ("use_x0", C.c_int32),
                ("record_history", C.c_int32), ("use_graphs", C.c_int32), ("timing", C.c_int32),
                ("split_spmm", C.c_int32), ("policy", C.c_int32), ("coeff_mode", C.c_int32),
                ("plan_reuse", C.c_int32), ("reserved", C.c_int32 * 3)]


class CsrStruct(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_begin", C.c_int64), ("n_loc", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


ALLRED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64))
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                          C.POINTER(C.c_int64))


class CommCallbacks(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allreduce", ALLRED_FN), ("alltoallv", ALLTOALLV_FN), ("exchange", EXCHANGE_FN)]


class Event(C.Structure):
    _fields_ = [("j", C.c_int64), ("col", C.c_int32), ("kind", C.c_int32), ("action", C.c_int32),
                ("pad", C.c_int32), ("ratio", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("p", C.c_int32), ("n", C.c_int64), ("iterations", C.c_int64),
                ("block_steps", C.c_int64), ("n_events", C.c_int64), ("slow_blocks", C.c_int64),
                ("history_len", C.c_int64), ("gpu_launches", C.c_int64),
                ("comp_res", C.c_double * MAX_P), ("true_res", C.c_double * MAX_P),
                ("solve_ms", C.c_double), ("loop_ms", C.c_double),
                ("phase_ms", C.c_double * NPHASE), ("phase_launches", C.c_int64 * NPHASE),
                ("bytes_per_block_step", C.c_double), ("spmm_bytes_per_launch", C.c_double),
                ("prec_true_res", C.c_double * MAX_P), ("preconditioned", C.c_int32), ("prec_levels", C.c_int32)]


_lib = None


def lib():
    """Load libbminres.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path) or _build.stale():
            _build.build()
        L = C.CDLL(path)
        L.bminres_default_options.argtypes = [C.POINTER(Options)]
        L.bminres_create.argtypes = [C.POINTER(Options), C.POINTER(C.c_void_p)]
        L.bminres_solve.argtypes = [C.c_void_p, C.POINTER(CsrStruct), C.c_void_p, C.c_void_p, C.c_int32,
                                    C.c_double, C.c_int64, C.c_double]
        L.bminres_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
        L.bminres_get_history.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.bminres_get_history.restype = C.c_int64
        L.bminres_get_events.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.bminres_get_events.restype = C.c_int64
        L.bminres_spmm.argtypes = [C.c_void_p, C.POINTER(CsrStruct), C.c_void_p, C.c_void_p, C.c_int32]
        L.bminres_random_vector.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64,
                                            C.c_int64, C.c_void_p, C.c_int64]
        L.bminres_workspace_bytes.argtypes = [C.c_int64, C.c_int32, C.c_int32]
        L.bminres_workspace_bytes.restype = C.c_size_t
        L.bminres_get_unique_id.argtypes = [C.c_void_p]
        L.bminres_init_nccl.argtypes = [C.c_void_p, C.c_void_p]
        L.bminres_set_comm_callbacks.argtypes = [C.c_void_p, C.POINTER(CommCallbacks)]
        L.bminres_halo_plan.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.bminres_interior_rows.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64)]
        L.bminres_set_preconditioner.argtypes = [C.c_void_p, C.POINTER(CsrStruct)]
        L.bminres_get_preconditioner.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.bminres_get_preconditioner.restype = C.c_int64
        L.bminres_precond_apply.argtypes = [C.c_void_p, C.POINTER(CsrStruct), C.c_void_p, C.c_void_p, C.c_int32,
                                            C.c_int32]
        L.bminres_last_error.argtypes = [C.c_void_p]
        L.bminres_last_error.restype = C.c_char_p
        L.bminres_destroy.argtypes = [C.c_void_p]
        L.bminres_destroy.restype = None
        _lib = L
    return _lib


EXPORTED = ["bminres_default_options", "bminres_create", "bminres_solve", "bminres_stats", "bminres_get_history",
            "bminres_get_events", "bminres_spmm", "bminres_random_vector", "bminres_workspace_bytes",
            "bminres_get_unique_id", "bminres_init_nccl", "bminres_set_comm_callbacks", "bminres_halo_plan",
            "bminres_interior_rows", "bminres_set_preconditioner", "bminres_get_preconditioner",
            "bminres_precond_apply", "bminres_last_error", "bminres_destroy"]


def _ptr(x):
    """Raw pointer of a torch tensor (device or host) or a numpy array."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise BminresError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise BminresError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(type(x))


@dataclass
class DeviceCsr:
    """CSR arrays resident on one CUDA device (torch tensors): int32 row_ptr/col_idx, fp64 values.
    n = rows held here; for a row partition (world > 1) rows [row_begin, row_begin + n) of an
    n_global x n_global matrix, column indices global."""
    n: int
    row_ptr: object
    col_idx: object
    values: object
    row_begin: int = 0
    n_global: int | None = None

    @property
    def nnz(self) -> int:
        return int(self.values.numel())

    @classmethod
    def from_host(cls, A, device="cuda"):
        import torch
        return cls(int(A.n), torch.from_numpy(np.ascontiguousarray(A.indptr, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(A.indices, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(A.data, dtype=np.float64)).to(device))

    @classmethod
    def rows_from_host(cls, A, row_begin: int, row_end: int, device="cuda"):
        """Rows [row_begin, row_end) of the host CSR A (global column indices kept)."""
        import torch
        ip = np.asarray(A.indptr, dtype=np.int64)
        k0, k1 = int(ip[row_begin]), int(ip[row_end])
        rp = (ip[row_begin:row_end + 1] - k0).astype(np.int32)
        return cls(row_end - row_begin, torch.from_numpy(rp).to(device),
                   torch.from_numpy(np.ascontiguousarray(A.indices[k0:k1], dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(A.data[k0:k1], dtype=np.float64)).to(device),
                   row_begin, int(A.n))


@dataclass
class HostCsrRows:
    """Rows [row_begin, row_begin + n) of an n_global x n_global host CSR (global columns):
    the host-memory form of one rank's rows (the library stages them)."""
    n: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    row_begin: int
    n_global: int

    @classmethod
    def from_host(cls, A, row_begin: int, row_end: int):
        ip = np.asarray(A.indptr, dtype=np.int64)
        k0, k1 = int(ip[row_begin]), int(ip[row_end])
        return cls(row_end - row_begin, (ip[row_begin:row_end + 1] - k0).astype(np.int32),
                   np.ascontiguousarray(A.indices[k0:k1], dtype=np.int32),
                   np.ascontiguousarray(A.data[k0:k1], dtype=np.float64), row_begin, int(A.n))


def _dtype_name(x) -> str:
    return str(x.dtype).replace("torch.", "")


def _check_panel(x, what, shape=None):
    """Row-major n x p fp64 panel (the layout every entry point takes)."""
    if _dtype_name(x) != "float64":
        raise BminresError(f"{what} must be float64, got {_dtype_name(x)}")
    if len(x.shape) != 2:
        raise BminresError(f"{what} must be 2-D (n x p), got shape {tuple(x.shape)}")
    if shape is not None and tuple(int(d) for d in x.shape) != tuple(int(d) for d in shape):
        raise BminresError(f"{what} has shape {tuple(x.shape)}, expected {tuple(shape)}")


def _check_csr(A):
    for nm, arr, want in (("row_ptr", A.row_ptr, "int32"), ("col_idx", A.col_idx, "int32"),
                          ("values", A.values, "float64")):
        if _dtype_name(arr) != want:
            raise BminresError(f"DeviceCsr.{nm} must be {want}, got {_dtype_name(arr)}")
    if int(A.row_ptr.numel()) != A.n + 1 or int(A.col_idx.numel()) != int(A.values.numel()):
        raise BminresError("DeviceCsr: row_ptr must hold n+1 offsets and col_idx / values nnz entries")


def _csr_struct(A) -> CsrStruct:
    s = CsrStruct()
    if isinstance(A, DeviceCsr):
        _check_csr(A)
        s.n, s.nnz = (A.n_global if A.n_global is not None else A.n), A.nnz
        s.row_ptr, s.col_idx, s.values = _ptr(A.row_ptr), _ptr(A.col_idx), _ptr(A.values)
        s.row_begin, s.n_loc = A.row_begin, A.n
        s._keep = (A,)
        return s
    else:  # host CSR (numpy): the library stages it
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        dv = np.ascontiguousarray(A.data, dtype=np.float64)
        s.n, s.nnz = int(A.n), int(ip[-1])
        s.row_ptr, s.col_idx, s.values = ip.ctypes.data, ix.ctypes.data, dv.ctypes.data
        keep = (ip, ix, dv)
    s.row_begin, s.n_loc = 0, s.n
    if isinstance(A, HostCsrRows):
        s.row_begin, s.n_loc, s.n = A.row_begin, A.n, A.n_global
    s._keep = keep
    return s


def halo_plan(world: int, rank: int, offsets, col_idx):
    """bminres_halo_plan (host only): (local_col, halo_rows, halo_count) of this rank's global
    column indices under the row partition `offsets` (world+1 int64)."""
    L = lib()
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    col = np.ascontiguousarray(col_idx, dtype=np.int32)
    nh = C.c_int64()
    rc = L.bminres_halo_plan(world, rank, off.ctypes.data, len(col), col.ctypes.data, None, None, C.byref(nh), None)
    if rc != 0:
        raise BminresError(f"bminres_halo_plan: {STATUS.get(rc, rc)}")
    local = np.zeros(max(len(col), 1), dtype=np.int32)
    rows = np.zeros(max(nh.value, 1), dtype=np.int64)
    cnt = np.zeros(world, dtype=np.int64)
    rc = L.bminres_halo_plan(world, rank, off.ctypes.data, len(col), col.ctypes.data, local.ctypes.data,
                             rows.ctypes.data, C.byref(nh), cnt.ctypes.data)
    if rc != 0:
        raise BminresError(f"bminres_halo_plan: {STATUS.get(rc, rc)}")
    return local[:len(col)], rows[:nh.value], cnt


def interior_rows(row_ptr, local_col):
    """bminres_interior_rows (host only): the longest run [lo, hi) of rows with only local columns."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    lc = np.ascontiguousarray(local_col, dtype=np.int32)
    if lc.size == 0:
        lc = np.zeros(1, dtype=np.int32)
    lo, hi = C.c_int64(), C.c_int64()
    rc = lib().bminres_interior_rows(len(rp) - 1, rp.ctypes.data, lc.ctypes.data, C.byref(lo), C.byref(hi))
    if rc != 0:
        raise BminresError(f"bminres_interior_rows: {STATUS.get(rc, rc)}")
    return lo.value, hi.value


@dataclass
class SolveResult:
    status: int
    iterations: int
    X: object
    history: np.ndarray
    events: list
    stats: dict = field(default_factory=dict)

    @property
    def status_name(self) -> str:
        return STATUS.get(self.status, str(self.status))


class TorchComm:
    """Host-callback transport over a torch.distributed process group (e.g. gloo): the testing
    transport of a row-partitioned solve (bminres_set_comm_callbacks).  Marshalling only; the
    allreduce is an all-gather summed in rank order, so every rank gets bitwise identical sums."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.cb = CommCallbacks(None, ALLRED_FN(self._allreduce), ALLTOALLV_FN(self._alltoallv),
                                EXCHANGE_FN(self._exchange))

    def _allreduce(self, ctx, buf, count):
        try:
            import torch
            a = np.ctypeslib.as_array(buf, shape=(count,))
            t = torch.from_numpy(a.copy())
            parts = [torch.empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(parts, t, group=self.group)
            tot = parts[0].clone()
            for q in range(1, self.world):
                tot += parts[q]
            a[:] = tot.numpy()
            return 0
        except Exception:   # noqa: BLE001 -- reported to the library as a transport error
            return 1

    def _p2p(self, send, scount, recv, rcount, dtype):
        import torch
        sc = [int(scount[q]) for q in range(self.world)]
        rc = [int(rcount[q]) for q in range(self.world)]
        s_arr = np.ctypeslib.as_array(send, shape=(max(sum(sc), 1),))
        r_arr = np.ctypeslib.as_array(recv, shape=(max(sum(rc), 1),))
        so = np.concatenate([[0], np.cumsum(sc)]).astype(int)
        ro = np.concatenate([[0], np.cumsum(rc)]).astype(int)
        reqs, bufs = [], []
        for q in range(self.world):
            if q == self.rank:
                r_arr[ro[q]:ro[q] + rc[q]] = s_arr[so[q]:so[q] + sc[q]]
                continue
            if sc[q]:
                reqs.append(self.dist.isend(torch.from_numpy(s_arr[so[q]:so[q] + sc[q]].copy()), q, group=self.group))
            if rc[q]:
                t = torch.empty(rc[q], dtype=dtype)
                bufs.append((q, t))
                reqs.append(self.dist.irecv(t, q, group=self.group))
        for r in reqs:
            r.wait()
        for q, t in bufs:
            r_arr[ro[q]:ro[q] + rc[q]] = t.numpy()

    def _alltoallv(self, ctx, send, scount, recv, rcount):
        try:
            import torch
            self._p2p(send, scount, recv, rcount, torch.int64)
            return 0
        except Exception:   # noqa: BLE001
            return 1

    def _exchange(self, ctx, send, scount, recv, rcount):
        try:
            import torch
            self._p2p(send, scount, recv, rcount, torch.float64)
            return 0
        except Exception:   # noqa: BLE001
            return 1


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().bminres_get_unique_id(C.addressof(buf))
    if rc != 0:
        raise BminresError(f"bminres_get_unique_id: {STATUS.get(rc, rc)}: {lib().bminres_last_error(None).decode()}")
    return bytes(buf)


class Solver:
    """One handle of the C ABI (bminres_create ... bminres_destroy).

    Row-partitioned solves (world > 1): pass rank/world and comm = "nccl" (the unique id is
    broadcast over the default torch.distributed group) or a TorchComm (host callbacks)."""

    def __init__(self, device: int = 0, *, pool_size: int = 1, seed: int = 0, use_graphs: bool = True,
                 timing: bool = False, record_history: bool = True, use_x0: bool = False, stream=None,
                 rank: int = 0, world: int = 1, comm=None, split_spmm: int = 0, policy: int = 0,
                 plan_reuse: bool = False):
        L = lib()
        o = Options()
        L.bminres_default_options(C.byref(o))
        o.device, o.pool_size, o.seed = device, pool_size, seed
        o.split_spmm = split_spmm
        o.policy, o.plan_reuse = policy, int(plan_reuse)
        o.use_graphs, o.timing, o.record_history, o.use_x0 = int(use_graphs), int(timing), int(record_history), int(use_x0)
        o.stream = stream
        o.rank, o.world = rank, world
        h = C.c_void_p()
        rc = L.bminres_create(C.byref(o), C.byref(h))
        if rc != 0:
            raise BminresError(f"bminres_create: {STATUS.get(rc, rc)}: {L.bminres_last_error(None).decode()}")
        self._h = h
        self.options = o
        self._comm = comm
        if comm == "nccl":
            uid = nccl_unique_id() if rank == 0 else None
            if world > 1:
                import torch.distributed as dist
                box = [uid]
                dist.broadcast_object_list(box, src=0)
                uid = box[0]
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            rc = L.bminres_init_nccl(self._h, C.addressof(buf))
            if rc != 0:
                raise BminresError(f"bminres_init_nccl: {STATUS.get(rc, rc)}: {self.last_error()}")
        elif comm is not None:
            rc = L.bminres_set_comm_callbacks(self._h, C.byref(comm.cb))
            if rc != 0:
                raise BminresError(f"bminres_set_comm_callbacks: {STATUS.get(rc, rc)}")

    def close(self):
        if getattr(self, "_h", None):
            lib().bminres_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def last_error(self) -> str:
        return lib().bminres_last_error(self._h).decode()

    def solve(self, A, B, X=None, *, tol=1e-8, maxit=1000, deflation_tol=1e-8, history=True, raise_on_error=True):
        """Solve A X = B.  A: DeviceCsr or host CSR (n, indptr, indices, data); B/X: torch CUDA
        tensors or numpy arrays (row-major n×p fp64).  Returns SolveResult (X is the array written)."""
        L = lib()
        p = int(B.shape[1])
        if X is None:
            if hasattr(B, "data_ptr"):
                import torch
                X = torch.zeros_like(B)
            else:
                X = np.zeros_like(B)
        _check_panel(B, "B")
        _check_panel(X, "X", B.shape)
        s = _csr_struct(A)
        if int(B.shape[0]) != s.n_loc:
            raise BminresError(f"B has {int(B.shape[0])} rows, A holds {s.n_loc}")
        rc = L.bminres_solve(self._h, C.byref(s), _ptr(B), _ptr(X), p, float(tol), int(maxit), float(deflation_tol))
        if rc < 0 and raise_on_error:
            raise BminresError(f"bminres_solve: {STATUS.get(rc, rc)}: {self.last_error()}")
        st = self.stats()
        hist = None
        if history and st["history_len"] > 0:
            hist = np.zeros((st["history_len"], p))
            L.bminres_get_history(self._h, hist.ctypes.data, st["history_len"])
        evs = []
        if st["n_events"] > 0:
            buf = (Event * st["n_events"])()
            c = L.bminres_get_events(self._h, C.addressof(buf), st["n_events"])
            evs = [dict(j=int(e.j), col=int(e.col), kind=int(e.kind), action=int(e.action), ratio=float(e.ratio))
                   for e in buf[:c]]
        return SolveResult(rc, st["iterations"], X, hist, evs, st)

    def stats(self) -> dict:
        s = Stats()
        lib().bminres_stats(self._h, C.byref(s))
        p = s.p
        return dict(status=s.status, p=p, n=s.n, iterations=s.iterations, block_steps=s.block_steps,
                    n_events=s.n_events, slow_blocks=s.slow_blocks, history_len=s.history_len,
                    gpu_launches=s.gpu_launches, comp_res=list(s.comp_res[:p]), true_res=list(s.true_res[:p]),
                    solve_ms=s.solve_ms, loop_ms=s.loop_ms,
                    phase_ms={PHASES[i]: s.phase_ms[i] for i in range(NPHASE)},
                    phase_launches={PHASES[i]: s.phase_launches[i] for i in range(NPHASE)},
                    bytes_per_block_step=s.bytes_per_block_step, spmm_bytes_per_launch=s.spmm_bytes_per_launch,
                    preconditioned=bool(s.preconditioned), prec_true_res=list(s.prec_true_res[:p]),
                    prec_levels=s.prec_levels)

    # ---- f3: IC(0) split preconditioning (bminres_set_preconditioner)

    def set_preconditioner(self, M):
        """Factor M (SPD CSR, DeviceCsr or host) with IC(0) and precondition later solves; None clears."""
        if M is None:
            rc = lib().bminres_set_preconditioner(self._h, None)
        else:
            s = _csr_struct(M)
            rc = lib().bminres_set_preconditioner(self._h, C.byref(s))
        if rc != 0:
            raise BminresError(f"bminres_set_preconditioner: {STATUS.get(rc, rc)}: {self.last_error()}")

    def get_preconditioner(self) -> np.ndarray:
        """The IC(0) factor's values in the order of M's lower-triangle entries (diagonal last per row)."""
        nz = int(lib().bminres_get_preconditioner(self._h, None, 0))
        out = np.zeros(max(nz, 1))
        lib().bminres_get_preconditioner(self._h, out.ctypes.data, nz)
        return out[:nz]

    def precond_apply(self, X, mode: int, A: DeviceCsr | None = None, Y=None):
        """mode 0: L^-1 X, 1: L^-T X, 2: L^-1 A L^-T X (device tensors)."""
        import torch
        if Y is None:
            Y = torch.empty_like(X)
        _check_panel(X, "X")
        _check_panel(Y, "Y", X.shape)
        s = _csr_struct(A) if A is not None else None
        rc = lib().bminres_precond_apply(self._h, C.byref(s) if s is not None else None, _ptr(X), _ptr(Y),
                                         int(X.shape[1]), int(mode))
        if rc != 0:
            raise BminresError(f"bminres_precond_apply: {STATUS.get(rc, rc)}: {self.last_error()}")
        return Y

    def spmm(self, A: DeviceCsr, X, Y=None):
        """Y = A X through the solver's SpMM kernel (device tensors)."""
        import torch
        if Y is None:
            Y = torch.empty_like(X)
        _check_panel(X, "X")
        _check_panel(Y, "Y", (A.n, X.shape[1]))
        s = _csr_struct(A)
        rc = lib().bminres_spmm(self._h, C.byref(s), _ptr(X), _ptr(Y), int(X.shape[1]))
        if rc != 0:
            raise BminresError(f"bminres_spmm: {STATUS.get(rc, rc)}: {self.last_error()}")
        return Y

    def random_vector(self, seed, stream, event, row_begin, n, out, stride=1):
        rc = lib().bminres_random_vector(self._h, seed, stream, event, row_begin, n, _ptr(out), stride)
        if rc != 0:
            raise BminresError(f"bminres_random_vector: {STATUS.get(rc, rc)}: {self.last_error()}")
        return out


def workspace_bytes(n: int, p: int, pool_size: int = 1) -> int:
    return int(lib().bminres_workspace_bytes(n, p, pool_size))
