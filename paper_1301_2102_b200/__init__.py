"""B200-native banded-Lanczos block MINRES (Soodhalter, arXiv:1301.2102) — hot path.

The product is ``libbminres.so`` (C ABI, include/bminres.h; CUDA sm_100a kernels in
``csrc/``).  This package only builds it (``_build``) and binds it (``binding``).
"""
from .binding import (BminresError, DeviceCsr, HostCsrRows, Solver, SolveResult, STATUS, SUPPORTED_P, TorchComm,  # noqa: F401
                      halo_plan, interior_rows, lib, nccl_unique_id, workspace_bytes)

__all__ = ["BminresError", "DeviceCsr", "HostCsrRows", "Solver", "SolveResult", "STATUS", "SUPPORTED_P", "TorchComm", "halo_plan",
           "interior_rows", "lib", "nccl_unique_id", "workspace_bytes"]
