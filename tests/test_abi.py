"""The C-ABI library builds, loads and exports every symbol include/bminres.h declares (CPU only)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "bminres.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bminres_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("bminres_create", "bminres_solve", "bminres_stats", "bminres_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1301_2102_b200 import binding
    L = binding.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(declared_functions()) == set(binding.EXPORTED)


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the header structs have the C sizes (compiled with gcc against the header)."""
    import ctypes
    import subprocess
    from paper_1301_2102_b200 import binding
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include "bminres.h"\nint main(){printf("%zu %zu %zu %zu %zu\\n",'
                 'sizeof(bminres_options), sizeof(bminres_stats_t), sizeof(bminres_event), sizeof(bminres_csr),'
                 'sizeof(bminres_comm_callbacks));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = subprocess.check_output([str(exe)]).decode().split()
    want = [ctypes.sizeof(binding.Options), ctypes.sizeof(binding.Stats), ctypes.sizeof(binding.Event),
            ctypes.sizeof(binding.CsrStruct), ctypes.sizeof(binding.CommCallbacks)]
    assert [int(x) for x in got] == want


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1301_2102_b200 import BminresError, Solver
    with pytest.raises(BminresError):
        Solver(0)


def test_product_does_not_import_oracle():
    """The product package never references the oracle (no CPU fallback path)."""
    pkg = os.path.join(ROOT, "paper_1301_2102_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "bminres_oracle" not in txt, f
