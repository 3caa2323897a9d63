#!/usr/bin/env python
"""Per-kernel SASS instruction summary of the built libbminres.so (static evidence of the fp64
tensor path, the bulk / 256-bit loads and the absence of local-memory spills).

  python profiles/sass_summary.py [lib.so] > profiles/r02_sass_summary.md

Reads `cuobjdump -sass` and `cuobjdump -res-usage`; counts static instructions per kernel for
the mnemonics that matter on this path: DMMA (fp64 mma.sync, the fp64 tensor-core path on
sm_100a -- tcgen05 has no f64 kind), DFMA, LDG.E.ENL2.256 (256-bit gathers), LDGSTS (cp.async),
UBLKCP (cp.async.bulk / TMA bulk copies), SYNCS (mbarrier), LDL / STL (local memory: spills).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(HERE), "paper_1301_2102_b200", "libbminres.so")
HOT = ("k1a_spmm", "k1_dmma", "k1u_update", "k2_dmma", "k2_row", "k3b_smallqr", "k_red2f", "k_reduce",
       "k1_ws", "k_trsv", "k_spmm_fwd")
OPS = [("DMMA", r"\bDMMA\b"), ("DFMA", r"\bDFMA\b"), ("LDG.256", r"LDG\.E\.ENL2\.256"),
       ("LDG", r"\bLDG\b"), ("LDGSTS", r"\bLDGSTS\b"), ("UBLKCP", r"\bUBLKCP\b"),
       ("SYNCS", r"\bSYNCS\b"), ("LDS", r"\bLDS\b"), ("STG", r"\bSTG\b"), ("LDL", r"\bLDL\b"),
       ("STL", r"\bSTL\b"), ("total", None)]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.strip().split("\n")


def main() -> None:
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", res):
        regs[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(5)))
    funcs = []
    cur, lines = None, []
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            if cur:
                funcs.append((cur, lines))
            cur, lines = m.group(1), []
        elif cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
            lines.append(ln)
    if cur:
        funcs.append((cur, lines))
    names = demangle([f for f, _ in funcs])
    print(f"# SASS summary of `{os.path.relpath(lib, os.path.dirname(HERE))}` (sm_100a)\n")
    print("Static instruction counts per kernel (hot kernels only); REG / STACK / LOCAL from "
          "`cuobjdump -res-usage` (STACK > 0 with LDL/STL = spills).\n")
    print("| kernel | REG | STACK | " + " | ".join(o for o, _ in OPS) + " |")
    print("|---|---|---|" + "---|" * len(OPS))
    for (mang, lines), name in zip(funcs, names):
        short = name.replace("bmr::", "").split("(")[0].removeprefix("void ")
        if not any(short.startswith(h) for h in HOT):
            continue
        body = "\n".join(lines)
        cnt = []
        for o, pat in OPS:
            cnt.append(str(len(lines)) if pat is None else str(len(re.findall(pat, body))))
        r = regs.get(mang, ("?", "?", "?"))
        print(f"| `{short}` | {r[0]} | {r[1]} | " + " | ".join(cnt) + " |")


if __name__ == "__main__":
    main()
