"""Per-SASS-instruction warp-stall samples of one kernel in an ncu report (first instance).

usage: python profiles/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    inst = []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if inst:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) > 3:
            inst.append(r)
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    tot = sum(int(r[si] or 0) for r in inst)
    byop = defaultdict(int)
    for r in inst:
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        byop[op.split(".")[0]] += int(r[si] or 0)
    print(f"total samples {tot}, instructions {len(inst)}")
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(byop.items(), key=lambda x: -x[1])[:12]))
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot_by = defaultdict(int)
    for r in inst:
        for i in stall_cols:
            tot_by[hdr[i][6:]] += int(r[i] or 0) if r[i].strip().isdigit() else 0
    print("by reason:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(tot_by.items(), key=lambda x: -x[1])[:8]))
    for idx, r in sorted(enumerate(inst), key=lambda x: -int(x[1][si] or 0))[:top]:
        rs = sorted(((int(r[i]) if r[i].strip().isdigit() else 0, hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
        why = " ".join(f"{n}:{v}" for v, n in rs if v)
        print(f"{100*int(r[si] or 0)/tot:6.2f}%  #{idx:5d} exec {r[ei]:>8}  {r[1].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main()
