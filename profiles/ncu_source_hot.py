"""Summarise an ncu report's source page: warp-stall samples per CUDA source line (-lineinfo builds).

usage: python profiles/ncu_source_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    samp_i = hdr.index("Warp Stall Sampling (All Samples)")
    inst_i = hdr.index("Instructions Executed")
    agg = defaultdict(lambda: [0, 0, ""])
    total = 0
    for r in rows[hi + 1:]:
        if len(r) <= samp_i or not r[0].strip().isdigit():
            if r and r[0] in ("File Path",):
                break
            continue
        line = int(r[0])
        try:
            smp = int(r[samp_i] or 0)
            ins = int(r[inst_i] or 0)
        except ValueError:
            continue
        agg[line][0] += smp
        agg[line][1] += ins
        agg[line][2] = r[1]
        total += smp
    print(f"total samples {total}")
    for line, (smp, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100.0 * smp / max(total, 1):6.2f}%  L{line:4d} inst {ins:9d}  {src.strip()[:110]}")


if __name__ == "__main__":
    main()
