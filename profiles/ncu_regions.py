"""Warp-stall samples of one kernel by SASS index range (prologue / loop / epilogue split).
usage: python profiles/ncu_regions.py REPORT KERNEL_REGEX [BUCKET]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
bucket = int(sys.argv[3]) if len(sys.argv) > 3 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, inst = None, []
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
si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in inst)
for i in range(0, len(inst), bucket):
    seg = inst[i:i + bucket]
    s = sum(int(r[si] or 0) for r in seg)
    ex = max(int(r[ei] or 0) for r in seg)
    top = max(seg, key=lambda r: int(r[si] or 0))
    print(f"{i:5d}-{i + bucket - 1:5d}: {100 * s / tot:5.1f}%  max_exec {ex:7d}  top: {top[1].strip()[:50]}")
