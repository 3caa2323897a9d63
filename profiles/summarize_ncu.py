"""Summarise ncu evidence for profiles/: per-kernel metrics of a --set full report and the
per-launch share table of a gpu__time_duration launch list.

usage: python profiles/summarize_ncu.py --rep R.ncu-rep [--launches L.csv] [--workload NAME]
                                        [--traffic-json profiles/traffic.json] > profiles/rNN_x.md
"""
import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe busy %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
]
KNAMES = {"k1_dmma": "spmm_fused", "k2_row": "orth", "k2_dmma": "orth", "k_reduce": "reduce", "k1_spmm": "spmm", "k2_orth": "orth", "k3b_smallqr": "smallqr", "k4a_basis": "basis",
          "k4b_update": "update", "k3_smallqr": "smallqr", "k4_update": "update"}


def short(name):
    m = re.search(r"(k\w+?)<", name) or re.search(r"(k\w+)", name)
    return m.group(1) if m else name


def raw(rep):
    if rep.endswith(".csv"):   # an `ncu -i R --page raw --csv` export
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_us(v, unit):
    f = float(v)
    return f * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True, help=".ncu-rep, or its --page raw --csv export")
    ap.add_argument("--launches")
    ap.add_argument("--workload", default="cfg2_lap3d_64_shift3")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    print(f"## ncu --set full: `{a.rep.split('/')[-1]}` (clock-control none)\n")
    print("| kernel | " + " | ".join(lbl for m, lbl in METRICS if m in idx) + " |")
    print("|---|" + "---|" * len(idx))
    traffic = {}
    for r in rows:
        cells = []
        for m, lbl in METRICS:
            if m not in idx:
                continue
            v, u = r[idx[m]], units[idx[m]]
            cells.append(f"{v} {u}".strip())
        k = short(r[kn])
        print(f"| {r[kn][:48]} | " + " | ".join(cells) + " |")
        if "dram__bytes_read.sum" in idx:
            tb = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]) + \
                 to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
            traffic[f"{a.workload}:{KNAMES.get(k, k)}"] = tb
    if a.traffic_json:
        try:
            old = json.load(open(a.traffic_json))
        except Exception:
            old = {}
        old.update(traffic)
        json.dump(old, open(a.traffic_json, "w"), indent=1, sort_keys=True)
    if a.launches:
        txt = open(a.launches).read()
        lines = [l for l in txt.splitlines() if l.startswith('"')]
        rows2 = list(csv.reader(io.StringIO("\n".join(lines))))
        h2 = rows2[0]
        ki, mi, vi, ui = h2.index("Kernel Name"), h2.index("Metric Name"), h2.index("Metric Value"), h2.index("Metric Unit")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows2[1:]:
            if r[mi] != "gpu__time_duration.sum":
                continue
            k = short(r[ki])
            tot[k] += to_us(r[vi].replace(",", ""), r[ui])
            cnt[k] += 1
        allt = sum(tot.values())
        print(f"\n## launch list `{a.launches.split('/')[-1]}` (ncu gpu__time_duration, cold-cache, serialised)\n")
        print("| kernel | launches | total us | mean us | share |")
        print("|---|---|---|---|---|")
        for k in sorted(tot, key=lambda x: -tot[x]):
            print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} | {100 * tot[k] / allt:.1f}% |")


if __name__ == "__main__":
    main()
