#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: launch-list shares and per-kernel
metrics (time, DRAM bytes, throughput, top stall reasons) of a --set full
capture.  Usage: tools/ncu_summary.py launches.csv [prof.ncu-rep]"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    cols = {"gpu__time_duration.sum": "time", "dram__bytes_read.sum": "dram rd", "dram__bytes_write.sum": "dram wr",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram %",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm %",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "warps act %",
            "launch__registers_per_thread": "regs", "smsp__inst_executed.sum": "warp inst"}
    out = ["| kernel | " + " | ".join(cols.values()) + " | top stalls |", "|" + "---|" * (len(cols) + 2)]
    for r in rows[2:]:
        vals = []
        for c in cols:
            i = hdr.index(c)
            vals.append(f"{r[i]} {units[i]}".strip())
        st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", "")))
              for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
              and not hdr[i].endswith("not_issued") and r[i] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:3])
        out.append(f"| {r[hdr.index('Kernel Name')].split('(')[0][:32]} | " + " | ".join(vals) + f" | {top} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print()
        print(full(sys.argv[2]))
