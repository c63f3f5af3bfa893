#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  ncu_summary.py report  X.ncu-rep  [--tag T]      -> markdown table of key metrics per launch
  ncu_summary.py launches X.csv     [--tag T]      -> per-kernel launch count / time / share
  ncu_summary.py traffic  X.ncu-rep KERNEL WORKLOAD -> update profiles/ncu_traffic.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def report(rep, tag):
    hdr, units, rows = raw_rows(rep)
    lines = [f"### {tag or os.path.basename(rep)}", "",
             "| kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---" * (len(KEYS) + 1) + "|"]
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0][-40:]
        vals = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
    print("\n".join(lines))


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}.get(unit, 1.0)
        k = r[hdr.index("Kernel Name")].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"### {tag or os.path.basename(path)}\n\n| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% |")


def traffic(rep, kernel, workload, n_gpus=1):
    hdr, units, rows = raw_rows(rep)
    out = []
    for r in rows:
        if kernel not in r[hdr.index("Kernel Name")]:
            continue
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[hdr.index("dram__bytes_read.sum")]) * mult[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(r[hdr.index("dram__bytes_write.sum")]) * mult[units[hdr.index("dram__bytes_write.sum")]]
        out.append(rd + wr)
    if not out:
        raise SystemExit("kernel not in report")
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[kernel] = {"workload": workload, "n_gpus": n_gpus, "dram_bytes_per_launch": sum(out) / len(out),
                 "launches": len(out), "report": os.path.basename(rep)}
    json.dump(d, open(p, "w"), indent=1)
    print(d[kernel])


if __name__ == "__main__":
    cmd = sys.argv[1]
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else None
    if cmd == "report":
        report(sys.argv[2], tag)
    elif cmd == "launches":
        launches(sys.argv[2], tag)
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
