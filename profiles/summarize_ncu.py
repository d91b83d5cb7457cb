#!/usr/bin/env python
"""Summarise ncu reports / launch lists into markdown (run here, no GPU needed).

    python profiles/summarize_ncu.py gpurun_out/prof_k3_TAG.ncu-rep [...]
    python profiles/summarize_ncu.py --launches gpurun_out/launches_TAG.csv --per-cycle 38 \
        [--cycle-index 0] [--sequence]
(launch lists from profiles/run_ncu.sh hold exactly one V-cycle: --cycle-index 0)
"""

import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def report(path):
    hdr, units, rows = raw(path)
    name_i = hdr.index("Kernel Name")
    print(f"### {path.split('/')[-1]}\n")
    for r in rows:
        print(f"- kernel `{r[name_i][:90]}`")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  - {label}: {r[i]} {units[i]}")
        print()


def launches(path, per_cycle, cycle_index=3, sequence=False):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi = hdr.index("Grid Size")
    data = [(r[ki], float(r[vi].replace(",", "")), r[gi]) for r in rows[h + 1:] if len(r) > vi]
    cyc = data[cycle_index * per_cycle:(cycle_index + 1) * per_cycle]
    tot = sum(d[1] for d in cyc)
    agg = defaultdict(lambda: [0.0, 0])
    for name, ns, _ in cyc:
        key = name.split("(")[0][:70]
        agg[key][0] += ns
        agg[key][1] += 1
    print(f"### one V-cycle from {path.split('/')[-1]} ({per_cycle} launches, "
          f"{tot / 1e3:.1f} us serialised, cold L2)\n")
    print("| kernel | launches | us | share |")
    print("|---|---|---|---|")
    for k, (ns, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"| `{k}` | {c} | {ns / 1e3:.1f} | {100 * ns / tot:.1f}% |")
    print()
    if sequence:
        print("| # | kernel | grid | us |")
        print("|---|---|---|---|")
        for i, (name, ns, grid) in enumerate(cyc):
            print(f"| {i} | `{name.split('(')[0][:60]}` | {grid} | {ns / 1e3:.1f} |")
        print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        per = int(args[args.index("--per-cycle") + 1]) if "--per-cycle" in args else 38
        ci = int(args[args.index("--cycle-index") + 1]) if "--cycle-index" in args else 3
        launches(args[1], per, ci, "--sequence" in args)
    else:
        for p in args:
            report(p)
