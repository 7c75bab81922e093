#!/usr/bin/env python
"""Summarize `ncu --page details --csv` exports: key SOL / memory / occupancy metrics per kernel."""
import csv
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Grid Size", "Block Size", "Executed Instructions", "Max Bandwidth", "Mem Busy"]


def summarize(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    out = {}
    name = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = name or d.get("Kernel Name")
        m = d.get("Metric Name")
        if m in KEYS and m not in out:
            out[m] = f"{d.get('Metric Value')} {d.get('Metric Unit')}".strip()
    return name, out


for p in sys.argv[1:]:
    name, out = summarize(p)
    print(f"== {p.split('/')[-1]}: {name[:90] if name else ''}")
    for k in KEYS:
        if k in out:
            print(f"   {k:40s} {out[k]}")
