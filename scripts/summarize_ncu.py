#!/usr/bin/env python
"""Summaries of ncu outputs for profiles/ (run in the build container).

    python scripts/summarize_ncu.py launches gpurun_out/fin_launches.csv "<command>"  > profiles/...txt
    python scripts/summarize_ncu.py full gpurun_out/fin_full.ncu-rep "<command>"      > profiles/...txt
    python scripts/summarize_ncu.py traffic gpurun_out/fin_full.ncu-rep <dtw_cells> > profiles/dtw_lane_traffic.json

`launches`: per-kernel launch count, total gpu__time_duration and share (the
--metrics gpu__time_duration.sum --clock-control none pass of
B200_PROFILING.md: cold-cache, serialised, so only the shares compare with
bench.py's CUDA-event phase times).  `full`: the metrics the roofline and
DESIGN.md cite, per captured launch, from `ncu --set full`.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
]


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    return name.split("(")[0]


def launches(path: str, cmd: str):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = re.sub(r"<.*", "", short(r["Kernel Name"]))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(
            r["Metric Unit"], 1e-6)
        tot[k] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    total = sum(tot.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none --csv of `{cmd}`")
    print("# cold-cache, serialised launches: compare shares, not absolute times")
    print()
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:45s} {cnt[k]:5d} launches {v:12.2f} ms {100 * v / total:6.1f}%")
    print(f"total {total:.1f} ms")


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[0]
    return [dict(zip(head, r)) for r in rows[2:]]


def full(rep: str, cmd: str):
    print(f"# ncu --set full --clock-control none --import-source on of `{cmd}`")
    for d in raw_rows(rep):
        print(f"== {short(d.get('Kernel Name', '?'))}")
        for k in FULL_KEYS:
            if k in d:
                print(f"  {k:62s} {d[k]}")
        st = [(k, v) for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:8]
        print("  stalls per issue: " + ", ".join(
            f"{k.split('stalled_')[1].split('_per_issue')[0]} {float(v):.2f}" for k, v in st))


def traffic(rep: str, cells: float):
    for d in raw_rows(rep):
        if "dtw_laner" in d.get("Kernel Name", ""):
            rd = float(d["dram__bytes_read.sum"]) * (1e9 if "Gbyte" in d.get("dram__bytes_read.sum", "") else 1)
            print(json.dumps({"source": rep, "kernel": short(d["Kernel Name"]), "dram_read": d["dram__bytes_read.sum"],
                              "dram_write": d["dram__bytes_write.sum"], "dtw_cells": cells}, indent=1))
            return


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif mode == "full":
        full(sys.argv[2], sys.argv[3])
    else:
        traffic(sys.argv[2], float(sys.argv[3]))
