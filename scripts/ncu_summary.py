#!/usr/bin/env python
"""Summarise an ncu capture (run here, no GPU needed):

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv]

Prints the per-launch duration, DRAM bytes read/written, DRAM and SM
throughput, occupancy and registers of each profiled kernel, plus (with
--launches) the kernel-time shares of a `--metrics gpu__time_duration.sum`
launch list.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "KB": 1e3, "MB": 1e6, "GB": 1e9}


def to_bytes(row, hdr, units, metric: str) -> float:
    """One byte metric in bytes, with ITS OWN unit (ncu picks a unit per
    metric: the read and write counters of one launch can differ)."""
    i = hdr.index(metric)
    u = units[i]
    if u not in _SCALE:
        raise ValueError(f"unknown unit {u!r} for {metric}")
    return float(row[i].replace(",", "")) * _SCALE[u]


def traffic(rep: str) -> list:
    """[(kernel, read bytes, write bytes, duration ns)] per profiled launch."""
    hdr, units, data = raw(rep)
    ni, ti = hdr.index("Kernel Name"), hdr.index("gpu__time_duration.sum")
    tscale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
              "second": 1e9, "s": 1e9}[units[ti]]
    return [(r[ni], to_bytes(r, hdr, units, "dram__bytes_read.sum"),
             to_bytes(r, hdr, units, "dram__bytes_write.sum"),
             float(r[ti].replace(",", "")) * tscale) for r in data]


def summarize(rep: str) -> str:
    hdr, units, data = raw(rep)
    lines = [f"ncu --set full capture: {rep}"]
    name_i = hdr.index("Kernel Name")
    for r in data:
        lines.append(f"- kernel: {r[name_i]}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"    {m} = {r[i]} {units[i]}")
        if "dram__bytes_read.sum" in hdr:
            rd = to_bytes(r, hdr, units, "dram__bytes_read.sum")
            wr = to_bytes(r, hdr, units, "dram__bytes_write.sum")
            lines.append(f"    dram read = {rd:.0f} bytes, dram write = {wr:.0f} bytes")
            lines.append(f"    traffic (read+write) = {rd + wr:.0f} bytes")
    return "\n".join(lines)


def launch_shares(path: str) -> str:
    tot = collections.Counter()
    cnt = collections.Counter()
    with open(path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 5]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    total = sum(tot.values())
    lines = [f"launch list {path}: {sum(cnt.values())} launches, {total / 1e3:.1f} us total"]
    for k, v in tot.most_common():
        lines.append(f"  {100 * v / total:6.2f}%  {cnt[k]:5d} x {v / cnt[k] / 1e3:9.2f} us  {k}")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.rep:
        print(summarize(a.rep))
    if a.launches:
        print(launch_shares(a.launches))


if __name__ == "__main__":
    sys.exit(main())
