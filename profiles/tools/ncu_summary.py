#!/usr/bin/env python
"""Summaries of the ncu captures committed under profiles/ (read here with
`ncu -i`; the .ncu-rep files themselves stay in gpurun_out/).

  ncu_summary.py full <report.ncu-rep> <title>      key metrics + stall mix
  ncu_summary.py launches <launches.csv> <title>   per-kernel share of a launch list
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def full(rep, title):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    print(f"# {title}")
    print(f"# source: {rep} (ncu --set full --clock-control none --import-source on)")
    print(f"{'Kernel Name':70s} {vals[hdr.index('Kernel Name')]}")
    for m in FULL_METRICS:
        if m in hdr:
            i = hdr.index(m)
            print(f"{m:70s} {vals[i]} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h = src[1]
    stall = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = {h[i]: sum(float(r[i] or 0) for r in src[2:]) for i in stall}
    s = sum(tot.values()) or 1.0
    print("# warp stall mix (sampled, % of samples)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
        print(f"  {k[6:]:24s} {100 * v / s:5.1f}")


def launches(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        ns = float(r[-1])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    print(f"# {title}")
    print(f"# {path}: {len(rows)} launches, {total / 1e6:.2f} ms (cold-cache, serialised: shares, not absolutes)")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k[:62]:62s} {n:4d} {ns / 1e6:9.3f} ms {100 * ns / total:6.1f}%  avg {ns / n / 1e3:9.2f} us")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
