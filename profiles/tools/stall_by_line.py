#!/usr/bin/env python
"""Warp-stall samples of one kernel aggregated per source line: joins the
ncu SASS page (per-instruction samples, address order) with nvdisasm
--print-line-info of the same build (the innermost inlined location).

  stall_by_line.py <report.ncu-rep> <all.sass from nvdisasm --print-line-info> <mangled kernel name> [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, sass, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                                   "sass"], capture_output=True, text=True).stdout)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
text = open(sass).read()
start = text.index(f".text.{fn}:")
end = text.find("//---------------------", start)
body = text[start:end if end > 0 else None].splitlines()
loc, locs = None, []
for ln in body:
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        loc = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", ln):
        locs.append(loc)
n = min(len(locs), len(data))
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
tot = 0.0
for k in range(n):
    r = data[k]
    s = float(r[iS] or 0)
    tot += s
    a = agg[locs[k]]
    a[0] += s
    a[1] += float(r[iI] or 0)
    for i in stall_cols:
        a[2][hdr[i][6:]] += float(r[i] or 0)
print(f"# {len(data)} SASS rows, {len(locs)} disassembled, {tot:.0f} samples")
for l, (s, ins, why) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    w = ", ".join(f"{k} {v / max(s, 1) * 100:.0f}%" for k, v in sorted(why.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{s / tot * 100:5.1f}%  {l:22s} inst {ins:9.0f}  {w}")
