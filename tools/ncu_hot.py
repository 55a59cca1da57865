#!/usr/bin/env python
"""Top SASS lines by warp-stall samples for one kernel of an ncu report.
Usage: python tools/ncu_hot.py rep.ncu-rep <kernel-regex> [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# first row: kernel name; second: header
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].strip().isdigit()]
tot = sum(int(r[ist]) for r in body) or 1
body.sort(key=lambda r: -int(r[ist]))
print(f"total samples {tot}")
for r in body[:n]:
    print(f"{int(r[ist]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:90]}")
