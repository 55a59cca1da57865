#!/usr/bin/env python
"""Instruction mix of one kernel from an ncu report's SASS source page:
executed warp-instructions per opcode and the hottest address ranges.
Usage: python tools/ncu_inst.py rep.ncu-rep <kernel-regex> [launch-index]"""
import collections
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sec = sections[which]
hdr = sec["rows"][0]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ith = hdr.index("Avg. Threads Executed")
body = [r for r in sec["rows"][1:] if len(r) == len(hdr) and r[iex].strip().isdigit()]
tot = sum(int(r[iex]) for r in body) or 1
print(sec["name"][:100], "total warp-inst", tot)
ops = collections.Counter()
for r in body:
    op = r[isrc].split()
    op = [t for t in op if not t.startswith("@")]
    ops[op[0].split(".")[0] if op else "?"] += int(r[iex])
for k, v in ops.most_common(25):
    print(f"  {k:10s} {v / tot * 100:5.1f}%")
# hottest 64-instruction windows
win = collections.Counter()
for i, r in enumerate(body):
    win[i // 32] += int(r[iex])
print("hot windows (32 SASS each):")
for w, v in win.most_common(8):
    seg = body[w * 32:(w + 1) * 32]
    thr = sum(float(r[ith]) * int(r[iex]) for r in seg) / max(1, sum(int(r[iex]) for r in seg))
    print(f"  [{seg[0][ia][-5:]}..{seg[-1][ia][-5:]}] {v / tot * 100:5.1f}%  avg threads {thr:4.1f}  "
          + " | ".join(r[isrc].strip()[:28] for r in seg[:6]))
