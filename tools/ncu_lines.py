#!/usr/bin/env python
"""Executed warp-instructions and average active threads per CUDA source line
for one kernel of an ncu report (SASS page joined with nvdisasm -g line info).
Usage: python tools/ncu_lines.py rep.ncu-rep <launch-index> <mangled-name> <file.cu>
(launch-index = position of the launch in the report, 0-based)"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, launch, mangled, fname = sys.argv[1:5]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_1804_10112_b200", "_lib", "libsl_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubin = os.path.join(tmp, os.path.splitext(os.path.basename(fname))[0] + ".sm_100a.cubin")
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
start = sass.index(f".text.{mangled}:")
lines, cur = {}, None
for l in sass[start:].split("\n")[1:]:
    if l.startswith(".text.") or "//---------------------" in l:
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
secs, cs = [], None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Kernel Name":
        cs = []
        secs.append(cs)
    elif cs is not None:
        cs.append(r)
print(secs and "")
hdr = secs[0][0]
ia, iex, ith = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Avg. Threads Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in secs[0][1:] if len(r) == len(hdr) and r[iex].strip().isdigit()]
base = int(body[0][ia], 16)
agg, thr, smp = collections.Counter(), collections.defaultdict(float), collections.Counter()
for r in body:
    key = lines.get(int(r[ia], 16) - base, ("?", 0))
    agg[key] += int(r[iex])
    thr[key] += int(r[iex]) * float(r[ith])
    smp[key] += int(r[ist]) if r[ist].strip().isdigit() else 0
tot, stot = sum(agg.values()) or 1, sum(smp.values()) or 1
srcs = {}
print(f"total warp-inst {tot}")
for key, v in agg.most_common(30):
    f, ln = key
    if f not in srcs:
        p = os.path.join(root, "paper_1804_10112_b200", "csrc", f)
        srcs[f] = open(p).read().split("\n") if os.path.exists(p) else []
    text = srcs[f][ln - 1].strip() if 0 < ln <= len(srcs[f]) else "?"
    print(f"{v / tot * 100:5.1f}% inst {smp[key] / stot * 100:5.1f}% stall thr {thr[key] / max(v, 1):4.1f} "
          f"{f}:{ln}: {text[:80]}")
