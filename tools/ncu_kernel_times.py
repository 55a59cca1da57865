#!/usr/bin/env python
"""Print kernel name + metric values from an `ncu --csv` launch list.
Usage: python tools/ncu_kernel_times.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iid = hdr.index("ID")
by = collections.OrderedDict()
for r in rows:
    if len(r) != len(hdr) or r is hdr or r[ik] == "Kernel Name":
        continue
    by.setdefault((r[iid], r[ik][:48]), {})[r[im]] = r[iv]
for (i, k), m in by.items():
    print(f"{i:>4} {k:48s} " + " ".join(f"{n.split('__')[-1][:28]}={v}" for n, v in m.items()))
