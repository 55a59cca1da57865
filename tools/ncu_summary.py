#!/usr/bin/env python
"""Summarise an ncu report: one row per kernel launch with the metrics the
roofline discussion needs.  Usage: python tools/ncu_summary.py rep.ncu-rep [--json out]"""
import csv
import json
import subprocess
import sys

COLS = {
    "time_us": ("gpu__time_duration.sum", 1e3),
    "dram_rd_MB": ("dram__bytes_read.sum", 1.0),
    "dram_wr_MB": ("dram__bytes_write.sum", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "stall_long_sb": ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
    "stall_barrier": ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", 1.0),
    "stall_lg_thr": ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", 1.0),
    "stall_mio": ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", 1.0),
    "stall_short_sb": ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1.0),
    "l2_rd_sectors_M": ("lts__t_sectors_srcunit_tex_op_read.sum", 1e-6),
    "inst_M": ("smsp__inst_executed.sum", 1e-6),
}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    res = []
    for r in rows[2:]:
        d = {"kernel": r[name_i].split("(")[0]}
        for k, (m, scale) in COLS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                    u = units[i]
                    if u == "Gbyte":
                        v *= 1e3
                    elif u == "Kbyte":
                        v *= 1e-3
                    elif u == "byte":
                        v *= 1e-6
                    if m == "gpu__time_duration.sum" and u == "usecond":
                        v /= 1e3
                    if m == "gpu__time_duration.sum" and u == "nsecond":
                        v /= 1e6
                    d[k] = round(v * scale, 3)
                except ValueError:
                    d[k] = None
        d["traffic_bytes"] = int(round((d.get("dram_rd_MB", 0) + d.get("dram_wr_MB", 0)) * 1e6))
        res.append(d)
    keys = ["kernel"] + list(COLS)
    print(" | ".join(keys))
    for d in res:
        print(" | ".join(str(d.get(k)) for k in keys))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
