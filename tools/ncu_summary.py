#!/usr/bin/env python3
"""Summarise an ncu --set full report (one row per captured launch) for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name")
    launches = []
    for r in data:
        d = {"kernel": r[name_i]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[m] = float(r[i].replace(",", ""))
                except ValueError:
                    d[m] = r[i]
                d[m + ":unit"] = units[i]
        launches.append(d)
    return launches


def main():
    path = sys.argv[1]
    launches = load(path)
    for m in METRICS:
        vals = [l.get(m) for l in launches]
        unit = launches[0].get(m + ":unit", "") if launches else ""
        print(f"{m:75s} {unit:10s} {vals}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(launches, fh, indent=1)


if __name__ == "__main__":
    main()
