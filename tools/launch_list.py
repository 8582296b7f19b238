#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: launch_list.py LAUNCHES.csv N_MODES [title]
Prints per-kernel launch counts / mean / total device time, then the last sweep (the last
N_MODES launches of the spMTTKRP kernels plus anything between them) and the streaming
kernels' share of it.  Times are ncu's (cold-cache, serialised): compare shares, not absolutes.
"""
import csv, io, sys
from collections import OrderedDict

path, nmodes = sys.argv[1], int(sys.argv[2])
title = sys.argv[3] if len(sys.argv) > 3 else path
text = open(path).read()
text = text[text.index('"ID"'):] if '"ID"' in text else text
rows = list(csv.DictReader(io.StringIO(text)))
launches = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "").strip()
    short = name.split("::")[-1]
    val = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = val / 1000.0 if unit == "ns" else (val * 1000.0 if unit == "ms" else val)
    launches.append((short, us))
agg = OrderedDict()
for k, us in launches:
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += us
print(f"# ncu launch list, {title}")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised per launch)")
print("# kernel, launches, mean us, total us")
for k, (cnt, tot) in agg.items():
    print(f"{k}, {cnt}, {tot / cnt:.2f}, {tot:.1f}")
hot = ("k_stream2", "k_sweep2", "k_mttkrp_stream", "k_mttkrp_tiles")
idx = [i for i, (k, _) in enumerate(launches) if k.startswith(hot)]
if any(launches[i][0].startswith("k_sweep2") for i in idx[-1:]):
    nmodes = 1  # the last sweep is one fused launch
if len(idx) >= nmodes:
    first = idx[-nmodes]
    # include the zeroing launches that precede the first hot launch of the sweep
    while first > 0 and launches[first - 1][0].startswith(("k_stream_zero", "k_zero_rows")):
        first -= 1
    sweep = launches[first:]
    tot = sum(us for _, us in sweep)
    hot_us = sum(us for k, us in sweep if k.startswith(hot))
    print("# last sweep (%d launches): " % len(sweep) + ", ".join(f"{k}={us:.1f}us" for k, us in sweep))
    print(f"# sweep share: streaming kernels {hot_us:.1f} us of {tot:.1f} us ({100 * hot_us / tot:.1f}%)")
