#!/usr/bin/env python3
"""Binding-roofline counters for bench.py's roofline.lsu.

  python tools/ncu_lsu.py --env BENCH.json CFG env vars forcing the bench run's plan for CFG
  python tools/ncu_lsu.py TAG CFG...           fold gpurun_out/TAG_lsu_CFG.csv into
                                               profiles/ncu_lsu.json

Per config the LAST sweep of the profiled run is kept (one k_sweep2 launch when fused, else
one launch per mode).  lsu_bytes_per_sweep = L1/SMEM data-pipe wavefronts x 128 B: every
wavefront is one cycle of the SM's 128 B/clk shared/L1 data path, so bytes / (128 B x SMs x
clock x time) is the fraction of that path's cycles the sweep kept busy.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def env_for(bench_json, cfg):
    d = json.load(open(bench_json))
    if not d["config"]["workload"].startswith(cfg + ":"):
        d = d["configs"][cfg]  # a sub-record of the headline line
    pm = d["roofline"]["per_mode"]
    ks, ker = [], []
    for m in pm:
        if "level-ordered" in m["kernel"]:
            ker.append("s2")
            ks.append(str(m.get("staged_levels", 0)))
        elif "fiber" in m["kernel"] or "k_mttkrp_stream" in m["kernel"]:
            ker.append("stream")
            ks.append("0")
        else:
            ker.append("tiles")
            ks.append("0")
    return f"MKB_FAST_KERNEL={','.join(ker)} MKB_FORCE_K={','.join(ks)}"


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[start]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = {}
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        L = launches.setdefault(int(r[iid]), {"kernel": r[ik]})
        try:
            L[r[im]] = float(r[iv].replace(",", ""))
        except ValueError:
            pass
    return [launches[k] for k in sorted(launches)]


def fold(tag, cfgs):
    from bench import CONFIGS
    out_path = os.path.join(ROOT, "profiles", "ncu_lsu.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for c in cfgs:
        L = load(os.path.join(ROOT, "gpurun_out", f"{tag}_lsu_{c}.csv"))
        n = 1 if "k_sweep2" in L[-1]["kernel"] else len(CONFIGS[c]["dims"])
        last = L[-n:]
        s = lambda k: sum(x.get(k, 0.0) for x in last)
        wf = s("l1tex__data_pipe_lsu_wavefronts.sum")
        t_ns = s("gpu__time_duration.sum")
        cyc = s("sm__cycles_elapsed.avg")
        out[c] = {
            "kernels": [x["kernel"].split("<")[0].split("::")[-1] for x in last],
            "lsu_wavefronts_per_sweep": wf,
            "lsu_shared_wavefronts_per_sweep": s("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "lsu_global_ld_wavefronts_per_sweep": s("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum"),
            "lsu_lgds_wavefronts_per_sweep": s("l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum"),
            "data_bank_reads_per_sweep": s("l1tex__data_bank_reads.sum"),
            "data_bank_writes_per_sweep": s("l1tex__data_bank_writes.sum"),
            "shared_ld_bank_conflicts_per_sweep": s("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
            "lsu_bytes_per_sweep": wf * 128.0,
            "dram_bytes_per_sweep": s("dram__bytes_read.sum") + s("dram__bytes_write.sum"),
            "l2_to_l1_bytes_per_sweep": s("l1tex__m_xbar2l1tex_read_bytes.sum"),
            "ncu_ms_per_sweep": t_ns / 1e6,
            "ncu_lsu_busy_frac": wf / (cyc * 148) if cyc else None,
            "sms": 148,
            "sm_mhz": (cyc / t_ns * 1e3) if t_ns else None,
            "source": f"profiles/r02_lsu/{tag}_lsu_{c}.csv (tools/ncu_lsu.sh; ncu --clock-control none, "
                      f"last sweep of bench.py --config {c} --profile)",
        }
        print(c, json.dumps(out[c])[:300])
    json.dump(out, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "--env":
        print(env_for(sys.argv[2], sys.argv[3]))
    else:
        fold(sys.argv[1], sys.argv[2:])
