#!/usr/bin/env python3
"""The paper's load-balancing experiment (§V-B: Scheme-1-only vs Scheme-2-only vs adaptive,
PAPER.md:369-381; the reference's bench_mttkrp.cpp:72-77) on one B200.

For each config and scheme policy (kappa = SM count, cyclic assignment) the mode copies are
built on the device and every mode is timed with
  * the partitioned executor (MK_EXEC_PARTITIONED: partition z of the plan on CTA z — the
    reference's work split, where the scheme decides the balance), and
  * the fast executor (equal-nnz slices whatever the scheme; only the copy order differs),
each the mean over --steps L2-flushed launches (CUDA events on the launch stream).  Prints one
JSON line per config; per mode: scheme, busy partitions, max/mean partition load, and ms.

usage: python tools/scheme_ablation.py [--configs cfg1,cfg2,...] [--steps 10]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2503_18198_b200 as mk
    from bench import CONFIGS, make_tensor

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    kappa = torch.cuda.get_device_properties(dev).multi_processor_count
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        t = make_tensor(mk, cfg)
        f = [m.data for m in mk.random_factors(cfg["dims"], cfg["rank"], 1)]
        rec = {"config": name, "desc": cfg["desc"], "kappa": kappa, "policies": {}}
        for policy in ("adaptive", "scheme1_only", "scheme2_only"):
            ctx = mk.Context(0)
            ctx.set_stream(stream.cuda_stream)
            ctx.upload_tensor(t)
            ctx.build_plans(kappa, mk.Strategy.cyclic, getattr(mk.SchemePolicy, policy))
            ctx.upload_factors(f)
            modes = []
            for d in range(len(cfg["dims"])):
                info = ctx.plan_info(d)
                offs = ctx.plan_export(d)["offsets"]
                loads = np.diff(offs.astype(np.int64))
                row = {"mode": d, "scheme": "scheme1" if info.scheme == 1 else "scheme2",
                       "busy": int((loads > 0).sum()),
                       "max_over_mean": float(loads.max() / (t.nnz / kappa)) if t.nnz else 1.0}
                for label, exec_code in (("partitioned_ms", mk.EXEC_PARTITIONED),
                                         ("fast_ms", mk.EXEC_FAST)):
                    ctx.mttkrp_mode_async(d, exec_code)  # warm-up (+ the fast path's plan choice)
                    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)]
                          for _ in range(args.steps)]
                    for s in range(args.steps):
                        ctx.flush_l2()
                        ev[s][0].record(stream)
                        ctx.mttkrp_mode_async(d, exec_code)
                        ev[s][1].record(stream)
                    torch.cuda.synchronize()
                    row[label] = float(np.mean([a.elapsed_time(b) for a, b in ev]))
                modes.append(row)
            ctx.synchronize()
            ctx.close()
            rec["policies"][policy] = {
                "modes": modes,
                "partitioned_total_ms": sum(m["partitioned_ms"] for m in modes),
                "fast_total_ms": sum(m["fast_ms"] for m in modes)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
