#!/usr/bin/env python3
"""Single-GPU evidence for the multi-GPU split: per-rank device time of each
rank's element-range shard, timed one rank at a time on ONE B200.

`gpurun` exposes one GPU, so no N > 1 run is possible here.  This times exactly the kernels a
rank runs in a sharded sweep (mk_set_shard(r, W): the rank's plan for its own element window,
the spMTTKRP over it, the pack of its touched rows, the unpack of all W blocks), with L2
flushed before each launch, for every rank r of W in {1, 2, 4, 8}.  Per mode the sharded
sweep waits for its slowest rank, so the compute part of a W-GPU sweep is
sum_d max_r t(d, r).  The all-gather is NOT timed (no peers): its bytes are reported, with an
estimate at an assumed 700 GB/s effective NVLink-5 all-gather bandwidth plus 15 us per
collective, labelled as such.

usage (GPU box): python tools/shard_projection.py [cfg5] > gpurun_out/shard_projection.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_18198_b200 as mk  # noqa: E402
from bench import CONFIGS, make_tensor  # noqa: E402

AG_GBS, AG_LAT_US = 700.0, 15.0


def timed(ctx, stream, fn, reps=3):
    best = 1e30
    for _ in range(reps):
        ctx.flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    cfg = CONFIGS[name]
    dims, R = cfg["dims"], cfg["rank"]
    t = make_tensor(mk, cfg)
    f = [m.data for m in mk.random_factors(dims, R, 1)]
    stream = torch.cuda.Stream()
    ctx = mk.Context()
    ctx.set_stream(stream.cuda_stream)
    ctx.upload_tensor(t)
    ctx.build_plans(torch.cuda.get_device_properties(0).multi_processor_count)
    ctx.upload_factors(f)
    n = len(dims)
    out = {"config": name, "dims": dims, "nnz": t.nnz, "rank": R, "worlds": []}
    for W in (1, 2, 4, 8):
        per_rank = []
        for r in range(W):
            ctx.set_shard(r, W)
            for d in range(n):  # one-time plan + kernel choice for this window
                ctx.mttkrp_mode_async(d)
            ctx.synchronize()
            rows = []
            for d in range(n):
                k0, k1 = ctx.shard_rows(d, r)
                ms = timed(ctx, stream, lambda: ctx.mttkrp_mode_async(d))
                buf = torch.empty(max(k1 - k0, 1) * R, device="cuda")
                pack_ms = timed(ctx, stream, lambda: ctx.shard_pack(d, buf)) if W > 1 else 0.0
                rows.append({"mode": d, "ms": ms, "pack_ms": pack_ms, "rows": k1 - k0,
                             "kernel": ctx.fast_path_info(d).as_dict()["kernel"]})
            per_rank.append(rows)
        modes = []
        for d in range(n):
            stride = max(max(ctx.shard_rows(d, r)[1] - ctx.shard_rows(d, r)[0] for r in range(W)), 1)
            recv = W * stride * R * 4 if W > 1 else 0
            unpack_ms = 0.0
            if W > 1:
                src = torch.zeros(W * stride * R, device="cuda")
                unpack_ms = timed(ctx, stream, lambda: ctx.shard_unpack(d, src, stride))
            t_max = max(per_rank[r][d]["ms"] for r in range(W))
            pack_max = max(per_rank[r][d]["pack_ms"] for r in range(W))
            ag_est = (recv / (AG_GBS * 1e9) * 1e3 + AG_LAT_US * 1e-3) if W > 1 else 0.0
            modes.append({"mode": d, "spmttkrp_ms_max_over_ranks": t_max,
                          "spmttkrp_ms_per_rank": [per_rank[r][d]["ms"] for r in range(W)],
                          "pack_ms_max": pack_max, "unpack_ms": unpack_ms,
                          "allgather_recv_bytes_per_rank": recv,
                          "allgather_ms_estimate": ag_est})
        compute = sum(m["spmttkrp_ms_max_over_ranks"] for m in modes)
        exch = sum(m["pack_ms_max"] + m["unpack_ms"] for m in modes)
        ag = sum(m["allgather_ms_estimate"] for m in modes)
        out["worlds"].append({"W": W, "modes": modes, "compute_ms": compute,
                              "pack_unpack_ms": exch, "allgather_ms_estimate": ag,
                              "sweep_ms_projection": compute + exch + ag})
        print(f"W={W}: spMTTKRP (max over ranks, per-mode launches) {compute:.3f} ms, "
              f"pack+unpack {exch:.3f} ms, all-gather estimate {ag:.3f} ms", file=sys.stderr)
    ctx.set_shard(0, 1)
    out["note"] = ("per-rank shard kernels timed one rank at a time on one B200 (L2 flushed); "
                   "all-gather not timed: estimate at %.0f GB/s + %.0f us per collective"
                   % (AG_GBS, AG_LAT_US))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
