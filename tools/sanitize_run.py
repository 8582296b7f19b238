#!/usr/bin/env python3
"""Small workload for compute-sanitizer (tools/sanitize.sh): every device code path of the
library once — format build, the fused level-ordered sweep, each fast kernel forced per mode,
the deterministic / partitioned / fp64 executors, CPD-ALS iterations (eager, captured and
replayed, side-stream inverse and serial), the cost-model plans, a simulated 2-rank
shard exchange and the one-rank NCCL sweep — on tensors small enough for the tools' overhead."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_18198_b200 as mk  # noqa: E402


def run(dims, nnz, R, gen="uniform"):
    t = mk.generate_powerlaw(dims, nnz, 1.0, seed=3) if gen == "powerlaw" else \
        mk.generate_synthetic(dims, nnz, seed=1)
    f = [m.data for m in mk.random_factors(dims, R, 1)]
    c = mk.Context()
    c.upload_tensor(t)
    c.build_plans(148)
    c.upload_factors(f)
    c.mttkrp_all_modes(False, False)   # one-time kernel choice + per-mode fast launches
    c.sweep_async(False, False)        # fused sweep when the plans allow it
    c.synchronize()
    for k in (0, 1, 2):                # every fast kernel
        c.set_fast_kernel(k)
        c.mttkrp_all_modes(False, False)
    c.set_fast_kernel(-1)
    c.mttkrp_all_modes(False, mk.EXEC_DETERMINISTIC)
    c.mttkrp_all_modes(False, mk.EXEC_PARTITIONED)
    c.upload_factors_f64([x.astype(np.float64) for x in f])
    c.mttkrp_all_modes_f64(False, True)
    c.mttkrp_all_modes_f64(False, False)
    c.upload_factors(f)
    if R <= 64:
        for _ in range(3):             # eager, graph capture, graph replay (side-stream inverse)
            c.cpd_als_iter()
        os.environ["MKB_ALS_OVERLAP"] = "0"
        c.cpd_als_iter()               # the serial update (inverse inside k_als_update)
        os.environ.pop("MKB_ALS_OVERLAP")
    c.set_plan_mode(mk.PLAN_MODEL)     # the cost model's plans (lead-2 pipeline where K = 1)
    c.sweep_async(False, False)
    c.set_plan_mode(mk.PLAN_TIMED)
    c.synchronize()
    # 2-rank exchange simulated with two contexts
    import torch
    ctxs = []
    for r in range(2):
        x = mk.Context()
        x.upload_tensor(t)
        x.build_plans(148)
        x.upload_factors(f)
        x.set_shard(r, 2)
        ctxs.append(x)
    for d in range(len(dims)):
        stride = max(max(k1 - k0 for k0, k1 in (ctxs[0].shard_rows(d, r) for r in range(2))), 1)
        buf = torch.zeros(2 * stride * R, device="cuda")
        for r, x in enumerate(ctxs):
            x.mttkrp_mode_async(d)
            s = torch.zeros(stride * R, device="cuda")
            x.shard_pack(d, s)
            x.synchronize()
            buf[r * stride * R:(r + 1) * stride * R] = s
        for x in ctxs:
            x.shard_unpack(d, buf, stride)
            x.synchronize()
    c.comm_init(1, 0, mk.Context.comm_unique_id())
    for _ in range(3):
        c.sweep_sharded()
    c.synchronize()
    print(f"ok {dims} nnz={nnz} R={R} {gen}", flush=True)


if __name__ == "__main__":
    run([60, 50, 40], 20_000, 32)
    run([300, 300, 300], 60_000, 32)
    run([50, 7, 40, 9], 20_000, 32)
    run([40, 30, 20, 17], 15_000, 64, "powerlaw")
    run([30, 20, 25, 15, 300], 10_000, 32)
