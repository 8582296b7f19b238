#!/usr/bin/env python3
"""Benchmark: all-mode spMTTKRP per CPD iteration on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config cfg2] [--impl ours|reference]

A step is one all-mode spMTTKRP sweep (Algorithm 1; the unit the
reference's run_timed measures, kernel.hpp:239-287) over the configured synthetic tensor.
Default workload: BASELINE configs[1] (uber-shaped 183x24x1140x1717, 3.3M nnz, R=32).

value      device time per sweep (ms, mean over K steps; CUDA events on the launch stream,
           tensor copies + factors resident in HBM, L2 flushed between steps)
e2e        the same sweep through the public C ABI with HOST buffers: H2D of every factor
           from pinned memory + sweep + D2H of every output, per step (mk_sweep_host)
roofline   HBM bound: algorithmic bytes per sweep (Σ_d nnz(4N+4) + 4R(Σ_{w≠d}D_w+I_d))
           ÷ the MTTKRP kernels' mean duration, vs MEASURED_PEAKS.json hbm_gbs
cpu_baseline  the reference compiled from its own sources (oracle/_ref) timed on this host
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "all-mode spMTTKRP ms/CPD-iter, HBM GB/s vs roofline; 1/2/4/8 B200 vs host CPU"

CONFIGS = {
    "cfg1": dict(desc="synthetic 3-mode 1000x1000x1000, 1M nnz uniform, R=32",
                 dims=[1000, 1000, 1000], nnz=1_000_000, rank=32, gen="uniform"),
    "cfg2": dict(desc="uber-shaped 4-mode 183x24x1140x1717, 3.3M nnz uniform, R=32",
                 dims=[183, 24, 1140, 1717], nnz=3_300_000, rank=32, gen="uniform"),
    "cfg3": dict(desc="nips-shaped 4-mode 2482x2862x14036x17, 3.1M nnz power-law, R=64",
                 dims=[2482, 2862, 14036, 17], nnz=3_100_000, rank=64, gen="powerlaw"),
    "cfg4": dict(desc="lbnl-shaped 5-mode 1605x4198x1631x4209x868131, 1.7M nnz, R=32",
                 dims=[1605, 4198, 1631, 4209, 868131], nnz=1_700_000, rank=32, gen="uniform"),
    "cfg5": dict(desc="nell-2-shaped 3-mode 12092x9184x28818, 77M nnz uniform, R=32",
                 dims=[12092, 9184, 28818], nnz=77_000_000, rank=32, gen="uniform"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_tensor(mk, cfg):
    if cfg["gen"] == "powerlaw":
        return mk.generate_powerlaw(cfg["dims"], cfg["nnz"], 1.0, 1)
    return mk.generate_synthetic(cfg["dims"], cfg["nnz"], seed=1)


def algorithmic_bytes(dims, nnz, rank, distinct):
    n = len(dims)
    per_mode = []
    for d in range(n):
        fac = sum(distinct[w] for w in range(n) if w != d) + dims[d]
        per_mode.append(nnz * (4 * n + 4) + 4 * rank * fac)
    return per_mode


class ClockSampler:
    """nvidia-smi-equivalent clocks/throttle sampling (NVML) during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.002):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(config_name):
    """dram bytes per sweep from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            entry = json.load(fh).get(config_name)
        return float(entry["dram_bytes_per_sweep"]) if entry else None
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def reference_arm(args, cfg, rank, world):
    if rank != 0:
        return 0
    import oracle
    t = None
    import paper_2503_18198_b200 as mk  # host generator only (bit-identical to the reference's)
    t = make_tensor(mk, cfg)
    f = [m.data for m in mk.random_factors(cfg["dims"], cfg["rank"], 1)]
    cores = os.cpu_count() or 1
    if oracle.reference_available():
        ref = oracle.Reference()
        totals, mode_min, plan_ms = ref.run_timed(cfg["dims"], t.coords, t.values, f, cores,
                                                  args.warmup + args.steps)
        timed = totals[args.warmup:]
        kind, sample = "reference", (f"full tensor, build_mode_plans(kappa=nproc={cores}) "
                                     f"+ run_timed {args.warmup}+{args.steps} iters")
    else:
        orc = oracle.Oracle()
        timed = []
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            for d in range(len(cfg["dims"])):
                orc.mttkrp(cfg["dims"], t.coords, t.values, f, d)
            if s >= args.warmup:
                timed.append((time.perf_counter() - t0) * 1e3)
        cores, kind, sample = 1, "port", "full tensor, oracle port (single thread)"
    v = float(np.mean(timed))
    line = {"metric": METRIC, "value": v, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "impl": "reference",
            "data": "synthetic (reference generator, seed 1)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "kappa": cores},
            "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample(cfg, t, factors):
    """Reference CPU path on a bounded sample of the same workload (rank 0, N=1)."""
    import oracle
    cores = os.cpu_count() or 1
    dims = cfg["dims"]
    sample_nnz = min(t.nnz, 4_000_000)
    coords, vals = t.coords[:sample_nnz], t.values[:sample_nnz]
    scale = t.nnz / sample_nnz
    if oracle.reference_available():
        ref = oracle.Reference()
        totals, _, plan_ms = ref.run_timed(dims, coords, vals, factors, cores, 3)
        v = float(np.median(totals)) * scale
        return {"value": v, "unit": "ms", "cores": cores, "kind": "reference",
                "sample": (f"first {sample_nnz} nnz of the workload, reference build_mode_plans("
                           f"kappa={cores}) + run_timed 3 iters (median), scaled by nnz x{scale:.2f};"
                           f" plan build {plan_ms:.0f} ms")}
    orc = oracle.Oracle()
    t0 = time.perf_counter()
    for d in range(len(dims)):
        orc.mttkrp(dims, coords, vals, factors, d)
    v = (time.perf_counter() - t0) * 1e3 * scale
    return {"value": v, "unit": "ms", "cores": 1, "kind": "port",
            "sample": f"first {sample_nnz} nnz, oracle port single-thread, scaled x{scale:.2f}"}


# ----------------------------------------------------------------------------- our arm
def our_arm(args, cfg, rank, world, local_rank):
    import torch
    import paper_2503_18198_b200 as mk

    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dims, R = cfg["dims"], cfg["rank"]
    n = len(dims)
    t = make_tensor(mk, cfg)
    factors = [m.data for m in mk.random_factors(dims, R, 1)]
    dev = torch.device("cuda", local_rank)
    # A dedicated (non-default) stream shared by torch's events and the library: the
    # legacy default stream's handle is NULL, which the C ABI reads as "own stream".
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0

    ctx = mk.Context(local_rank)
    ctx.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    ctx.upload_tensor(t)
    torch.cuda.synchronize()
    upload_ms = (time.perf_counter() - t0) * 1e3
    kappa = torch.cuda.get_device_properties(dev).multi_processor_count
    t0 = time.perf_counter()
    ctx.build_plans(kappa, mk.Strategy.cyclic, mk.SchemePolicy.adaptive)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    infos = [ctx.plan_info(d) for d in range(n)]
    distinct = [int(i.distinct_rows) for i in infos]
    ctx.upload_factors(factors)

    # quick parity gate on the benchmarked workload: fast vs deterministic (bitwise ==
    # the reference oracle, tests/test_gpu_mttkrp.py) within 1e-5
    det = ctx.mttkrp_all_modes(False, True)
    fast = ctx.mttkrp_all_modes(False, False)
    parity = max(mk.verify_against(a, b)[0] for a, b in zip(fast, det))

    bytes_mode = algorithmic_bytes(dims, t.nnz, R, distinct)
    b_iter = float(sum(bytes_mode))

    # N > 1: row-range shards per mode + NCCL all-gather of each mode's rows
    ex = None
    if world > 1:
        from paper_2503_18198_b200.distributed import ShardExchange
        ex = ShardExchange(ctx, R, dims, device=dev)

    def sweep_timed(n_steps, flush, record):
        """Per mode launches with events between them (the per-mode breakdown)."""
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(n_steps)]
        evk = [[torch.cuda.Event(enable_timing=True) for _ in range(n)] for _ in range(n_steps)]
        for s in range(n_steps):
            if flush:
                ctx.flush_l2()
            ev[s][0].record(stream)
            for d in range(n):
                ctx.mttkrp_mode_async(d, False)
                evk[s][d].record(stream)
                if ex is not None:
                    ex.gather_mode(d)
                ev[s][d + 1].record(stream)
        return ev, evk

    def sweep_fused_timed(n_steps, flush):
        """Whole sweeps through the public sweep entry (one fused launch when applicable)."""
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n_steps)]
        for s in range(n_steps):
            if flush:
                ctx.flush_l2()
            ev[s][0].record(stream)
            sweep_once()
            ev[s][1].record(stream)
        return ev

    def sweep_once():
        if ex is not None:
            ex.sweep()
        else:
            ctx.sweep_async(False, False)

    for _ in range(max(args.warmup, 3)):
        sweep_once()
    ctx.synchronize()
    if args.profile:
        # short, L2-flushed sweeps for ncu (never a bench number)
        for _ in range(args.steps):
            ctx.flush_l2()
            sweep_once()
        ctx.synchronize()
        log(f"profile run done: {args.steps} sweeps of {n} modes")
        return 0

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        w0 = time.perf_counter()
        evf = sweep_fused_timed(args.steps, True)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
    ctx.synchronize()  # non-finite check
    fused_lib = ex is None and ctx.last_sweep_fused()  # the library's own record of the launch
    step_ms = [evf[s][0].elapsed_time(evf[s][1]) for s in range(args.steps)]
    ms = float(np.mean(step_ms))
    # per-mode breakdown (separate launches per mode, L2 flushed per sweep)
    ev, evk = sweep_timed(args.steps, True, True)
    torch.cuda.synchronize()
    mode_ms = np.array([[ev[s][d].elapsed_time(evk[s][d]) for d in range(n)]
                        for s in range(args.steps)])  # spMTTKRP kernels only
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # warm (no flush) for reference
    evw = sweep_fused_timed(args.steps, False)
    torch.cuda.synchronize()
    warm_ms = float(np.mean([evw[s][0].elapsed_time(evw[s][1]) for s in range(args.steps)]))

    # e2e through the C ABI with pinned host buffers
    # one pinned allocation per direction, matrices packed in mode order: the C ABI then moves
    # all factors (outputs) in one copy instead of one per mode (~6 us of PCIe latency each)
    offs = np.cumsum([0] + [(d * R + 31) // 32 * 32 for d in dims])
    arena_f = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    arena_o = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    pin_f = [arena_f[offs[w]:offs[w] + d * R].view(d, R) for w, d in enumerate(dims)]
    pin_o = [arena_o[offs[w]:offs[w] + d * R].view(d, R) for w, d in enumerate(dims)]
    for p_, f_ in zip(pin_f, factors):
        p_.copy_(torch.from_numpy(f_))
    f_np = [p.numpy() for p in pin_f]
    o_np = [p.numpy() for p in pin_o]
    def e2e_step():
        if ex is None:
            ctx.sweep_host(f_np, o_np)
        else:  # H2D factors, sharded sweep + all-gathers, D2H outputs
            ctx.upload_factors(f_np)
            ex.sweep()
            for d in range(n):
                o_np[d][...] = ctx.output(d)

    for _ in range(2):
        e2e_step()
    e2e = []
    for s in range(args.steps):
        ctx.flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2e))
    h2d = int(sum(d * R * 4 for d in dims))

    # CPD-ALS iteration (MTTKRP + on-device Gram/solve/normalise/fit), reported alongside
    als_ms = None
    if R <= 64:
        ctx.upload_factors(factors)
        als_iter = ex.cpd_als_iter if ex is not None else ctx.cpd_als_iter
        als_iter()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            als_iter()
        b.record(stream)
        b.synchronize()
        als_ms = a.elapsed_time(b) / 3

    if rank != 0:
        return 0
    peak, peak_src = measured_peaks()
    fast_info_all = [ctx.fast_path_info(d).as_dict() for d in range(n)]
    # the timed sweep is all streaming-kernel time when fused (one launch); otherwise the
    # per-mode kernel events
    fused = bool(fused_lib)
    kern_ms = ms if fused else float(mode_ms.sum(axis=1).mean())
    achieved = b_iter / (kern_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config)
    fast = fast_info_all
    launches_per_sweep = 1 if fused else sum(f["launches"] for f in fast)
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator, seed 1; factors random_factors seed 1)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "kappa": kappa,
                   "policy": "adaptive", "strategy": "cyclic",
                   "schemes": [int(i.scheme) for i in infos],
                   "l2": "flushed between timed steps (memset 2x L2 on the launch stream)",
                   "parallelism": f"row-range shards x{world}" if world > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_sweep": b_iter,
                     "kernel": sorted({f["kernel"] for f in fast}), "kernel_ms_per_sweep": kern_ms,
                     "per_mode": fast},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": h2d, "path": "mk_sweep_host (C ABI), pinned host buffers"},
        "gpu_launches": (launches_per_sweep + (2 * n if ex is not None else 0)) * args.steps,
        "allgather_bytes_per_sweep": ex.bytes_per_sweep() if ex is not None else 0,
        "clocks": clk.summary(),
        "per_mode_ms": mode_ms.mean(axis=0).tolist(),
        "per_mode_note": "separate launch per mode (the timed sweep is one fused launch when every "
                         "mode runs k_stream2 with one specialisation)",
        "fused_sweep": fused,
        "warm_ms_per_step": warm_ms,
        "wall_ms_timed_region": wall,
        "format_build_ms": build_ms, "tensor_upload_ms": upload_ms,
        "cpd_als_ms_per_iter": als_ms,
        "parity_fast_vs_deterministic_max_rel_err": parity,
    }
    if world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(cfg, t, factors)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "ms", "cores": None, "kind": "reference",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true",
                    help="skip the cpu_baseline sample (kernel-tuning runs only)")
    ap.add_argument("--profile", action="store_true",
                    help="only build + run --steps flushed sweeps (for ncu); prints no JSON")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local_rank = dist_env()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)
    return our_arm(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
