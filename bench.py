#!/usr/bin/env python3
"""Benchmark: all-mode spMTTKRP per CPD iteration on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config cfg5] [--only] [--impl ours|reference]

A step is one all-mode spMTTKRP sweep (Algorithm 1; the unit the
reference's run_timed measures, kernel.hpp:239-287) over the configured synthetic tensor.
Headline workload: BASELINE configs[4] (nell-2-shaped 12092x9184x28818, 77M nnz, R=32) — the
config the metric's "1/2/4/8 B200" is quoted on and the largest single-GPU one.  The other
BASELINE configs (cfg1-cfg4) follow as sub-records of the same JSON line ("configs"), each with
its own roofline and CPU baseline, unless --only is given.

value      device time per sweep (ms, mean over K steps; CUDA events on the launch stream,
           tensor copies + factors resident in HBM, L2 flushed between steps)
e2e        the same sweep through the public C ABI with HOST buffers: H2D of every factor
           from pinned memory + sweep + D2H of every output, per step (mk_sweep_host)
roofline   HBM bound: algorithmic bytes per sweep (Σ_d nnz(4N+4) + 4R(Σ_{w≠d}D_w+I_d))
           ÷ the MTTKRP kernels' mean duration, vs MEASURED_PEAKS.json hbm_gbs
parity     after the timed loop: the last timed sweep's outputs vs the device fp64 deterministic
           result (bitwise = the reference's oracle_mttkrp<double>, tests/test_gpu_parity_full.py)
cpu_baseline  the reference compiled from its own sources (oracle/_ref) timed on this host:
           run_timed on the FULL tensor at kappa = nproc and kappa = 148 (plans from the
           oracle's bit-identical planner, pinned against the reference's build_mode_plans)
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
HEADLINE = "cfg5"

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
CPU_BUDGET_S = 45.0  # per (config, kappa) of timed reference sweeps


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
    """dram bytes per sweep from the committed ncu captures (the round's counter capture of the
    timed plan, profiles/ncu_lsu.json; else the older --set full summary), if present."""
    for fname in ("ncu_lsu.json", "ncu_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", fname)) as fh:
                entry = json.load(fh).get(config_name)
            if entry and entry.get("dram_bytes_per_sweep"):
                return float(entry["dram_bytes_per_sweep"])
        except Exception:
            pass
    return None


def lsu_roofline(config_name, kern_ms, sm_mhz=None):
    """Secondary (binding) roofline: bytes through the SM's L1/shared-memory data path per
    sweep (l1tex data-pipe wavefronts x 128 B from the committed ncu capture of the timed
    plan, tools/ncu_lsu.sh) against the chip's 128 B/clk/SM x 148 SMs x the SM clock sampled
    during this run's timed region."""
    path = os.path.join(ROOT, "profiles", "ncu_lsu.json")
    try:
        with open(path) as fh:
            entry = json.load(fh).get(config_name)
        if not entry:
            return None
        mhz = sm_mhz or entry["sm_mhz"]
        peak = 128.0 * entry["sms"] * mhz * 1e6 / 1e9  # GB/s
        achieved = entry["lsu_bytes_per_sweep"] / (kern_ms * 1e-3) / 1e9
        return {"bound": "l1/smem data path (128 B/clk/SM)", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "sm_mhz": mhz,
                "bytes_per_sweep": entry["lsu_bytes_per_sweep"], "source": entry.get("source")}
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU reference
def ref_generate(cfg):
    """The workload's tensor from the ORACLE generators (bit-identical to the reference's,
    pinned in tests/test_oracle.py; the product library is not loaded in the reference arm)."""
    import oracle
    orc = oracle.Oracle()
    if cfg["gen"] == "powerlaw":
        c, v = orc.generate_powerlaw(cfg["dims"], cfg["nnz"], 1.0, 1)
    else:
        c, v = orc.generate_synthetic(cfg["dims"], cfg["nnz"], 0, 0, 2, 1)
    f = orc.random_factors(cfg["dims"], cfg["rank"], 1)
    return c, v, f


def cpu_reference(cfg, coords, values, factors, max_steps, warmup):
    """The reference's own run_timed (oracle/_ref, kernel.hpp:239-287) on the full tensor, at
    kappa = nproc (the CLI default, mttkrp_bench.cpp:54-57) and kappa = 148.
    Plans come from the oracle's planner (bit-identical to build_mode_plans, pinned), so the
    reference's ~90 s single-threaded plan sort at 77M nnz stays out of the run.  Each kappa
    gets `warmup` untimed sweeps and up to `max_steps` timed ones within CPU_BUDGET_S."""
    import oracle
    cores = os.cpu_count() or 1
    orc = oracle.Oracle()
    dims = cfg["dims"]
    if not oracle.reference_available():
        # no compiled reference: the single-threaded C port of the oracle (kind "port")
        t0 = time.perf_counter()
        for d in range(len(dims)):
            orc.mttkrp(dims, coords, values, factors, d)
        v = (time.perf_counter() - t0) * 1e3
        return {"value": v, "unit": "ms", "cores": 1, "kind": "port",
                "sample": "full tensor, 1 sweep of the oracle port (single thread)",
                "cpu_model": cpu_model()}
    ref = oracle.Reference()
    rows = {}
    for kappa in sorted({cores, 148}):
        t0 = time.perf_counter()
        plans = orc.build_plans_all(dims, coords, kappa)
        plan_s = time.perf_counter() - t0
        # one probe sweep to size the sample, then warm-up + timed sweeps
        tot, _, _ = ref.run_timed_plans(dims, coords, values, factors, kappa, plans, 1)
        per = max(float(tot[0]) / 1e3, 1e-3)
        steps = int(max(2, min(max_steps, CPU_BUDGET_S // per)))
        w = max(0, min(warmup, int(10.0 // per)))
        tot, mode_min, ident = ref.run_timed_plans(dims, coords, values, factors, kappa, plans,
                                                   w + steps)
        timed = [float(x) for x in tot[w:]]
        rows[kappa] = {"kappa": kappa, "ms_mean": float(np.mean(timed)),
                       "ms_min": float(np.min(timed)), "steps": len(timed), "warmup": w + 1,
                       "mode_min_ms": [float(x) for x in mode_min],
                       "outputs_bit_identical": ident, "plan_build_s": plan_s}
        del plans
    best = min(rows.values(), key=lambda r: r["ms_mean"])
    return {"value": best["ms_mean"], "unit": "ms", "cores": cores, "kind": "reference",
            "kappa": best["kappa"], "cpu_model": cpu_model(),
            "sample": (f"full tensor ({cfg['nnz']} nnz); reference run_timed (oracle/_ref) at "
                       f"kappa=nproc={cores} and kappa=148, adaptive/cyclic, P=32; value = mean "
                       f"of the faster kappa's timed sweeps (kappa={best['kappa']}, "
                       f"{best['steps']} timed after {best['warmup']} untimed)"),
            "per_kappa": list(rows.values())}


def reference_arm(args, cfg, rank, world):
    if rank != 0:
        return 0
    c, v, f = ref_generate(cfg)
    cb = cpu_reference(cfg, c, v, f, args.steps, args.warmup)
    val = cb["value"]
    line = {"metric": METRIC, "value": val, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "impl": "reference",
            "data": "synthetic (oracle generator = the reference's generate_synthetic, seed 1)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "kappa": cb.get("kappa")},
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def make_tensor(mk, cfg):
    if cfg["gen"] == "powerlaw":
        return mk.generate_powerlaw(cfg["dims"], cfg["nnz"], 1.0, 1)
    return mk.generate_synthetic(cfg["dims"], cfg["nnz"], seed=1)


def run_config(args, name, rank, world, local_rank, stream, with_cpu):
    """Our arm on one config; returns the JSON record (rank 0) or None."""
    import torch
    import paper_2503_18198_b200 as mk

    cfg = CONFIGS[name]
    dims, R = cfg["dims"], cfg["rank"]
    n = len(dims)
    dev = torch.device("cuda", local_rank)
    t = make_tensor(mk, cfg)
    factors = [m.data for m in mk.random_factors(dims, R, 1)]

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
    if args.plan == "model":  # reproducible plans: the cost model's choice, no timed autotune
        ctx.set_plan_mode(mk.PLAN_MODEL)
    b_iter = float(sum(algorithmic_bytes(dims, t.nnz, R, distinct)))

    ex = None
    if world > 1:  # NCCL inside the library (comm.cu): sharded sweep captured in a CUDA graph
        from paper_2503_18198_b200.distributed import NcclExchange
        ex = NcclExchange(ctx)

    def sweep_once():
        if ex is not None:
            ex.sweep()
        else:
            ctx.sweep_async(False, False)

    def timed_sweeps(n_steps, flush):
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n_steps)]
        for s in range(n_steps):
            if flush:
                ctx.flush_l2()
            ev[s][0].record(stream)
            sweep_once()
            ev[s][1].record(stream)
        return ev

    # first fast call: the one-time plan choice (mttkrp.cu choose_fast_kernel), then warm-up
    ctx.mttkrp_all_modes(False, False)
    for _ in range(args.warmup):
        sweep_once()
    ctx.synchronize()
    if args.profile:
        for _ in range(args.steps):  # short, L2-flushed sweeps for ncu (never a bench number)
            ctx.flush_l2()
            sweep_once()
        ctx.synchronize()
        log(f"profile run done: {args.steps} sweeps of {n} modes ({name})")
        return None

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        w0 = time.perf_counter()
        evf = timed_sweeps(args.steps, True)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
    ctx.synchronize()  # non-finite check of the timed sweeps
    fused = ctx.last_sweep_fused()  # sharded: the local part of every rank's sweep
    step_ms = [evf[s][0].elapsed_time(evf[s][1]) for s in range(args.steps)]
    ms = float(np.mean(step_ms))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # parity of the timed sweep: its outputs vs the device fp64 deterministic result
    # (bitwise = the reference's oracle_mttkrp<double>) and vs the fp32 deterministic one
    # (bitwise = the reference's oracle_mttkrp<float>)
    timed_out = [ctx.output(d) for d in range(n)]
    parity = {}
    if ex is None:
        det = ctx.mttkrp_all_modes(False, True)
        ctx.upload_factors_f64([f.astype(np.float64) for f in factors])
        det64 = ctx.mttkrp_all_modes_f64(False, True)
        e64 = [float((np.abs(a.astype(np.float64) - b) / np.maximum(1.0, np.abs(b))).max())
               for a, b in zip(timed_out, det64)]
        e32 = [mk.verify_against(a, b)[0] for a, b in zip(timed_out, det)]
        parity = {"timed_sweep_vs_fp64_max_rel_err": max(e64),
                  "timed_sweep_vs_reference_fp32_max_rel_err": max(e32),
                  "per_mode_vs_fp64": e64, "tolerance": 1e-4, "pass": max(e64) <= 1e-4}
        del det, det64
        ctx.upload_factors(factors)
        ctx.sweep_async(False, False)  # re-establish the timed state after the parity calls

    # per-mode breakdown (separate launch per mode, L2 flushed per sweep)
    evm = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(args.steps)]
    for s in range(args.steps):
        ctx.flush_l2()
        evm[s][0].record(stream)
        for d in range(n):
            ctx.mttkrp_mode_async(d, False)
            evm[s][d + 1].record(stream)
    torch.cuda.synchronize()
    mode_ms = np.array([[evm[s][d].elapsed_time(evm[s][d + 1]) for d in range(n)]
                        for s in range(args.steps)])

    evw = timed_sweeps(args.steps, False)  # warm L2, reported alongside
    torch.cuda.synchronize()
    warm_ms = float(np.mean([evw[s][0].elapsed_time(evw[s][1]) for s in range(args.steps)]))

    # e2e through the C ABI: pinned host buffers packed like the device arenas (one copy per
    # direction), and the reference-API-shaped variant with one pageable array per mode
    offs = np.cumsum([0] + [(d * R + 31) // 32 * 32 for d in dims])
    arena_f = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    arena_o = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    pin_f = [arena_f[offs[w]:offs[w] + d * R].view(d, R) for w, d in enumerate(dims)]
    pin_o = [arena_o[offs[w]:offs[w] + d * R].view(d, R) for w, d in enumerate(dims)]
    for p_, f_ in zip(pin_f, factors):
        p_.copy_(torch.from_numpy(f_))
    f_np = [p.numpy() for p in pin_f]
    o_np = [p.numpy() for p in pin_o]
    pg_f = [f.copy() for f in factors]
    pg_o = [np.empty_like(f) for f in factors]

    def e2e_step(fs, os_):
        if ex is None:
            ctx.sweep_host(fs, os_)
        else:  # H2D factors, sharded sweep + all-gathers, D2H outputs
            ctx.upload_factors(fs)
            ex.sweep()
            for d in range(n):
                os_[d][...] = ctx.output(d)

    def e2e_time(fs, os_):
        for _ in range(2):
            e2e_step(fs, os_)
        out = []
        for s in range(args.steps):
            ctx.flush_l2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step(fs, os_)
            b.record(stream)
            b.synchronize()
            out.append(a.elapsed_time(b))
        return float(np.mean(out))

    e2e_ms = e2e_time(f_np, o_np)
    e2e_pageable_ms = e2e_time(pg_f, pg_o)
    h2d = int(sum(d * R * 4 for d in dims))

    # CPD-ALS iteration (MTTKRP + on-device Gram/solve/normalise/fit), reported alongside
    als_ms = None
    if R <= 64:
        ctx.upload_factors(factors)
        als_iter = ex.cpd_als_iter if ex is not None else ctx.cpd_als_iter
        for _ in range(2):  # eager iteration (one-time plan choices), then the graph capture
            als_iter()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(5):
            als_iter()
        b.record(stream)
        b.synchronize()
        als_ms = a.elapsed_time(b) / 5

    if rank != 0:
        return None
    peak, peak_src = measured_peaks()
    fast = [ctx.fast_path_info(d).as_dict() for d in range(n)]
    kern_ms = ms if fused else float(mode_ms.sum(axis=1).mean())
    achieved = b_iter / (kern_ms * 1e-3) / 1e9
    launches_per_sweep = 1 if fused else sum(f["launches"] for f in fast)
    rec = {
        "value": ms, "unit": "ms", "ms_per_step": ms,
        "config": {"workload": f"{name}: {cfg['desc']}", "kappa": kappa, "plan": args.plan,
                   "policy": "adaptive", "strategy": "cyclic",
                   "schemes": [int(i.scheme) for i in infos],
                   "l2": "flushed between timed steps (memset 2x L2 on the launch stream)",
                   "parallelism": f"row-range shards x{world}" if world > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(name),
                     "peak_source": peak_src, "algorithmic_bytes_per_sweep": b_iter,
                     "kernel": sorted({f["kernel"] for f in fast}), "kernel_ms_per_sweep": kern_ms,
                     "lsu": lsu_roofline(name, kern_ms, clk.summary().get("sm_mhz")),
                     "per_mode": fast},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": h2d, "path": "mk_sweep_host (C ABI), pinned host buffers; H2D / kernel / D2H pipelined above 2 MB of copies",
                "pageable_per_mode_ms": e2e_pageable_ms},
        "gpu_launches": (launches_per_sweep + (2 * n if ex is not None else 0)) * args.steps,
        "allgather_bytes_per_sweep": ex.bytes_per_sweep(R, n) if ex is not None else 0,
        "clocks": clk.summary(),
        "per_mode_ms": mode_ms.mean(axis=0).tolist(),
        "fused_sweep": bool(fused),
        "warm_ms_per_step": warm_ms,
        "wall_ms_timed_region": wall,
        "format_build_ms": build_ms, "tensor_upload_ms": upload_ms,
        "cpd_als_ms_per_iter": als_ms,
        "parity": parity,
    }
    ctx.close()
    if with_cpu:
        try:
            rec["cpu_baseline"] = cpu_reference(cfg, t.coords, t.values, factors,
                                                min(args.steps, 5), 1)
        except Exception as e:  # pragma: no cover
            rec["cpu_baseline"] = {"value": None, "unit": "ms", "cores": None,
                                   "kind": "reference", "sample": f"failed: {e}"}
    return rec


def our_arm(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    dev = torch.device("cuda", local_rank)
    # A dedicated (non-default) stream shared by torch's events and the library: the
    # legacy default stream's handle is NULL, which the C ABI reads as "own stream".
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    with_cpu = world == 1 and not args.no_cpu
    head = run_config(args, args.config, rank, world, local_rank, stream, with_cpu)
    if head is None:
        return 0
    subs = {}
    if not args.only and world == 1:
        for name in sorted(CONFIGS):
            if name != args.config:
                subs[name] = run_config(args, name, rank, world, local_rank, stream, with_cpu)
    line = {"metric": METRIC, "value": head["value"], "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["value"],
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generator restated bit-identically, seed 1; factors "
                    "random_factors seed 1)"}
    line.update({k: v for k, v in head.items() if k not in ("value", "unit", "ms_per_step")})
    line["gpu_launches"] = head["gpu_launches"]
    if subs:
        line["configs"] = subs
    print(json.dumps(line), flush=True)
    return 0


def spawn(args):
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (one per GPU)."""
    import torch
    have = torch.cuda.device_count()
    if args.gpus > have:
        print(json.dumps({"error": f"--gpus {args.gpus} requested, {have} GPU(s) visible"}),
              flush=True)
        log(f"bench: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}")
        return 2
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={29500 + os.getpid() % 1000}"] + sys.argv
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--only", action="store_true",
                    help="only the --config workload (no cfg1-cfg4 sub-records)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--plan", default="timed", choices=["timed", "model"],
                    help="fast-path plan choice: timed autotune (default) or the cost model only")
    ap.add_argument("--no-cpu", action="store_true",
                    help="skip the cpu_baseline (kernel-tuning runs only)")
    ap.add_argument("--profile", action="store_true",
                    help="only build + run --steps flushed sweeps (for ncu); prints no JSON")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local_rank = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if world != args.gpus and args.impl == "ours":
        log(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
        return 2
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)
    return our_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
