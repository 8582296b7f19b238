"""Generate tests/golden/golden.json from the REFERENCE itself.

Run in the build container only (needs /root/reference and oracle/_ref, the reference
library compiled from its own sources by oracle/Makefile):

    python tests/golden/make_golden.py               # everything
    python tests/golden/make_golden.py cfg3_nips,cfg5_nell2   # re-pin some configs only

Contents (everything is produced by the reference's own code path through
oracle/_ref/libmttkrp_ref.so, except the reference's checked-in fixtures which are read
from /root/reference/proj/tests/fixtures):
  tiny3        tiny3.tns + factors_tiny3.json + the expected outputs (test_oracle.cpp:79-90)
  kat          partition KATs of test_layout.cpp:58-99 recomputed by the reference
  configs      sha256 pins of generator output, plans (order/offsets/owned per mode),
               oracle_mttkrp<float> and oracle_mttkrp<double> outputs (the fp64 truth the
               fast path is gated against, oracle.hpp:20-43) for every BASELINE config, and
               the reference fp32 oracle's own max relative deviation from its fp64 result
The GPU box has no /root/reference, so GPU parity tests compare against these pins.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Oracle, Reference  # noqa: E402

FIX = "/root/reference/proj/tests/fixtures"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tensor_with_mode0_degrees(degrees):  # tests/support.hpp:63-72
    maxd = max([1] + list(degrees))
    coords = [(v, k) for v, d in enumerate(degrees) for k in range(d)]
    return [len(degrees), maxd], np.array(coords, dtype=np.uint32).reshape(-1, 2)


PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
# name, dims, nnz, rank, kappas of the format pins, strategies (0 cyclic, 1 LPT), generator
CONFIGS = [
    ("cfg1", [1000, 1000, 1000], 1_000_000, 32, [148, 8], [0, 1], "uniform"),
    ("cfg2_uber", [183, 24, 1140, 1717], 3_300_000, 32, [148], [0, 1], "uniform"),
    ("cfg3_nips", [2482, 2862, 14036, 17], 3_100_000, 64, [148, 16], [0, 1], "powerlaw"),
    ("cfg4_lbnl", [1605, 4198, 1631, 4209, 868131], 1_700_000, 32, [148], [0, 1], "uniform"),
    ("cfg5_nell2", [12092, 9184, 28818], 77_000_000, 32, [148, 16], [0], "uniform"),
    ("adaptive_kat", [6186, 24, 77, 32], 20_000, 8, [82], [0, 1], "uniform"),
]


def main():
    ref = Reference()
    only = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else set()
    old = json.load(open(PATH)) if only and os.path.exists(PATH) else {}
    out = {"generator": "tests/golden/make_golden.py (reference via oracle/_ref)"}

    # tiny3 (FROSTT 1-based -> 0-based) + golden factors
    lines = [l.split() for l in open(os.path.join(FIX, "tiny3.tns")) if l.strip() and
             not l.startswith("#")]
    coords = [[int(x) - 1 for x in l[:-1]] for l in lines]
    vals = [float(l[-1]) for l in lines]
    dims = [max(c[h] for c in coords) + 1 for h in range(len(coords[0]))]
    g = json.load(open(os.path.join(FIX, "factors_tiny3.json")))
    factors = [np.array(f, dtype=np.float32) for f in g["factors"]]
    got = [ref.oracle_mttkrp(dims, np.array(coords, np.uint32), np.array(vals, np.float32),
                             factors, d).tolist() for d in range(len(dims))]
    assert got == [[[float(x) for x in r] for r in m] for m in g["expected"]]
    out["tiny3"] = {"dims": dims, "coords": coords, "values": vals, "rank": g["rank"],
                    "factors": g["factors"], "expected": g["expected"]}

    # partition KATs (test_layout.cpp:58-99), recomputed by the reference
    kat = []
    for degrees, kappa, strategy, policy in [([5, 4, 3, 2, 1], 2, 0, 1), ([5, 4, 3, 2, 1], 2, 1, 1),
                                             ([1, 3, 2], 1, 0, 1), ([10], 3, 0, 2),
                                             ([6], 3, 0, 2), ([2], 5, 0, 2), ([37], 7, 0, 2)]:
        d, c = tensor_with_mode0_degrees(degrees)
        p = ref.build_plan(d, c, 0, kappa, strategy, policy)
        kat.append({"degrees": degrees, "kappa": kappa, "strategy": strategy, "policy": policy,
                    "scheme": p["scheme"], "order": p["order"].tolist(),
                    "offsets": p["offsets"].tolist(), "owned": p["owned"].tolist(),
                    "owned_offsets": p["owned_offsets"].tolist()})
    out["kat"] = kat

    # config pins (every BASELINE config; cfg3 has no reference generator: its tensor comes
    # from the DESIGN.md §5 power-law generator of the oracle, pinned by its own sha)
    pins = [c for c in old.get("configs", []) if c["name"] not in only] if only else []
    for name, dims, nnz, rank, kappas, strategies, gen in CONFIGS:
        if only and name not in only:
            continue
        seed = 9 if name == "adaptive_kat" else 1
        if gen == "powerlaw":
            c, v = Oracle().generate_powerlaw(dims, nnz, 1.0, seed)
        else:
            c, v = ref.generate_synthetic(dims, nnz, 0, 0, 2, seed)
        print(name, "generated", flush=True)
        f = ref.random_factors(dims, rank, 1)
        entry = {"name": name, "dims": dims, "nnz": nnz, "seed": seed, "gen": gen,
                 "rank": rank, "coords_sha": sha(c), "values_sha": sha(v),
                 "factors_sha": [sha(m) for m in f], "plans": [], "mttkrp_sha": [],
                 "mttkrp64_sha": [], "ref32_vs_64_max_rel_err": []}
        for kappa in kappas:
            for strategy in strategies:
                plans, ms = ref.build_plans_all(dims, c, v, kappa, strategy, 0)
                for d, p in enumerate(plans):
                    entry["plans"].append({"kappa": kappa, "strategy": strategy, "mode": d,
                                           "scheme": p["scheme"], "order_sha": sha(p["order"]),
                                           "offsets_sha": sha(p["offsets"]),
                                           "owned_sha": sha(p["owned"]),
                                           "owned_offsets_sha": sha(p["owned_offsets"])})
                print(name, kappa, strategy, [p["scheme"] for p in plans], f"{ms:.0f} ms",
                      flush=True)
                del plans
        for d in range(len(dims)):
            want32 = ref.oracle_mttkrp(dims, c, v, f, d)
            want64 = ref.oracle_mttkrp_f64(dims, c, v, f, d)
            entry["mttkrp_sha"].append(sha(want32))
            entry["mttkrp64_sha"].append(sha(want64))
            err = np.abs(want32.astype(np.float64) - want64) / np.maximum(1.0, np.abs(want64))
            entry["ref32_vs_64_max_rel_err"].append(float(err.max()) if err.size else 0.0)
            print(name, "mode", d, "ref fp32 vs fp64", entry["ref32_vs_64_max_rel_err"][-1],
                  flush=True)
        pins.append(entry)
        order = [x[0] for x in CONFIGS]
        pins.sort(key=lambda e: order.index(e["name"]) if e["name"] in order else 99)
        out["configs"] = pins
        with open(PATH, "w") as fh:  # checkpoint after every config (cfg5 takes minutes)
            json.dump(out, fh, indent=1)
    out["configs"] = pins
    with open(PATH, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", PATH)


if __name__ == "__main__":
    main()
