#!/usr/bin/env python3
"""Per-sweep device time of each executor (mk_run_timed, L2 flushed): fast, deterministic,
reference contract (Scheme 1 modes deterministic, Scheme 2 fast) and partitioned.
usage (GPU box): python tools/exec_modes.py cfg2 cfg5"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_18198_b200 as mk  # noqa: E402
from bench import CONFIGS, make_tensor  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    cfg = CONFIGS[name]
    t = make_tensor(mk, cfg)
    f = [m.data for m in mk.random_factors(cfg["dims"], cfg["rank"], 1)]
    c = mk.Context()
    c.upload_tensor(t)
    c.build_plans(148)
    c.upload_factors(f)
    row = [name]
    for label, ex in (("fast", mk.EXEC_FAST), ("deterministic", mk.EXEC_DETERMINISTIC),
                      ("reference", mk.EXEC_REFERENCE), ("partitioned", mk.EXEC_PARTITIONED)):
        c.run_timed(1, ex)  # one-time choices
        _, total = c.run_timed(5, ex)
        row.append(f"{label} {np.median(total):.3f} ms")
    print("  ".join(row), flush=True)
