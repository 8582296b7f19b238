"""GPU probe: CPD-ALS iteration timing (events) for a config; run under ncu for a launch list."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2503_18198_b200 as mk
from bench import CONFIGS, make_tensor
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
t = make_tensor(mk, cfg)
f = [m.data for m in mk.random_factors(cfg["dims"], cfg["rank"], 1)]
ctx = mk.Context()
ctx.upload_tensor(t); ctx.build_plans(148); ctx.upload_factors(f)
for _ in range(3):
    ctx.cpd_als_iter()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    fit, _ = ctx.cpd_als_iter()
torch.cuda.synchronize()
print("wall ms/iter %.3f fit %.5f" % ((time.perf_counter() - t0) * 1e3 / 5, fit))
