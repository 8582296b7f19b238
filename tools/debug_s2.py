"""GPU debug: fast (streaming) vs deterministic MTTKRP per mode on configurable shapes."""
import os, sys, numpy as np
sys.path.insert(0, '.')
os.environ.setdefault("MKB_DEBUG", "1")
import paper_2503_18198_b200 as mk
cases = [([12092, 9184, 28818], 2_000_000, 32), ([2482, 2862, 14036, 17], 500_000, 64),
         ([183, 24, 1140, 1717], 500_000, 32), ([1000, 1000, 1000], 300_000, 32)]
for dims, nnz, R in cases:
    t = mk.generate_synthetic(dims, nnz, seed=3)
    f = [m.data for m in mk.random_factors(dims, R, 1)]
    plans = mk.build_mode_plans(t, 148)
    det = mk.mttkrp_all_modes(t, plans, f, mk.ExecConfig(148, 32, True), False)
    fast = mk.mttkrp_all_modes(t, plans, f, mk.ExecConfig(148), False)
    for d in range(len(dims)):
        err = mk.verify_against(fast[d], det[d].data)[0]
        bad = np.where(np.abs(fast[d].data - det[d].data).max(axis=1) > 1e-3 * (1 + np.abs(det[d].data).max(axis=1)))[0]
        print(dims, R, "mode", d, "err %.2e" % err, "bad rows", len(bad), bad[:8], flush=True)
        if len(bad):
            r = bad[0]
            print("  fast", fast[d].data[r, :4], " det", det[d].data[r, :4], " ratio", (fast[d].data[r, :4] / det[d].data[r, :4]))
