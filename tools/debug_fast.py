import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_18198_b200 as mk
from oracle import Oracle
orc = Oracle()
cases = [(6, 16), (6, 32), (6, 64), (12, 16), (2, 64), (8, 32)]
for seed, rank in cases:
    g = np.random.default_rng(seed)
    n = int(g.integers(3, 6)); dims = [int(x) for x in g.integers(1, 33, size=n)]
    nnz = int(g.integers(0, min(int(np.prod(dims)), 2000) + 1))
    t0 = mk.generate_synthetic(dims, nnz, seed=seed)
    sign = np.where(g.integers(0, 2, size=nnz) == 1, 1, -1).astype(np.float32)
    t = mk.SparseTensorCOO(dims, t0.coords, t0.values * sign)
    g.choice([2]); kappa = int(g.choice([1, 3, 8])); pol = mk.SchemePolicy(int(g.integers(0, 3)))
    f = [m.data for m in mk.random_factors(dims, rank, seed + 11)]
    plans = mk.build_mode_plans(t, kappa, mk.Strategy.cyclic, pol)
    for d in range(n):
        want = orc.mttkrp(dims, t.coords, t.values, f, d)
        fast = mk.mttkrp_mode(t, plans[d], f, mk.ExecConfig(kappa)).data
        err = mk.verify_against(fast, want)
        if err[0] > 1e-5:
            bad = np.where(np.abs(fast - want).max(axis=1) > 1e-4)[0]
            print("seed", seed, "R", rank, "dims", dims, "nnz", nnz, "mode", d, "err", err, "bad rows", bad[:10], "of", len(bad))
            r = bad[0]; print(" fast", fast[r, :8], "\n want", want[r, :8])
        else:
            print("ok seed", seed, "R", rank, "mode", d)
