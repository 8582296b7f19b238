"""GPU: CPD-ALS on the device vs the fp64 restatement (oracle/als.py).  Parity for this
subsystem is unpinned against the reference (it has no ALS)."""
import numpy as np
import pytest

from oracle import als as als_oracle

pytestmark = pytest.mark.gpu


def dense_lowrank_tensor(mk, dims, rank, seed):
    g = np.random.default_rng(seed)
    A = [g.normal(size=(d, rank)) for d in dims]
    X = np.einsum("ir,jr,kr->ijk", *A)
    coords = np.argwhere(np.ones(dims, bool)).astype(np.uint32)
    vals = X[tuple(coords.T)].astype(np.float32)
    return mk.SparseTensorCOO(dims, coords, vals)


def check_against_fp64(ctx, dims, coords, values, f0, tol=1e-4):
    """Factors, lambda and fit of one device iteration against the fp64 restatement, with the
    north star's 1e-4 relative bound (verify.hpp:21-39 error |g-w|/max(1,|w|)); returns the
    worst factor error."""
    fit, lam = ctx.cpd_als_iter()
    Y, lam64, fit64, _ = als_oracle.als_iteration(dims, coords, values, f0)
    worst = 0.0
    for d in range(len(dims)):
        got = ctx.download_factor(d).astype(np.float64)
        worst = max(worst, float((np.abs(got - Y[d]) / np.maximum(1.0, np.abs(Y[d]))).max()))
    lam_err = float((np.abs(lam - lam64) / np.maximum(1.0, np.abs(lam64))).max())
    assert worst <= tol, worst
    assert lam_err <= tol, lam_err
    assert abs(fit - fit64) <= tol, (fit, fit64)
    return worst


@pytest.mark.parametrize("rank,seed", [(4, 0), (8, 1), (16, 2), (32, 3), (64, 4)])
def test_one_iteration_matches_fp64(mk, rank, seed):
    g = np.random.default_rng(seed)
    dims = [30, 40, 50]
    t = mk.generate_synthetic(dims, 6000, seed=seed)
    f0 = [g.normal(size=(d, rank)).astype(np.float32) for d in dims]  # well-conditioned Grams
    plans = mk.build_mode_plans(t, 8)
    ctx = plans[0]._ctx
    ctx.upload_factors(f0)
    check_against_fp64(ctx, dims, t.coords, t.values, f0)


def test_cfg3_shaped_r64_update(mk):
    """k_als_update<64, 1024> (the R = 64 path of cfg3's "full CPD-ALS R=64") on cfg3-shaped
    power-law data (nips extents, 4 modes, 300 K nnz), one iteration at 1e-4."""
    dims = [2482, 2862, 14036, 17]
    t = mk.generate_powerlaw(dims, 300_000, 1.0, 3)
    g = np.random.default_rng(11)
    f0 = [g.normal(size=(d, 64)).astype(np.float32) for d in dims]
    plans = mk.build_mode_plans(t, 148)
    ctx = plans[0]._ctx
    ctx.upload_factors(f0)
    check_against_fp64(ctx, dims, t.coords, t.values, f0)


def test_rank_change_resets_accumulators(mk):
    """after an odd number of mode updates at one rank, a lower-rank upload on the
    same context must not read stale MᵀM sums (als.cu als_prepare)."""
    dims = [30, 40, 50]
    t = mk.generate_synthetic(dims, 6000, seed=9)
    plans = mk.build_mode_plans(t, 8)
    ctx = plans[0]._ctx
    g = np.random.default_rng(5)
    ctx.upload_factors([g.normal(size=(d, 64)).astype(np.float32) for d in dims])
    ctx.cpd_als_iter()  # N = 3 updates: the ping-pong ends on slot 1
    f0 = [g.normal(size=(d, 16)).astype(np.float32) for d in dims]
    ctx.upload_factors(f0)
    check_against_fp64(ctx, dims, t.coords, t.values, f0)


def test_exact_lowrank_recovered(mk):
    t = dense_lowrank_tensor(mk, [12, 14, 16], 3, 7)
    plans = mk.build_mode_plans(t, 8)
    g = np.random.default_rng(1)
    f0 = [g.normal(size=(d, 3)).astype(np.float32) for d in t.dims]
    fit, iters, lam, _ = mk.cpd_als(t, plans, f0, 200, 1e-9)
    assert fit > 0.999, (fit, iters)


def test_fit_monotone_on_random_tensor(mk):
    t = mk.generate_synthetic([60, 70, 80], 20000, seed=4)
    plans = mk.build_mode_plans(t, 148)
    ctx = plans[0]._ctx
    f0 = [m.data for m in mk.random_factors(t.dims, 16, 2)]
    ctx.upload_factors(f0)
    fits = [ctx.cpd_als_iter()[0] for _ in range(8)]
    assert all(b >= a - 1e-4 for a, b in zip(fits, fits[1:])), fits
    Y = [ctx.download_factor(d) for d in range(3)]
    for y in Y:  # columns normalised
        assert np.allclose(np.linalg.norm(y, axis=0), 1.0, atol=1e-4)


def test_rank_deficient_uses_pinv(mk):
    # duplicate columns make V singular: the device falls back to the pseudo-inverse
    dims = [20, 20, 20]
    t = mk.generate_synthetic(dims, 3000, seed=5)
    g = np.random.default_rng(3)
    f0 = []
    for d in dims:
        a = g.normal(size=(d, 2)).astype(np.float32)
        f0.append(np.concatenate([a, a[:, :1]], axis=1))
    plans = mk.build_mode_plans(t, 8)
    ctx = plans[0]._ctx
    ctx.upload_factors(f0)
    fit, lam = ctx.cpd_als_iter()
    Y, lam64, fit64, _ = als_oracle.als_iteration(dims, t.coords, t.values, f0)
    assert np.isfinite(fit) and abs(fit - fit64) < 5e-3


@pytest.mark.parametrize("overlap", ["0", "1"])
def test_overlapped_inverse_matches_serial(mk, monkeypatch, overlap):
    """The side-stream V_d⁻¹ (k_als_inverse during mode d's spMTTKRP on SM count - 1 CTAs)
    gives the same iteration as the serial update: factors, lambda and fit to the fast
    spMTTKRP's own run-to-run spread (its atomics are not bit-reproducible)."""
    dims = [300, 200, 150, 40]
    t = mk.generate_powerlaw(dims, 80_000, 1.0, 5)
    f0 = [m.data for m in mk.random_factors(dims, 64, 2)]
    res = []
    for ov in ("0", overlap):
        monkeypatch.setenv("MKB_ALS_OVERLAP", ov)
        ctx = mk.Context()
        ctx.upload_tensor(t)
        ctx.build_plans(148)
        ctx.upload_factors(f0)
        fit, lam = ctx.cpd_als_iter()
        res.append((fit, lam, [ctx.download_factor(d) for d in range(4)]))
    (f_a, l_a, y_a), (f_b, l_b, y_b) = res
    # a wrong or stale inverse is an O(1) error; the spread of two fast runs is ~1e-4
    assert abs(f_a - f_b) <= 1e-4
    assert np.allclose(l_a, l_b, rtol=1e-3)
    for d in range(4):
        assert mk.verify_against(y_b[d], y_a[d])[0] <= 1e-3


@pytest.mark.parametrize("rank", [32, 64])
def test_graph_replay_matches_eager(mk, monkeypatch, rank):
    """The captured CPD-ALS iteration (eager, capture, then replays) follows the eager
    iteration, also across a re-plan in between (an unchained sweep re-plans the level-ordered
    kernel for every SM; the stale graph must not be replayed)."""
    dims = [400, 300, 200]
    t = mk.generate_synthetic(dims, 120_000, seed=4)
    f0 = [m.data for m in mk.random_factors(dims, rank, 3)]
    fits = {}
    for g in ("0", "1"):
        monkeypatch.setenv("MKB_GRAPH", g)
        ctx = mk.Context()
        ctx.upload_tensor(t)
        ctx.build_plans(148)
        ctx.upload_factors(f0)
        seq = []
        for it in range(6):
            if it == 3:
                ctx.sweep_async(False, False)
            seq.append(ctx.cpd_als_iter()[0])
        fits[g] = (seq, [ctx.download_factor(d) for d in range(3)])
    assert np.allclose(fits["0"][0], fits["1"][0], rtol=0, atol=1e-6), fits
    for d in range(3):
        assert mk.verify_against(fits["1"][1][d], fits["0"][1][d])[0] <= 1e-4
