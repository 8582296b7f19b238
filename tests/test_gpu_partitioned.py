"""GPU: the partitioned executor (MK_EXEC_PARTITIONED) — partition z of the
plan on CTA z, the reference's for_each_partition work split (parallel.hpp:16-49) — against
the reference's oracle_mttkrp (fp32, verify_tolerance 1e-5) for every scheme policy and
assignment strategy, including empty partitions (kappa > extent), Scheme 2 rows that
straddle partitions, skewed modes and kappa = 1."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POLICIES = ["adaptive", "scheme1_only", "scheme2_only"]


def _check_all(mk, orc, t, R, kappa, strategy, policy, seed=1):
    f = [m.data for m in mk.random_factors(t.dims, R, seed)]
    plans = mk.build_mode_plans(t, kappa, strategy, getattr(mk.SchemePolicy, policy))
    cfg = mk.ExecConfig(kappa, 32, False, partitioned=True)
    for d in range(t.mode_count()):
        got = mk.mttkrp_mode(t, plans[d], f, cfg)
        want = orc.mttkrp(t.dims, t.coords, t.values, f, d)
        err = mk.verify_against(got, want)[0]
        assert err <= 1e-5, (policy, strategy, kappa, d, err)


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("strategy", ["cyclic", "least_loaded"])
def test_partitioned_uniform(mk, orc, policy, strategy):
    t = mk.generate_synthetic([183, 24, 114, 171], 60_000, seed=2)
    _check_all(mk, orc, t, 32, 148, getattr(mk.Strategy, strategy), policy)


@pytest.mark.parametrize("policy", POLICIES)
def test_partitioned_skewed_and_ranks(mk, orc, policy):
    t = mk.generate_synthetic([300, 3, 200], 20_000, dist="mode_skewed", skew_mode=1,
                              skew_distinct=2, seed=4)
    for R in (8, 16, 32, 64):
        _check_all(mk, orc, t, R, 148, mk.Strategy.cyclic, policy)


@pytest.mark.parametrize("kappa", [1, 7, 148, 1000])
def test_partitioned_kappa(mk, orc, kappa):
    """kappa = 1 (one CTA), kappa > every extent (empty partitions), kappa > SM count."""
    t = mk.generate_powerlaw([120, 90, 17], 30_000, 1.0, seed=3)
    for policy in POLICIES:
        _check_all(mk, orc, t, 32, kappa, mk.Strategy.cyclic, policy)


def test_partitioned_run_timed_and_all_modes(mk, orc):
    t = mk.generate_synthetic([1000, 1000, 1000], 200_000, seed=1)
    f = [m.data for m in mk.random_factors(t.dims, 32, 1)]
    plans = mk.build_mode_plans(t, 148)
    cfg = mk.ExecConfig(148, 32, False, partitioned=True)
    outs = mk.mttkrp_all_modes(t, plans, f, cfg, False)
    rep, last = mk.run_timed(t, plans, f, cfg, 3)
    for d in range(3):
        want = orc.mttkrp(t.dims, t.coords, t.values, f, d)
        assert mk.verify_against(outs[d], want)[0] <= 1e-5
        assert mk.verify_against(last[d], want)[0] <= 1e-5
    assert all(len(m.wall_ms) == 3 for m in rep.modes)
