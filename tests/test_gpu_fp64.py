"""GPU: the fp64 path (the reference's T = double instantiation).

* SparseTensorCOO<double> / FactorMatrix<double> through mk_tensor_upload_f64 /
  mk_factors_upload_f64; deterministic exec bitwise equal to oracle_mttkrp<double>
  (oracle.hpp:20-43: element order, term = val; term *= Y_w for w ascending) — restated in
  fp64 numpy (oracle/als.py mttkrp64, whose np.add.at accumulates in element order);
* fast exec within verify_tolerance<double> = 1e-12 (verify.hpp:42-45), the reference's
  f64 acceptance bar (acceptance.cpp:35-77 at T = double);
* T is not mixed: fp32 calls on an fp64 tensor fail, as the reference's templates would not
  compile.
"""
import numpy as np
import pytest

from oracle import als as als_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(6))
def test_fp64_tensor_random(mk, seed):
    g = np.random.default_rng(40 + seed)
    n = int(g.integers(3, 6))
    dims = [int(x) for x in g.integers(1, 33, size=n)]
    nnz = int(g.integers(0, min(int(np.prod(dims)), 2000) + 1))
    t32 = mk.generate_synthetic(dims, nnz, seed=seed, dtype=np.float64)
    assert t32.values.dtype == np.float64
    vals = t32.values * np.where(g.integers(0, 2, size=nnz) == 1, 1.0, -1.0)  # signed
    t = mk.SparseTensorCOO(dims, t32.coords, vals)
    rank = int(g.choice([2, 8, 32, 40]))
    f = mk.random_factors(dims, rank, seed + 3, dtype=np.float64)
    assert f[0].data.dtype == np.float64
    kappa = int(g.choice([1, 3, 8]))
    plans = mk.build_mode_plans(t, kappa, mk.Strategy(int(g.integers(0, 2))),
                                mk.SchemePolicy(int(g.integers(0, 3))))
    det = mk.mttkrp_all_modes(t, plans, f, mk.ExecConfig(kappa, 32, True), False)
    fast = mk.mttkrp_all_modes(t, plans, f, mk.ExecConfig(kappa, 32, False), False)
    for d in range(n):
        want = als_oracle.mttkrp64(dims, t.coords, t.values, [m.data for m in f], d)
        assert det[d].data.dtype == np.float64
        assert np.array_equal(det[d].data.view(np.uint64), want.view(np.uint64)), d
        assert mk.verify_against(fast[d], want)[0] <= 1e-12, d
        one = mk.mttkrp_mode(t, plans[d], f, mk.ExecConfig(kappa, 32, True))
        assert np.array_equal(one.data.view(np.uint64), want.view(np.uint64))


def test_fp64_generators_widen_fp32(mk):
    """generate_synthetic<double> / random_factors<double> draw the same sequence as the fp32
    versions (rng.hpp:37-39 casts the same double)."""
    dims = [50, 60, 70]
    a = mk.generate_synthetic(dims, 5000, seed=4)
    b = mk.generate_synthetic(dims, 5000, seed=4, dtype=np.float64)
    assert np.array_equal(a.coords, b.coords)
    assert np.array_equal(a.values, b.values.astype(np.float32))
    fa = mk.random_factors(dims, 8, 2)
    fb = mk.random_factors(dims, 8, 2, dtype=np.float64)
    for x, y in zip(fa, fb):
        assert np.array_equal(x.data, y.data.astype(np.float32))


def test_fp64_on_fp32_tensor_is_exact_widening(mk, orc):
    """The device fp64 path on an fp32 tensor with widened fp32 factors is the fp64 truth the
    fast fp32 path is gated against: bitwise = orc.mttkrp_f64 (= the reference's
    oracle_mttkrp<double>, pinned in test_oracle.py)."""
    dims = [183, 24, 1140, 1717]
    t = mk.generate_synthetic(dims, 200_000, seed=2)
    f = [m.data for m in mk.random_factors(dims, 32, 1)]
    c = mk.Context()
    c.upload_tensor(t)
    c.build_plans(148)
    c.upload_factors_f64([m.astype(np.float64) for m in f])
    det = c.mttkrp_all_modes_f64(False, True)
    for d in range(4):
        want = orc.mttkrp_f64(dims, t.coords, t.values, f, d)
        assert np.array_equal(det[d].view(np.uint64), want.view(np.uint64)), d


def test_types_are_not_mixed(mk):
    dims = [5, 6, 7]
    t = mk.generate_synthetic(dims, 50, seed=1, dtype=np.float64)
    plans = mk.build_mode_plans(t, 2)
    f32 = mk.random_factors(dims, 4, 1)
    with pytest.raises(mk.MttkrpError, match="fp64 tensor needs fp64 factor"):
        mk.mttkrp_mode(t, plans[0], f32, mk.ExecConfig(2))
    c = plans[0]._ctx
    c.upload_factors([m.data for m in f32])
    with pytest.raises(mk.MttkrpError, match="holds fp64 values"):
        c.mttkrp_mode(0)
    t32 = mk.generate_synthetic(dims, 50, seed=1)
    p32 = mk.build_mode_plans(t32, 2)
    with pytest.raises(mk.MttkrpError, match="fp64 factor matrices need an fp64 tensor"):
        mk.mttkrp_mode(t32, p32[0], mk.random_factors(dims, 4, 1, dtype=np.float64),
                       mk.ExecConfig(2))


def test_fp64_nonfinite_reported(mk):
    dims = [3, 4, 5]
    coords = np.array([[0, 0, 0], [1, 2, 3], [2, 3, 4]], np.uint32)
    t = mk.SparseTensorCOO(dims, coords, np.array([1.0, 1e200, 2.0]))
    plans = mk.build_mode_plans(t, 1)
    f = [np.full((d, 2), 1e200) for d in dims]
    with pytest.raises(mk.MttkrpError, match="non-finite partial product"):
        mk.mttkrp_mode(t, plans[0], [mk.FactorMatrix(i, m) for i, m in enumerate(f)],
                       mk.ExecConfig(1, 32, True))
