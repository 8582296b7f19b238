"""GPU: the device format builder + partitioner (layout.cpp:76-183) is bit-exact with the
reference: order, partition_offsets, owned_indices and the materialised SoA copy."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def device_plans(mk, dims, coords, kappa, strategy, policy, values=None):
    if values is None:
        values = np.ones(coords.shape[0], np.float32)
    t = mk.SparseTensorCOO(dims, coords, values)
    ctx = mk.Context()
    ctx.upload_tensor(t)
    ctx.build_plans(kappa, strategy, policy)
    return ctx


def test_partition_kats(mk, golden):
    # test_layout.cpp:58-99 (cyclic {9,6} owned {0,2,4},{1,3}; LPT {0,3,4},{1,2}; S2 ceil-first)
    for k in golden["kat"]:
        deg = k["degrees"]
        coords = np.array([(v, j) for v, d in enumerate(deg) for j in range(d)], np.uint32)
        ctx = device_plans(mk, [len(deg), max(deg)], coords, k["kappa"], k["strategy"], k["policy"])
        p = ctx.plan_export(0)
        assert p["scheme"] == k["scheme"]
        assert p["order"].tolist() == k["order"]
        assert p["offsets"].tolist() == k["offsets"]
        assert p["owned"].tolist() == k["owned"]
        assert p["owned_offsets"].tolist() == k["owned_offsets"]


@pytest.mark.parametrize("seed", range(12))
def test_random_plans_match_oracle(mk, orc, seed):
    g = np.random.default_rng(100 + seed)
    n = int(g.integers(2, 6))
    dims = [int(x) for x in g.integers(1, 40, size=n)]
    nnz = int(g.integers(0, min(int(np.prod(dims)), 3000) + 1))
    t = mk.generate_synthetic(dims, nnz, seed=seed)
    ctx = mk.Context()
    ctx.upload_tensor(t)
    for kappa in (1, 3, 8, 82, 148):
        for strategy in (0, 1):
            for policy in (0, 1, 2):
                ctx.build_plans(kappa, strategy, policy)
                for d in range(n):
                    a = ctx.plan_export(d)
                    b = orc.build_plan(dims, t.coords, d, kappa, strategy, policy)
                    for key in b:
                        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), \
                            (kappa, strategy, policy, d, key)
                    assert np.array_equal(ctx.mode_degrees(d),
                                          np.bincount(t.coords[:, d].astype(np.int64),
                                                      minlength=dims[d]).astype(np.uint64))


def test_materialised_copy(mk):
    t = mk.generate_synthetic([183, 24, 1140, 1717], 200_000, seed=1)
    ctx = mk.Context()
    ctx.upload_tensor(t)
    ctx.build_plans(148)
    for d in range(4):
        p = ctx.plan_export(d)
        idx, vals = ctx.copy_export(d)
        o = p["order"].astype(np.int64)
        assert np.array_equal(idx, t.coords[o].T)
        assert np.array_equal(vals, t.values[o])
        # one contiguous run per output row (what the fast kernel relies on)
        rows = idx[d]
        starts = np.flatnonzero(np.r_[True, rows[1:] != rows[:-1]])
        assert len(np.unique(rows)) == len(starts)


def test_adaptive_selection_kat(mk):
    # acceptance.cpp:192-202: 6186x24x77x32 at kappa=82 -> s1,s2,s2,s2
    t = mk.generate_synthetic([6186, 24, 77, 32], 20000, seed=9)
    plans = mk.build_mode_plans(t, 82)
    assert [p.scheme for p in plans] == [mk.Scheme.scheme1, mk.Scheme.scheme2,
                                         mk.Scheme.scheme2, mk.Scheme.scheme2]


@pytest.mark.parametrize("name", ["cfg1", "cfg2_uber", "cfg3_nips", "cfg4_lbnl", "cfg5_nell2",
                                  "adaptive_kat"])
def test_config_plans_match_reference_pins(mk, golden, name):
    """Every BASELINE config at full size, format bit-exact against the reference's own
    build_mode_plans (sha256 of order / partition_offsets / owned_indices, computed by the
    reference in tests/golden/make_golden.py) at kappa = 148 and a second kappa (8 or 16),
    cyclic and LPT."""
    e = [c for c in golden["configs"] if c["name"] == name][0]
    if e.get("gen") == "powerlaw":
        t = mk.generate_powerlaw(e["dims"], e["nnz"], 1.0, e["seed"])
    else:
        t = mk.generate_synthetic(e["dims"], e["nnz"], seed=e["seed"])
    assert sha(t.coords) == e["coords_sha"] and sha(t.values) == e["values_sha"]
    ctx = mk.Context()
    ctx.upload_tensor(t)
    built = None
    for p in e["plans"]:
        if built != (p["kappa"], p["strategy"]):
            ctx.build_plans(p["kappa"], p["strategy"], 0)
            built = (p["kappa"], p["strategy"])
        q = ctx.plan_export(p["mode"])
        assert q["scheme"] == p["scheme"]
        assert sha(q["order"]) == p["order_sha"], (name, p)
        assert sha(q["offsets"]) == p["offsets_sha"]
        assert sha(q["owned"]) == p["owned_sha"]
        assert sha(q["owned_offsets"]) == p["owned_offsets_sha"]


def test_tensor_upload_validation_on_device(mk):
    ctx = mk.Context()
    dims = np.array([2, 3], np.uint32)
    coords = np.array([[0, 0], [1, 7]], np.uint32)
    vals = np.array([1.0, 2.0], np.float32)
    with pytest.raises(mk.MttkrpError, match="coordinate 7 out of range for mode 1"):
        mk.load_library()
        mk._check(ctx.lib.mk_tensor_upload(ctx.h, 2, dims.ctypes.data, 2, coords.ctypes.data,
                                           vals.ctypes.data))
    vals = np.array([np.nan, 2.0], np.float32)
    coords = np.array([[0, 0], [1, 1]], np.uint32)
    with pytest.raises(mk.MttkrpError, match="non-finite element value"):
        mk._check(ctx.lib.mk_tensor_upload(ctx.h, 2, dims.ctypes.data, 2, coords.ctypes.data,
                                           vals.ctypes.data))
    with pytest.raises(mk.MttkrpError, match="kappa must be at least 1"):
        mk._check(ctx.lib.mk_build_plans(ctx.h, 0, 0, 0))
