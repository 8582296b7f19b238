"""CPU: pin the oracle (oracle/oracle.c) before trusting it.

The oracle is checked against (a) the reference's own golden fixtures and KATs
(tests/golden/golden.json, produced by tests/golden/make_golden.py from the reference) and
(b) the reference itself compiled from its sources (oracle/_ref) when present.
"""
import hashlib

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_tiny3_golden_exact(orc, golden):
    # test_oracle.cpp:79-90 (golden fixture agrees exactly)
    g = golden["tiny3"]
    f = [np.array(m, np.float32) for m in g["factors"]]
    for d in range(len(g["dims"])):
        out = orc.mttkrp(g["dims"], np.array(g["coords"], np.uint32),
                         np.array(g["values"], np.float32), f, d)
        assert out.tolist() == g["expected"][d]


def test_single_nonzero_kat(orc):
    # test_kernel.cpp:57-77: mode0 row0 = [6,6]; mode1 row1 = [6,3]; mode2 row1 = [3,6]
    dims, c, v = [1, 2, 2], np.array([[0, 1, 1]], np.uint32), np.array([3.0], np.float32)
    f = [np.array([[1, 1]], np.float32), np.array([[7, 8], [1, 2]], np.float32),
         np.array([[6, 7], [2, 1]], np.float32)]
    assert orc.mttkrp(dims, c, v, f, 0).tolist() == [[6, 6]]
    assert orc.mttkrp(dims, c, v, f, 1).tolist() == [[0, 0], [6, 3]]
    assert orc.mttkrp(dims, c, v, f, 2).tolist() == [[0, 0], [3, 6]]


def test_partition_kats(orc, golden):
    # test_layout.cpp:58-99 recomputed by the reference
    for k in golden["kat"]:
        deg = k["degrees"]
        coords = np.array([(v, j) for v, d in enumerate(deg) for j in range(d)], np.uint32)
        p = orc.build_plan([len(deg), max(deg)], coords, 0, k["kappa"], k["strategy"], k["policy"])
        assert p["scheme"] == k["scheme"]
        assert p["order"].tolist() == k["order"]
        assert p["offsets"].tolist() == k["offsets"]
        assert p["owned"].tolist() == k["owned"]
        assert p["owned_offsets"].tolist() == k["owned_offsets"]
    # the hand-stated KATs themselves
    cyc, lpt = golden["kat"][0], golden["kat"][1]
    assert np.diff(cyc["offsets"]).tolist() == [9, 6]
    assert cyc["owned"] == [0, 2, 4, 1, 3]
    assert lpt["owned"] == [0, 3, 4, 1, 2]
    assert np.diff(golden["kat"][3]["offsets"]).tolist() == [4, 3, 3]
    assert np.diff(golden["kat"][5]["offsets"]).tolist() == [1, 1, 0, 0, 0]


def test_config_pins_small(orc, golden):
    # generator, factors, plans and oracle MTTKRP of the adaptive KAT config
    e = [c for c in golden["configs"] if c["name"] == "adaptive_kat"][0]
    c, v = orc.generate_synthetic(e["dims"], e["nnz"], 0, 0, 2, e["seed"])
    assert sha(c) == e["coords_sha"] and sha(v) == e["values_sha"]
    f = orc.random_factors(e["dims"], e["rank"], 1)
    assert [sha(m) for m in f] == e["factors_sha"]
    for p in e["plans"]:
        q = orc.build_plan(e["dims"], c, p["mode"], p["kappa"], p["strategy"], 0)
        assert q["scheme"] == p["scheme"]
        assert sha(q["order"]) == p["order_sha"]
        assert sha(q["offsets"]) == p["offsets_sha"]
        assert sha(q["owned"]) == p["owned_sha"]
    assert [p["scheme"] for p in e["plans"][:4]] == [1, 2, 2, 2]  # acceptance.cpp:192-202
    for d in range(len(e["dims"])):
        assert sha(orc.mttkrp(e["dims"], c, v, f, d)) == e["mttkrp_sha"][d]


@pytest.mark.parametrize("name", ["adaptive_kat", "cfg2_uber"])
def test_oracle_f64_matches_reference_pins(orc, golden, name):
    """oracle.hpp:20-43 with T = double: the C restatement (row-parallel) is bitwise equal to the
    reference's own oracle_mttkrp<double> (sha256 computed by the reference); the recorded
    deviation of the reference's fp32 result from it is what the fast path is compared with."""
    e = [c for c in golden["configs"] if c["name"] == name][0]
    c, v = orc.generate_synthetic(e["dims"], e["nnz"], 0, 0, 2, e["seed"])
    f = orc.random_factors(e["dims"], e["rank"], 1)
    for d in range(len(e["dims"])):
        got = orc.mttkrp_f64(e["dims"], c, v, f, d)
        assert sha(got) == e["mttkrp64_sha"][d], (name, d)
        want32 = orc.mttkrp(e["dims"], c, v, f, d)
        assert abs(orc.max_rel_err_f64(want32, got) - e["ref32_vs_64_max_rel_err"][d]) < 1e-12


@pytest.mark.slow
def test_config_pins_cfg1(orc, golden):
    e = [c for c in golden["configs"] if c["name"] == "cfg1"][0]
    c, v = orc.generate_synthetic(e["dims"], e["nnz"], 0, 0, 2, e["seed"])
    assert sha(c) == e["coords_sha"] and sha(v) == e["values_sha"]
    f = orc.random_factors(e["dims"], e["rank"], 1)
    for p in e["plans"][:3]:
        q = orc.build_plan(e["dims"], c, p["mode"], p["kappa"], p["strategy"], 0)
        assert sha(q["order"]) == p["order_sha"] and sha(q["offsets"]) == p["offsets_sha"]
    assert sha(orc.mttkrp(e["dims"], c, v, f, 0)) == e["mttkrp_sha"][0]


@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_random(orc, ref, seed):
    # randomized equivalence in the style of acceptance.cpp:35-77 / test_layout.cpp:180-210
    g = np.random.default_rng(seed)
    n = int(g.integers(2, 6))
    dims = [int(x) for x in g.integers(1, 33, size=n)]
    cap = int(np.prod(dims))
    nnz = int(g.integers(0, min(cap, 2000) + 1))
    c, v = ref.generate_synthetic(dims, nnz, 0, 0, 2, seed)
    c2, v2 = orc.generate_synthetic(dims, nnz, 0, 0, 2, seed)
    assert np.array_equal(c, c2) and np.array_equal(v, v2)
    v = v * np.where(g.integers(0, 2, size=nnz) == 1, 1, -1).astype(np.float32)
    rank = int(g.choice([2, 8, 32]))
    f = ref.random_factors(dims, rank, seed + 7)
    for kappa in (1, 3, 8):
        for strategy in (0, 1):
            for policy in (0, 1, 2):
                for d in range(n):
                    a = orc.build_plan(dims, c, d, kappa, strategy, policy)
                    b = ref.build_plan(dims, c, d, kappa, strategy, policy, values=v)
                    for k in a:
                        assert np.array_equal(a[k], b[k]), (kappa, strategy, policy, d, k)
    for d in range(n):
        a = orc.mttkrp(dims, c, v, f, d)
        b = ref.oracle_mttkrp(dims, c, v, f, d)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        a64 = orc.mttkrp_f64(dims, c, v, f, d, threads=3)
        b64 = ref.oracle_mttkrp_f64(dims, c, v, f, d)
        assert np.array_equal(a64.view(np.uint64), b64.view(np.uint64))


def test_skewed_generator_matches_reference(orc, ref):
    for dims, nnz, sm, sd, seed in [([100, 2, 100], 500, 1, 2, 13), ([60, 2, 40], 900, 1, 2, 77),
                                    ([50, 7, 9], 300, 1, 3, 4)]:
        c, v = ref.generate_synthetic(dims, nnz, 1, sm, sd, seed)
        c2, v2 = orc.generate_synthetic(dims, nnz, 1, sm, sd, seed)
        assert np.array_equal(c, c2) and np.array_equal(v, v2)
        assert len(np.unique(c[:, sm])) == min(sd, dims[sm])
