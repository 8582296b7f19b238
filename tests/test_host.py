"""CPU: the C-ABI library loads and exports every symbol include/mttkrp_b200.h declares;
host-side ingest (generator, factor init) is bit-identical to the reference; host
validation reproduces the reference's error messages.  No GPU compute calls here."""
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mttkrp_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(mk_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol(mk):
    lib = ctypes.CDLL(mk.library_path())
    syms = header_symbols()
    assert len(syms) >= 29
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(mk.EXPORTED_SYMBOLS) == syms
    assert b"sm_100a" in mk.load_library().mk_version()


def test_library_is_sm100a_cubin(mk):
    data = open(mk.library_path(), "rb").read()
    assert b"sm_100a" in data


def test_generator_bit_identical_to_reference_pins(mk, golden):
    for e in golden["configs"]:
        if e["nnz"] > 2_000_000:
            continue
        t = mk.generate_synthetic(e["dims"], e["nnz"], seed=e["seed"])
        assert sha(t.coords) == e["coords_sha"], e["name"]
        assert sha(t.values) == e["values_sha"], e["name"]
        f = mk.random_factors(e["dims"], e["rank"], 1)
        assert [sha(m.data) for m in f] == e["factors_sha"]


@pytest.mark.parametrize("spec", [([4, 4, 4], 64, 0, 0, 2, 5), ([30, 7, 50], 400, 0, 0, 2, 99),
                                  ([100, 2, 100], 500, 1, 1, 2, 11), ([60, 2, 40], 900, 1, 1, 2, 77),
                                  ([12092, 9184, 28818], 50_000, 0, 0, 2, 1),
                                  ([6186, 24, 77, 32], 20000, 0, 0, 2, 9)])
def test_generator_matches_oracle(mk, orc, spec):
    dims, nnz, dist, sm, sd, seed = spec
    t = mk.generate_synthetic(dims, nnz, dist, sm, sd, seed)
    c, v = orc.generate_synthetic(dims, nnz, dist, sm, sd, seed)
    assert np.array_equal(t.coords, c)
    assert np.array_equal(t.values.view(np.uint32), v.view(np.uint32))


def test_generator_errors(mk):
    with pytest.raises(mk.MttkrpError, match="exceeds index capacity"):
        mk.generate_synthetic([2, 2], 5)
    with pytest.raises(mk.MttkrpError, match="zero extent"):
        mk.generate_synthetic([2, 0], 1)
    with pytest.raises(mk.MttkrpError, match="skew mode out of range"):
        mk.generate_synthetic([2, 2], 1, "mode_skewed", skew_mode=3)
    with pytest.raises(mk.MttkrpError, match="rank must be at least 1"):
        mk.random_factors([2, 2], 0, 1)


def test_powerlaw_generator_matches_oracle(mk, orc):
    dims = [248, 286, 1403, 17]
    t = mk.generate_powerlaw(dims, 20000, 1.0, 3)
    c, v = orc.generate_powerlaw(dims, 20000, 1.0, 3)
    assert np.array_equal(t.coords, c) and np.array_equal(t.values, v)
    # distinct tuples, heavy head
    assert len({tuple(r) for r in t.coords.tolist()}) == 20000
    counts = np.bincount(t.coords[:, 2], minlength=dims[2])
    assert counts.max() > 20 * counts.mean()


def test_tensor_validation_messages(mk):
    # tensor.hpp:97-106
    with pytest.raises(mk.MttkrpError, match="coordinate 5 out of range for mode 1"):
        mk.SparseTensorCOO([2, 3], [[0, 0], [1, 5]], [1.0, 2.0])
    with pytest.raises(mk.MttkrpError, match="non-finite element value"):
        mk.SparseTensorCOO([2, 3], [[0, 0], [1, 1]], [1.0, np.inf])
    with pytest.raises(mk.MttkrpError, match="storage size mismatch"):
        mk.SparseTensorCOO([2, 3], [[0, 0], [1, 1]], [1.0])
    with pytest.raises(mk.MttkrpError, match="zero extent"):
        mk.SparseTensorCOO([2, 0])
    with pytest.raises(mk.MttkrpError, match="at least one mode"):
        mk.SparseTensorCOO([])


def test_exec_config_validation(mk):
    with pytest.raises(mk.MttkrpError, match="kappa must be at least 1"):
        mk.ExecConfig(0, 32).validate()
    with pytest.raises(mk.MttkrpError, match="batch size P must be at least 1"):
        mk.ExecConfig(2, 0).validate()


def test_verify_metric(mk):
    g = np.array([[1.0, 2.0], [100.0, 0.5]], np.float32)
    w = np.array([[1.0, 2.5], [101.0, 0.5]], np.float32)
    err, row, col = mk.verify_against(g, w)
    assert abs(err - 0.5 / 2.5) < 1e-7 and (row, col) == (0, 1)
    assert mk.verify_tolerance(np.float32) == 1e-5
    assert mk.verify_tolerance(np.float64) == 1e-12


def test_no_cpu_fallback_without_gpu(mk):
    # the product never computes on the CPU: without a device, compute entry points fail loudly
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mk.MttkrpError):
        mk.Context()


def test_element_update(mk):
    """kernel.hpp:133-153 via test_kernel.cpp:39-55 (host arithmetic, API parity)."""
    ones = mk.SparseTensorCOO([2, 2, 2], [[0, 1, 0]], [1.0])
    all_ones = [np.ones((2, 2), np.float32)] * 3
    assert mk.element_update(ones, 0, all_ones, 2).tolist() == [1, 1]
    t = mk.SparseTensorCOO([1, 2, 1], [[0, 1, 0]], [3.0])
    f = [np.array(m, np.float32) for m in ([[1, 2]], [[9, 9], [2, 1]], [[5, 5]])]
    assert mk.element_update(t, 0, f, 2).tolist() == [6, 6]
    t2 = mk.SparseTensorCOO([1, 2, 1], [[0, 1, 0]], [2.0])
    disjoint = [np.array(m, np.float32) for m in ([[1, 0]], [[9, 9], [0, 1]], [[5, 5]])]
    assert mk.element_update(t2, 0, disjoint, 2).tolist() == [0, 0]
    with pytest.raises(mk.MttkrpError, match="disagree on rank"):
        mk.element_update(t, 0, [f[0], np.zeros((2, 3), np.float32), f[2]], 2)
