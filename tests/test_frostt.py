"""FROSTT ingest and the binary tensor cache, host-only (no GPU).

The product's multithreaded parser/writer (csrc/frostt.cpp via the C ABI) is checked against
the reference's own sequential implementation (frostt.hpp:74-206, compiled into oracle/_ref)
on randomized texts — coordinates, values (bitwise), duplicate counts and error messages must
be identical for every thread count — plus the reference's own test cases
(tests/test_frostt.cpp:8-100).
"""
import os

import numpy as np
import pytest

import oracle
import paper_2503_18198_b200 as mk

ref_needed = pytest.mark.skipif(not oracle.reference_available(),
                                reason="oracle/_ref (the compiled reference) not built")


# ---------------------------------------------------------------- reference test cases
def test_basic_parse():  # test_frostt.cpp:8-19
    r = mk.parse_frostt("1 1 1 2.0\n2 2 2 3.0\n")
    t = r.tensor
    assert t.dims == [2, 2, 2] and t.nnz == 2
    assert t.coords[0, 0] == 0 and t.values[0] == 2.0
    assert t.index(1, 2) == 1 and t.values[1] == 3.0
    assert r.duplicates_merged == 0


def test_duplicates_merge_or_reject():  # test_frostt.cpp:21-33
    m = mk.parse_frostt("1 1 1 2.0\n1 1 1 3.0\n")
    assert m.tensor.nnz == 1 and m.tensor.values[0] == 5.0 and m.duplicates_merged == 1
    with pytest.raises(mk.MttkrpError, match="duplicate"):
        mk.parse_frostt("1 1 1 2.0\n1 1 1 3.0\n", mk.FrosttOptions(merge_duplicates=False))


def test_comments_blank_scientific():  # test_frostt.cpp:35-40
    r = mk.parse_frostt("# header comment\n\n  \n1 2 1.5e2\n#tail\n2 1 -3e-1\n", dtype=np.float64)
    assert r.tensor.dims == [2, 2]
    assert r.tensor.values[0] == 150.0 and r.tensor.values[1] == -0.3


@pytest.mark.parametrize("text,needle", [
    ("", "empty"), ("# comments only\n\n", "empty"), ("1 1 1 1\n1 1 1\n", "line 2"),
    ("1 x 1 1\n", "non-numeric"), ("1 1 1 abc\n", "bad value"), ("0 1 1 1\n", "< 1"),
    ("1\n", "need at least one index"), ("1 1 1 inf\n", "non-finite"),
    ("5000000000 1 1 1\n", "32-bit"),
])
def test_malformed(text, needle):  # test_frostt.cpp:42-53
    with pytest.raises(mk.MttkrpError, match=needle):
        mk.parse_frostt(text)


def test_dims_override():  # test_frostt.cpp:55-66
    r = mk.parse_frostt("1 1 1 1\n", mk.FrosttOptions(dims_override=[4, 4, 4]))
    assert r.tensor.dims == [4, 4, 4]
    with pytest.raises(mk.MttkrpError, match="below largest index"):
        mk.parse_frostt("1 2 0.5\n", mk.FrosttOptions(dims_override=[1, 1]))
    with pytest.raises(mk.MttkrpError, match="dims override has 1 modes"):
        mk.parse_frostt("1 2 0.5\n", mk.FrosttOptions(dims_override=[1]))


def test_writer_shortest_round_trip():  # test_frostt.cpp:68-77
    t = mk.SparseTensorCOO([1, 1, 1], [[0, 0, 0]], np.array([2.0], dtype=np.float32))
    assert mk.write_frostt_string(t) == "1 1 1 2\n"
    u = mk.SparseTensorCOO([2, 3], [[1, 2], [0, 0]], np.array([0.1, -1e30]))
    assert mk.write_frostt_string(u) == "2 3 0.1\n1 1 -1e+30\n"


def test_empty_body_does_not_reparse():  # test_frostt.cpp:79-83
    t = mk.SparseTensorCOO([2, 2])
    assert mk.write_frostt_string(t) == ""
    with pytest.raises(mk.MttkrpError):
        mk.parse_frostt(mk.write_frostt_string(t))


# ---------------------------------------------------------------- randomized vs the reference
def _random_text(rng, n, extent, m, dup_frac=0.2, noise=True, prec=32):
    coords = rng.integers(1, extent + 1, size=(m, n))
    ndup = int(m * dup_frac)
    if ndup and m > 1:
        src = rng.integers(0, m, size=ndup)
        dst = rng.integers(0, m, size=ndup)
        coords[dst] = coords[src]
    lines = []
    for i in range(m):
        if noise and rng.random() < 0.05:
            lines.append(rng.choice(["# comment", "", "   ", "\t", "#x 1 2 3"]))
        kind = rng.integers(0, 5)
        if kind == 0:
            v = str(int(rng.integers(-5, 6)))
        elif kind == 1:
            v = f"{rng.normal():.{int(rng.integers(1, 12))}f}"
        elif kind == 2:
            v = f"{rng.normal() * 10.0 ** int(rng.integers(-30, 30)):.{int(rng.integers(1, 17))}e}"
        elif kind == 3:
            v = repr(float(np.float32(rng.normal())))
        else:
            v = repr(float(rng.normal()))
        sep = rng.choice([" ", "  ", "\t", " \t "]) if noise else " "
        lead = rng.choice(["", " ", "\t"]) if noise else ""
        tail = rng.choice(["", " ", "\r"]) if noise else ""
        lines.append(lead + sep.join(str(int(c)) for c in coords[i]) + sep + v + tail)
    return "\n".join(lines) + ("\n" if rng.random() < 0.7 else "")


def _same(ours, ref_out):
    dims, coords, vals, dups = ref_out
    assert ours.tensor.dims == dims
    assert np.array_equal(ours.tensor.coords, coords)
    assert ours.tensor.values.dtype == vals.dtype
    assert np.array_equal(ours.tensor.values.view(np.uint8), vals.view(np.uint8))
    assert ours.duplicates_merged == dups


@ref_needed
@pytest.mark.parametrize("seed", range(12))
def test_parse_matches_reference(seed):
    ref = oracle.Reference()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 6))
    m = int(rng.integers(1, 3000))
    extent = int(rng.integers(1, 40))
    for prec in (32, 64):
        text = _random_text(rng, n, extent, m, prec=prec)
        dt = np.float64 if prec == 64 else np.float32
        want = ref.frostt_parse(text, prec=prec)
        for threads in (1, 2, 3, 7, 16):
            _same(mk.parse_frostt(text, dtype=dt, threads=threads), want)


def _ref_error(ref, text, **kw):
    try:
        ref.frostt_parse(text, **kw)
    except oracle.OracleError as e:
        return str(e)
    return None


@ref_needed
@pytest.mark.parametrize("seed", range(10))
def test_errors_match_reference(seed):
    """The earliest failing line wins across chunks; a strict-mode duplicate before a parse
    error is reported first (frostt.hpp:96-142 order)."""
    ref = oracle.Reference()
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 5))
    m = 400
    text = _random_text(rng, n, 6, m, dup_frac=0.0 if seed % 2 else 0.01, noise=False)
    lines = text.split("\n")
    bad = ["1 " * (n - 1) + "1", "1 " * n + "nan", "0 " * n + "1", "x " * n + "1",
           "1 " * n + "1 2", "9999999999 " + "1 " * (n - 1) + "1", "1 " * n + "1e999"]
    for k in range(int(rng.integers(1, 4))):
        lines[int(rng.integers(0, m))] = bad[int(rng.integers(0, len(bad)))]
    text = "\n".join(lines)
    for merge in (True, False):
        want = _ref_error(ref, text, merge=merge)
        for threads in (1, 4, 9):
            try:
                mk.parse_frostt(text, mk.FrosttOptions(merge_duplicates=merge), threads=threads)
                got = None
            except mk.MttkrpError as e:
                got = str(e)
            assert got == want, (merge, threads)


@ref_needed
@pytest.mark.parametrize("seed", range(8))
def test_writer_matches_reference(seed):
    ref = oracle.Reference()
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(1, 6))
    m = int(rng.integers(0, 2000))
    dims = [int(x) for x in rng.integers(1, 5000, size=n)]
    coords = np.stack([rng.integers(0, d, size=m) for d in dims], axis=1).astype(np.uint32) \
        if m else np.zeros((0, n), dtype=np.uint32)
    if m:  # distinct tuples (a strict re-parse rejects duplicates), in random order
        coords = np.unique(coords, axis=0)
        coords = coords[rng.permutation(coords.shape[0])]
        m = coords.shape[0]
    for dt in (np.float32, np.float64):
        bits = rng.integers(0, 2 ** 62, size=m, dtype=np.int64)
        vals = (rng.normal(size=m) * np.exp(rng.uniform(-60, 60, size=m))).astype(dt)
        vals[::7] = bits[::7].astype(dt)  # integral values
        t = mk.SparseTensorCOO(dims, coords, vals)
        s = mk.write_frostt_string(t, threads=5)
        assert s == ref.frostt_write(dims, coords, vals)
        if m:  # round trip: strict parse with the dims restores the tensor exactly
            back = mk.parse_frostt(s, mk.FrosttOptions(False, dims), dtype=dt, threads=3)
            assert np.array_equal(back.tensor.coords, t.coords)
            assert np.array_equal(back.tensor.values.view(np.uint8), t.values.view(np.uint8))


def test_file_io_and_cache(tmp_path):
    t = mk.generate_synthetic([50, 7, 30], 5000, seed=3)
    p = tmp_path / "t.tns"
    mk.write_frostt_file(t, p)
    r = mk.read_frostt_file(p)
    assert r.duplicates_merged == 0
    assert np.array_equal(r.tensor.coords, t.coords)
    assert np.array_equal(r.tensor.values, t.values)
    c = tmp_path / "t.mkbt"
    mk.save_tensor_cache(t, c)
    back = mk.load_tensor_cache(c)
    assert back.dims == t.dims and np.array_equal(back.coords, t.coords)
    assert np.array_equal(back.values, t.values)
    # corruption is detected
    raw = bytearray(c.read_bytes())
    raw[40] ^= 0x10
    c.write_bytes(bytes(raw))
    with pytest.raises(mk.MttkrpError, match="checksum"):
        mk.load_tensor_cache(c)
    c.write_bytes(bytes(raw[:30]))
    with pytest.raises(mk.MttkrpError, match="truncated"):
        mk.load_tensor_cache(c)
    with pytest.raises(mk.MttkrpError, match="cannot open"):
        mk.read_frostt_file(tmp_path / "missing.tns")
    # load_tensor: parse once, then served from <path>.mkbt
    r1 = mk.load_tensor(p)
    assert os.path.exists(str(p) + ".mkbt")
    r2 = mk.load_tensor(p)
    assert np.array_equal(r2.tensor.coords, r1.tensor.coords)
    assert np.array_equal(r2.tensor.values, r1.tensor.values)
    r64 = mk.load_tensor(p, dtype=np.float64)  # precision mismatch: re-parsed
    assert r64.tensor.values.dtype == np.float64


def test_fp64_cache_round_trip(tmp_path):
    t = mk.generate_synthetic([9, 8, 7], 200, seed=5, dtype=np.float64)
    mk.save_tensor_cache(t, tmp_path / "d.mkbt")
    back = mk.load_tensor_cache(tmp_path / "d.mkbt")
    assert back.values.dtype == np.float64
    assert np.array_equal(back.values, t.values)
