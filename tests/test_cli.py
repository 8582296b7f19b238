"""mttkrp-bench --backend gpu: the reference's CLI tests (tests/test_cli.cpp)
restated against the GPU binary, plus byte-equality of `gen` with the reference's own
generator + FROSTT writer.  gen and argument/ingest errors need no GPU; run/inspect do."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2503_18198_b200", "bin", "mttkrp-bench")


@pytest.fixture(scope="module")
def cli(mk):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2503_18198_b200")], check=True)
    return CLI


def run_cli(cli, args, env=None):
    e = dict(os.environ)
    e.pop("SPMTTKRP_WORKERS", None)
    if env:
        e.update(env)
    return subprocess.run([cli] + args, capture_output=True, text=True, env=e, timeout=600)


def test_gen_reproducible_and_counts(cli, tmp_path):  # test_cli.cpp:56-70
    tns = tmp_path / "t.tns"
    assert run_cli(cli, ["gen", "--dims", "16,16,16", "--nnz", "1000", "--seed", "1", "--out",
                         str(tns)]).returncode == 0
    first = tns.read_text()
    assert first.count("\n") == 1000
    assert run_cli(cli, ["gen", "--dims", "16,16,16", "--nnz", "1000", "--seed", "1", "--out",
                         str(tns)]).returncode == 0
    assert tns.read_text() == first
    assert run_cli(cli, ["gen", "--dims", "2,2", "--nnz", "5", "--seed", "1", "--out",
                         str(tns)]).returncode != 0


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dims,nnz,seed", [([40, 6, 30], 800, 3), ([100, 2, 100], 500, 5),
                                           ([6186, 24, 77, 32], 5000, 8)])
def test_gen_bytes_equal_reference(cli, tmp_path, dims, nnz, seed):
    """gen = the reference's generate_synthetic + write_frostt_file, byte for byte."""
    tns = tmp_path / "g.tns"
    assert run_cli(cli, ["gen", "--dims", ",".join(map(str, dims)), "--nnz", str(nnz), "--seed",
                         str(seed), "--out", str(tns)]).returncode == 0
    ref = oracle.Reference()
    c, v = ref.generate_synthetic(dims, nnz, 0, 0, 2, seed)
    assert tns.read_text() == ref.frostt_write(dims, c, v)


def test_errors_exit_nonzero_with_json(cli, tmp_path):  # test_cli.cpp:226-237
    rep = tmp_path / "report.json"
    assert run_cli(cli, ["run", "--tensor", str(tmp_path / "missing.tns")]).returncode != 0
    bad = tmp_path / "bad.tns"
    bad.write_text("1 1 oops\n")
    r = run_cli(cli, ["run", "--tensor", str(bad), "--json", str(rep)])
    assert r.returncode == 1
    assert "error" in json.loads(rep.read_text())
    assert run_cli(cli, ["run", "--tensor", str(bad), "--backend", "cpu"]).returncode != 0
    assert run_cli(cli, ["frobnicate"]).returncode != 0


def test_gen_binary_cache_output(cli, tmp_path, mk):
    out = tmp_path / "t.mkbt"
    assert run_cli(cli, ["gen", "--dims", "30,20,10", "--nnz", "500", "--seed", "2", "--out",
                         str(out)]).returncode == 0
    t = mk.load_tensor_cache(out)
    g = mk.generate_synthetic([30, 20, 10], 500, seed=2)
    assert np.array_equal(t.coords, g.coords) and np.array_equal(t.values, g.values)


# ---------------------------------------------------------------- GPU (device build + kernels)
@pytest.mark.gpu
def test_run_verify_schema(cli, tmp_path):  # test_cli.cpp:72-106
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "40,6,30", "--nnz", "800", "--seed", "3", "--out",
                         str(tns)]).returncode == 0
    r = run_cli(cli, ["run", "--tensor", str(tns), "--rank", "8", "--kappa", "4", "--iters", "2",
                      "--verify", "--deterministic", "--json", str(rep)])
    assert r.returncode == 0, r.stderr
    j = json.loads(rep.read_text())
    assert j["nnz"] == 800 and j["kappa"] == 4 and j["backend"] == "gpu"
    assert len(j["timing"]["modes"]) == 3
    for m in j["timing"]["modes"]:
        assert "scheme" in m and len(m["wall_ms"]) == 2 and "busy_workers" in m
        assert len(m["elements_per_worker"]) == 4
    assert len(j["timing"]["total_ms"]) == 2
    assert j["timing"]["outputs_bit_identical"] is True
    for bm in j["balance"]:
        assert {"loads", "owned_index_counts", "max_over_mean"} <= set(bm)
    assert {"bits_per_element", "total_copy_bits", "total_copy_bytes",
            "factor_matrix_bytes"} <= set(j["memory"])
    assert j["verify"]["passed"] is True and j["verify"]["max_rel_err"] <= 1e-5
    # the fast executor verifies too
    r = run_cli(cli, ["run", "--tensor", str(tns), "--rank", "32", "--verify", "--iters", "3",
                      "--json", str(rep)])
    assert r.returncode == 0, r.stderr
    j = json.loads(rep.read_text())
    assert j["verify"]["passed"] is True


@pytest.mark.gpu
def test_policy_override_busy_workers(cli, tmp_path):  # test_cli.cpp:108-137
    tns, rep = tmp_path / "skew.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "100,2,100", "--nnz", "500", "--dist", "skewed",
                         "--skew-mode", "1", "--seed", "5", "--out", str(tns)]).returncode == 0
    base = ["run", "--tensor", str(tns), "--rank", "4", "--kappa", "8", "--json", str(rep)]
    assert run_cli(cli, base + ["--policy", "s1"]).returncode == 0
    s1 = json.loads(rep.read_text())
    assert s1["timing"]["modes"][1]["scheme"] == "scheme1"
    assert s1["timing"]["modes"][1]["busy_workers"] == 2
    assert run_cli(cli, base + ["--policy", "adaptive"]).returncode == 0
    ad = json.loads(rep.read_text())
    assert ad["timing"]["modes"][1]["scheme"] == "scheme2"
    assert ad["timing"]["modes"][1]["busy_workers"] == 8
    assert run_cli(cli, base + ["--policy", "s2"]).returncode == 0
    assert all(m["scheme"] == "scheme2" for m in json.loads(rep.read_text())["timing"]["modes"])


@pytest.mark.gpu
def test_deterministic_reruns_reproduce(cli, tmp_path):  # test_cli.cpp:139-170
    tns = tmp_path / "t.tns"
    assert run_cli(cli, ["gen", "--dims", "20,3,20", "--nnz", "300", "--seed", "9", "--out",
                         str(tns)]).returncode == 0
    args = ["run", "--tensor", str(tns), "--rank", "8", "--kappa", "4", "--seed", "11",
            "--verify", "--deterministic", "--json"]
    outs = []
    for k in range(2):
        p = tmp_path / f"r{k}.json"
        assert run_cli(cli, args + [str(p)]).returncode == 0
        j = json.loads(p.read_text())
        for m in j["timing"]["modes"]:
            for key in ("wall_ms", "min_ms", "median_ms"):
                m.pop(key)
        for key in ("total_ms", "total_min_ms", "total_median_ms"):
            j["timing"].pop(key)
        j.pop("tensor")
        outs.append(j)
    assert outs[0] == outs[1]


@pytest.mark.gpu
def test_inspect_memory_formula(cli, tmp_path):  # test_cli.cpp:172-188
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "4,4,4", "--nnz", "10", "--seed", "2", "--out",
                         str(tns)]).returncode == 0
    assert run_cli(cli, ["inspect", "--tensor", str(tns), "--kappa", "2", "--rank", "2",
                         "--json", str(rep)]).returncode == 0
    j = json.loads(rep.read_text())
    assert j["memory"]["bits_per_element"] == 38
    assert j["memory"]["total_copy_bits"] == 1140
    for m in j["modes"]:
        assert m["scheme"] == "scheme1" and "distinct_indices" in m and "extent" in m


@pytest.mark.gpu
def test_chicago_narrow_modes_scheme2(cli, tmp_path):  # test_cli.cpp:190-206
    tns, rep = tmp_path / "c.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "6186,24,77,32", "--nnz", "5000", "--seed", "8",
                         "--out", str(tns)]).returncode == 0
    assert run_cli(cli, ["inspect", "--tensor", str(tns), "--kappa", "82", "--json",
                         str(rep)]).returncode == 0
    modes = json.loads(rep.read_text())["modes"]
    assert [m["scheme"] for m in modes] == ["scheme1", "scheme2", "scheme2", "scheme2"]


@pytest.mark.gpu
def test_f64_tight_tolerance(cli, tmp_path):  # test_cli.cpp:208-222
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "12,13,14", "--nnz", "400", "--seed", "10",
                         "--precision", "f64", "--out", str(tns)]).returncode == 0
    assert run_cli(cli, ["run", "--tensor", str(tns), "--rank", "4", "--kappa", "3",
                         "--precision", "f64", "--verify", "--json", str(rep)]).returncode == 0
    j = json.loads(rep.read_text())
    assert j["verify"]["tolerance"] == 1e-12 and j["verify"]["max_rel_err"] <= 1e-12


@pytest.mark.gpu
def test_kappa1_scheme1_and_env_workers(cli, tmp_path):  # test_cli.cpp:224-260
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "3,2,3", "--nnz", "8", "--seed", "4", "--out",
                         str(tns)]).returncode == 0
    assert run_cli(cli, ["inspect", "--tensor", str(tns), "--kappa", "1", "--json",
                         str(rep)]).returncode == 0
    assert all(m["scheme"] == "scheme1" for m in json.loads(rep.read_text())["modes"])
    t2 = tmp_path / "t2.tns"
    assert run_cli(cli, ["gen", "--dims", "10,10,10", "--nnz", "50", "--seed", "6", "--out",
                         str(t2)]).returncode == 0
    assert run_cli(cli, ["run", "--tensor", str(t2), "--rank", "2", "--json", str(rep)],
                   env={"SPMTTKRP_WORKERS": "3"}).returncode == 0
    assert json.loads(rep.read_text())["kappa"] == 3
    # default kappa on the GPU backend: the SM count
    assert run_cli(cli, ["run", "--tensor", str(t2), "--rank", "2", "--json",
                         str(rep)]).returncode == 0
    import torch
    assert json.loads(rep.read_text())["kappa"] == \
        torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.gpu
def test_cached_tensor_run(cli, tmp_path):
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "50,40,30", "--nnz", "3000", "--seed", "7", "--out",
                         str(tns)]).returncode == 0
    for _ in range(2):  # parse + write the cache, then read it
        r = run_cli(cli, ["run", "--tensor", str(tns), "--cache", "--verify", "--json", str(rep)])
        assert r.returncode == 0, r.stderr
        assert json.loads(rep.read_text())["verify"]["passed"] is True
    assert os.path.exists(str(tns) + ".mkbt")
    r = run_cli(cli, ["run", "--tensor", str(tns) + ".mkbt", "--verify", "--json", str(rep)])
    assert r.returncode == 0 and json.loads(rep.read_text())["nnz"] == 3000


@pytest.mark.gpu
def test_run_exec_reference_and_fast(cli, tmp_path):
    """`run` keeps the reference's executor contract by default (exec "reference": Scheme 1
    modes bitwise equal to --deterministic); `--fast` selects the B200 fast path;
    both verify against the deterministic executor."""
    tns, rep = tmp_path / "t.tns", tmp_path / "report.json"
    assert run_cli(cli, ["gen", "--dims", "300,200,160", "--nnz", "50000", "--seed", "4", "--out",
                         str(tns)]).returncode == 0
    for flags, want in (([], "reference"), (["--fast"], "fast"), (["--deterministic"], "deterministic")):
        r = run_cli(cli, ["run", "--tensor", str(tns), "--rank", "32", "--verify", "--iters", "2",
                          "--json", str(rep)] + flags)
        assert r.returncode == 0, r.stderr
        j = json.loads(rep.read_text())
        assert j["exec"] == want and j["verify"]["passed"] is True
        if want != "fast":  # every extent >= kappa (SM count): all modes Scheme 1, bitwise
            assert j["timing"]["outputs_bit_identical"] is True
            assert j["verify"]["max_rel_err"] == 0.0
