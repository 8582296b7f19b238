"""The C++ drop-in header (include/mttkrp_b200/mttkrp.hpp) compiles and links against the
C ABI (CPU), and the reference's own test cases re-stated against it pass (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2503_18198_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_binary():
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lmttkrp_b200", f"-Wl,-rpath,{LIBDIR}", "-o", BIN],
                   check=True)


def test_dropin_header_compiles_and_links(mk):
    build_binary()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_cases_pass_on_gpu(mk):
    build_binary()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
