import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configuration")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def orc():
    """The C oracle (test infrastructure).  Built on demand (gcc is in the image)."""
    import oracle
    if not os.path.exists(oracle.Oracle.path):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"),
                        os.path.join(ROOT, "oracle", "liboracle.so")], check=True)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref (reference compiled from /root/reference) not present")
    return oracle.Reference()


@pytest.fixture(scope="session")
def mk():
    import paper_2503_18198_b200 as mk
    mk.load_library()
    return mk
