import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_built():
    lib = os.path.join(REPO, "paper_2404_02218_b200", "lib", "libhalogen_b200.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-s", "-C", os.path.join(REPO, "paper_2404_02218_b200"),
                               "-j8"])
    port = os.path.join(REPO, "oracle", "libhg_oracle.so")
    if not os.path.exists(port):
        subprocess.check_call(["make", "-s", "-C", os.path.join(REPO, "oracle"), "port"])


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(REPO, "tests", "golden", "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import REF_PATH, Ref
    if not os.path.exists(REF_PATH):
        pytest.skip("oracle/_ref/libhalogen_ref.so not built (needs /root/reference)")
    return Ref()
