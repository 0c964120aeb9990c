import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: multi-GB state")


@pytest.fixture(scope="session")
def oracle():
    """The CPU restatement (oracle/tso.py + oracle/ts_oracle.c) — checker only."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle-only"], check=True,
                   stdout=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import tso

    return tso


@pytest.fixture(scope="session")
def native():
    from paper_2601_16956_b200 import build

    build.build()
    from paper_2601_16956_b200 import _native

    return _native


def golden_recipes():
    d = os.path.join(GOLDEN, "trees")
    return sorted(os.listdir(d))


def read_tree(root):
    out = {}
    for dp, _, fs in os.walk(root):
        for fn in fs:
            p = os.path.join(dp, fn)
            with open(p, "rb") as f:
                out[os.path.relpath(p, root)] = f.read()
    return out


@pytest.fixture
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
