import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def kat():
    return np.load(GOLDEN / "kat.npz")


@pytest.fixture(scope="session")
def c0():
    return dict(np.load(GOLDEN / "c0.npz"))


@pytest.fixture(scope="session")
def hbpq_rig():
    return dict(np.load(GOLDEN / "hbpq.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    orc.lib()
    return orc
