"""Shared fixtures.  `-m gpu` tests need a B200 (cuda:0); everything else runs on CPU."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


@pytest.fixture(scope="session")
def engine():
    from paper_1706_06940_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle


def rng(seed):
    return np.random.default_rng(seed)
