import gzip
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str):
    with gzip.open(GOLDEN / name, "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("golden_small.json.gz")


@pytest.fixture(scope="session")
def golden_medium():
    return load_golden("golden_medium.json.gz")


@pytest.fixture(scope="session")
def golden_protein():
    return load_golden("golden_protein.json.gz")


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)
