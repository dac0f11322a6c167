import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs the CUDA path through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name):
    """Rows of a golden text file: whitespace-split fields before '#'."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            body = line.split("#", 1)[0].strip()
            if body:
                rows.append(body.split())
    return rows


@pytest.fixture(scope="session")
def golden():
    return read_golden
