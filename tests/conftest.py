import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(TESTS, "golden")
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_kats():
    return load_golden("kats.json")


@pytest.fixture(scope="session")
def golden_instances():
    return load_golden("instances.json")


@pytest.fixture(scope="session")
def golden_datagen():
    return load_golden("datagen.json")


@pytest.fixture(scope="session")
def golden_configs():
    return load_golden("configs.json")


@pytest.fixture(scope="session")
def ctx():
    """Device context; the GPU tests must run on the CUDA path (no fallback)."""
    from paper_0905_2203_b200 import Context
    c = Context(0)
    yield c
    c.close()
