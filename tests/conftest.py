import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "libstdcxx_streams.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ctx():
    import paper_1505_07570_b200 as rn
    c = rn.Context(0)
    yield c
    c.close()
