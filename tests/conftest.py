import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the engine")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    import json
    from common import GOLDEN
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_configs():
    import json
    from common import GOLDEN
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle.ref import Port
    return Port()


@pytest.fixture(scope="session")
def reference():
    from oracle.ref import Reference, reference_available
    if not reference_available():
        pytest.skip("reference library oracle/_ref not built here")
    return Reference()
