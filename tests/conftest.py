import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gpu():
    """One GpuExecutor on cuda:0 for the whole session (fails loudly without a device)."""
    from paper_2502_11129_b200 import GpuExecutor
    ex = GpuExecutor(0)
    yield ex
    ex.ctx.close()


@pytest.fixture(scope="session")
def gpu_generic():
    """The reference-order generic kernel variant (the in-tree cross-check)."""
    from paper_2502_11129_b200 import GpuExecutor
    ex = GpuExecutor(0, kernel=1)
    yield ex
    ex.ctx.close()
