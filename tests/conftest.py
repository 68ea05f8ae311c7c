import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name + ".npz"))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure; never the product path)."""
    from oracle import oracle as orc

    orc.lib()
    return orc


def coeff_d(x, y, z):
    return 1.0 / np.sqrt(1.0 + x * x + y * y)


def pytest_sessionfinish(session, exitstatus):
    """Tear down the world-size-1 NCCL group some GPU tests create."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:  # pragma: no cover - best effort at exit
        pass
