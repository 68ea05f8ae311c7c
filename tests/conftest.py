import os
import sys

# The emulated multi-rank peer-memory tests run several ranks' series on one
# device, each on its own stream, and the ranks spin-wait on each other: their
# streams must not share a hardware work queue (read at CUDA context creation).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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


def fresh_stream():
    """A newly created non-blocking CUDA stream (not one of torch's pooled
    streams, which may share a hardware queue with earlier work)."""
    import torch
    from cuda.bindings import runtime as rt

    err, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
    assert err == rt.cudaError_t.cudaSuccess, err
    return torch.cuda.ExternalStream(int(s))


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
