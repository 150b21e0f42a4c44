import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running full-size check")


@pytest.fixture(scope="session")
def fc():
    import paper_2512_17574_b200 as fcmod
    from paper_2512_17574_b200 import build
    build.build()
    return fcmod


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test without a CUDA device")
    torch.cuda.set_device(0)
    return torch


@pytest.fixture(params=["tc", "mma"])
def kernel(request, monkeypatch):
    """Which fused kernel serves NV12 / fp32 requests: "mma" (the mma.sync
    kernel, the default) or "tc" (the tcgen05 kernel, FC_TC=1, wherever its
    shared-memory plan fits).  libfc reads FC_TC at every launch."""
    monkeypatch.setenv("FC_TC", "1" if request.param == "tc" else "0")
    return request.param
