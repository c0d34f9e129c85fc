import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# Forward schedules go to a per-session plan cache (plan_cache.cpp), so the
# suite neither reads nor fills the user's ~/.cache/radon_b200.
if "RK_PLAN_CACHE" not in os.environ:
    import tempfile

    os.environ["RK_PLAN_CACHE"] = tempfile.mkdtemp(prefix="rk_plan_cache_")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


@pytest.fixture(scope="session")
def oracle():
    """The reference compiled in place when built (oracle/_ref), else the C restatement."""
    from oracle import default_oracle

    return default_oracle()


@pytest.fixture(scope="session")
def port():
    from oracle import PortOracle

    return PortOracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefOracle

    try:
        return RefOracle()
    except (FileNotFoundError, OSError):
        pytest.skip("reference oracle (oracle/_ref) not built")


@pytest.fixture(scope="session")
def rk():
    import paper_2009_14788_b200 as rk

    return rk


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA (run -m 'not gpu' here)")
    return torch.device("cuda:0")


def to_np(t):
    return t.detach().cpu().numpy()
