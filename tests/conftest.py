import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libvoxrf_b200 kernels)")
    config.addinivalue_line("markers", "ref: needs the reference build in oracle/_ref")
    config.addinivalue_line("markers", "slow: config-shaped parity (seconds to a minute each)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc
    return orc.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle as orc
    try:
        return orc.RefLib()
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def ctx():
    """A device context. No skip: on the GPU box a missing library or device is a failure."""
    from paper_2307_03404_b200 import Context
    return Context(0)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
