import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle_engine():
    import helpers
    return helpers.oracle_engine()


@pytest.fixture(scope="session")
def sim_engine():
    import helpers
    return helpers.sim_engine()


@pytest.fixture(scope="session")
def cuda_engine():
    import helpers
    return helpers.cuda_engine()


@pytest.fixture(scope="session")
def sim_tile_engine():
    """context whose plain post-SSA runs take the tile kernels (the default; fused only for match lists)"""
    import helpers
    return helpers.sim_engine(fused=False)


@pytest.fixture(scope="session")
def cuda_tile_engine():
    import helpers
    return helpers.cuda_engine(fused=False)


@pytest.fixture(scope="session")
def sim_fused_engine():
    """context whose post-SSA runs all take the function-resident fused kernels"""
    import helpers
    return helpers.sim_engine(fused=True)


@pytest.fixture(scope="session")
def cuda_fused_engine():
    import helpers
    return helpers.cuda_engine(fused=True)
